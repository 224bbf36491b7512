import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) == 1:
    for flags in ["8", "14", "22", "30"]:
        r = subprocess.run([sys.executable, __file__, flags], capture_output=True, text=True, timeout=120)
        print("flags", flags, (r.stdout + r.stderr).strip().splitlines()[-1:])
    sys.exit(0)
os.environ["AFDK_DEBUG_SYNC"] = "1"
os.environ["AFDK_DEBUG_FLAGS"] = sys.argv[1]
from paper_2507_19427_b200 import Context
from tests.test_moe_gpu import run_moe
from tests.helpers import rel_err
ctx = Context(0)
try:
    got, ref = run_moe(ctx, 33, 256, 256, 8, 2, 1)
    print("small rel_err", rel_err(got, ref))
except Exception as e:
    print("ERR", e)
