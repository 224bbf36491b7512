"""Print the MoE parity errors (vs the oracle) of the GPU tests' cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_19427_b200 import Context
from tests.helpers import rel_err
from tests.test_moe_gpu import run_moe
from tests.test_moe_mx_gpu import run_moe_mx

ctx = Context(0)
for args in [(33, 256, 256, 8, 2, 1), (40, 7168, 5120, 8, 3, 2), (300, 256, 384, 4, 2, 3)]:
    got, ref = run_moe(ctx, *args)
    print("fp8", args, rel_err(got, ref))
for pair in ("0", "1"):
    os.environ["AFDK_MX_PAIR"] = pair
    for args in [(33, 512, 512, 8, 2, 1), (40, 7168, 5120, 8, 3, 2), (400, 7168, 5120, 4, 2, 5)]:
        got, ref = run_moe_mx(ctx, *args)
        print("mx pair=" + pair, args, rel_err(got, ref))
