import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_19427_b200 import Context
from tests.test_mfa_decode_gpu import run_case

for nsm in [0, 1, 3]:
    ctx = Context(0, nsm)
    for sl in [[65], [128], [64, 64], [1, 63, 64, 65], [200], [4096]]:
        for poison in [False, True]:
            got, lse, ref, ref_lse = run_case(ctx, sl, poison=poison)
            errs = []
            for b in range(len(sl)):
                e = np.max(np.abs(got[b] - ref[b])) / max(np.max(np.abs(ref[b])), 1e-9)
                ratio = np.median(got[b] / np.where(np.abs(ref[b]) > 1e-3, ref[b], np.nan)[..., None].squeeze()) if True else 0
                errs.append(f"{e:.1e}/r{np.nanmedian(got[b]/np.where(np.abs(ref[b])>1e-2, ref[b], np.nan)):.3f}/lse{np.max(np.abs(lse[b]-ref_lse[b])):.1e}")
            print(f"nsm={ctx.num_sms} sl={sl} poison={poison}: {errs}", flush=True)
    ctx.close()
