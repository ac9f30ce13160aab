"""Quick on-GPU sanity sweep: every rung x split of a few plans on integer inputs vs the
fp64 oracle.  Prints one line per case; exit 1 on any mismatch.  (Debug aid; the real
parity suite is tests/test_gpu_parity.py.)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2409_01075_b200 as vx
import synth


def main():
    bad = 0
    torch.cuda.init()
    desc = vx.device_probe(0)
    print("desc", desc.to_json(), flush=True)
    cases = [(384, 512, "nk"), (384, 512, "kn")]
    for N, K, bl in cases:
        p = vx.Plan(N, K, "bf16", "fp32", bl)
        dump = p.dump()
        for M in (1, 129, 300):
            A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="int", seed=M)
            ref = oracle.gemm(A, B, bl)
            Ad, Bd = A.cuda(), B.cuda()
            for r in dump["rungs"]:
                if r["family"] == 3 and M > r["bm"]:
                    continue
                for s in r["splits"]:
                    t0 = time.time()
                    C = p.gemm(Ad, Bd, force=(r["rung_id"], s))
                    torch.cuda.synchronize()
                    got = C.cpu().double().numpy()
                    err = np.abs(got - ref).max()
                    ok = err == 0
                    bad += not ok
                    print("N=%d K=%d %s M=%d rung=%d fam=%d bn=%d split=%d maxerr=%g %s (%.2fs)" % (
                        N, K, bl, M, r["rung_id"], r["family"], r["bn"], s, err,
                        "OK" if ok else "FAIL", time.time() - t0), flush=True)
    print("BAD", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
