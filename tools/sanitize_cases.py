"""One small launch per schedule of the ladder, checked against the oracle, for running
under compute-sanitizer (memcheck / racecheck / synccheck; SURVEY 5 aux subsystems):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: persistent (128x128, swapped 128x32), split-K cluster (DSMEM reduce), stream-K
(flag protocol), cta_group::2 pair, TMA-multicast cluster, GEMV, fused gather epilogue."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2409_01075_b200 as vx
import synth


def main():
    M, N, K = 200, 512, 512
    p = vx.Plan(N, K, "bf16", "fp32", "nk")
    rungs = p.dump()["rungs"]
    A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=3)
    want = oracle.gemm(A, B, "nk")
    Ad, Bd = A.cuda(), B.cuda()

    def pick(**kw):
        for r in rungs:
            if all(r[k] == v for k, v in kw.items()):
                return r["rung_id"]
        raise KeyError(kw)

    cases = [("persistent 128x128", pick(family=0, bm=128, bn=128, mc=1), 1),
             ("persistent swap 128x32", pick(family=1, bn=32, mc=1), 1),
             ("split-K 2 (DSMEM reduce)", pick(family=0, bm=128, bn=64, mc=1), 2),
             ("stream-K", pick(family=0, bm=128, bn=128, mc=1), 0),
             ("pair 256x128", pick(family=0, bm=256, bn=128), 1),
             ("pair 256x256 stream-K", pick(family=0, bm=256, bn=256), 0),
             ("multicast mc2 128x128", pick(family=0, bm=128, bn=128, mc=2), 1),
             ("multicast mc4 swap 128x64", pick(family=1, bn=64, mc=4), 1)]
    ok = True
    for name, rid, s in cases:
        C, ch = p.gemm(Ad, Bd, force=(rid, s), want_choice=True)
        torch.cuda.synchronize()
        good = np.array_equal(C.cpu().double().numpy(), want)
        ok &= good
        print("%-28s rung %2d split %d grid %3d  %s" % (name, rid, s, ch["grid"], "ok" if good else "MISMATCH"), flush=True)
    A1, B1 = synth.gemm_inputs(3, N, K, "bf16", "nk", kind="int", seed=4)
    g = pick(family=3, bm=4)
    C = p.gemm(A1.cuda(), Bd if False else B1.cuda(), force=(g, 1))
    torch.cuda.synchronize()
    good = np.array_equal(C.cpu().double().numpy(), oracle.gemm(A1, B1, "nk"))
    ok &= good
    print("%-28s %s" % ("GEMV MT=4", "ok" if good else "MISMATCH"))
    bufs = [torch.zeros((M, N), dtype=torch.float32, device="cuda") for _ in range(2)]
    for lo, hi in ((0, 100), (100, M)):
        p.gemm_gather(Ad[lo:hi].contiguous(), Bd, bufs, lo)
    torch.cuda.synchronize()
    good = all(np.array_equal(b.cpu().double().numpy(), want) for b in bufs)
    ok &= good
    print("%-28s %s" % ("fused gather (2 dst)", "ok" if good else "MISMATCH"))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
