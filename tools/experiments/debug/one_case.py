"""Run one forced (rung, split) case and compare with the oracle (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2409_01075_b200 as vx

def main(N, K, bl, M, rung, split, out="fp32", batch=None):
    p = vx.Plan(N if batch is None else 0, K, "bf16", out, bl)
    A, B = synth.gemm_inputs(M, N, K, "bf16", bl, kind="int", seed=M, batch=batch)
    ref = oracle.gemm(A, B, bl)
    C, ch = p.gemm(A.cuda(), B.cuda(), force=(rung, split), want_choice=True)
    torch.cuda.synchronize()
    got = C.cpu().double().numpy()
    print(ch, "maxerr", np.abs(got - ref).max(), flush=True)

if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]), int(a[1]), a[2], int(a[3]), int(a[4]), int(a[5]))
