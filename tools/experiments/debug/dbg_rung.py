"""Launch one forced (rung, split) once with integer data and compare with the oracle (debug)."""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import paper_2409_01075_b200 as vx, synth, oracle
M, N, K, bn, s = (int(v) for v in sys.argv[1:6])
out = sys.argv[6] if len(sys.argv) > 6 else "fp32"
p = vx.Plan(N, K, "bf16", out, "nk")
r = [x for x in p.dump()["rungs"] if x["family"] == 0 and x["bm"] == 128 and x["bn"] == bn and x["mc"] == 1][0]
A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="int", seed=1)
C, ch = p.gemm(A.cuda(), B.cuda(), force=(r["rung_id"], s), want_choice=True)
torch.cuda.synchronize()
want = oracle.gemm(A, B, "nk")
got = C.cpu().double().numpy()
print(M, N, K, bn, s, out, "exact" if np.array_equal(got, want) else "MISMATCH %g" % np.abs(got - want).max(), flush=True)
