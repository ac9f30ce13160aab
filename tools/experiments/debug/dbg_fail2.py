import sys, torch, time
sys.path.insert(0, '.')
import paper_2409_01075_b200 as vx, synth
N, K = int(sys.argv[1]), 4096
M = int(sys.argv[2])
p = vx.Plan(N, K, "bf16", "bf16", "nk")
A, B = synth.gemm_inputs(M, N, K, "bf16", "nk", kind="normal", seed=M, device="cuda")
for i in range(int(sys.argv[3])):
    C = p.gemm(A, B)
torch.cuda.synchronize()
print("ok", N, M, p.select(M))
