"""Launch torch.mm (cuBLAS) on given shapes, R times each, for an ncu launch list (informational)."""
import sys
import torch
shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]]
for M, N, K in shapes:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = torch.mm(a, b.t())
    torch.cuda.synchronize()
