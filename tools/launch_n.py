"""Launch one (M, N, K) GEMM R times back to back (selected or forced rung), for ncu captures.

    python tools/launch_n.py M N K [rung split] [--R 8] [--out bf16]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2409_01075_b200 as vx
import synth


def main():
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    R = int(sys.argv[sys.argv.index("--R") + 1]) if "--R" in sys.argv else 8
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else "bf16"
    a = [x for x in a if x not in (str(R), out)]
    M, N, K = int(a[0]), int(a[1]), int(a[2])
    force = (int(a[3]), int(a[4])) if len(a) > 4 else (-1, 0)
    p = vx.Plan(N, K, "bf16", out, "nk")
    print("selected", p.select(M))
    A = synth.matrix((M, K), "bf16", seed=1, device="cuda")
    B = synth.matrix((N, K), "bf16", seed=2, scale=K ** -0.5, device="cuda")
    C = torch.empty((M, N), dtype={"bf16": torch.bfloat16, "fp32": torch.float32}[out], device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ch = vx.Choice()
    for _ in range(R):
        st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, A.data_ptr(), M * K, B.data_ptr(), N * K,
                               C.data_ptr(), M * N, force[0], force[1], sp, ctypes.byref(ch))
        assert st == 0, vx.lib.vx_last_error()
    torch.cuda.synchronize()
    print(ch.as_dict())


if __name__ == "__main__":
    main()
