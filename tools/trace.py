"""Phase trace of one launch: %globaltimer stamps per CTA (debug hook vx_debug_set_trace).
    python tools/trace.py M N K [rung split] [--batch B]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_01075_b200 as vx
import synth

PH = ["entry", "setup", "prod_done", "first_full", "mma_done", "acc_ready", "epi/sync2", "reduced",
      "dep_released", "exit", "first_issue", "-"]
NS = 40        # slots per CTA (vx_umma.cuh trace_at)

def main():
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    M, N, K = int(a[0]), int(a[1]), int(a[2])
    force = (int(a[3]), int(a[4])) if len(a) > 4 else (-1, 0)
    dev = torch.device("cuda", 0)
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    A = synth.matrix((M, K), "bf16", seed=1, device=dev)
    B = synth.matrix((N, K), "bf16", seed=2, scale=K ** -0.5, device=dev)
    C = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    buf = torch.zeros(NS * 4096, dtype=torch.int64, device=dev)
    fl = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    vx.lib.vx_debug_set_trace.argtypes = [ctypes.c_void_p]
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for rep in range(4):
        fl.zero_(); fl.view(torch.int32).sum()
        buf.zero_()
        vx.lib.vx_debug_set_trace(buf.data_ptr())
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        ch = vx.Choice()
        e0.record()
        st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, A.data_ptr(), M * K, B.data_ptr(), N * K,
                               C.data_ptr(), M * N, force[0], force[1], sp, ctypes.byref(ch))
        e1.record()
        torch.cuda.synchronize()
        vx.lib.vx_debug_set_trace(None)
        assert st == 0, vx.lib.vx_last_error()
    g = ch.grid
    t = buf[: NS * g].view(g, NS).cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print("M=%d N=%d K=%d choice=%s event=%.2fus" % (M, N, K, ch.as_dict(), e0.elapsed_time(e1) * 1e3))
    if "--late" in sys.argv:
        order = np.argsort(-rel[:, 6])[:12]
        for c in order:
            print("  cta %3d " % c + " ".join("%7.2f" % x for x in rel[c]))
    for i, nm in enumerate(PH):
        col = rel[:, i]
        col = col[t[:, i] > 0]
        if len(col):
            print("  %-10s min %7.2f  med %7.2f  max %7.2f us" % (nm, col.min(), np.median(col), col.max()))

if __name__ == "__main__":
    main()
