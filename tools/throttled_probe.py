"""Per-launch time of forced (rung, split) choices in a POWER-CAPPED context (measurement tool).

The bench's sweep is one long step dominated by large GEMMs, so its small launches run at the
~1 kW power cap (SM clock ~1.3 GHz).  Here each measured batch of R launches of
the shape (fresh arena slices) is preceded, in the same CUDA graph, by a heater of large
GEMMs (M=16384, N=12288, K=4096) that holds the GPU at the cap; events bracket only the
measured launches.  Prints the ranking under heat next to a cold (no heater) ranking.

    python tools/throttled_probe.py "16,11008,4096;128,768,768" [--R 48] [--heat 24]
"""
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2409_01075_b200 as vx


def main():
    shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1].split(";")]
    R = int(sys.argv[sys.argv.index("--R") + 1]) if "--R" in sys.argv else 48
    H = int(sys.argv[sys.argv.index("--heat") + 1]) if "--heat" in sys.argv else 24
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    GiB = 1 << 30
    aA = torch.randn(GiB // 2, dtype=torch.bfloat16, device=dev)
    aB = torch.randn(GiB // 2, dtype=torch.bfloat16, device=dev) * 0.02
    aC = torch.empty(GiB // 2, dtype=torch.bfloat16, device=dev)
    hM, hN, hK = 16384, 12288, 4096
    hp = vx.Plan(hN, hK, "bf16", "bf16", "nk")
    hA = torch.randn(hM, hK, device=dev).to(torch.bfloat16)
    hB = (torch.randn(hN, hK, device=dev) * 0.02).to(torch.bfloat16)
    hC = torch.empty(hM, hN, dtype=torch.bfloat16, device=dev)
    side = torch.cuda.Stream(dev)
    for M, N, K in shapes:
        p = vx.Plan(N, K, "bf16", "bf16", "nk")
        sel = p.select(M)
        cands = [(r["rung_id"], s) for r in p.dump()["rungs"] for s in r["splits"]
                 if not (r["family"] == 3 and M > r["bm"])]
        res = []
        for rid, s in cands:
            out = {}
            for heat in (0, H):
                views = []
                for i in range(R):
                    oa = (i * M * K) % (aA.numel() - M * K) // 64 * 64
                    ob = (i * N * K) % (aB.numel() - N * K) // 64 * 64
                    oc = (i * M * N) % (aC.numel() - M * N) // 64 * 64
                    views.append((aA[oa:oa + M * K], aB[ob:ob + N * K], aC[oc:oc + M * N]))
                e0 = torch.cuda.Event(enable_timing=True, external=True)
                e1 = torch.cuda.Event(enable_timing=True, external=True)
                side.wait_stream(stream)
                with torch.cuda.stream(side):
                    sp = ctypes.c_void_p(side.cuda_stream)
                    a, b, c = views[0]
                    st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, a.data_ptr(), M * K, b.data_ptr(),
                                           N * K, c.data_ptr(), M * N, rid, s, sp, None)
                    if st:
                        raise RuntimeError(vx.lib.vx_last_error().decode())
                    side.synchronize()
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=side):
                        cs = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
                        for _ in range(heat):
                            hp.gemm(hA, hB, out=hC)
                        e0.record()
                        for a, b, c in views:
                            vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, a.data_ptr(), M * K,
                                              b.data_ptr(), N * K, c.data_ptr(), M * N, rid, s, cs,
                                              None)
                        e1.record()
                stream.wait_stream(side)
                ts = []
                for rep in range(4):
                    g.replay()
                    torch.cuda.synchronize()
                    if rep:
                        ts.append(e0.elapsed_time(e1) * 1e3 / R)
                out[heat] = statistics.median(ts)
                del g
            res.append((out[H], out[0], rid, s))
        res.sort()
        print("M=%d N=%d K=%d  selected (%d,%d)" % (M, N, K, sel["rung_id"], sel["split"]))
        for hot, cold, rid, s in res[:8]:
            print("   rung %2d split %d   hot %7.2f us   cold %7.2f us%s" % (
                rid, s, hot, cold, "   <- selected" if (rid, s) == (sel["rung_id"], sel["split"]) else ""))
        for hot, cold, rid, s in res:
            if (rid, s) == (sel["rung_id"], sel["split"]):
                print("   selected: hot %.2f (best hot %.2f, regret %.3f)" % (hot, res[0][0], res[0][0] / hot))


if __name__ == "__main__":
    main()
