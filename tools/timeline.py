"""Steady-state launch timeline: R back-to-back launches of one (rung, split) captured in a
CUDA graph on rotating cold buffers (as tools/sweep.py --method graph), each launch with its
own %globaltimer trace slice (vx_debug_set_trace).  Prints, per phase, the median over
launches 1..R-1 of the time relative to the PREVIOUS launch's last CTA exit -- where the
per-launch floor goes.  NOTE: %globaltimer ticks every ~0.256 us on B200, so single phase
stamps are quantised to that; cycle counters (slots 12-14) are exact.

    python tools/timeline.py M N K [rung split] [--R 32] [--hot]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2409_01075_b200 as vx
import synth

PH = ["entry", "setup", "prod_done", "first_full", "mma_done", "acc_ready", "epi_done",
      "pre_teardown", "dep_released", "exit", "2nd_issue", "1st_issue", "-", "-", "-", "-", "split_sync1", "split_posted", "-", "-"] + ["-"] * 20
NS = 56   # slots per CTA; 12-15 = MMA-issuer cycle counters (wait, issue, commit, n), 18-31 cycle stamps


def main():
    a = [x for x in sys.argv[1:] if not x.startswith("--")]
    R = 32
    if "--R" in sys.argv:
        R = int(sys.argv[sys.argv.index("--R") + 1])
        a = [x for x in a if x != str(R)]
    M, N, K = int(a[0]), int(a[1]), int(a[2])
    force = (int(a[3]), int(a[4])) if len(a) > 4 else (-1, 0)
    dev = torch.device("cuda", 0)
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    hot = "--hot" in sys.argv          # same buffers every launch (L2-resident operands)
    nb = 1 if hot else R
    A = synth.matrix((nb, M * K), "bf16", seed=1, device=dev)
    B = synth.matrix((nb, N * K), "bf16", seed=2, scale=K ** -0.5, device=dev)
    C = torch.empty((nb, M * N), dtype=torch.bfloat16, device=dev)
    ch = vx.Choice()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, A[0].data_ptr(), M * K, B[0].data_ptr(), N * K,
                           C[0].data_ptr(), M * N, force[0], force[1], sp, ctypes.byref(ch))
    assert st == 0, vx.lib.vx_last_error()
    torch.cuda.synchronize()
    g = ch.grid
    buf = torch.zeros((R, NS * max(g, 1)), dtype=torch.int64, device=dev)
    vx.lib.vx_debug_set_trace.argtypes = [ctypes.c_void_p]
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for i in range(R):
                vx.lib.vx_debug_set_trace(buf[i].data_ptr())
                j = i % nb
                st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, A[j].data_ptr(), M * K,
                                       B[j].data_ptr(), N * K, C[j].data_ptr(), M * N, force[0],
                                       force[1], sp, None)
                assert st == 0, vx.lib.vx_last_error()
            vx.lib.vx_debug_set_trace(None)
    torch.cuda.current_stream().wait_stream(side)
    for rep in range(3):
        buf.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
    t = buf.view(R, g, NS).cpu().numpy().astype(np.int64)
    print("M=%d N=%d K=%d choice=%s  graph per-launch %.2f us" % (
        M, N, K, ch.as_dict(), e0.elapsed_time(e1) * 1e3 / R))
    rows = {nm: [] for nm in PH}
    per_launch = []
    for i in range(1, R):
        prev_exit = t[i - 1, :, 9].max()
        per_launch.append((t[i, :, 9].max() - prev_exit) / 1e3)
        for j, nm in enumerate(PH):
            if nm == "-":
                continue
            col = t[i, :, j]
            col = col[col > 0]
            if len(col):
                rows[nm].append(((col.min() - prev_exit) / 1e3, (np.median(col) - prev_exit) / 1e3,
                                 (col.max() - prev_exit) / 1e3))
    print("  exit-to-exit median %.2f us (relative to previous launch's last exit):" %
          np.median(per_launch))
    cy = t[1:, :, 12:16].reshape(-1, 4)
    cy = cy[cy[:, 3] > 0]
    if len(cy):
        n = cy[:, 3].astype(float)
        print("  MMA issuer cycles per k-block: wait-full %.0f  issue %.0f  commit %.0f" % (
            np.median(cy[:, 0] / n), np.median(cy[:, 1] / n), np.median(cy[:, 2] / n)))
    CY = {18: "prod: dep-wait -> 1st issue", 20: "prod: createpolicy", 21: "prod: WorkIter",
          22: "prod: next+decode", 23: "prod: 1st empty wait", 24: "setup: bar init (entry+)",
          25: "setup: L2 prefetch (entry+)", 26: "setup: synced (entry+)",
          27: "setup: dep released (entry+)", 28: "tmem alloc", 29: "epi: 1st tmem ld",
          30: "epi: chunks issued / split push", 31: "epi: bulk wait read",
          19: "split: push + own-rows barrier", 29: "split: reduce + C store",
          32: "last tile: owner flag acquire", 33: "last tile: accumulator wait",
          34: "last tile: epilogue chunks", 35: "epi: final bulk wait"}
    for sl, nm in CY.items():
        c = t[1:, :, sl].reshape(-1)
        c = c[c > 0]
        if len(c):
            print("  cyc %-30s median %7.0f  max %7.0f" % (nm, np.median(c), c.max()))
    iss = t[1:, :, 40:48].reshape(-1, 8).astype(float)
    arr = t[1:, :, 48:56].reshape(-1, 8).astype(float)
    if (iss[:, 0] > 0).any():
        dep = t[1:, :, 27].reshape(-1).astype(float)       # dependency released (entry+)
        ok = iss[:, 0] > 0
        print("  units 0-7, cycles after the dependency release (median over CTAs):")
        print("    issued  " + " ".join("%6.0f" % np.median(iss[ok, u] - dep[ok]) for u in range(8)
                                       if (iss[ok, u] > 0).any()))
        ok2 = arr[:, 0] > 0
        print("    landed  " + " ".join("%6.0f" % np.median(arr[ok2, u] - dep[ok2]) for u in range(8)
                                       if (arr[ok2, u] > 0).any()))
    for nm in PH:
        if nm != "-" and rows[nm]:
            v = np.median(np.array(rows[nm]), axis=0)
            print("  %-13s first %7.2f  median %7.2f  last %7.2f" % (nm, v[0], v[1], v[2]))


if __name__ == "__main__":
    main()
