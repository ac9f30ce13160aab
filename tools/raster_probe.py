"""Raster group size A/B on the large pair-rung shapes (VX_GROUP_P is read once at library load,
so every group size runs in its own process).

    python tools/raster_probe.py [--gp 4,8,16,32] [--flags 0,524288] [--shapes 0,1] [--R 64] [--ncu]
    (child) python tools/raster_probe.py --child M N K R

Per (group, shape): device time per launch of R back-to-back launches in one CUDA graph on
fresh operand slices (>= 1 GiB arenas: cold L2 per launch, the bench's timing), median of 5
replays after a 3-replay warm-up that brings the GPU to its power-capped steady state.
With --ncu, one launch per (group, shape) is captured for dram__bytes_read/write.
"""
import ctypes
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(16383, 12288, 4096), (16384, 11008, 4096), (8192, 12288, 4096), (4096, 4096, 4096),
          (10000, 11008, 4096)]


def child(M, N, K, R):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2409_01075_b200 as vx
    p = vx.Plan(N, K, "bf16", "bf16", "nk")
    ch = p.select(M)
    a_el, b_el, c_el = M * K, N * K, M * N
    slots = max(2, min(R, (1 << 30) // (2 * max(a_el, c_el)) + 1))
    A = torch.randn(slots * a_el, device="cuda").to(torch.bfloat16)
    B = (torch.randn(slots * b_el, device="cuda") * K ** -0.5).to(torch.bfloat16)
    C = torch.empty(slots * c_el, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = vx.Choice()

    def launch(i):
        j = i % slots
        st = vx.lib.vx_gemm_ex(p.handle, 1, M, N, K, A.data_ptr() + 2 * j * a_el, M * K,
                               B.data_ptr() + 2 * j * b_el, N * K, C.data_ptr() + 2 * j * c_el,
                               M * N, -1, 0, sp, ctypes.byref(out))
        assert st == 0, vx.lib.vx_last_error()

    if os.environ.get("RASTER_NCU"):
        with torch.cuda.stream(s):
            launch(0)
        torch.cuda.synchronize()
        return
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        launch(0)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                launch(i)
    ts = []
    for rep in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        if rep >= 3:
            ts.append(e0.elapsed_time(e1) * 1000 / R)
    print(json.dumps({"M": M, "N": N, "K": K, "rung": out.as_dict().get("rung_id"),
                      "us": statistics.median(ts), "us_all": ts}))


def main():
    if "--child" in sys.argv:
        i = sys.argv.index("--child")
        child(*(int(x) for x in sys.argv[i + 1:i + 5]))
        return
    gps = [int(x) for x in (sys.argv[sys.argv.index("--gp") + 1] if "--gp" in sys.argv
                            else "4,8,16,24,32").split(",")]
    R = int(sys.argv[sys.argv.index("--R") + 1]) if "--R" in sys.argv else 64
    flags = [int(x) for x in (sys.argv[sys.argv.index("--flags") + 1] if "--flags" in sys.argv
                              else "0").split(",")]
    shapes = [SHAPES[int(x)] for x in sys.argv[sys.argv.index("--shapes") + 1].split(",")] \
        if "--shapes" in sys.argv else SHAPES
    res = []
    for (M, N, K), gp, fl in [(s_, g_, f_) for s_ in shapes for g_ in gps for f_ in flags]:
        if True:
            env = dict(os.environ, VX_GROUP_P=str(gp), VX_DEBUG_FLAGS=str(fl))
            o = subprocess.run([sys.executable, __file__, "--child", str(M), str(N), str(K), str(R)],
                               env=env, capture_output=True, text=True, timeout=600)
            line = [x for x in o.stdout.splitlines() if x.startswith("{")]
            r = json.loads(line[-1]) if line else {"err": o.stderr[-400:]}
            r["gp"] = gp
            r["flags"] = fl
            if "--ncu" in sys.argv:
                env["RASTER_NCU"] = "1"
                q = subprocess.run(["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,"
                                    "gpu__time_duration.sum", "--clock-control", "none", "-k",
                                    "regex:vx_umma", "-c", "1", "--csv", sys.executable, __file__,
                                    "--child", str(M), str(N), str(K), "1"],
                                   env=env, capture_output=True, text=True, timeout=600)
                for ln in q.stdout.splitlines():
                    f = [x.strip('"') for x in ln.split('","')]
                    if len(f) > 3 and f[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                                "gpu__time_duration.sum"):
                        r[f[-3] + " (" + f[-2] + ")"] = f[-1]
            print(json.dumps(r), flush=True)
            res.append(r)
    if "--out" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--out") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
