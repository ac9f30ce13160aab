"""Per-launch cost of switching kernels: total graph time / launches for (a) one shape
repeated, (b) two shapes alternating, (c) blocks of R launches with an event node between
blocks.  Cold operands (rotating arena slices as in bench.py)."""
import ctypes, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2409_01075_b200 as vx

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev); side = torch.cuda.Stream(dev)
S1 = (512, 4096, 4096); S2 = (128, 3072, 768); S3 = (512, 11008, 4096)
plans = {}
for M, N, K in (S1, S2, S3):
    plans[(N, K)] = vx.Plan(N, K, "bf16", "bf16", "nk", device=0)
arenas = bench.make_arenas([("x", M, N, K) for M, N, K in (S1, S2, S3)], dev, 0)
aA, aB, aC = arenas

def graph_time(seq, events_every=0, reps=5):
    work = [(s, aA.take(s[0] * s[2]), aB.take(s[1] * s[2]), aC.take(s[0] * s[1])) for s in seq]
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        sp = ctypes.c_void_p(side.cuda_stream)
        for (M, N, K), a, b, c in work[:4]:
            plans[(N, K)].gemm_ptr(1, M, N, K, a, M * K, b, N * K, c, M * N, sp)
        side.synchronize()
        g = torch.cuda.CUDAGraph()
        evs = []
        with torch.cuda.graph(g, stream=side):
            cs = torch.cuda.current_stream(); sp = ctypes.c_void_p(cs.cuda_stream)
            for i, ((M, N, K), a, b, c) in enumerate(work):
                if events_every and i % events_every == 0:
                    e = torch.cuda.Event(enable_timing=True, external=True); e.record(cs); evs.append(e)
                plans[(N, K)].gemm_ptr(1, M, N, K, a, M * K, b, N * K, c, M * N, sp)
    stream.wait_stream(side)
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream); g.replay(); e1.record(stream); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)

n = 64
t11 = graph_time([S1] * n); t22 = graph_time([S2] * n); t33 = graph_time([S3] * n)
print("S1 x%d: %.2f us/launch   S2: %.2f   S3: %.2f" % (n, t11 / n, t22 / n, t33 / n))
t12 = graph_time([S1, S2] * (n // 2))
print("S1,S2 alternating: %.2f us/pair (sum of singles %.2f)" % (t12 / (n // 2), (t11 + t22) / n))
t13 = graph_time([S1, S3] * (n // 2))
print("S1,S3 alternating: %.2f us/pair (sum of singles %.2f)" % (t13 / (n // 2), (t11 + t33) / n))
for R in (1, 8):
    t = graph_time([S1] * n, events_every=R)
    print("S1 x%d with an event node every %d launches: %.2f us/launch" % (n, R, t / n))
t = graph_time(([S1] * 8 + [S2] * 8) * 4)
print("S1x8,S2x8 blocks: %.2f us per 16 (sum singles %.2f)" % (t / 4, 8 * (t11 + t22) / n))
