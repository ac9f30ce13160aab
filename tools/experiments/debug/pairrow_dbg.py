"""pair-row store debug: each (s, rung, split) in its own process so a fault names its case."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import torch
    import paper_2409_01075_b200 as vx
    s, d, rung, split = (int(x) for x in sys.argv[2:6])
    p = vx.Plan(0, d, "bf16", "bf16", "nk")
    Q = torch.randint(-3, 4, (2, s, d), device="cuda").to(torch.bfloat16)
    K = torch.randint(-3, 4, (2, s, d), device="cuda").to(torch.bfloat16)
    out = p.gemm(Q, K, force=None if rung < 0 else (rung, split))
    torch.cuda.synchronize()
    ref = torch.bmm(Q.float(), K.float().transpose(1, 2)).to(torch.bfloat16)
    print("OK" if torch.equal(out, ref) else "MISMATCH %d" % (out != ref).sum().item())
    sys.exit(0)
import torch  # noqa
import paper_2409_01075_b200 as vx
for d in (64,):
    rungs = vx.Plan(0, d, "bf16", "bf16", "nk").dump()["rungs"]
    for s in (100,):
        for r in [{"rung_id": -1, "splits": [1]}] + rungs[:2]:
            for sp in r["splits"]:
                o = subprocess.run([sys.executable, __file__, "--one", str(s), str(d), str(r["rung_id"]), str(sp)],
                                   capture_output=True, text=True, timeout=120)
                res = o.stdout.strip().splitlines()[-1:] or [o.stderr.strip().splitlines()[-1] if o.stderr.strip() else "?"]
                print(s, d, r["rung_id"], r.get("bm"), r.get("bn"), r.get("family"), sp, res[0][:100], flush=True)
