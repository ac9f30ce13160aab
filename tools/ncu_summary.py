"""Summarise an `ncu --set full` report into a small text file for profiles/ and, with
--traffic KEY, record dram read+write bytes per launch into profiles/ncu_traffic.json
(bench.py's roofline.traffic)."""
import csv, io, json, os, subprocess, sys

WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__cluster_dim_x", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__warps_active.avg.per_cycle_active"]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    lines = ["# ncu --set full --clock-control none summary of %s" % os.path.basename(rep),
             "kernel: %s" % vals[hdr.index("Kernel Name")]]
    got = {}
    for i, h in enumerate(hdr):
        if h in WANT:
            lines.append("%-66s %-14s %s" % (h, units[i], vals[i]))
            got[h] = (units[i], vals[i])
    open(out, "w").write("\n".join(lines) + "\n")
    if key:
        def to_bytes(u, v):
            f = float(v.replace(",", ""))
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        t = to_bytes(*got["dram__bytes_read.sum"]) + to_bytes(*got["dram__bytes_write.sum"])
        pj = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        d = json.load(open(pj)) if os.path.exists(pj) else {}
        d[key] = int(t)
        json.dump(d, open(pj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
