# Round-2 (session 2) evidence: GPU tests, the default bench line + per-point results, the
# reference arm, ncu --set full of the dominant / BERT / decode / multicast kernels, and the
# ncu launch list of one bench replay.   gpurun -- 'bash tools/experiments/gpurun/r2_evidence.sh'
set -x
mkdir -p gpurun_out/ev3 /tmp/ncu
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/ev3/gpu_tests.log 2>&1
tail -2 gpurun_out/ev3/gpu_tests.log
python bench.py --points-out gpurun_out/ev3/bench_points.json > gpurun_out/ev3/bench.json 2> gpurun_out/ev3/bench.err
tail -c 300 gpurun_out/ev3/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev3/bench_reference.json 2> gpurun_out/ev3/bench_reference.err
for spec in "dominant:16383 12288 4096:2:vx_umma" "bert:128 3072 768:4:vx_umma" "decode16:16 11008 4096:4:vx_" "mc2:128 11008 4096:4:vx_umma"; do
  IFS=: read name shape skip kre <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/ncu/$name -f python tools/launch_n.py $shape --R 8 > gpurun_out/ev3/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/ncu/$name.ncu-rep gpurun_out/ev3/ncu_$name.txt --traffic "$(echo $shape | tr ' ' '_')" >> gpurun_out/ev3/ncu_$name.log 2>&1
done
cp profiles/ncu_traffic.json gpurun_out/ev3/ncu_traffic.json
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file /tmp/ncu/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-cublas --no-extra > gpurun_out/ev3/launches_bench.log 2>&1
python - <<'PY'
import csv, json
rows = [r for r in csv.reader(open('/tmp/ncu/launches.csv')) if len(r) > 10]
hdr = rows[0]; idx = {h: i for i, h in enumerate(hdr)}
recs = [(int(r[idx['ID']]), r[idx['Kernel Name']], r[idx['Grid Size']], float(r[idx['Metric Value']]))
        for r in rows[1:] if r[idx['Metric Name']] == 'gpu__time_duration.sum']
with open('gpurun_out/ev3/launches_trim.csv', 'w') as f:
    w = csv.writer(f); w.writerow(['ID', 'Kernel Name', 'Grid Size', 'ns'])
    for rec in recs:
        w.writerow([rec[0], rec[1][:90], rec[2], rec[3]])
# launches 192 .. 192 + 192*48 - 1 = the first full sweep replay (the first 192 are capture-time
# warm-up launches), 48 per point in sweep order; the dominant point is the largest group
R = 48
rep = recs[192:192 + 192 * R]
groups = [rep[i * R:(i + 1) * R] for i in range(len(rep) // R)]
tot = sum(x[3] for x in rep)
best = max(range(len(groups)), key=lambda i: sum(x[3] for x in groups[i]))
g = groups[best]
json.dump({"replay_total_ms": tot / 1e6, "dominant_group_index": best,
           "dominant_ms": sum(x[3] for x in g) / 1e6,
           "dominant_share": sum(x[3] for x in g) / tot,
           "dominant_per_launch_us": sum(x[3] for x in g) / len(g) / 1e3,
           "kernel": g[0][1][:120], "grid": g[0][2], "launches": len(rep)},
          open('gpurun_out/ev3/launches_share.json', 'w'), indent=1)
PY
gzip -f gpurun_out/ev3/launches_trim.csv
ls -la gpurun_out/ev3
timeout 900 python tools/sweep.py --method graph --shapes all --out gpurun_out/ev3/heldout_sweep.json > gpurun_out/ev3/heldout.log 2>&1
tail -1 gpurun_out/ev3/heldout.log
