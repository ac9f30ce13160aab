timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests_r2g.log 2>&1
tail -2 gpurun_out/gpu_tests_r2g.log
python bench.py --steps 10 --warmup 3 --points-out gpurun_out/bench_points_r2d.json > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err
tail -c 300 gpurun_out/bench_r2d.err
mkdir -p gpurun_out/ncu /tmp/ncu
for spec in "dominant:16383 12288 4096:2:vx_umma" "bert:128 3072 768:4:vx_umma" "decode16:16 11008 4096:4:vx_" "mc2:128 11008 4096:4:vx_umma"; do
  IFS=: read name shape skip kre <<< "$spec"
  ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/ncu/r02_$name -f python tools/launch_n.py $shape --R 8 > gpurun_out/ncu/$name.log 2>&1
  ncu -i /tmp/ncu/r02_$name.ncu-rep --page raw --csv > gpurun_out/ncu/r02_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/r02_$name.ncu-rep --page details --csv > gpurun_out/ncu/r02_${name}_details.csv 2>/dev/null
done
ncu -i /tmp/ncu/r02_bert.ncu-rep --page source --csv > gpurun_out/ncu/r02_bert_source.csv 2>/dev/null
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file /tmp/ncu/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-cublas --no-extra > gpurun_out/ncu/launches_bench.log 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('/tmp/ncu/launches.csv')) if len(r)>10]
hdr=rows[0]; idx={h:i for i,h in enumerate(hdr)}
out=open('gpurun_out/ncu/r02_launches_trim.csv','w')
w=csv.writer(out); w.writerow(['ID','Kernel Name','Grid Size','Block Size','gpu__time_duration.sum(ns)'])
for r in rows[1:]:
    if r[idx['Metric Name']]=='gpu__time_duration.sum':
        w.writerow([r[idx['ID']], r[idx['Kernel Name']][:90], r[idx['Grid Size']], r[idx['Block Size']], r[idx['Metric Value']]])
PY
du -sh gpurun_out; ls -la gpurun_out/ncu
