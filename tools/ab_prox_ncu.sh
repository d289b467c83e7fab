# per-launch durations of the prox kernels (ncu launch list, serialised) for each variants/*.so, C5-shaped solve (T = 20)
mkdir -p gpurun_out/abp
for f in variants/*.so; do
  cp $f paper_1904_04884_b200/libholo_b200.so
  b=$(basename $f .so)
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_prox_strip --csv --log-file gpurun_out/abp/$b.csv python tools/run_solve.py 1024 1024 512 2 20 > gpurun_out/abp/$b.log 2>&1
done
python - <<'PY'
import csv, glob, collections, os
for f in sorted(glob.glob("gpurun_out/abp/*.csv")):
    d = collections.defaultdict(list)
    for r in csv.DictReader(l for l in open(f) if l.startswith('"')):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            d[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    print(os.path.basename(f))
    for k, v in d.items():
        v = sorted(v)
        print(f"   {k[:60]:60s} n={len(v):3d} median {v[len(v)//2]/1e6 if max(v) > 1e5 else v[len(v)//2]:.3f}")
PY
