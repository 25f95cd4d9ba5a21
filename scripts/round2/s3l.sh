# session 3: k-tail trimming A/B on one box with serialised ncu launch times (wgrad kernels)
mkdir -p gpurun_out
for i in 1 2; do for t in 0 1; do
MOE_NO_KTRIM=$t ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm2 --csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E '"gpu__time_duration' > gpurun_out/s3l_notrim${t}_$i.csv
done; done
for f in gpurun_out/s3l_*.csv; do python - "$f" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
acc = collections.defaultdict(list)
for r in rows:
    name = r[4] if len(r) > 4 else ''
    kind = name.split('<')[1].split(',')[0] if '<' in name else name
    try: acc[kind].append(float(r[-1]))
    except ValueError: pass
print(sys.argv[1], {k: round(sum(v) / len(v), 1) for k, v in sorted(acc.items())})
PY
done
