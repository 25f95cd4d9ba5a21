# session 3 (reverted experiment, the switch is gone): dispatch tiles in reverse order (MOE_DISPATCH_REV=1: x rows the gate streamed last
# are still in L2) -- alternating c3 A/B and the dispatch kernel's DRAM bytes without cache control
mkdir -p gpurun_out
for i in 1 2 3 4; do
MOE_DISPATCH_REV=0 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3c_fwd_$i.json 2>/dev/null
MOE_DISPATCH_REV=1 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s3c_rev_$i.json 2>/dev/null
done
for r in 0 1; do
MOE_DISPATCH_REV=$r ncu --cache-control none --clock-control none -k regex:dispatch_kernel -s 2 -c 1 \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/s3c_ncu_rev$r.txt 2>&1
done
for f in gpurun_out/s3c_*.json; do python scripts/summ.py $f all < $f; done
grep -E 'dram__|gpu__time|lts__' gpurun_out/s3c_ncu_rev*.txt
# the fused cached-mode gate + dispatch kernel (c5): full set with source
KREGEX=gate_fwd_tc NAME=s3c_gate_cdisp BENCH_ARGS="--config c5" SKIP=2 bash scripts/ncu_kernel.sh
ncu -i gpurun_out/s3c_gate_cdisp.ncu-rep --page details --csv > gpurun_out/s3c_gate_cdisp_details.csv 2>/dev/null
ncu -i gpurun_out/s3c_gate_cdisp.ncu-rep --page source --csv --print-source sass > gpurun_out/s3c_gate_cdisp_source.csv 2>/dev/null
ls -la gpurun_out/s3c_gate_cdisp*
