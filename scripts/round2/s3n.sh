# session 3: ncu --set full of the c2 (fp32 split-tf32) FWD1 / FWD2 GEMMs
mkdir -p gpurun_out
KBASE=demangled KREGEX='tf32' NAME=s3n_c2_tf32 SKIP=300 COUNT=2 BENCH_ARGS="--config c2" OUT=/tmp/s3n bash scripts/ncu_kernel.sh
ncu -i /tmp/s3n/s3n_c2_tf32.ncu-rep --page details --csv > gpurun_out/s3n_details.csv 2>/dev/null
ncu -i /tmp/s3n/s3n_c2_tf32.ncu-rep --page source --csv --print-source sass > gpurun_out/s3n_source.csv 2>/dev/null
ncu -i /tmp/s3n/s3n_c2_tf32.ncu-rep --page raw --csv > gpurun_out/s3n_raw.csv 2>/dev/null
tail -3 /tmp/s3n/s3n_c2_tf32.log; ls -la gpurun_out/s3n*
