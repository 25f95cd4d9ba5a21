# session 3: ncu --set full of the FWD2 and DGRAD_A GEMMs (c3): L2 / smem / stall picture
mkdir -p gpurun_out
KBASE=demangled KREGEX='tc_gemm2_kernel<.int.1,' NAME=s3h_fwd2 SKIP=2 bash scripts/ncu_kernel.sh
KBASE=demangled KREGEX='tc_gemm2_kernel<.int.2,' NAME=s3h_dgradA SKIP=2 bash scripts/ncu_kernel.sh
for r in s3h_fwd2 s3h_dgradA; do
ncu -i gpurun_out/$r.ncu-rep --page details --csv > gpurun_out/${r}_details.csv 2>/dev/null
ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out/s3h*
