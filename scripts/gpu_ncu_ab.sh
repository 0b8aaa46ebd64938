# DRAM / L2 / time of the GEMM kernel under several env variants (ncu metrics pass).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python scripts/one_gemm.py ${N:-16384} 2 > gpurun_out/plain.log 2>&1 || { echo plain failed; tail gpurun_out/plain.log; exit 1; }
for v in $SWEEP; do
  echo "== $v"
  env ${v//,/ } timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tf32 -s 1 -c 1 python scripts/one_gemm.py ${N:-16384} 2 2>&1 | grep -E "dram__|lts__|gpu__time|cycles_elapsed|tensor_cycles" 
done
