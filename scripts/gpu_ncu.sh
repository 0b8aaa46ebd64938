# ncu evidence for the bench command, one capture per gpurun call (ncu replays
# every kernel; the plain command runs first and must exit 0):
#   gpurun -- 'bash scripts/gpu_ncu.sh list'   -> gpurun_out/launches.csv
#   gpurun -- 'bash scripts/gpu_ncu.sh full'   -> gpurun_out/gemm_full.ncu-rep
# then: python scripts/ncu_summary.py gpurun_out/gemm_full.ncu-rep gpurun_out/launches.csv --out profiles/<name>
mkdir -p gpurun_out
A="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/plain.log 2>&1 || { echo "plain bench failed"; tail gpurun_out/plain.log; exit 1; }
case "$1" in
  list) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tf32|split" --csv \
          --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?" ;;
  full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 1 -c 1 \
          -o gpurun_out/gemm_full -f python bench.py $A > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?" ;;
  *) echo "usage: bash scripts/gpu_ncu.sh list|full"; exit 2 ;;
esac
