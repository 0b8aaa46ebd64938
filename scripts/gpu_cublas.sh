mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python scripts/cublas_compare.py 16384 fp32
timeout 300 python scripts/cublas_compare.py 16384 tf32
CUBLAS_EMULATE_SINGLE_PRECISION=1 timeout 300 python scripts/cublas_compare.py 16384 fp32
CUBLAS_EMULATE_SINGLE_PRECISION=1 CUBLAS_EMULATION_STRATEGY=performant timeout 300 python scripts/cublas_compare.py 16384 fp32
CUBLAS_EMULATE_SINGLE_PRECISION=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -s 3 -c 3 python scripts/cublas_compare.py 16384 fp32 2>&1 | grep -E "^  [a-zA-Z_]|dram__|lts__|gpu__time|cycles_elapsed" | head -30
