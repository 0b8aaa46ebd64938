# Refresh every measured artifact with the current code (one GPU call).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo "smoke failed"; tail gpurun_out/smoke.log; exit 1; }
tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 900 python scripts/bench_configs.py > gpurun_out/configs.md 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 600 python scripts/bench_ext.py > gpurun_out/ext.md 2>&1; timeout 600 python scripts/bench_ext.py dgemm >> gpurun_out/ext.md 2>&1; echo "ext rc=$?"
A="--steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 python bench.py $A > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tf32|split" --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 1 -c 1 -o gpurun_out/gemm_full python bench.py $A > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 python scripts/mode_speed.py > gpurun_out/modes.txt 2>&1; echo "modes rc=$?"
