# Refresh measured artifacts (no ncu in this call).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo "smoke failed"; tail gpurun_out/smoke.log; exit 1; }
tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 900 python scripts/bench_configs.py > gpurun_out/configs.md 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 600 python scripts/bench_c5.py >> gpurun_out/configs.md 2>> gpurun_out/configs.err; echo "c5 rc=$?"
timeout 600 python scripts/bench_ext.py > gpurun_out/ext.md 2>&1; timeout 600 python scripts/bench_ext.py dgemm >> gpurun_out/ext.md 2>&1; echo "ext rc=$?"
timeout 600 python scripts/mode_speed.py > gpurun_out/modes.txt 2>&1; echo "modes rc=$?"
