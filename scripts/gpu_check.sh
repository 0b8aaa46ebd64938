# Quick GPU validation: smoke, probes, parity subset, short bench.  Fail fast.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "build failed"; tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -3 gpurun_out/smoke.log
[ $rc -eq 0 ] || exit 1
if [ -z "$SKIP_PROBE" ]; then
timeout 180 python -m pytest tests/test_probe.py -x -q -s > gpurun_out/probe.log 2>&1; echo "probe rc=$?"; grep -E "probe|3xTF32|passed|failed" gpurun_out/probe.log | tail -8
fi
timeout ${PARITY_TIMEOUT:-600} python -m pytest tests/test_parity.py tests/test_inputs.py -x -q ${PARITY_K:+-k "$PARITY_K"} > gpurun_out/parity.log 2>&1; rc=$?; echo "parity rc=$rc"
tail -15 gpurun_out/parity.log
[ $rc -eq 0 ] || [ -n "$BENCH_ANYWAY" ] || exit 1
timeout 600 python bench.py --steps ${BENCH_STEPS:-5} --warmup 3 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
