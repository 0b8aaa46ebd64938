# Build, smoke, quick parity, then an interleaved in-process A/B sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail -5 gpurun_out/smoke.log; exit 1; }
if [ -n "$PARITY_K" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -k "$PARITY_K" > gpurun_out/parity.log 2>&1; rc=$?; echo "parity rc=$rc"; tail -3 gpurun_out/parity.log
[ $rc -eq 0 ] || exit 1
fi
timeout 900 python scripts/sweep_inproc.py --rounds ${ROUNDS:-4} --steps ${STEPS:-5} $SWEEP_ARGS $SWEEP 2>&1 | tail -20
