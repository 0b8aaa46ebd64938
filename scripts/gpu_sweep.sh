# Sweep env knobs with short benches (device-timed, no e2e/cpu baseline).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo smoke failed; tail gpurun_out/smoke.log; exit 1; }
for v in $SWEEP; do
  echo "== $v"
  env ${v//,/ } timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS 2>gpurun_out/sweep.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"value {d['value']:.1f} TF/s  ms {d['ms_per_step']:.2f}  gemm {r['gemm_ms_per_launch']:.2f} ms  split {r['split_ms_per_step']:.3f} ms  clk {d['clocks']['sm_mhz']} {d['clocks']['reasons']} P {d['clocks'].get('power_w_max')}  par {d['parity_sample_max_err_units_2^-20']:.3f}\")
" || tail -3 gpurun_out/sweep.err
done
