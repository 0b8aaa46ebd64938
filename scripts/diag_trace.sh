# Per-CTA phase timestamps of the GEMM (diagnostics build) for small shapes:
#   bash scripts/diag_trace.sh "256 256 256" "1000 2000 1500" ...
# Rebuilds libla.so with LA_BUILD_DIAGNOSTICS=1 in place (run it last in a
# gpurun call: the box's copy of the repo is scratch).
LA_BUILD_DIAGNOSTICS=1 python paper_1306_6192_b200/_build.py --force > /dev/null || exit 1
for s in "$@"; do
  echo "== $s"
  LA_DIAG_TRACE=1 python scripts/one_shape.py $s 3 2>&1 | tail -9
done
