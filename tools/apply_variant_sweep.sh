# Apply-kernel variants (build_variants/lib_*.so, optional env overrides) on config 5:
# per-apply microseconds from bench.py (sensitivity, density), two passes to see the noise.
for pass in $(seq ${PASSES:-2}); do
for spec in ${SPECS:-paper_2012_08208_b200/libtopofilt.so build_variants/lib_*.so} $EXTRA_SPECS; do
  set -- ${spec//,/ }
  l=$1; shift
  echo -n "$pass $(basename $l) $* "
  env TOPOFILT_LIB=$l "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-build-cell-list 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['apply']['sensitivity_us'],1), round(d['apply']['density_us'],1), round(d['value'],1))"
done
done
