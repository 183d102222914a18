# Apply-kernel build variants (build_variants/lib_*.so) on config 5: per-apply microseconds.
for l in paper_2012_08208_b200/libtopofilt.so build_variants/lib_*.so; do
  echo -n "$l "
  TOPOFILT_LIB=$l timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['apply']['sensitivity_us'],1), round(d['apply']['density_us'],1))"
done
