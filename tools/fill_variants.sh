for l in paper_2012_08208_b200/libtopofilt.so build_variants/lib_fill_co100.so build_variants/lib_fill_co100_minb9.so build_variants/lib_fill_co100_minb10.so; do
  echo $l; TOPOFILT_TRACE=1 TOPOFILT_LIB=$l timeout 300 python bench.py --steps 3 --warmup 2 --applies 1 --no-e2e --no-cpu-baseline 2>&1 >/dev/null | grep trace | tail -2 | grep -o "count [0-9.]*\|fill [0-9.]*" | tr '\n' ' '; echo
done
