# Apply G/U sweep on one config (default 4): per-apply microseconds from bench.py (hot, in-step).
CFG=${CFG:-4}
for gu in "2 4" "2 8" "4 4" "4 8" "8 4" "8 8"; do
  set -- $gu
  echo -n "cfg $CFG G=$1 U=$2: "
  TOPOFILT_APPLY_G=$1 TOPOFILT_APPLY_U=$2 timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --applies 20 --no-e2e --no-cpu-baseline --no-build-cell-list 2>/dev/null | \
    python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['apply']['sensitivity_us'],1), round(d['apply']['density_us'],1))"
done
