# one gpurun call: smoke, GPU parity tests, bench, ncu launch list (same bench command)
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
CMD="python bench.py --steps 1 --warmup 0 --applies 2 --no-e2e --no-cpu-baseline"
if [ "${NCU:-1}" = "1" ]; then
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
fi
if [ -n "${NCU_FULL:-}" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -c ${NCU_COUNT:-4} -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
fi
