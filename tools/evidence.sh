# Round evidence in one gpurun call: tests, bench (default args), clocks, ncu launch list and
# full captures of the dominant kernels (each ncu only after the same command exited 0).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev_gpu.csv
timeout 300 python __graft_entry__.py smoke > gpurun_out/ev_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev_pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ev_pytest_gpu.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/ev_clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo bench=$?
kill $SMI
timeout 900 python bench.py --impl reference > gpurun_out/ev_bench_ref.json 2> gpurun_out/ev_bench_ref.err; echo ref=$?
timeout 600 python tools/bench_configs.py > gpurun_out/ev_configs.jsonl 2> gpurun_out/ev_configs.err; echo cfg=$?
# launch list of one step (build + 2 applies), without the build_cell_list leg
CMDL="python bench.py --steps 1 --warmup 0 --applies 2 --no-e2e --no-cpu-baseline --no-build-cell-list"
timeout 300 $CMDL > gpurun_out/ev_prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMDL > gpurun_out/ev_ncu_launch.log 2>&1; echo ncu1=$?
CMD="python bench.py --steps 1 --warmup 0 --applies 2 --no-e2e --no-cpu-baseline"
# the step's lattice fill and two applies, then the cell-list count and fill (bench's build_cell_list leg)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_fill|k_count|k_lat_fill_exact" -c 8 -o gpurun_out/ev_prof $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo ncu2=$?
timeout 300 python tools/helm_probe.py > gpurun_out/ev_helm_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hz_apply -c 1 -o gpurun_out/ev_hz python tools/helm_probe.py ncu > gpurun_out/ev_ncu_hz.log 2>&1; echo ncu_hz=$?
timeout 300 python tools/matrix_free_probe.py > gpurun_out/ev_mf_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(k_stencil|k_lattice)$" -c 2 -o gpurun_out/ev_mf python tools/matrix_free_probe.py > gpurun_out/ev_ncu_mf.log 2>&1; echo ncu_mf=$?
timeout 600 python tools/shard_probe.py 2 4 8 > gpurun_out/ev_shard_probe.jsonl 2> gpurun_out/ev_shard_probe.err; echo shard=$?
