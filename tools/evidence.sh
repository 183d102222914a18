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
CMDL="python bench.py --steps 1 --warmup 0 --applies 2 --no-e2e --no-cpu-baseline --no-build-cell-list --no-check"
timeout 300 $CMDL > gpurun_out/ev_prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMDL > gpurun_out/ev_ncu_launch.log 2>&1; echo ncu1=$?
CMD="python bench.py --steps 1 --warmup 0 --applies 2 --no-e2e --no-cpu-baseline --no-check"
# the step's lattice fill and two applies, then the cell-list count and fill (bench's build_cell_list leg)
# (step: k_lat_fill_exact, 2 x (k_tpass, k_spmv<1>, k_spmv<0>); the path-stats build's k_lat_fill_exact; then the
# cell-list leg's k_cl_count, k_cl_fill)
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spmv|k_cl_fill|k_cl_count|k_lat_fill_exact|k_tpass" -c 16 -o gpurun_out/ev_prof $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo ncu2=$?
# the report is too large to bring back (gpurun_out <= 64 MiB): export the pages here, drop the report
ncu -i gpurun_out/ev_prof.ncu-rep --page raw --csv > gpurun_out/ev_prof_raw.csv 2>/dev/null
for k in k_spmv k_cl_fill k_cl_count k_lat_fill_exact; do
ncu -i gpurun_out/ev_prof.ncu-rep --page source --csv --print-source cuda,sass -k regex:$k -c 1 > gpurun_out/ev_src_$k.csv 2>/dev/null
done
rm -f gpurun_out/ev_prof.ncu-rep
# instructions per query of the cell-list build kernels: group kernels vs the per-bin kernels (config 5)
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_cl_count|k_cl_fill|k_count|k_fill" --csv --log-file gpurun_out/ev_build_inst_groups.csv python tools/cl_one.py 5 cell_list > /dev/null 2>&1; echo ncu3=$?
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_count|k_fill" --csv --log-file gpurun_out/ev_build_inst_bins.csv python tools/cl_one.py 5 cell_list_bins > /dev/null 2>&1; echo ncu4=$?
TOPOFILT_TRACE=1 BUILD_PATHS=lattice,cell_list python tools/build_paths.py 1 2 3 4 5 > gpurun_out/ev_build_paths.jsonl 2> gpurun_out/ev_build_trace.log; echo paths=$?
python tools/cl_check.py 3 4 5 > gpurun_out/ev_cl_check.jsonl 2>&1; echo clcheck=$?
python tools/apply_mid_probe.py > gpurun_out/ev_apply_mid.jsonl 2>&1; echo mid=$?
timeout 900 python bench.py --gpus 2 --dry-run --steps 3 --warmup 3 > gpurun_out/ev_bench_dry2.json 2> gpurun_out/ev_bench_dry2.err; echo dry2=$?
timeout 900 python bench.py --gpus 4 --dry-run --config 3 --steps 3 --warmup 3 > gpurun_out/ev_bench_dry4_c3.json 2> gpurun_out/ev_bench_dry4_c3.err; echo dry4=$?
timeout 300 python tools/helm_probe.py > gpurun_out/ev_helm_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hz_apply -c 1 -o gpurun_out/ev_hz python tools/helm_probe.py ncu > gpurun_out/ev_ncu_hz.log 2>&1; echo ncu_hz=$?
timeout 300 python tools/matrix_free_probe.py > gpurun_out/ev_mf_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(k_stencil|k_lattice)$" -c 2 -o gpurun_out/ev_mf python tools/matrix_free_probe.py > gpurun_out/ev_ncu_mf.log 2>&1; echo ncu_mf=$?
timeout 600 python tools/shard_probe.py 2 4 8 > gpurun_out/ev_shard_probe.jsonl 2> gpurun_out/ev_shard_probe.err; echo shard=$?
timeout 600 python tools/dense_probe.py > gpurun_out/ev_dense_probe.jsonl 2> gpurun_out/ev_dense_probe.err; echo dense=$?
