# quick iteration on the cell-list build: bitwise check + timing (configs 3 4 5), group-kernel tests,
# optional ncu metrics (NCU_CFG=4|5)
set -x
python tools/cl_check.py ${CFGS:-3 4 5} > gpurun_out/cl_check.jsonl 2>&1; echo clcheck=$?; cat gpurun_out/cl_check.jsonl | cut -c1-420
TOPOFILT_TRACE=1 BUILD_PATHS=cell_list python tools/build_paths.py 4 5 2>&1 | grep -v '^{' | tail -4
timeout 900 python -m pytest tests/test_gpu_cl_groups.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/cl_tests.log 2>&1; echo pytest=$?; tail -3 gpurun_out/cl_tests.log
for c in ${NCU_CFG:-}; do
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"k_cl_count|k_cl_fill|k_cl_groups|k_cl_units|k_radix|k_gather|k_keys|k_bbox|k_tile|k_scan|k_cellstart|k_plan" --csv --log-file gpurun_out/cl_ncu_c$c.csv python tools/cl_one.py $c cell_list > /dev/null 2>&1; echo ncu=$?
done
