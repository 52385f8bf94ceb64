# ncu L2 reduction traffic of the product backward vs the K13 port.
# Plain run first (must exit 0), then the metric capture on the same command.
set -e
python tools/atomics_probe.py > gpurun_out/atom_plain.log 2>&1
M=gpu__time_duration.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_atom.sum,lts__t_sectors_op_atom.sum,sm__sass_inst_executed_op_global_red.sum,sm__sass_inst_executed_op_global_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_red.sum.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
ncu --metrics $M --clock-control none -k regex:"k_render_bwd|k_naive_render_bwd|naive" --csv \
    --log-file gpurun_out/atomics_r02.csv python tools/atomics_probe.py > gpurun_out/atom_ncu.log 2>&1
echo atomics done
