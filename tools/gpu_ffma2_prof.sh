# ncu instruction counts / issue / duration of the render kernels for two library builds
for L in ${LIBS:-libgsr_noffma2.so libgsr.so}; do
  GSR_LIB=$L ncu --clock-control none -k regex:"k_render_(fwd|bwd)" -s 4 -c 4 --csv \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum \
    python tools/stage_probe.py --views 1 --chunk 1 --reps 3 > gpurun_out/ffma2_$L.csv 2>&1
done
