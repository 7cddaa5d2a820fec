# ncu --set full (with source) of the C2 top kernels, one serial time point
ncu --set full --clock-control none --import-source on -k "regex:tc_pass|median3_bits|mrf_stream_v4|edt_pass_zr|edt_y_build|ccl_run_union|tab_voxels_w" -c 10 -o gpurun_out/full_c2 python tools/profile_stages.py --reps 1 > gpurun_out/ncu_c2f.log 2>&1
exit 0
