# ncu --set full of the C3 (u16) cell-channel kernels (one time point, serial)
ncu --set full --clock-control none --import-source on -k "regex:tc_pass|median3_bits|mrf_stream_nz|otsu_kernel" -c 8 -o gpurun_out/full_c3 python tools/profile_stages.py --config C3 --reps 1 > gpurun_out/ncu_c3f.log 2>&1
exit 0
