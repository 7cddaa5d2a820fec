# Round-end profile set (run under gpurun): per-stage CUDA-event times, the ncu
# launch list of one C2 time point (durations + DRAM bytes), the bench's own
# launch list, and one `ncu --set full` capture of the top kernels.
set -x
python tools/profile_stages.py --reps 2 > gpurun_out/stages.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_stages.py --reps 1 > gpurun_out/ncu_l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_b.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tc_pass|edt_pass_zr|median3_bits|mrf_decide_walk|edt_y_build|edt_pass_x_seg4|ccl_run_union|tab_voxels_w" -c 12 -o gpurun_out/full_final python tools/profile_stages.py --reps 1 > gpurun_out/ncu_f.log 2>&1
ls -la gpurun_out
