timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_n56.csv python tools/profile_pass.py --n 56 --reps 2 --mixed > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/r01_conv2 python tools/profile_pass.py --n 96 --reps 1 > gpurun_out/ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gather_rows|compact_index|segment_mean|pool3" -c 4 -o gpurun_out/r01_hbm python tools/profile_pass.py --n 96 --reps 1 > gpurun_out/ncu_full2.log 2>&1
