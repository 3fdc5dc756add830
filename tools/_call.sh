timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 2 -c 1 -o gpurun_out/r01_conv2_halo python tools/profile_pass.py --n 96 --reps 1 > gpurun_out/ncu_full1.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
