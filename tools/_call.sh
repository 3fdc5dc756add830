timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python tools/policy_bench.py > gpurun_out/policy_bench.txt 2>&1
