timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python tools/op_times.py --n 32 --mask 2 --top 10 > gpurun_out/op32f.txt 2>&1
