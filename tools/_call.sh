timeout 900 python -m pytest tests -m gpu -x -q -k "model or pool" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python tools/op_times.py --n 64 --mask 1 --top 60 > gpurun_out/op64r.txt 2>&1
