python tools/op_times.py --n 32 --top 200 > gpurun_out/op32g.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "pool or model" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
