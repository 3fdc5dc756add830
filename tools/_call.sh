timeout 600 python -m pytest tests -m gpu -x -q -k "gather or compact or model" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
python - > gpurun_out/compact_t.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import bench
from paper_2310_18481_b200.executor import build_tbn_model
m = build_tbn_model(max_req=96, n_slots=192)
print(bench.compaction_roofline(m, 6546.9, 96))
PY
