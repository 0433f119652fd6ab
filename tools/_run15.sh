python - <<'PY'
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2305_07165_b200 import volume as pv
from tools.prof_volume import build
tree, vals, plan, t_tree, t_plan = build()
for i in range(4):
    t0 = time.perf_counter(); u = pv.fgt_box(tree, vals, 1e-4, 1e-10, plan=plan); dt = time.perf_counter() - t0
    print("e2e plan reused ms", round(dt * 1e3, 2))
t0 = time.perf_counter(); leaves, V = pv._stack_values(tree, vals, 16, pinned=True); print("stack ms", round((time.perf_counter() - t0) * 1e3, 2))
PY
python -m pytest tests/test_gpu_volume.py -m gpu -x -q 2>&1 | tail -2
