# new: device Alg 3 pieces, Alg 5 from retained psi
python -m pytest tests/test_gpu_output_tree.py tests/test_gpu_volume.py -q -x -s > gpurun_out/r02y_pytest.log 2>&1; tail -25 gpurun_out/r02y_pytest.log
python - <<'PY'
import time, torch, numpy as np
from paper_2305_07165_b200 import volume as pv
from tools.prof_volume import config4_density_torch
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    tree, vals, _ = pv.build_density_tree(config4_density_torch(), 3, 16, 1e-10, device="cuda")
    torch.cuda.synchronize(); print("config-4 device density tree", round(time.perf_counter()-t,4), "s", tree.n_boxes)
PY
