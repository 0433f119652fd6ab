"""Two transforms of a BASELINE point config (launch lists / traces): python tools/cfg_step.py 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.run_config import CONFIGS, generate  # noqa: E402
from paper_2305_07165_b200 import fgt_points_device  # noqa: E402

c = int(sys.argv[1])
cfg = CONFIGS[c]
y, q, x = generate(c, cfg["N"])
dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
for _ in range(2):
    u, t = fgt_points_device(dy, dq, dx, cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"], return_times=True)
torch.cuda.synchronize()
print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()})
