"""Two config-2 transforms of one strong-scaling share (rank r of P) for launch lists.

    python tools/share_step.py RANK SIZE
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools import configs  # noqa: E402
from paper_2305_07165_b200 import fgt_points_device  # noqa: E402

r, P = int(sys.argv[1]), int(sys.argv[2])
y, q, x = configs.config2(1_000_000, 1_000_000)
dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
for _ in range(2):
    u, t = fgt_points_device(dy, dq, dx, 1e-4, 1e-9, 200, return_times=True, share=(r, P))
torch.cuda.synchronize()
print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()})
