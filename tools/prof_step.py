"""Two config-2 steps through fgt_points_device (for ncu launch lists / captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.configs import config2  # noqa: E402
from paper_2305_07165_b200 import fgt_points_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
y, q, x = config2(n, n)
dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
for _ in range(2):
    u, t = fgt_points_device(dy, dq, dx, 1e-4, 1e-9, 200, return_times=True)
torch.cuda.synchronize()
print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()})
