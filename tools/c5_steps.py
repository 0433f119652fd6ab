import sys, time, json
sys.path.insert(0, '.')
import torch
from tools.run_config import generate, CONFIGS
from paper_2305_07165_b200 import fgt_points_device
cfg = CONFIGS[5]
y, q, x = generate(5, cfg["N"])
dy, dq, dx = (torch.from_numpy(a).cuda() for a in (y, q, x))
del y, q, x
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    u, t = fgt_points_device(dy, dq, dx, cfg["delta"], cfg["eps"], cfg["n_s"], return_times=True)
    torch.cuda.synchronize()
    print(i, {k: round(t[k], 1) for k in ("total_ms", "tree_ms", "form_ms", "k_form_ms", "gather_ms", "eval_ms", "direct_ms")},
          "mem GB", round(torch.cuda.memory_allocated() / 1e9, 1), flush=True)
