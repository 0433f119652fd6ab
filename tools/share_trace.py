"""FGT_TRACE timeline of one rank's exchange-path begin at a BASELINE config (share planning)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools import configs  # noqa: E402
from paper_2305_07165_b200.point_fgt import fgt_points_exchange_begin  # noqa: E402

cid, P, r = (int(a) for a in sys.argv[1:4])
cfg = configs.CONFIGS[cid]
y, q, x = configs.generate(cid)
dy, dq, dx = (torch.from_numpy(v).cuda() for v in (y, q, x))
args = (cfg["delta"], cfg["eps"], cfg["n_s"], cfg["boundary"])
for _ in range(2):
    run = fgt_points_exchange_begin(dy, dq, dx, *args, share=(r, P))
    recv = torch.zeros(sum(run.recv_counts) * run.slot, dtype=torch.float64, device="cuda")
    run.unpack(recv)
    u, t = run.finish(return_times=True)
    torch.cuda.synchronize()
    print({k: round(t[k], 2) for k in ("tree_ms", "lists_ms", "form_ms", "gather_ms", "eval_ms", "direct_ms", "total_ms")})
    del run
