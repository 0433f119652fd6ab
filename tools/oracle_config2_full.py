"""One full CPU-oracle transform of config 2 (N = M = 10^6), timed per phase, with the
host's CPU model and core count.  Prints one JSON line (profiles/r02_oracle_config2_full.json)."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import point_fgt as op  # noqa: E402
from tools.configs import config2  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


y, q, x = config2()
tm = {}
t0 = time.perf_counter()
u = op.fgt_points(y, q, x, 1e-4, 1e-9, 200, timings=tm)
sec = time.perf_counter() - t0
sub = np.sort(np.random.default_rng(123).choice(x.shape[0], 2000, replace=False))
ex = op.direct_oracle(y, q, x[sub], 1e-4)
err = float(np.linalg.norm(u[sub] - ex) / np.linalg.norm(ex))
print(json.dumps({"what": "oracle Alg 2 (numpy restatement of the reference), config 2, full transform",
                  "seconds": sec, "points_per_s": 2e6 / sec, "phases_s": tm,
                  "rel_l2_vs_direct_2000": err, "cpu": cpu_model(), "nproc": os.cpu_count(),
                  "threads": "1 process (numpy einsum single-threaded; BLAS default)"}))
