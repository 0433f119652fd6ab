"""Config 4 (volume FGT, d=3, k=16, delta=1e-4, eps=1e-10): build tree + plan on the host,
then time fgt_box_device steps (for profiling and the bench's volume leg)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def config4_density():
    r = np.random.default_rng(0)
    c = r.uniform(-0.3, 0.3, (5, 3))
    a = r.uniform(0.5, 1.5, 5)
    w = np.geomspace(0.01, 0.1, 5)
    return lambda p: sum(ai * np.exp(-np.sum((p - ci) ** 2, axis=-1) / wi ** 2)
                         for ci, ai, wi in zip(c, a, w))


def config4_density_torch():
    """The same density as a torch function (GPU evaluation in build_density_tree)."""
    import torch
    r = np.random.default_rng(0)
    c = torch.from_numpy(r.uniform(-0.3, 0.3, (5, 3)))
    a = r.uniform(0.5, 1.5, 5)
    w = np.geomspace(0.01, 0.1, 5)

    def f(p):
        cc = c.to(p.device)
        return sum(float(ai) * torch.exp(-torch.sum((p - cc[i]) ** 2, dim=-1) / float(wi) ** 2)
                   for i, (ai, wi) in enumerate(zip(a, w)))
    return f


def build(k=16, eps_tree=1e-10, delta=1e-4, eps=1e-10):
    from paper_2305_07165_b200 import volume as pv
    t0 = time.perf_counter()
    tree, vals, _ = pv.build_density_tree(config4_density(), 3, k, eps_tree)
    t1 = time.perf_counter()
    plan = pv.BoxPlan(tree, delta, eps, k, False)
    t2 = time.perf_counter()
    return tree, vals, plan, t1 - t0, t2 - t1


if __name__ == "__main__":
    import torch
    from paper_2305_07165_b200 import volume as pv
    tree, vals, plan, t_tree, t_plan = build()
    leaves, V = pv._stack_values(tree, vals, 16)
    print(f"boxes {tree.n_boxes} leaves {len(leaves)} grid points {V.size} n_pw {plan.n_pw} "
          f"n_f {plan.n_f} l_c {plan.l_c} d_pairs {plan.d_tgt.size} gather {plan.n_gather_pairs} "
          f"tree {t_tree:.2f}s plan {t_plan:.2f}s")
    dv = torch.from_numpy(V).cuda()
    for _ in range(3):
        u, t = pv.fgt_box_device(plan, dv, return_times=True)
    torch.cuda.synchronize()
    print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items() if v})
