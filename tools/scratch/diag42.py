import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
from paper_2305_07165_b200 import volume as pv
from oracle import volume as ov
d, k, delta, eps = 2, 8, 4e-3, 1e-12
C = np.array([[0.1, 0.02], [-0.15, -0.2]])
W, A = [1e-2, 1e-2], [1.0, 1.0]
dens = lambda p: sum(np.exp(-np.sum((p - c) ** 2, axis=-1) / w ** 2) for c, w in zip(C, W))
tree, vals, _ = pv.build_density_tree(dens, d, k, eps)
u, state = pv.fgt_box(tree, vals, delta, eps, retain=True)
basis = pv.LegendreBasis(k)
leaves = sorted(u)
# node accuracy
nerr = []; 
for b in leaves:
    ex = ov.gaussian_box_convolution(pv.leaf_grid(tree, b, basis).reshape(-1, d), delta, C, W, A).reshape(k, k)
    nerr.append(np.max(np.abs(u[b] - ex)))
print("max node error", max(nerr), "scale", max(np.abs(v).max() for v in u.values()))
te = pv.tail_errors(np.stack([u[b] for b in leaves]), d, k)
# interpolation error per leaf at a 12x12 uniform grid inside
ie = []
t = (np.arange(12) + 0.5) / 12 - 0.5
for b in leaves:
    c = tree.centers(b); s = tree.side(tree.level[b])
    X = np.stack(np.meshgrid(c[0] + s * t, c[1] + s * t, indexing="ij"), -1).reshape(-1, 2)
    ex = ov.gaussian_box_convolution(X, delta, C, W, A)
    ie.append(np.max(np.abs(pv.interp_at(tree, u, X) - ex)))
ie = np.array(ie); lv = tree.level[leaves]
order = np.argsort(-ie)[:15]
for i in order:
    print("leaf", leaves[i], "level", lv[i], "center", tree.centers(leaves[i]), "interp err", ie[i], "tail", te[i])
print("leaves with tail > eps:", int((te > eps).sum()), "leaves with interp err > 1e-11:", int((ie > 1e-11).sum()))
for l in range(lv.max()+1):
    m = lv == l
    if m.any(): print("level", l, "n", m.sum(), "max ie", ie[m].max(), "max tail", te[m].max())
