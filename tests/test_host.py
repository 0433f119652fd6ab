"""Host-side tests (no GPU): parameters, the C-ABI library surface, partitioning, and
the multi-process share logic over gloo (world_size 2)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def lib():
    from paper_2305_07165_b200 import _build, _lib
    if not os.path.exists(_lib.LIB_PATH):
        _build.build()
    return _lib.load()


def test_product_params_bit_identical_to_reference():
    from paper_2305_07165_b200 import planewave as pp
    g = np.load(os.path.join(GOLD, "params.npz"))
    for i, e in enumerate(g["eps"]):
        assert pp.cutoff_factor(e) == g["D0"][i]
        for k, f in enumerate((2.0, 3.0, 4.0)):
            q = pp.pw_params(e, 1e-3, R=f * pp.cutoff_factor(e), dim=2)
            assert q.n_f == g["nf"][k, i] and q.h == g["h"][k, i]
    assert np.array_equal(pp.pw_params(1e-6, 1e-3, dim=3).weights_1d, g["w30"])
    for c, out in zip(g["cl_cases"], g["cl_out"]):
        assert pp.cutoff_level(c[0], c[1], c[2], "point" if c[3] else "density") == (out[0], out[1])


def test_param_errors():
    from paper_2305_07165_b200 import planewave as pp
    with pytest.raises(ValueError):
        pp.pw_params(0.5, 1e-3)
    with pytest.raises(ValueError):
        pp.pw_params(1e-6, -1.0)
    with pytest.raises(ValueError):
        pp.pw_params(1e-6, 1e-3, dim=4)
    with pytest.raises(ValueError):
        pp.pw_params(1e-6, 1e-3, R=1.0)
    assert pp.clamp_tolerance(1e-20) == 1e-14 and pp.clamp_tolerance(0.5) == 0.099


def header_functions():
    src = open(os.path.join(ROOT, "include", "fgt_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fgt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(lib):
    from paper_2305_07165_b200 import _lib
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
        assert n in _lib.SIGNATURES, f"{n} has no ctypes signature"
    assert lib.fgt_version().decode().endswith("sm_100a")


def test_sm100a_only_cubin(lib):
    """The shipped library carries sm_100a SASS (and no other GPU arch)."""
    import subprocess
    from paper_2305_07165_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_\d+a?", out.stdout))
    assert archs == {"sm_100a"}, archs


def bounds(lib, cost, parts):
    from paper_2305_07165_b200 import _lib
    c = np.ascontiguousarray(cost, dtype=np.float64)
    b = np.zeros(parts + 1, dtype=np.int64)
    _lib.check(lib.fgt_partition_bounds(_lib.ptr(c), c.size, parts, _lib.ptr(b)))
    return b


def test_partition_bounds(lib):
    r = np.random.default_rng(0)
    for n, parts in ((0, 1), (1, 4), (10, 3), (1000, 8), (37, 37), (5, 8)):
        cost = r.exponential(size=n)
        b = bounds(lib, cost, parts)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        if n >= parts and n > 0:
            share = [cost[b[i]:b[i + 1]].sum() for i in range(parts)]
            assert max(share) <= cost.sum() / parts + cost.max() + 1e-12
    with pytest.raises(ValueError):
        bounds(lib, np.array([1.0, -1.0]), 2)


def test_status_codes_map_to_exceptions(lib):
    from paper_2305_07165_b200 import _lib
    with pytest.raises(ValueError):
        _lib.check(lib.fgt_partition_bounds(None, 3, 0, None))
    assert "bad arguments" in lib.fgt_last_error().decode()


def _share_worker(rank, world, port, q):
    """One gloo rank: evaluates its target-leaf share with the oracle; all_reduce sums."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_07165_b200 import _lib
        from oracle import point_fgt as ofgt
        lib = _lib.load()
        r = np.random.default_rng(5)
        y = r.uniform(-0.5, 0.5, (3000, 2))
        x = r.uniform(-0.5, 0.5, (3000, 2))
        qq = r.uniform(-1, 1, 3000)
        a = ofgt.Alg2(y, qq, x, 1e-3, 1e-6, 40)
        t = a.build_tree()
        a.form()
        leaves = a.tleaves
        cost = t.tgt_count[leaves].astype(float)
        b = bounds(lib, cost, world)
        mine = leaves[b[rank]:b[rank + 1]]
        a.gather_eval(mine)
        a.direct(mine)
        u = torch.from_numpy(a.potentials())
        mask = torch.zeros(x.shape[0], dtype=torch.int64)
        for T in mine:
            mask[t.tgt_perm[t.tgt_start[T]:t.tgt_start[T] + t.tgt_count[T]]] += 1
        dist.all_reduce(u)
        dist.all_reduce(mask)
        full = ofgt.fgt_points(y, qq, x, 1e-3, 1e-6, 40)
        q.put((rank, bool(torch.all(mask == 1)),
               float(np.linalg.norm(u.numpy() - full) / np.linalg.norm(full))))
    finally:
        dist.destroy_process_group()


def test_two_rank_shares_gloo():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_share_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, tiled, err in res:
        assert tiled, f"rank {rank}: targets not covered exactly once"
        assert err < 1e-13, err


def _exchange_worker(rank, world, port, q):
    """One gloo rank of the expansion-halo all-to-all (TorchExchange) on CPU tensors: the
    counts matrix is known to every rank (as the replicated lists make it on the GPU), the
    payload encodes (source rank, destination rank, slot)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_07165_b200.point_fgt import TorchExchange
        slot = 3
        C = [[0 if a == b else (a + 2 * b) % 4 for b in range(world)] for a in range(world)]  # C[src][dst]
        send_counts, recv_counts = C[rank], [C[p][rank] for p in range(world)]
        send = torch.cat([torch.tensor([[rank * 100 + dst * 10 + k] * slot for k in range(C[rank][dst])],
                                       dtype=torch.float64).reshape(-1) for dst in range(world)])
        recv = torch.empty(sum(recv_counts) * slot, dtype=torch.float64)
        TorchExchange()(send, recv, send_counts, recv_counts, slot)
        want = torch.cat([torch.tensor([[src * 100 + rank * 10 + k] * slot for k in range(C[src][rank])],
                                       dtype=torch.float64).reshape(-1) for src in range(world)])
        q.put((rank, bool(torch.equal(recv, want))))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_all_to_all_gloo():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert ok, f"rank {rank}: halo blocks out of place"


def _assemble_worker(rank, world, port, q):
    """One gloo rank of the result assembly: the rank holds the potentials of its own
    targets and exact zeros elsewhere; TorchExchange.assemble leaves the whole transform on
    every rank, bit for bit."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_07165_b200.point_fgt import TorchExchange
        full = torch.from_numpy(np.random.default_rng(5).standard_normal(1001))
        owner = torch.from_numpy(np.random.default_rng(6).integers(0, world, 1001))
        mine = torch.where(owner == rank, full, torch.zeros_like(full))
        out = TorchExchange().assemble(mine.clone())
        q.put((rank, bool(torch.equal(out, full))))
    finally:
        dist.destroy_process_group()


def test_result_assembly_gloo():
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    procs = [ctx.Process(target=_assemble_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert ok, f"rank {rank}: assembled potentials differ from the whole transform"
