"""Row-cluster sharding on CPU (world_size 2, gloo): the library's shard plan driven through a real
two-process exchange, with the oracle's dense operators standing in for the GPU kernels.

SURVEY.md §8(e) / DESIGN.md §7: rank r owns tree node r at level log2(G) (a contiguous internal-order
row range); the hot path exchanges padded vector segments (maxc per rank) by allgather:
    flux:  allgather T -> y = (L^-1) rows (w = eps T^4) -> allgather y -> z = (U^-1) rows ->
           allgather z -> q rows = sigma (eps/A)(F z - eta g)
The plan (ranges, maxc, block ownership) comes from the C library on a host-only context
(device = -1, no CUDA); the arithmetic is the oracle's (TEST INFRASTRUCTURE), so this checks the
partition and the exchange schedule, not the kernels (tests/test_gpu_shard.py does those on a GPU).
"""
import os
import socket

import numpy as np
import pytest

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import scipy.linalg as sla
    import paper_2305_06891_b200 as hm
    from oracle import viewfactor as vf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.make_config(2, geometry=synth.icosphere(3))
        f = cfg.facets
        n = f.n
        ctx = hm.hm_init(-1, rank, world)                       # host-only: trees + plan
        g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=cfg.n_min, eta=cfg.eta)
        perm = hm.hm_export_perm(g)
        beg, end, maxc, owner = hm.hm_shard_plan(g, world)
        b0, e0 = hm.hm_local_range(g, rank, world)
        assert (b0, e0) == (beg[rank], end[rank])
        # dense oracle operators in internal order
        Fd, C, _ = vf.dense_operators(f, cfg.emissivity)
        Fi = Fd[np.ix_(perm, perm)]
        Ci = C[np.ix_(perm, perm)]
        P, Lf, Uf = sla.lu(Ci)                                    # Ci = P L U
        Linv = np.linalg.solve(Lf, P.T)                           # L^-1 P^T
        Uinv = np.linalg.inv(Uf)
        eps_i = cfg.emissivity[perm]
        A_i = f.area[perm]
        g_i = Fi @ (Uinv @ (Linv @ eps_i))                        # g = F C^-1 eps
        T_i = cfg.T[perm, 0]
        rows = np.arange(b0, e0)

        def allgather(local):
            seg = torch.zeros(maxc, dtype=torch.float64)
            seg[: len(local)] = torch.from_numpy(np.asarray(local))
            parts = [torch.zeros(maxc, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, seg)
            full = np.empty(n)
            for q in range(world):
                full[beg[q]:end[q]] = parts[q].numpy()[: end[q] - beg[q]]
            return full

        T_full = allgather(T_i[rows])                             # exchange 1
        w = eps_i * T_full ** 4
        y_loc = Linv[rows] @ w
        y = allgather(y_loc)                                      # exchange 2
        z_loc = Uinv[rows] @ y
        z = allgather(z_loc)                                      # exchange 3
        eta = T_i[rows] ** 4
        q_loc = vf.SIGMA_SB * (eps_i[rows] / A_i[rows]) * (Fi[rows] @ z - eta * g_i[rows])
        q_all = allgather(q_loc)
        if rank == 0:
            q_ext = np.empty(n)
            q_ext[perm] = q_all
            qo = vf.flux_from_dense(Fd, C, f.area, cfg.emissivity, cfg.T[:, 0])[:, 0]
            out.put(dict(err=float(np.linalg.norm(q_ext - qo) / np.linalg.norm(qo)),
                         beg=beg.tolist(), end=end.tolist(), maxc=int(maxc), n=n,
                         owner_min=int(owner.min()), nblk=len(owner)))
    finally:
        dist.destroy_process_group()


def test_shard_plan_and_exchange_schedule_world2():
    import torch.multiprocessing as mp
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = res["n"]
    assert res["beg"][0] == 0 and res["end"][-1] == n and res["beg"][1] == res["end"][0]   # ranges tile [0, n)
    assert res["maxc"] >= max(e - b for b, e in zip(res["beg"], res["end"])) and res["maxc"] % 2 == 0
    assert res["owner_min"] >= 0            # no block straddles the two ranks (admissible blocks start deeper)
    assert res["err"] <= 1e-12


def test_shard_plan_ranges_world_1_to_8():
    import paper_2305_06891_b200 as hm
    ctx = hm.hm_init(-1)
    f = synth.icosphere(4)
    g = hm.hm_build_geometry(ctx, f.centroid, f.normal, f.area, f.aabb, n_min=64)
    nb = hm.hm_export_partition(g).shape[0]
    for world in (1, 2, 4, 8):
        b, e, maxc, owner = hm.hm_shard_plan(g, world)
        assert b[0] == 0 and e[-1] == f.n and (b[1:] == e[:-1]).all()
        assert (e - b).max() <= maxc and maxc % 2 == 0
        # balanced median splits: n / G each (n = 5120 is a power-of-two multiple)
        assert ((e - b) == f.n // world).all()
        assert owner.shape == (nb,) and (owner >= 0).all()
    with pytest.raises(hm.HMError):
        hm.hm_shard_plan(g, 3)                 # world must be a power of two
    with pytest.raises(hm.HMError):
        hm.hm_assemble_aca(ctx, g)             # host-only context: no compute
