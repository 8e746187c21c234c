"""World-size-2 CPU tests (gloo) of the multi-GPU host logic.

On the GPU box every rank runs the library and one ncclAllReduce of the
unnormalised [g; ℓ] per F evaluation.  Here the same row
sharding (paper_2503_19925_b200.dist) drives the fp64 oracle on each rank's
row block, gloo plays the allreduce, and the result must equal the
single-process oracle: F is a sum over rows (Eq. operator),
so the sharded sum is the full operator up to summation order, and the
replicated projection keeps every rank's iterate bit-identical.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import configs as G


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _body(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _allreduce(vec):
    t = torch.tensor(vec, dtype=torch.float64)
    dist.all_reduce(t)
    return t.numpy()


def _body(rank, world):
    import oracle
    from oracle import workloads as OW
    from paper_2503_19925_b200 import dist as D

    out = {}
    oracle.set_threads(2)
    # strong sharding of C1 (fp64): the local problem keeps n_norm = n_global
    cfg = G.C1
    gcfg, row0, n_local, scaling = D.shard(cfg, rank, world, strong=True)
    assert scaling == "strong" and gcfg.n == cfg.n
    rows = np.arange(row0, row0 + n_local)
    wl = OW.build(cfg, rows=rows)
    wf = OW.build(cfg)
    pl, pf = wl["problem"], wf["problem"]
    assert pl.n_norm == cfg.n
    x = 0.7 * wf["x_star"]
    gl, ll = pl.F(x)
    red = _allreduce(np.concatenate([gl, [ll]]))
    gf, lf = pf.F(x)
    out["F_err"] = float(np.linalg.norm(red[:-1] - gf) / np.linalg.norm(gf))
    out["loss_err"] = abs(red[-1] - lf) / abs(lf)
    out["rows"] = (row0, row0 + n_local)

    # EXACT with the allreduce inside each F (Eq. extragrad-method), every rank
    # projecting the same reduced bits
    gam, _ = OW.step_size(pf, wf["s"], wf["mu"], cfg.I_bar)
    xd = pf.project(np.zeros(cfg.d))
    for _ in range(20):
        g1 = _allreduce(pl.F(xd)[0])
        xh = pl.project(xd - gam * g1)
        g2 = _allreduce(pl.F(xh)[0])
        xd = pl.project(xd - gam * g2)
    xs, _, bad = pf.solve(20, gam)
    assert bad == 0
    out["solve_err"] = float(np.linalg.norm(xd - xs) / np.linalg.norm(xs))
    gathered = [None] * world
    dist.all_gather_object(gathered, xd.tobytes())
    out["replicas_identical"] = all(b == gathered[0] for b in gathered)

    # weak sharding: rank r holds rows [r n, (r+1) n) of the n*world problem
    wcfg, wr0, wn, sc = D.shard(G.scaled(G.C1F, 500), rank, world, strong=False)
    out["weak"] = (wcfg.n, wr0, wn, sc)

    # timing / byte reductions and the id exchange
    out["max"] = D.max_over_ranks(1.0 + rank, world, device="cpu")
    out["sum"] = D.sum_over_ranks(10.0 * (rank + 1), world, device="cpu")
    out["id"] = D.exchange_id(lambda: b"\x07" * 128, rank, world)
    # K9's window-handle exchange: 64 bytes per rank, concatenated in rank order
    out["handles"] = D.gather_handles(bytes([rank + 1]) * 64, rank, world)
    return out


def test_row_block_partition():
    from paper_2503_19925_b200 import dist as D
    for n in (0, 1, 7, 2000, 8_000_000):
        for world in (1, 2, 3, 8):
            blocks = [D.row_block(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.row_block(10, 2, 2)


def test_gloo_world2_sharded_oracle_matches_full():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    assert res[0]["rows"] == (0, 1000) and res[1]["rows"] == (1000, 2000)
    for r in range(world):
        o = res[r]
        assert o["F_err"] <= 1e-13, o["F_err"]
        assert o["loss_err"] <= 1e-13
        assert o["solve_err"] <= 1e-12, o["solve_err"]
        assert o["replicas_identical"]
        assert o["weak"] == (1000, 500 * r, 500, "weak")
        assert o["max"] == 2.0 and o["sum"] == 30.0
        assert o["id"] == b"\x07" * 128
        assert o["handles"] == b"\x01" * 64 + b"\x02" * 64


def _fd_worker(rank, world, port, name, path, q):
    """poly_share_fd, the same-node hand-off poly_nvls_open uses for the
    multicast object's descriptor: rank 0 shares an open file, the other ranks
    read the shared content through the descriptor they receive."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2503_19925_b200 as P
        fd = os.open(path, os.O_RDONLY) if rank == 0 else -1
        got = P.poly_share_fd(rank, world, name, fd, timeout_s=30.0)
        # the ranks' descriptors share one open file description (SCM_RIGHTS), hence one file
        # offset: a positioned read, not lseek + read, which races between ranks
        data = os.pread(got, 64, 0)
        if rank != 0:
            os.close(got)
        dist.barrier()
        q.put((rank, data.decode()))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_share_fd_world(tmp_path, world):
    path = tmp_path / "payload.txt"
    path.write_text("multicast-object")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    name = f"poly-test-{os.getpid()}-{world}"
    ps = [ctx.Process(target=_fd_worker, args=(r, world, PORTS[world], name,
                                               str(path), q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    assert all(v == "multicast-object" for v in res.values()), res


PORTS = {2: _free_port(), 3: _free_port()}


def test_share_fd_timeout():
    """A rank whose peer never shows up returns POLY_ENCCL after the timeout
    instead of blocking (the 'abort instead of hang' rule)."""
    import paper_2503_19925_b200 as P
    with pytest.raises(P.PolyError) as ei:
        P.poly_share_fd(1, 2, f"poly-nobody-{os.getpid()}", -1, timeout_s=0.3)
    assert ei.value.code == P.POLY_ENCCL
