"""World-size-2 CPU test of the multi-GPU host logic (gloo): track sharding
(ShardPlan), the Z_k / theta_k broadcast and the column-block all-gather of C_k,
with each rank's block computed by the oracle.  The gathered matrix must equal
the single-process C_k exactly (columns are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_id, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2512_06230_b200.dist import ShardPlan, allgather_columns, broadcast_measurements
        from paper_2512_06230_b200.scenes import make_scene
        oracle.set_num_threads(1)
        full = make_scene(cfg_id, steps=1)
        c = full.cfg
        Tk = c.T + c.B
        plan = ShardPlan(Tk, world, c.B)
        surv, births = plan.surv(rank), plan.births(rank)
        cols = list(surv) + [c.T + b for b in births]
        # Z_k, theta_k live on rank 0 and are broadcast
        M = len(full.Z[0])
        Z = torch.from_numpy(full.Z[0].copy()) if rank == 0 else torch.zeros(M, 2)
        th = torch.from_numpy(full.theta[0].copy()) if rank == 0 else torch.zeros(M, dtype=torch.int32)
        broadcast_measurements(Z, th, src=0)
        Z, th = Z.numpy(), th.numpy()
        # this rank's particles: survivors from the generator, births (split evenly) from the oracle
        s = make_scene(cfg_id, rows=surv, steps=1)
        bidx = list(births)
        xs, ys, ws = [s.x], [s.y], [s.w]
        if bidx:
            bo = oracle.birth(full.birth_mean[bidx], full.birth_chol[bidx], full.birth_gid[bidx],
                              c.P, c.seed, 0)
            xs.append(bo[0].astype(np.float32)); ys.append(bo[1].astype(np.float32))
            ws.append(bo[5].astype(np.float32))
        x, y, w = (np.concatenate(a) if len(cols) else np.zeros((0, c.P), np.float32)
                   for a in (xs, ys, ws))
        loc = oracle.compat(x, y, w, Z, c.R, c.p_d, c.kappa, c.gamma)
        ldc = M
        block = torch.zeros(plan.per_rank, ldc, dtype=torch.float64)
        block[:len(cols)] = torch.from_numpy(loc["C_tracks"])
        gathered = torch.zeros(plan.per_rank * world, ldc, dtype=torch.float64)
        allgather_columns(block, gathered)
        # the reweight block per contiguous run of global columns (survivors, then births)
        ln = np.zeros(len(cols))
        for a, b, off in ((0, len(surv), surv.start), (len(surv), len(cols), c.T + births.start)):
            if b > a:
                ln[a:b] = oracle.reweight(x[a:b], y[a:b], w[a:b], Z, c.R, th, col_offset=off)[1]
        lnb = torch.zeros(plan.per_rank, dtype=torch.float64)
        lnb[:len(cols)] = torch.from_numpy(ln)
        lng = torch.zeros(plan.per_rank * world, dtype=torch.float64)
        allgather_columns(lnb, lng)
        if rank == 0:
            rows = plan.global_rows()
            out_q.put((gathered.numpy()[rows], lng.numpy()[rows], cols, plan.per_rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_id,world", [(0, 2), (1, 2), (1, 3)])
def test_sharded_C_equals_single_process(orc, cfg_id, world):
    import oracle
    from paper_2512_06230_b200.scenes import make_scene
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_id, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, ln_g, cols0, per = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    full = make_scene(cfg_id, steps=1)
    c = full.cfg
    bo = oracle.birth(full.birth_mean, full.birth_chol, full.birth_gid, c.P, c.seed, 0)
    x = np.concatenate([full.x, bo[0].astype(np.float32)])
    y = np.concatenate([full.y, bo[1].astype(np.float32)])
    w = np.concatenate([full.w, bo[5].astype(np.float32)])
    ref = orc.compat(x, y, w, full.Z[0], c.R, c.p_d, c.kappa, c.gamma)
    np.testing.assert_array_equal(gathered, ref["C_tracks"])
    _, ln_ref, _ = orc.reweight(x, y, w, full.Z[0], c.R, full.theta[0], 0)
    np.testing.assert_array_equal(ln_g, ln_ref)
    assert cols0[0] == 0 and len(cols0) <= per


def test_shard_plan_covers_columns_once():
    from paper_2512_06230_b200.dist import ShardPlan
    for n, B in ((0, 0), (1, 0), (7, 0), (64, 0), (68, 4), (1040, 16), (4096, 0), (21, 5), (3, 3)):
        for world in (1, 2, 3, 4, 8):
            plan = ShardPlan(n, world, B)
            seen = sorted(c for r in range(world) for c in plan.cols(r))
            assert seen == list(range(n))
            assert all(len(plan.cols(r)) <= plan.per_rank for r in range(world))
            # births split evenly: no rank holds more than ceil(B / W)
            assert all(len(plan.births(r)) <= -(-B // world) for r in range(world))
            rows = plan.global_rows()
            assert len(set(rows.tolist())) == n and (rows < world * plan.per_rank).all()
            for col in range(n):
                r = plan.owner(col)
                assert col in list(plan.cols(r))
                assert rows[col] == r * plan.per_rank + list(plan.cols(r)).index(col)
            if B == 0 or world == 1:      # one contiguous block per rank: gathered = global order
                assert (rows == np.arange(n)).all()
