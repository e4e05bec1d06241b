"""The multi-GPU step (dist.ShardedStep) at world size 2 with the REAL CUDA kernels: two
processes (gloo, collectives on host-staged copies), both ranks launching their shard's
predict / birth / compat / reweight on cuda:0 -- the kernels of one rank never wait on the
other's, so one GPU runs them safely (B200_PROFILING: no cross-rank device waits on one GPU).
The gathered C_k, gate words, log-normalisers and flags of every step, and each rank's
particles, must be bit-identical to the single-GPU step (Philox keyed by the
global track id, launch shapes that depend on (M, P) only)."""
import os
import socket

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_id, steps, side, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_06230_b200 import _lib as L
        from paper_2512_06230_b200.dist import ShardedStep
        L.glmb_init(0)
        sh = ShardedStep(cfg_id, device="cuda:0", stage_on_host=True, steps=steps)
        stream = torch.cuda.Stream()
        side_s = torch.cuda.Stream() if side else None
        outs = {}
        for k in range(steps):
            M = sh.load_measurements(k, stream=stream)
            sh.step(k, M, stream=stream, side=side_s)
            torch.cuda.synchronize()
            outs[f"C{k}"] = sh.C_all().cpu().numpy()[:, :M]
            outs[f"G{k}"] = sh.gate_all().cpu().numpy()[:, :(M + 31) // 32]
            outs[f"ln{k}"] = sh.log_norm_all().cpu().numpy()
            outs[f"fl{k}"] = sh.flags_all().cpu().numpy()
        st = sh.st
        outs["particles"] = torch.cat([st.particles.data[:5], st.weights()[None]]).cpu().numpy()[:, :st.T_local]
        outs["col_of_row"] = st.col_of_row
        outs["rows"] = sh.plan.global_rows()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **outs)
    finally:
        dist.destroy_process_group()


def _single_gpu(cfg_id, steps):
    """The W = 1 reference: the same four stages through GlmbStep on the whole scene."""
    import torch
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200.scenes import make_scene
    from paper_2512_06230_b200.step import GlmbStep
    from paper_2512_06230_b200.build import build
    build()
    torch.cuda.set_device(0)
    L.glmb_init(0)
    s = make_scene(cfg_id, steps=steps)
    st = GlmbStep(s)
    ref = {}
    for k in range(steps):
        M = len(s.Z[k % len(s.Z)])
        st.predict(k)
        st.birth(k)
        st.compat(k)
        st.reweight(k)
        torch.cuda.synchronize()
        ref[f"C{k}"] = st.out.C_tracks.cpu().numpy()[:, :M]
        ref[f"G{k}"] = st.out.gate.cpu().numpy()[:, :(M + 31) // 32]
        ref[f"ln{k}"] = st.out.log_norm.cpu().numpy()
        ref[f"fl{k}"] = st.out.flags.cpu().numpy()
    ref["particles"] = st.particles.data.cpu().numpy()
    return ref


@pytest.mark.parametrize("cfg_id,steps,side", [(1, 3, False), (1, 3, True), (3, 2, True)])
def test_sharded_step_world2_bit_identical(cfg_id, steps, side, tmp_path):
    import torch.multiprocessing as mp
    ref = _single_gpu(cfg_id, steps)
    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_id, steps, side, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    rows = ranks[0]["rows"]
    Tk = len(rows)
    for k in range(steps):
        for key in ("C", "G", "ln", "fl"):
            for r in range(world):        # every rank holds the whole gathered C_k
                got = ranks[r][f"{key}{k}"][rows]
                np.testing.assert_array_equal(got.view(np.uint32), ref[f"{key}{k}"][:Tk].view(np.uint32),
                                              err_msg=f"{key} step {k} rank {r}")
    for r in range(world):
        cr = ranks[r]["col_of_row"]
        np.testing.assert_array_equal(ranks[r]["particles"].view(np.uint32),
                                      ref["particles"][:, cr].view(np.uint32))
    if cfg_id in (1, 3):   # births split over both ranks
        assert all((r["col_of_row"] >= Tk - {1: 4, 3: 16}[cfg_id]).sum() > 0 for r in ranks)


def _worker_host(rank, world, port, cfg_id, steps, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_06230_b200 import _lib as L
        from paper_2512_06230_b200.dist import ShardedStep
        L.glmb_init(0)
        sh = ShardedStep(cfg_id, device="cuda:0", stage_on_host=True, steps=steps)
        stream, side = torch.cuda.Stream(), torch.cuda.Stream()
        outs = {}
        for k in range(steps):
            zi = k % len(sh.scene.Z)
            Zh = torch.from_numpy(sh.scene.Z[zi]).pin_memory()
            th = torch.from_numpy(sh.scene.theta[zi]).pin_memory()
            nnz, h2d, d2h = sh.step_host_csr(k, Zh, th, stream=stream, side=side, first_copy=3)
            if rank == 0:
                b = sh._csr
                M = Zh.shape[0]
                outs[f"rp{k}"] = b["rp_h"][:M + 1].numpy().copy()
                outs[f"col{k}"] = b["col_h"][:nnz].numpy().copy()
                outs[f"val{k}"] = b["val_h"][:nnz].numpy().copy()
                outs[f"ln{k}"] = b["ln_h"].numpy().reshape(world, 2, -1)[:, 0].reshape(-1).copy()
                assert h2d == M * 12 and d2h > 0
            else:
                assert (nnz, h2d, d2h) == (0, 0, 0)
        outs["rows"] = sh.plan.global_rows()
        if rank == 0:
            np.savez(os.path.join(out_dir, "host.npz"), **outs)
    finally:
        dist.destroy_process_group()


def test_sharded_step_host_csr_world2(tmp_path):
    """The N > 1 end-to-end entry point (ShardedStep.step_host_csr, what bench.py's e2e leg
    times at N > 1): rank 0's CSR of the gathered C_k (column = gathered row; a speculative first
    copy of 3 entries, the rest in the second copy) and the gathered log-normalisers equal the
    single-GPU C_k's gated entries and log_norm, mapped through ShardPlan.row_of."""
    import torch.multiprocessing as mp
    cfg_id, steps, world = 1, 2, 2
    ref = _single_gpu(cfg_id, steps)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker_host, args=(r, world, port, cfg_id, steps, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    got = np.load(tmp_path / "host.npz")
    rows = got["rows"]
    col_of_row = np.full(rows.max() + 1, -1)
    col_of_row[rows] = np.arange(len(rows))
    for k in range(steps):
        C = ref[f"C{k}"]
        bits = ((ref[f"G{k}"].view(np.uint32)[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(
            C.shape[0], -1)[:, :C.shape[1]].astype(bool)
        rp = got[f"rp{k}"]
        M = len(rp) - 1
        assert rp[M] == bits.sum() > 3
        for i in range(M):
            cols = col_of_row[got[f"col{k}"][rp[i]:rp[i + 1]]]
            np.testing.assert_array_equal(np.sort(cols), np.nonzero(bits[:, i])[0])
            order = np.argsort(cols)
            np.testing.assert_array_equal(got[f"val{k}"][rp[i]:rp[i + 1]][order], C[np.sort(cols), i])
        np.testing.assert_array_equal(got[f"ln{k}"][rows].view(np.uint32), ref[f"ln{k}"].view(np.uint32))
