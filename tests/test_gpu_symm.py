"""The symmetric-memory plumbing of the fused compat + all-gather at world size 1 on one GPU
(the only size one GPU can run without ranks waiting on one another): rendezvous, the
device pointer table, the kernel's peer stores and the device barrier, vs glmb_compat."""
import os

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA GPU")]


def test_symmetric_columns_world1():
    import torch
    import torch.distributed as dist
    from paper_2512_06230_b200 import _lib as L
    from paper_2512_06230_b200._lib import Particles
    from paper_2512_06230_b200 import scenes
    from paper_2512_06230_b200.build import build
    build()
    torch.cuda.set_device(0)
    L.glmb_init(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        from paper_2512_06230_b200.symm import SymmetricColumns
        sc = scenes.make_scene(1, steps=1)
        cfg = sc.cfg
        p = Particles.from_arrays([sc.x, sc.y, sc.v, sc.psi, sc.omega, sc.w])
        Z = torch.from_numpy(sc.Z[0]).cuda()
        M = Z.shape[0]
        ldc, ldg = (M + 31) // 32 * 32, (M + 31) // 32
        S = ldc + (ldg + 31) // 32 * 32                  # dist.ShardedStep's packed row
        try:
            cols = SymmetricColumns(p.T, S, ldc, torch.device("cuda", 0))
        except Exception as e:  # noqa: BLE001
            pytest.skip(f"symmetric memory unavailable: {e}")
        C0 = torch.zeros(p.T, ldc, device="cuda")
        G0 = torch.zeros(p.T, ldg, dtype=torch.int32, device="cuda")
        L.glmb_compat(p, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma, None, C0, G0)
        for k in (0, 1):                                 # both copies of the double buffer
            cols.compat(p, Z, cfg.R, cfg.p_d, cfg.kappa, cfg.gamma, None, 0, k)
            cols.barrier(k)
            torch.cuda.synchronize()
            buf = cols.buffer(k)
            np.testing.assert_array_equal(buf.cpu().numpy()[:, :M], C0.cpu().numpy()[:, :M])
            np.testing.assert_array_equal(buf.view(torch.int32)[:, ldc:ldc + ldg].cpu().numpy(), G0.cpu().numpy())
        assert cols.buffer(0).data_ptr() != cols.buffer(1).data_ptr()
    finally:
        dist.destroy_process_group()
