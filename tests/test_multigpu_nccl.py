"""N>1 path on the GPU (-m gpu): min(#GPUs, 2) NCCL ranks, one per GPU, each running sks_sum over its slice range
[r P / G, (r+1) P / G) through the C-ABI, combined by the one all-reduce of parallel.distributed_sliced_sum (Alg. 1's
average).  Rank 0's result is compared with oracle (b).  Skips when fewer than 2 GPUs
are visible (the gloo twin, tests/test_multiproc_gloo.py, covers the host logic on CPU)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from paper_2401_08260_b200 import inputs as I  # noqa: E402

CASES = [("cfg2", dict(N=20000, M=2000, P=32), 1e-5), ("paper_gauss", dict(N=3000, M=800, P=32), 1e-4),
         ("paper_laplace", dict(N=3000, M=800, P=32), 1e-4)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200.parallel import distributed_sliced_sum
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        for name, size, _ in CASES:
            cfg = I.scaled(I.CONFIGS[name], **size)
            x, y, w = (torch.from_numpy(a).cuda() for a in (I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)))
            param = I.kernel_param(cfg) if cfg.kind != "negdist" else 1.0
            s = distributed_sliced_sum(lambda p0, p1: S.sks_sum(x, y, w, cfg.kind, param, cfg.P, cfg.dir_seed, p0, p1,
                                                                cfg.matern_p), cfg.P)
            if rank == 0:
                np.save(os.path.join(out_dir, f"{name}.npy"), s.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_nccl_ranks_match_oracle(tmp_path):
    import torch.multiprocessing as mp
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip(f"{ngpu} GPU visible: the NCCL path needs 2 (host logic: tests/test_multiproc_gloo.py)")
    from paper_2401_08260_b200 import build
    build.build()
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for name, size, tol in CASES:
        cfg = I.scaled(I.CONFIGS[name], **size)
        x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
        param = I.kernel_param(cfg) if cfg.kind != "negdist" else 0.0
        tgt = I.target_subset(cfg.M, 200)
        ref = O.sliced_sum(cfg.kind, param, x, y, w, cfg.P, cfg.dir_seed, targets=tgt, matern_p=cfg.matern_p)
        got = np.load(tmp_path / f"{name}.npy")[tgt].astype(np.float64)
        assert np.max(np.abs(got - ref)) / np.abs(w.astype(np.float64)).sum() <= tol, name
