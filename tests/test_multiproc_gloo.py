"""N>1 path on CPU (-m "not gpu"): world-size-2 gloo process group running the slice-parallel driver
(paper_2401_08260_b200.parallel) with the oracle as the compute function.  Checks that the partitioned
partial sums, combined by one all-reduce, reproduce the single-process sliced estimator (Alg. 1)
for every kernel, and that the slice ranges tile [0, P)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2401_08260_b200 import inputs as I
from paper_2401_08260_b200.parallel import distributed_sliced_sum, slice_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [("paper_negdist", 0.0), ("paper_gauss", 1.0), ("paper_laplace", 2.0), ("paper_matern", 1.0)]


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for name, param in CASES:
            cfg = I.scaled(I.CONFIGS[name], N=300, M=40, P=13)
            x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)

            def compute(p0, p1):
                part = O.sliced_sum(cfg.kind, param, x, y, w, cfg.P, cfg.dir_seed, p0=p0, p1=p1,
                                    matern_p=cfg.matern_p)
                return torch.from_numpy(part)

            s = distributed_sliced_sum(compute, cfg.P)
            if rank == 0:
                np.save(os.path.join(out_dir, f"{name}.npy"), s.numpy())
    finally:
        dist.destroy_process_group()


def test_slice_range_tiles():
    for P in (1, 7, 64, 512):
        for G in (1, 2, 3, 8):
            rs = [slice_range(r, G, P) for r in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == P
            assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_two_rank_gloo_matches_single_process(tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    for name, param in CASES:
        cfg = I.scaled(I.CONFIGS[name], N=300, M=40, P=13)
        x, y, w = I.points(cfg, "x"), I.points(cfg, "y"), I.weights(cfg)
        ref = O.sliced_sum(cfg.kind, param, x, y, w, cfg.P, cfg.dir_seed, matern_p=cfg.matern_p)
        got = np.load(tmp_path / f"{name}.npy")
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(ref).max()))
