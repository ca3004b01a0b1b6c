"""Point sharding of the large-N Fourier path (include/sks.h sks_exchange_fn; parallel.point_sharded_sum).

-m gpu: two ranks, each calling sks_sum through the C-ABI with its own rows of x, w and y and the full slice range;
the three exchanges inside the call (rank 0's centre, the norm words' maxima, the grids' sum) go through
torch.distributed.  With 2 GPUs the ranks run one per GPU over NCCL; with 1 GPU both ranks use cuda:0 over gloo
(host-mediated collectives between kernels: no kernel waits on another rank).  The concatenated result is compared
with oracle (b) and with the unsharded call.
-m "not gpu": the row ranges tile [0, n); the exchange callback's three operations on a workspace tensor (gloo,
world size 2, CPU tensors)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402
from paper_2401_08260_b200 import inputs as I  # noqa: E402
from paper_2401_08260_b200.parallel import make_exchange, point_range  # noqa: E402

CFG = I.Config("points", "gaussian", 100, 600_011, 4001, 40, 41, 141, "mixture10", "pm1", param=30.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_point_range_tiles():
    for n in (1, 7, 600_011):
        for G in (1, 2, 3, 8):
            if G > n:
                continue
            rs = [point_range(r, G, n) for r in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(G - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def _xchg_worker(rank, world, port, out_dir):
    import torch.distributed as dist

    from paper_2401_08260_b200 import _lib
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ws = torch.zeros(4096, dtype=torch.uint8)
        ws[256:256 + 24].view(torch.float64)[:] = torch.tensor([1.5, -2.0, 3.25]) * (rank + 1)
        ws[512:512 + 16].view(torch.int32)[:] = torch.tensor([5, 1, 7, 0]) if rank == 0 else torch.tensor([2, 9, 7, 3])
        ws[1024:1024 + 12].view(torch.float32)[:] = torch.tensor([1.0, 2.0, 3.0]) * (1 + rank)
        fn, errors = make_exchange(ws)
        base = ws.data_ptr()
        assert fn(None, _lib.XCHG_BCAST_F64, base + 256, 3, None) == 0
        assert fn(None, _lib.XCHG_MAX_I32, base + 512, 4, None) == 0
        assert fn(None, _lib.XCHG_SUM_F32, base + 1024, 3, None) == 0
        assert fn(None, _lib.XCHG_SUM_F32, base + 4090, 3, None) == 1 and errors   # outside the workspace: refused
        np.save(os.path.join(out_dir, f"ws{rank}.npy"), ws.numpy())
    finally:
        dist.destroy_process_group()


def test_exchange_callback_gloo(tmp_path):
    import torch.multiprocessing as mp
    mp.start_processes(_xchg_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    for rank in range(2):
        ws = torch.from_numpy(np.load(tmp_path / f"ws{rank}.npy"))
        assert ws[256:280].view(torch.float64).tolist() == [1.5, -2.0, 3.25]          # rank 0's values
        assert ws[512:528].view(torch.int32).tolist() == [5, 9, 7, 3]                 # maxima
        assert ws[1024:1036].view(torch.float32).tolist() == [3.0, 6.0, 9.0]          # sums


def _worker(rank, world, port, out_dir, backend):
    import torch.distributed as dist

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200.parallel import point_sharded_sum
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y, w = I.points(CFG, "x"), I.points(CFG, "y"), I.weights(CFG)
        n0, n1 = point_range(rank, world, CFG.N)
        m0, m1 = point_range(rank, world, CFG.M)
        xl, yl, wl = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x[n0:n1], y[m0:m1], w[n0:n1]))
        s = point_sharded_sum(S.sks_sum, S.sks_workspace_size, xl, yl, wl, CFG.kind, CFG.param, CFG.P, CFG.dir_seed)
        assert S.sks_last_plan()["fused"] == 1
        np.save(os.path.join(out_dir, f"s{rank}.npy"), s.cpu().numpy())
        with pytest.raises(S.SKSError) as e:   # a shard too small for the fused path: refused, not silently wrong
            point_sharded_sum(S.sks_sum, S.sks_workspace_size, xl[:1000], yl, wl[:1000], CFG.kind, CFG.param, CFG.P,
                              CFG.dir_seed)
        assert e.value.status == 2
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_point_sharded_match_oracle(tmp_path):
    import torch.multiprocessing as mp

    import paper_2401_08260_b200 as S
    from paper_2401_08260_b200 import build
    build.build()
    assert torch.cuda.is_available()
    backend = "nccl" if torch.cuda.device_count() >= 2 else "gloo"
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), backend), nprocs=2, join=True,
                       start_method="spawn")
    got = np.concatenate([np.load(tmp_path / f"s{r}.npy") for r in range(2)]).astype(np.float64)
    assert got.shape == (CFG.M,)
    x, y, w = I.points(CFG, "x"), I.points(CFG, "y"), I.weights(CFG)
    sw = np.abs(w.astype(np.float64)).sum()
    # targets of both ranks' shards
    tgt = np.concatenate([I.target_subset(CFG.M // 2, 12), CFG.M // 2 + I.target_subset(CFG.M - CFG.M // 2, 12)])
    ref = O.sliced_sum(CFG.kind, CFG.param, x, y, w, CFG.P, CFG.dir_seed, targets=tgt)
    err = float(np.max(np.abs(got[tgt] - ref)) / sw)
    one = S.sks_sum(*(torch.from_numpy(a).cuda() for a in (x, y, w)), CFG.kind, CFG.param, CFG.P,
                    CFG.dir_seed).cpu().numpy().astype(np.float64)
    diff = float(np.max(np.abs(got - one)) / sw)
    print(f"point-sharded ({backend}, 2 ranks): vs oracle {err:.3e}, vs the unsharded call {diff:.3e}")
    assert err <= 1e-4, err
    # the same estimator: the shards' centre and footprints differ from the unsharded call's only in rounding
    assert diff <= 1e-6, diff
