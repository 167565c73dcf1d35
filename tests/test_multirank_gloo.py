"""World-size-2 gloo test of the distributed resampling host logic: each rank quantizes
its shard, all-gathers the integer masses Q_r, computes its slot range with cdms_resample_plan (the
library's host code), resolves the ancestors of those slots from its local CDF, exchanges them per the
plan's send counts, and the assembled global ancestors must equal the oracle's single-process
systematic resampling bit for bit."""
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


def _worker(rank, world, port, w_all, u_bits, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_19723_b200 import cdms
    P_local = len(w_all) // world
    w = w_all[rank * P_local:(rank + 1) * P_local]
    # global max via the collective (max is exact), then the integer quantization of C-amb-15
    wmax = torch.tensor([w.max()], dtype=torch.float64)
    dist.all_reduce(wmax, op=dist.ReduceOp.MAX)
    q = np.rint(np.ldexp(w / wmax.item(), 36)).astype(np.uint64)
    C = np.cumsum(q, dtype=np.uint64)
    Qr = torch.tensor([int(C[-1])], dtype=torch.int64)
    Qs = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(Qs, Qr)
    Q = [int(x.item()) for x in Qs]
    lo, hi, counts = cdms.resample_plan(Q, rank, P_local, u_bits)
    Qt, O, P = sum(Q), sum(Q[:rank]), P_local * world
    anc = np.empty(hi - lo, dtype=np.int64)
    for k, i in enumerate(range(lo, hi)):
        t = (u_bits + i * 2**32) * Qt // (P * 2**32) - O
        anc[k] = rank * P_local + int(np.searchsorted(C, t, side="right"))
    # exchange: rank d receives the ancestors of its slots from every source rank
    recv_counts = []
    for s in range(world):
        lo_s, hi_s, _ = cdms.resample_plan(Q, s, P_local, u_bits)
        recv_counts.append(max(0, min(hi_s, (rank + 1) * P_local) - max(lo_s, rank * P_local)))
    send = torch.from_numpy(anc)
    recv = torch.empty(P_local, dtype=torch.int64)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=counts)
    gathered = [torch.empty(P_local, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, recv)
    if rank == 0:
        np.save(out_path, torch.cat(gathered).numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["random", "skewed", "onehot_rank1"])
def test_distributed_resampling_equals_oracle(tmp_path, orc, case):
    from paper_2604_19723_b200 import build as B
    B.build()
    world, P_local = 2, 37
    rng = np.random.default_rng({"random": 1, "skewed": 2, "onehot_rank1": 3}[case])
    w = rng.exponential(size=world * P_local)
    if case == "skewed":
        w[:P_local] *= 1e-3
    if case == "onehot_rank1":
        w[:] = 0.0
        w[P_local + 5] = 1.0
    w = w / w.sum()
    u_bits = int(rng.integers(0, 2**32))
    out = str(tmp_path / "anc.npy")
    mp.start_processes(_worker, args=(world, _free_port(), w, u_bits, out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    st, ref = orc.resample(w, u_bits)
    assert st == 0
    assert np.array_equal(got, ref)
