"""Host logic of the multi-GPU path (row e) on CPU, no GPU needed.

* the 2D block-cyclic maps: local shapes and index sets partition the matrix;
* the distributed QR plan (intra-domain levels per process row + the inter-domain head merges in
  slot indices, hlq_dist_plan) is exactly the single-device greedy tree of the oracle (qr_plan);
* across gloo ranks (world size 2 and 4, one process per rank as under torchrun): every
  communicator's exchange sizes agree (hlq_dist_counts — a disagreement would deadlock NCCL), the
  root of every broadcast and the owner of every step are unique, and a block-cyclic
  scatter / gather round trip of a seeded matrix reassembles it exactly.
"""
import os
import socket

import numpy as np
import pytest

import hlq_inputs as I
import paper_1401_5522_b200 as H
from oracle import hlq_oracle as O


@pytest.mark.parametrize("N,nb,P,Q", [(1000, 64, 2, 3), (1024, 128, 2, 2), (131072, 320, 2, 4),
                                      (100, 128, 2, 2), (777, 64, 3, 1)])
def test_local_shapes_partition(N, nb, P, Q):
    nbe = min(nb, N)
    assert sum(H.local_shape(N, nb, P, Q, p, 0)[0] for p in range(P)) == N
    assert sum(H.local_shape(N, nb, P, Q, 0, q)[1] for q in range(Q)) == N
    if N <= 4096:
        rows = np.concatenate([H.cyclic_rows(N, nbe, P, p) for p in range(P)])
        assert np.array_equal(np.sort(rows), np.arange(N))
        for p in range(P):
            assert len(H.cyclic_rows(N, nbe, P, p)) == H.local_shape(N, nb, P, Q, p, 0)[0]


def _global_plan(n, P, D, k):
    """Map every rank's local plan back to global tile indices."""
    plans = [H.dist_plan(n, P, D, p, k) for p in range(P)]
    c = D // P
    intra = {}
    slot_head = {}
    owners = []
    for p, pl in enumerate(plans):
        li0 = pl["li0"]
        owners += [(li0 + j) * P + p for j in range(pl["ms"])]
        for lv, pairs in enumerate(pl["intra"]):
            intra.setdefault(lv, set()).update(
                ((li0 + a) * P + p, (li0 + b) * P + p) for a, b in pairs)
        for t, (hl, hg) in enumerate(pl["heads"]):
            slot_head[p * c + t] = hg
            if hl >= 0:
                assert (li0 + hl) * P + p == hg
        assert pl["diag"] == (1 if k % P == p else 0)
    inter = [[(slot_head[a], slot_head[b]) for a, b in lv] for lv in plans[0]["inter"]]
    for pl in plans[1:]:
        assert pl["inter"] == plans[0]["inter"]  # every rank merges the heads identically
    return sorted(owners), intra, inter


@pytest.mark.parametrize("n,P,D", [(16, 1, 2), (16, 2, 2), (17, 2, 4), (9, 3, 3), (410, 2, 2),
                                   (7, 2, 2), (5, 4, 4)])
def test_distributed_plan_is_the_greedy_tree(n, P, D):
    for k in range(n):
        owners, intra, inter = _global_plan(n, P, D, k)
        assert owners == list(range(k, n))  # every panel tile has exactly one owner
        _, _, levels = O.qr_plan(k, n, D, tree="greedy")
        depth = len(intra)
        for lv in range(depth):
            assert intra[lv] == set(levels[lv]), (k, lv)
        assert inter == levels[depth:], k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, P, Q, port, N, nb, D, result_dir):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        p, q = divmod(rank, Q)
        n = -(-N // nb)
        # 1. exchange sizes: gather every rank's counts of every step
        cnt = torch.tensor([H.dist_counts(N, nb, P, Q, D, p, q, k) for k in range(n)],
                           dtype=torch.int64)
        allc = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(allc, cnt)
        ok = True
        for k in range(n):
            for r in range(world):
                pr, qr = divmod(r, Q)
                for r2 in range(world):
                    p2, q2 = divmod(r2, Q)
                    a, b = allc[r][k], allc[r2][k]
                    if qr == q2 == k % Q and (a[0] != b[0] or a[1] != b[1]):
                        ok = False  # X1 / X2 allgather in the panel column
                    if pr == p2 and a[2] != b[2]:
                        ok = False  # X3 broadcast in a process row
                    if qr == q2 and a[3] != b[3]:
                        ok = False  # X4 allgather in a process column
        # 2. block-cyclic scatter / gather round trip of the seeded matrix
        A = I.uniform_matrix(2, N)
        L = H.scatter_block_cyclic(A, nb, P, Q, p, q)
        m, nl = H.local_shape(N, nb, P, Q, p, q)
        ok = ok and L.shape == (m, nl)
        cap = max(H.local_shape(N, nb, P, Q, pp, qq)[0] * H.local_shape(N, nb, P, Q, pp, qq)[1]
                  for pp in range(P) for qq in range(Q))
        buf = torch.zeros(cap, dtype=torch.float64)
        buf[:L.size] = torch.from_numpy(np.ascontiguousarray(L).reshape(-1))
        gathered = [torch.zeros(cap, dtype=torch.float64) for _ in range(world)] if rank == 0 \
            else None
        dist.gather(buf, gathered, dst=0)
        if rank == 0:
            locs = {}
            for r in range(world):
                pp, qq = divmod(r, Q)
                mm, nn = H.local_shape(N, nb, P, Q, pp, qq)
                locs[(pp, qq)] = gathered[r][:mm * nn].numpy().reshape(mm, nn)
            ok = ok and np.array_equal(H.gather_block_cyclic(locs, N, nb, P, Q), A)
        # 3. max-over-ranks timing reduction as bench.py does it
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = ok and float(t.item()) == float(world)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int64)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if rank == 0:
            with open(os.path.join(result_dir, "ok"), "w") as fh:
                fh.write(str(int(flag.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,P,Q,N,nb,D", [(2, 1, 2, 1000, 64, 2), (2, 2, 1, 1000, 64, 2),
                                              (4, 2, 2, 777, 64, 2), (4, 2, 2, 1024, 128, 4)])
def test_gloo_ranks_agree(tmp_path, world, P, Q, N, nb, D):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(world, P, Q, port, N, nb, D, str(tmp_path)), nprocs=world, join=True)
    assert (tmp_path / "ok").read_text() == "1"
