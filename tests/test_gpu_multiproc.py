"""Row e across PROCESSES (-m gpu): hlq_factor_dist with one process per rank on the per-rank code
path (the same branch the NCCL grid takes), the collectives handed to torch.distributed gloo on the
host through the host-staged backend (hlq_grid_create_host).  Two processes share the one B200 of
this run; no kernel ever waits on another process (every exchange is a host collective between
stream synchronisations), so the ranks cannot deadlock on the GPU.

Each rank factors its block-cyclic local array of a 1 x 2 or 2 x 1 grid, solves, and writes its
local factors; the parent gathers them and compares with the oracle run with the same QR-tree
domains D = P (decisions identical, factors within 1e-10, HPL3 <= 16)."""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import hlq_inputs as I  # noqa: E402
from oracle import hlq_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, P, Q, port, N, nb, crit, alpha, forced, outdir, pivot="tile"):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_1401_5522_b200 as H
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    p, q = divmod(rank, Q)
    # communicators: the process row (Q members, index q) and column (P members, index p)
    rows = [dist.new_group([pp * Q + qq for qq in range(Q)]) for pp in range(P)]
    cols = [dist.new_group([pp * Q + qq for pp in range(P)]) for qq in range(Q)]

    def group(comm):
        if comm == H.COMM_ROW:
            return rows[p], [p * Q + qq for qq in range(Q)]
        if comm in (H.COMM_COL, H.COMM_COL_PANEL):
            return cols[q], [pp * Q + q for pp in range(P)]
        return None, list(range(world))

    def allgather(comm, send, recv):
        g, members = group(comm)
        outs = [torch.empty(send.size, dtype=torch.float64) for _ in members]
        dist.all_gather(outs, torch.from_numpy(send.copy()), group=g)
        for t, o in enumerate(outs):
            recv[t * send.size:(t + 1) * send.size] = o.numpy()

    def broadcast(comm, buf, root):
        g, members = group(comm)
        t = torch.from_numpy(buf.copy())
        dist.broadcast(t, src=members[root], group=g)
        buf[:] = t.numpy()

    def allreduce(comm, buf, op):
        g, _ = group(comm)
        t = torch.from_numpy(buf.copy())
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM, group=g)
        buf[:] = t.numpy()

    grid = H.grid_host(world, rank, P, Q, allgather, broadcast, allreduce)
    A = I.uniform_matrix(11, N)
    b = I.uniform_rhs(11, N)
    L = H.scatter_block_cyclic(A, nb, P, Q, p, q)
    dA = H.to_colmajor(L) if L.size else torch.zeros(0, dtype=torch.float64, device="cuda")
    kw = dict(tree_domains=P)
    if pivot == "domain":
        kw["pivot_scope"] = H.PIVOT_DOMAIN
    if forced is not None:
        kw["forced"] = forced
    f = H.hlq_factor_dist(grid, [dA], N, nb, crit, alpha, **kw)
    x = f.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             F=H.from_colmajor(dA) if L.size else np.zeros((0, 0)), dec=f.decisions(), x=x,
             growth=f.growth(), hinted=f.info()["hinted"])
    f.free()
    grid.free()
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def cuda_ok():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True


@pytest.mark.parametrize("P,Q,N,nb,crit,alpha,f_qr,pivot", [
    (1, 2, 1000, 64, O.CRIT_MAX, 1.2e4, None, "tile"),   # criterion-decided LU/QR mix, ragged tile
    (2, 1, 1000, 64, O.CRIT_MAX, 1.2e4, None, "tile"),   # two process rows: cross-rank TT merges
    (1, 2, 768, 128, O.CRIT_MAX, 1.0, 0.5, "tile"),      # forced Bernoulli pattern
    (2, 1, 768, 64, O.CRIT_MAX, 1.0, 1.0, "tile"),       # all QR, D = 2
    (2, 1, 1000, 64, O.CRIT_MAX, 300.0, None, "domain"),  # diagonal-domain pivoting (NEXT f1)
    (1, 2, 1000, 64, O.CRIT_MAX, 300.0, None, "domain"),
])
def test_two_process_grid_against_oracle(cuda_ok, P, Q, N, nb, crit, alpha, f_qr, pivot):
    import torch.multiprocessing as mp
    import paper_1401_5522_b200 as H
    n = (N + nb - 1) // nb
    forced = I.bernoulli_pattern(30, n, f_qr) if f_qr is not None else None
    A = I.uniform_matrix(11, N)
    b = I.uniform_rhs(11, N)
    fo = O.hybrid_factor(A, nb, crit, alpha, D=P, forced=forced, pivot_scope=pivot)
    assert not np.any(np.isfinite(fo.margin) & (np.abs(fo.margin) < 1e-10))  # no hints needed
    with tempfile.TemporaryDirectory() as td:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank_main, args=(r, P * Q, P, Q, port, N, nb, crit, alpha,
                                                        forced, td, pivot)) for r in range(P * Q)]
        for pr in procs:
            pr.start()
        for pr in procs:
            pr.join(timeout=600)
        assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
        res = [np.load(os.path.join(td, f"rank{r}.npz")) for r in range(P * Q)]
    for r in res:
        np.testing.assert_array_equal(r["dec"], fo.dec)
        assert int(r["hinted"]) == 0
        assert float(r["growth"]) == pytest.approx(fo.growth, rel=1e-10)
    F = H.gather_block_cyclic({divmod(r, Q): res[r]["F"] for r in range(P * Q)}, N, nb, P, Q)
    assert O.factor_diff(F, fo.A) <= 1e-10, O.factor_diff(F, fo.A)
    for r in res:  # x is returned on every rank
        assert O.hpl3(A, r["x"], b) <= 16.0
        assert np.linalg.norm(r["x"] - O.solve(fo, b)) <= 1e-8 * np.linalg.norm(O.solve(fo, b))
