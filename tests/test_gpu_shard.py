"""The row-sharded (world > 1) code path on ONE GPU, through virtual-rank handles
(fde_create_virtual_rank): each rank's local work runs exactly as it would in a
G-process job; only the ncclAllGather itself is replaced by stacking the ranks'
local results in the all-gather layout.

Invariant (SURVEY.md §8(c) "Sharding"): every rank's rows, the gathered matvec
and the replicated H-matrix / H-LU are BITWISE equal to the world = 1 ones.
"""
import numpy as np
import pytest

import fde_inputs as fi
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fde():
    from paper_1808_02937_b200 import fde as F
    return F


@pytest.fixture(scope="module")
def h(fde):
    return fde.Handle(0)


def metric_A(Ag, Ao):
    d = np.sqrt(np.abs(np.diag(Ao)))
    return np.max(np.abs(Ag - Ao) / (d[:, None] * d[None, :]))


def ragged():
    # N = 37 elements over 4 or 8 ranks: unequal shards, a rank boundary inside
    # every cluster level
    nodes = np.concatenate([[0.0], np.sort(np.random.default_rng(11).uniform(0, 1, 36)), [1.0]])
    return fi.Problem("ragged37", 0.0, 1.0, 1.55, 0.35, 0.7, 0.0, 0.0, nodes, 5, 6, n_min=4,
                      forcings=[fi.random_legendre_forcing(5)])


CASES = [(fi.config4(), 2), (fi.config4(), 4), (fi.config4(), 8), (ragged(), 4), (ragged(), 8)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].name}-G{c[1]}")
def test_shard_rows_and_gathered_matvec_bitwise(fde, h, case):
    """Sharded assembly (rank g: its element rows, the row triangle plus the
    transposed column band, api.cpp) gives rows [r0, r1) of the world = 1
    operator bit for bit; the local GEMVs stacked in the all-gather layout and
    compacted by the library's post-all-gather kernel give the world = 1 A x."""
    p, G = case
    op1 = fde.assemble_problem(h, p)
    A1 = fde.operator_rows_internal(h, op1)
    rng = np.random.default_rng(G)
    for nrhs in (1, 3):
        x = torch.tensor(rng.standard_normal((nrhs, p.n)), device="cuda")
        y1 = fde.stiffness_matvec(h, op1, x, path=fde.PATH_DENSE)
        locs = []
        rows_max = fde.shard_rows(p.N, p.P, G, 0)[2]
        keep = None
        for g in range(G):
            hg = fde.Handle(0, virtual=True, rank=g, world=G)
            opg = fde.assemble_problem(hg, p)
            r0, r1, rm = fde.shard_rows(p.N, p.P, G, g)
            assert rm == rows_max
            inf = opg.info
            assert (inf.row_begin, inf.row_end) == (r0, r1)
            if nrhs == 1:
                Ag = fde.operator_rows_internal(hg, opg)
                assert torch.equal(Ag, A1[r0:r1]), f"rank {g}: rows differ"
            locs.append(fde.shard_matvec(hg, opg, x, rows_max))
            with pytest.raises(fde.FdeError) as e:       # the collective is not there
                fde.stiffness_matvec(hg, opg, x, path=fde.PATH_DENSE)
            assert e.value.name == "FDE_ENCCL"
            if g == 0:
                keep = (hg, opg)          # rank 0 runs the compaction below
            else:
                opg.free()
                hg.close()
        gathered = torch.stack(locs)                      # (G, nrhs, rows_max)
        y = fde.compact_gather(keep[0], keep[1], gathered, nrhs)
        assert torch.equal(y, y1)
        keep[1].free()
        keep[0].close()
    op1.free()


@pytest.mark.parametrize("case", [(fi.config4(N=256, P=8), 2), (ragged(), 4)], ids=lambda c: f"{c[0].name}-G{c[1]}")
def test_recompute_path_hmatrix_and_replicated_hlu(fde, h, case):
    """At world > 1 the near-field (inadmissible) leaves are recomputed from pair
    moments (hmatrix.cu recompute path) instead of copied from the resident A:
    the resulting A~ equals the copy-path A~ (M-A <= 1e-14) and the oracle's A~
    (M-A <= 1e-10); every rank builds the SAME H-matrix and H-LU bit for bit
    (the replicas must agree for the ranks to run the same Krylov iterations)."""
    p, G = case
    n_min = p.n_min if p.N > 64 else 4
    op1 = fde.assemble_problem(h, p)
    hm1 = fde.hmatrix_build(h, op1, p.R, p.lam, n_min)
    At1 = fde.hmatrix_dense_paper(h, hm1).cpu().numpy()
    Z = []
    r = torch.tensor(np.random.default_rng(3).standard_normal((2, p.n)), device="cuda")
    Ats = []
    for g in range(G):
        hg = fde.Handle(0, virtual=True, rank=g, world=G)
        opg = fde.assemble_problem(hg, p)
        hmg = fde.hmatrix_build(hg, opg, p.R, p.lam, n_min)
        Ats.append(fde.hmatrix_dense_paper(hg, hmg).cpu().numpy())
        lug = fde.hlu_factor(hg, hmg, 1e-3)
        Z.append(fde.precond_apply(hg, lug, r).cpu().numpy())
        for o in (lug, hmg, opg):
            o.free()
        hg.close()
    for g in range(1, G):
        assert np.array_equal(Ats[g], Ats[0]), f"rank {g} H-matrix differs from rank 0"
        assert np.array_equal(Z[g], Z[0]), f"rank {g} preconditioner differs from rank 0"
    assert metric_A(Ats[0], At1) <= 1e-14
    if p.N <= 64:
        so = O.assemble_system(p)
        Ato, _ = O.hmatrix_dense(p, so, R=p.R, lam=p.lam, n_min=n_min)
        assert metric_A(Ats[0], Ato) <= 1e-10
    hm1.free()
    op1.free()


def test_compact_gather_synthetic(fde, h):
    """k_compact_gather on a synthetic all-gather buffer whose entry encodes
    (rank, column, local row): the output must hold, in paper order, the value
    of the rank that owns each internal row (padding rows never read)."""
    p = ragged()
    G = 8
    hv = fde.Handle(0, virtual=True, rank=3, world=G)
    op = fde.assemble_problem(hv, p)
    r0s = [fde.shard_rows(p.N, p.P, G, g) for g in range(G)]
    rows_max = r0s[0][2]
    nrhs = 3
    buf = np.full((G, nrhs, rows_max), np.nan)
    expect_internal = np.zeros((nrhs, p.n))
    for g, (r0, r1, _) in enumerate(r0s):
        for c in range(nrhs):
            vals = 1000.0 * g + 100.0 * c + np.arange(r1 - r0)
            buf[g, c, :r1 - r0] = vals
            expect_internal[c, r0:r1] = vals
            buf[g, c, r1 - r0:] = -1.0          # padding: must not appear
    y = fde.compact_gather(hv, op, torch.tensor(buf, device="cuda"), nrhs).cpu().numpy()
    perm = fde.internal_to_paper_index(p.N, p.P)
    expect = np.zeros_like(expect_internal)
    expect[:, perm] = expect_internal
    assert np.array_equal(y, expect)
    op.free()
    hv.close()


@pytest.mark.parametrize("nrhs", [1, 3])
def test_nccl_one_rank_allgather_path(fde, h, nrhs):
    """The world > 1 matvec's communication calls on real NCCL (one-rank
    communicator: dlopen'ed libnccl, ncclGetUniqueId, ncclCommInitRank,
    ncclAllGather of the padded local rows, k_compact_gather): bitwise the
    world-1 A x."""
    p = fi.config4(N=256, P=8)
    op = fde.assemble_problem(h, p)
    x = torch.tensor(np.random.default_rng(nrhs).standard_normal((nrhs, p.n)), device="cuda")
    y1 = fde.stiffness_matvec(h, op, x, path=fde.PATH_DENSE)
    y = fde.comm_selftest(h, op, x)
    assert torch.equal(y, y1)
    op.free()


@pytest.mark.parametrize("NPG", [(8, 3, 8), (5, 2, 8), (3, 4, 4)], ids=lambda t: f"N{t[0]}P{t[1]}G{t[2]}")
def test_more_ranks_than_elements(fde, h, NPG):
    """One element per rank, and more ranks than elements (empty shards: a rank
    with no rows must skip its GEMV instead of launching an empty grid -- found
    and fixed in round 2): the gathered matvec is still bitwise the world-1 A x,
    and every rank builds the H-matrix (recompute path)."""
    N, P, G = NPG
    p = fi.Problem(f"s{N}", 0.0, 1.0, 1.5, 0.5, 1.0, 0.0, 0.0, fi.uniform_mesh(0, 1, N), P, 3, n_min=1,
                   forcings=[fi.random_legendre_forcing(1)])
    op1 = fde.assemble_problem(h, p)
    x = torch.tensor(np.random.default_rng(0).standard_normal((2, p.n)), device="cuda")
    y1 = fde.stiffness_matvec(h, op1, x, path=fde.PATH_DENSE)
    rm = fde.shard_rows(N, P, G, 0)[2]
    locs, keep = [], None
    for g in range(G):
        hg = fde.Handle(0, virtual=True, rank=g, world=G)
        opg = fde.assemble_problem(hg, p)
        locs.append(fde.shard_matvec(hg, opg, x, rm))
        hm = fde.hmatrix_build(hg, opg, 3, 1.0, 1)
        hm.free()
        if g == 0:
            keep = (hg, opg)
        else:
            opg.free()
            hg.close()
    y = fde.compact_gather(keep[0], keep[1], torch.stack(locs), 2)
    assert torch.equal(y, y1)
    keep[1].free()
    keep[0].close()
    op1.free()
