"""Pins of the oracle's smoothed-aggregation setup (a4): the strength rule (D2), the MIS(2)/aggregate rules
(D3) and the damped prolongator (D5), against
  * tests/golden/sa_level.txt -- a 12-node matrix with an exact 0.25 ratio, a 0.28 ratio, weak entries to lump,
    a positive off-diagonal, a z-block boundary, an isolated row and a phase-2 tie, hand-checked in its header
    (written by tests/golden/make_sa_level.py, numpy only);
  * tests/sa_ref.py -- an independent numpy statement of the same readings on dense matrices, on random
    3-component 27-point matrices and on the SDC part of a generated A_uu.
Each of these one-line changes to oracle/oracle.c fails at least one test here (checked when the pins were
written): theta 0.25 -> 0.3; '>=' -> '>' in the strength test; no lumping of weak entries into the diagonal;
omega = 2/(3 rho); phase-2 ties to the largest aggregate id.  CPU only."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
import sa_ref

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sa_level.txt")


def _read_golden():
    g = dict(entries=[], edges=set(), state={}, ph1={}, agg={}, P={})
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        t = line.split()
        if t[0] == "n":
            g["n"] = int(t[1])
        elif t[0] == "zb":
            g["zb"] = np.array([int(x) for x in t[1:]], np.int32)
        elif t[0] == "entry":
            g["entries"].append((int(t[1]), int(t[2]), float(t[3])))
        elif t[0] == "edge":
            g["edges"].add((int(t[1]), int(t[2])))
        elif t[0] in ("state", "ph1", "agg"):
            g[t[0]][int(t[1])] = int(t[2])
        elif t[0] in ("rho", "omega"):
            g[t[0]] = float(t[1])
        elif t[0] == "P":
            g["P"][(int(t[1]), int(t[2]))] = float(t[3])
    n = g["n"]
    rows = [[] for _ in range(n)]
    for i, j, a in g["entries"]:
        rows[i].append((j, a))
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.array([j for r in rows for j, _ in sorted(r)], np.int32)
    v = np.array([a for r in rows for _, a in sorted(r)])
    g["csr"] = (rp, ci, v)
    return g


@pytest.fixture(scope="module")
def gold():
    return _read_golden()


def test_golden_file_is_the_script_output(gold):
    """The committed golden equals what make_sa_level.py's numpy statement gives today."""
    rp, ci, v = gold["csr"]
    A = sp.csr_matrix((v, ci, rp), shape=(gold["n"],) * 2).toarray()[None]
    r = sa_ref.level(A, gold["zb"])
    assert {(i, j) for i, j in zip(*np.nonzero(np.triu(r["E"])))} == gold["edges"]
    assert [gold["agg"][i] for i in range(gold["n"])] == list(r["agg"])
    assert float(r["omega"][0]) == gold["omega"]


def test_strength_golden(gold):
    """D2: |a_ij| >= 0.25 max_k!=i |a_ik| (equality counts), same z-block only, symmetrised S u S^T."""
    rp, ci, v = gold["csr"]
    E = oracle.strength(rp, ci, v, gold["zb"], 0.25)
    got = set()
    for i in range(gold["n"]):
        for q in range(rp[i], rp[i + 1]):
            if E[q] and i < ci[q]:
                got.add((i, int(ci[q])))
    assert got == gold["edges"]


def test_aggregation_golden(gold):
    """D3: MIS(2) states, phase-1 aggregates (root + strong neighbours, numbered by ascending root) and
    phase-2 assignment (strongest neighbour, tie -> smallest aggregate id) of the hand-checked matrix."""
    rp, ci, v = gold["csr"]
    amg = oracle.Amg(rp, ci, v, gold["zb"], amg_coarse_max=2)
    st, ph1, om = amg.detail(0)
    n = gold["n"]
    assert list(st) == [gold["state"][i] for i in range(n)]
    assert list(ph1) == [gold["ph1"][i] for i in range(n)]
    assert list(amg.levels()[0]["agg"]) == [gold["agg"][i] for i in range(n)]
    assert gold["agg"][4] == 0 and gold["ph1"][4] == -1      # the tie of the header: aggregate 0, not 2


def test_prolongator_golden(gold):
    """D5: rho over the filtered, lumped A^F; omega = 4/(3 rho) = 12/17; P = P_tent - omega D_F^-1 A^F P_tent
    (the header derives P_4,0 = 49/85 and P_4,2 = 24/85 by hand)."""
    rp, ci, v = gold["csr"]
    amg = oracle.Amg(rp, ci, v, gold["zb"], amg_coarse_max=2)
    _, _, om = amg.detail(0)
    assert om[0] == pytest.approx(12.0 / 17.0, rel=1e-15)
    assert gold["omega"] == pytest.approx(12.0 / 17.0, rel=1e-15)
    L0 = amg.levels()[0]
    got = {}
    for i in range(gold["n"]):
        for q in range(L0["P_rp"][i], L0["P_rp"][i + 1]):
            got[(i, int(L0["P_ci"][q]))] = float(L0["P_v"][q, 0])
    got = {k: x for k, x in got.items() if x != 0.0}
    assert set(got) == set(gold["P"])
    for k, x in gold["P"].items():
        assert got[k] == pytest.approx(x, rel=2e-15, abs=1e-16), k
    assert got[(4, 0)] == pytest.approx(49.0 / 85.0, rel=1e-15)
    assert got[(4, 2)] == pytest.approx(24.0 / 85.0, rel=1e-15)


def _grid27_random(nx, ny, nz, nc, seed):
    """Random 27-point values (mixed signs off the diagonal, dominant diagonal) on a node grid."""
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    idx = np.arange(n).reshape(nz, ny, nx)
    rows = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                r = []
                for dk in (-1, 0, 1):
                    for dj in (-1, 0, 1):
                        for di in (-1, 0, 1):
                            ii, jj, kk = i + di, j + dj, k + dk
                            if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                                r.append(idx[kk, jj, ii])
                rows.append(sorted(r))
    rp = np.zeros(n + 1, np.int32)
    rp[1:] = np.cumsum([len(r) for r in rows])
    ci = np.concatenate(rows).astype(np.int32)
    v = rng.standard_normal((len(ci), nc)) * rng.choice([0.05, 1.0], size=(len(ci), 1))
    v = np.where(rng.random((len(ci), 1)) < 0.8, -np.abs(v), np.abs(v))
    diag = np.repeat(np.arange(n), np.diff(rp)) == ci
    rowsum = np.add.reduceat(np.abs(v) * ~diag[:, None], rp[:-1])
    v[diag] = rowsum * rng.uniform(0.9, 1.3, (n, 1))
    zb = (np.arange(n) // (nx * ny) // 3).astype(np.int32)
    return rp, ci, v, zb


def _dense(rp, ci, v, n):
    nc = v.shape[1]
    A = np.zeros((nc, n, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    for c in range(nc):
        A[c, rows, ci] = v[:, c]
    return A


def _compare_level(rp, ci, v, zb, **amg_kw):
    n = len(rp) - 1
    A = _dense(rp, ci, v, n)
    ref = sa_ref.level(A, zb)
    E = oracle.strength(rp, ci, v, zb)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.array_equal(E, ref["E"][rows, ci])
    amg = oracle.Amg(rp, ci, v, zb, **amg_kw)
    st, ph1, om = amg.detail(0)
    L0 = amg.levels()[0]
    assert np.array_equal(st, ref["st"])
    assert np.array_equal(ph1, ref["ph1"])
    assert np.array_equal(L0["agg"], ref["agg"]) and L0["nagg"] == ref["nagg"]
    np.testing.assert_allclose(om, ref["omega"], rtol=1e-14)
    for c in range(v.shape[1]):
        P = sp.csr_matrix((L0["P_v"][:, c], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
        scale = np.abs(ref["P"][c]).max()
        assert np.abs(P - ref["P"][c]).max() <= 1e-14 * scale
    # the stored pattern is exactly the aggregates of {i} U strong(i)
    for i in range(n):
        want = set() if ref["agg"][i] < 0 else {ref["agg"][j] for j in np.flatnonzero(ref["E"][i]) if ref["agg"][j] >= 0} | {ref["agg"][i]}
        assert set(L0["P_ci"][L0["P_rp"][i]:L0["P_rp"][i + 1]]) == want
    return ref


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_three_component_level_matches_numpy(seed):
    """Strength with the SDC measure sum_c |a^c_ij| (D2), shared aggregates and one damped
    prolongator per component (D5) equal the dense numpy statement on a random 3-component 27-point matrix."""
    rp, ci, v, zb = _grid27_random(6, 5, 7, 3, seed)
    ref = _compare_level(rp, ci, v, zb, amg_coarse_max=8)
    assert ref["nagg"] >= 3 and len(set(ref["omega"])) == 3


def test_sdc_level0_of_a_generated_problem_matches_numpy():
    """Level 0 of the oracle's mechanics hierarchy (SDC of A_uu; node z-blocks R-zblock) equals the
    dense numpy statement of D2-D5 on the same three value sets."""
    pb = synth.generate(nx=4, ny=3, nz=18, recipe=2, perm_sigma=2.0)
    o = oracle.Oracle(pb, zblock=16).setup()
    L0 = o.level(0, 0)
    rp, ci, v = L0["A_rp"], L0["A_ci"], L0["A_v"]
    # a2: the SDC values are the xx, yy, zz entries of A_uu's 3x3 blocks
    assert np.array_equal(v, pb.uu_val.reshape(-1, 9)[:, [0, 4, 8]])
    k = np.arange(pb.Nn) // ((pb.nx + 1) * (pb.ny + 1))
    zb = (np.minimum(k, pb.nz - 1) // 16).astype(np.int32)
    n = len(rp) - 1
    ref = sa_ref.level(_dense(rp, ci, v, n), zb)
    assert np.array_equal(L0["agg"], ref["agg"])
    for c in range(3):
        P = sp.csr_matrix((L0["P_v"][:, c], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
        assert np.abs(P - ref["P"][c]).max() <= 1e-14 * np.abs(ref["P"][c]).max()


def test_pressure_level0_of_a_generated_problem_matches_numpy():
    """Level 0 of the oracle's pressure hierarchy (S_pp) against the dense numpy statement."""
    pb = synth.generate(nx=5, ny=4, nz=18, recipe=2, perm_sigma=2.0)
    o = oracle.Oracle(pb, zblock=16).setup()
    L0 = o.level(1, 0)
    rp, ci, v = L0["A_rp"], L0["A_ci"], L0["A_v"]
    zb = ((np.arange(pb.Nc) // (pb.nx * pb.ny)) // 16).astype(np.int32)
    n = len(rp) - 1
    ref = sa_ref.level(_dense(rp, ci, v, n), zb)
    assert np.array_equal(L0["agg"], ref["agg"])
    P = sp.csr_matrix((L0["P_v"][:, 0], L0["P_ci"], L0["P_rp"]), shape=(n, L0["nagg"])).toarray()
    assert np.abs(P - ref["P"][0]).max() <= 1e-14 * np.abs(ref["P"][0]).max()
