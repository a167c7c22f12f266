"""Writes tests/golden/sa_level.txt: one smoothed-aggregation level of a 12-node matrix built to exercise each
reading of SURVEY.md D2-D5 (DESIGN.md R-strength, R-mis2, R-agg, R-prolong).  Calls only numpy (tests/sa_ref.py,
written from the readings, never from the oracle).  The hand checks of the interesting entries are in the
golden file's header.  Run:  python tests/golden/make_sa_level.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import sa_ref  # noqa: E402

N = 12
# off-diagonal entries a_ij (row i, column j); the pattern is structurally symmetric
OFF = {
    # chain 10 - 2 - 4 - 7 - 5: roots 10 and 5 (the two highest fmix32 priorities), node 4 is left for phase 2
    (10, 2): -4.0, (2, 10): -4.0,
    (2, 4): -4.0, (4, 2): -2.0,
    (4, 7): -2.0, (7, 4): -4.0,          # |a_42| == |a_47|: phase-2 tie -> the smaller aggregate id
    (7, 5): -4.0, (5, 7): -4.0,
    (2, 7): -1.12, (7, 2): -1.12,        # ratio 0.28 in both rows: strong at theta = 0.25, weak at 0.3
    # second group 9 - 1 - 8 - 3 - 11
    (9, 1): -4.0, (1, 9): -4.0,
    (1, 8): -1.0, (8, 1): -1.0,          # row 1: exactly 0.25 * 4 (strong only through '>='); row 8: 1/5 < 0.25
    (8, 3): -5.0, (3, 8): -5.0,
    (3, 11): 4.0, (11, 3): -4.0,         # a positive off-diagonal: strength uses |a_ij|
    (5, 9): -0.5, (9, 5): -0.5,          # weak both ways (0.125): lumped into d_5 and d_9
    # z-block boundary: node 6 lives in z-block 1, its only coupling (to 11) is not a strength edge
    (6, 11): -3.0, (11, 6): -3.0,
    # node 0 has no off-diagonal (a Dirichlet-like row): isolated
}
DIAG = {0: 1.0, 1: 6.0, 2: 12.0, 3: 11.0, 4: 5.0, 5: 5.0, 6: 4.0, 7: 12.0, 8: 7.0, 9: 5.0, 10: 5.0, 11: 8.0}
ZB = np.array([0] * 6 + [1] + [0] * 5)


def matrix():
    A = np.zeros((1, N, N))
    for (i, j), v in OFF.items():
        A[0, i, j] = v
    for i, v in DIAG.items():
        A[0, i, i] = v
    return A


def main():
    A = matrix()
    r = sa_ref.level(A, ZB, 0.25)
    L = []
    L.append("# One smoothed-aggregation level (SURVEY.md D2-D5; DESIGN.md R-strength, R-mis2, R-agg, R-prolong),")
    L.append("# written by tests/golden/make_sa_level.py (numpy only, tests/sa_ref.py).  Read by tests/test_oracle_sa.py.")
    L.append("# Hand checks (single component, theta = 0.25):")
    L.append("#  priorities fmix32(i): 10 > 5 > 9 > 11 > 3 > 1 > 8 > 2 > 4 > 7 > 0 (6 and 0 are isolated, never ranked)")
    L.append("#  row 1: m = 4 (col 9); |a_18| = 1 = 0.25 * 4 -> strong by '>='; row 8: m = 5, 1 < 1.25 -> weak; E(1,8) via row 1")
    L.append("#  rows 2 and 7: m = 4, |a_27| = |a_72| = 1.12 = 0.28 m -> strong at 0.25 (weak at 0.3)")
    L.append("#  rows 5, 9: |a_59| = 0.5 = 0.125 m -> weak, lumped: d_5 = 5 - 0.5 = 4.5, d_9 = 5 - 0.5 = 4.5")
    L.append("#  row 11: |a_11,6| = 3 >= 1 but zb(6) = 1 != zb(11) = 0 -> weak, lumped: d_11 = 8 - 3 = 5; node 6 isolated")
    L.append("#  greedy MIS(2): 10 root (decides 2, 4, 7); 5 root (distance 3 from 10 through 2-7); 9 root (decides 1, 8);")
    L.append("#    11 root (distance 4 from 9: 9-1-8-3-11; decides 3, 8)  => roots 5, 9, 10, 11 -> aggregates 0, 1, 2, 3")
    L.append("#  phase 1: {5, 7} = 0, {9, 1} = 1, {10, 2} = 2, {11, 3} = 3; phase 2: node 4 ties (|a_42| = |a_47| = 2) between")
    L.append("#    aggregate 2 (via 2) and aggregate 0 (via 7) -> 0 (smallest id); node 8: |a_83| = 5 > |a_81| = 1 -> aggregate 3")
    L.append("#  rho = max_i sum_j |a^F_ij| / |a^F_ii|: rows 2, 7 = 21.12 / 12 = 1.76; row 4 = 9 / 5 = 1.8; row 1 = 11 / 6;")
    L.append("#    row 3 = 20 / 11; row 8 = (7 + 1 + 5) / 7 = 13 / 7; rows 5, 9 = (4.5 + 4) / 4.5 = 17 / 9 (the max, set by the lumping)")
    L.append("#    -> rho = 17/9, omega = 4 / (3 rho) = 12/17 = 0.70588235...")
    L.append("#  P_4,0 = 1 - (omega / 5) (5 + a_47) = 1 - (12/85) * 3 = 0.576470588...; P_4,2 = -(12/85) * (-2) = 0.28235294...")
    L.append("# format: 'n N', 'zb ...', 'entry i j a_ij' (row-major, ascending j), 'edge i j' (i < j), 'state i s'")
    L.append("# (-1 isolated, 1 root, 2 out), 'ph1 i a', 'agg i a', 'rho x', 'omega x', 'P i J value' (nonzeros, repr)")
    L.append(f"n {N}")
    L.append("zb " + " ".join(str(int(z)) for z in ZB))
    for i in range(N):
        for j in range(N):
            if A[0, i, j] != 0.0 or i == j:
                L.append(f"entry {i} {j} {float(A[0, i, j])!r}")
    E = r["E"]
    for i in range(N):
        for j in range(i + 1, N):
            if E[i, j]:
                L.append(f"edge {i} {j}")
    for i in range(N):
        L.append(f"state {i} {int(r['st'][i])}")
    for i in range(N):
        L.append(f"ph1 {i} {int(r['ph1'][i])}")
    for i in range(N):
        L.append(f"agg {i} {int(r['agg'][i])}")
    L.append(f"rho {float(r["rho"][0])!r}")
    L.append(f"omega {float(r["omega"][0])!r}")
    P = r["P"][0]
    for i in range(N):
        for J in range(r["nagg"]):
            if P[i, J] != 0.0:
                L.append(f"P {i} {J} {float(P[i, J])!r}")
    with open(os.path.join(HERE, "sa_level.txt"), "w") as f:
        f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    main()
