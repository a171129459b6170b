"""The paper's byte model (Tables 1-4) re-derived under the conventions of SURVEY.md
App. B and compared with every printed cell (rounded as printed).  This pins the accounting the
bench and DESIGN.md use for context (B200 speed-of-light figures come from the same formulas).

Conventions (App. B): MB = 1e6 B; 100^3 hexes, N = 101^3 nodes; bandwidths implied by the
tables: V100 900 GB/s, A100 1935 GB/s, MI250X 1638.4 GB/s; nnz = 27 / 81 per row; 12 B per
non-zero; the Table 1 totals include 8-B row offsets; Table 2 ranges = each nodal value
read once .. read once per incident cell (8); Table 3 quadrature storage 8 values per cell x 6 /
21 doubles; Table 4 = two streams of N c doubles per row; throughputs are computed from the
printed (rounded) MB totals.
"""
from __future__ import annotations

import pytest

E = 100 ** 3
N = 101 ** 3
BW = {"V100": 900e9, "A100": 1935e9, "MI250X": 1638.4e9}
MB = 1e6


def close(value, printed, sig):
    """`value` rounds to the printed number at its printed precision (sig = decimals)."""
    return round(value, sig) == pytest.approx(printed, abs=0.5 * 10 ** -sig + 1e-12)


def table1(c):
    rows = N * c
    nnz = 27 * c * rows
    matrix = nnz * 12
    offsets = (rows + 1) * 8
    vectors = 2 * rows * 8
    total = matrix + offsets + vectors
    return rows, matrix, offsets, vectors, total


def test_table1_spmv():
    rows, matrix, off, vec, total = table1(1)
    assert rows == 1_030_301
    assert close((matrix + off) / MB, 342.1, 1)          # printed 343 (App. B: incl. offsets)
    assert round(vec / MB) == 16 and round(total / MB) == 359
    t = {k: total / b * 1e3 for k, b in BW.items()}
    assert close(t["V100"], 0.40, 2) and close(t["A100"], 0.19, 2) and close(t["MI250X"], 0.22, 2)
    gd = {k: rows / (total / b) / 1e9 for k, b in BW.items()}
    assert close(gd["V100"], 2.6, 1) and close(gd["A100"], 5.6, 1) and close(gd["MI250X"], 4.7, 1)
    rows, matrix, off, vec, total = table1(3)
    assert rows == 3_090_903
    assert round(matrix / MB) == 3004 and round(vec / MB) == 49 and round(total / MB) == 3079
    t = {k: total / b * 1e3 for k, b in BW.items()}
    assert close(t["V100"], 3.4, 1) and close(t["A100"], 1.6, 1) and close(t["MI250X"], 1.9, 1)
    gd = {k: rows / (total / b) / 1e9 for k, b in BW.items()}
    assert close(gd["V100"], 0.90, 2) and close(gd["A100"], 1.9, 1) and close(gd["MI250X"], 1.6, 1)


def mf_range(c, cell_const):
    node_map = E * 8 * 4
    best = node_map + cell_const * E + N * 24 + 3 * N * c * 8
    worst = node_map + cell_const * E + E * 8 * 24 + 3 * E * 8 * c * 8
    return best, worst


def test_table2_matrix_free():
    assert round(E * 8 * 4 / MB) == 32
    for c, C, tot, gd in [(1, 0, (81, 416), {"V100": (11, 2.2), "A100": (25, 4.8), "MI250X": (21, 4.1)}),
                          (3, 16, (147, 816), {"V100": (19, 3.4), "A100": (41, 7.3), "MI250X": (34, 6.2)})]:
        best, worst = mf_range(c, C)
        assert round(best / MB) == tot[0] and round(worst / MB) == tot[1]
        for k, b in BW.items():  # throughputs follow the PRINTED (rounded) totals
            hi, lo = N * c / (tot[0] * MB / b) / 1e9, N * c / (tot[1] * MB / b) / 1e9
            assert close(hi, gd[k][0], 0 if gd[k][0] >= 10 else 1), (k, hi)
            assert close(lo, gd[k][1], 1), (k, lo)


def test_table3_partial_assembly():
    for c, vals, qmb, tot in [(1, 6, 384, (441, 608)), (3, 21, 1344, (1450, 1952))]:
        q = E * 8 * vals * 8
        assert round(q / MB) == qmb
        node_map = E * 8 * 4
        best = node_map + q + 3 * N * c * 8
        worst = node_map + q + 3 * E * 8 * c * 8
        # (App. B: the elasticity totals leave out the 16 MB cell-constant line)
        assert round(best / MB) == tot[0] and round(worst / MB) == tot[1]


def test_table4_cg_streams():
    assert close(2 * N * 1 * 8 / MB, 16.5, 1)
    assert close(2 * N * 3 * 8 / MB, 49.5, 1)
