"""CPU check of the rotated blocked form the sm_100a kernels run for L = 3, 4 (bondr_step, one
pair per thread) and L = 5 (deep_sweep_bondr, one thread per 2 x 2-block column): lower-level
passes on the block rows and columns, then per block the L = 2-type step whose eight
coefficients are chosen by the top-level selectors (TR, TC) — the branch-free table
bondr_coef in qk_sweep.cu — restated in numpy and checked against the reference's own golden
amplitudes.  Row and column passes are applied in the alternating order of the L = 5 kernel
(they commute).  Test-only restatement: the product computes these on the GPU."""
import numpy as np
import pytest

from conftest import load_golden


def coef(tr, tc, C, D, p1, q1, p2, q2):
    """(a0, b0, a1, b1, a2, b2, a3, b3) of qk_sweep.cu bondr_coef."""
    opc, cm1 = 1.0 + C, C - 1.0
    if tr == tc:
        s = -1.0 if tr else 1.0
        return opc, s * q1, cm1, s * p2, s * p1, -D, s * q2, D
    s = 1.0 if tr else -1.0
    return s * D, p1, s * D, -q2, -q1, s * opc, p2, -s * cm1


def rotate(V, axis, k, c, s):
    """Level k on block index `axis` (0 rows, 1 columns): pairs differing in bit k, selected by
    bit k - 1 (qk_sweep.cu rot_pair)."""
    H = V.shape[axis]
    out = V.copy()
    for b in range(H):
        if b & (1 << k):
            continue
        b1 = b | (1 << k)
        sel = 0 if k == 0 else (b >> (k - 1)) & 1
        p, q = (-s, c) if sel else (c, s)
        x0 = V[b] if axis == 0 else V[:, b]
        x1 = V[b1] if axis == 0 else V[:, b1]
        y0, y1 = p * x0 + q * x1, q * x0 + p * x1
        if axis == 0:
            out[b], out[b1] = y0, y1
        else:
            out[:, b], out[:, b1] = y0, y1
    return out


def blocked_amplitude(xi, xj, layers):
    M = layers - 1
    H = 1 << (M - 1)
    V = np.zeros((H, H, 4))
    V[0, 0, 0] = V[0, 0, 2] = 1.0
    for q in range(len(xi)):
        ci, si, cj, sj = np.cos(xi[q] / 2), np.sin(xi[q] / 2), np.cos(xj[q] / 2), np.sin(xj[q] / 2)
        ai, bi = ci * ci - si * si, 2 * ci * si
        aj, bj = cj * cj - sj * sj, 2 * cj * sj
        C, D = bi * bj + ai * aj, ai * bj - bi * aj
        p1, q1, p2, q2 = ai + aj, bi + bj, bj - bi, ai - aj
        sides = [(0, ci, si), (1, cj, sj)]
        for axis, c, s in (sides if q % 2 == 0 else sides[::-1]):
            for k in range(M - 1):
                V = rotate(V, axis, k, c, s)
        W = V.copy()
        for r in range(H):
            for cc in range(H):
                a0, b0, a1, b1, a2, b2, a3, b3 = coef((r >> (M - 2)) & 1, (cc >> (M - 2)) & 1,
                                                      C, D, p1, q1, p2, q2)
                S, Dg, T, E = V[r, cc]
                W[r, cc] = (a0 * S + b0 * Dg, a1 * T + b1 * E, a2 * T + b2 * E, a3 * S + b3 * Dg)
        V = W
    return float((V[..., 0] + V[..., 1]).sum()) * 2.0 ** -len(xi)


@pytest.mark.parametrize("name", ["gram_n6_L3", "gram_n5_L4", "gram_n5_L5", "pairs_n24_L4",
                                  "pairs_n24_L5"])
def test_blocked_form_matches_reference_golden(name):
    g = load_golden(name)
    L = int(g["layers"])
    pairs = g["pairs"][:12]
    for (p, q), want in zip(pairs, g["amp_re"][:12]):
        got = blocked_amplitude(g["A"][p], g["B"][q], L)
        assert abs(got - want) <= 1e-12 * max(1.0, abs(want)), (name, p, q, got, want)


def test_coefficient_table_is_the_four_block_steps():
    """bondr_coef's branch-free table against the four specialised block_step variants."""
    rng = np.random.default_rng(0)
    C, D, p1, q1, p2, q2 = rng.normal(size=6)
    S, Dg, T, E = rng.normal(size=4)
    ref = {
        (0, 0): (C * S + S + q1 * Dg, p2 * E + C * T - T, p1 * T - D * E, q2 * S + D * Dg),
        (0, 1): (p1 * Dg - D * S, -q2 * E - D * T, -q1 * T - (C * E + E), p2 * S + C * Dg - Dg),
        (1, 0): (p1 * Dg + D * S, -q2 * E + D * T, -q1 * T + C * E + E, p2 * S - C * Dg + Dg),
        (1, 1): (C * S + S - q1 * Dg, -p2 * E + C * T - T, -D * E - p1 * T, D * Dg - q2 * S),
    }
    for (tr, tc), want in ref.items():
        a0, b0, a1, b1, a2, b2, a3, b3 = coef(tr, tc, C, D, p1, q1, p2, q2)
        got = (a0 * S + b0 * Dg, a1 * T + b1 * E, a2 * T + b2 * E, a3 * S + b3 * Dg)
        assert np.allclose(got, want, rtol=1e-13, atol=1e-13), (tr, tc)
