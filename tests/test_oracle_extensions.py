"""Known-answer tests pinning the oracle's EXTENSION semantics (no reference counterpart:
RK4, logistic, Lotka-Volterra, bracket search, bilinear maps, closed-form weights, tree
composition). These are "parity unpinned" against the reference; the KATs below are what pins them.
"""
import math

import numpy as np
import pytest

import oracle as O


def logistic_exact(y0, t, r=1.0, K=1.0):
    return K * y0 * math.exp(r * t) / (K + y0 * (math.exp(r * t) - 1.0))


def test_logistic_rk4_matches_exact_solution():
    _, _, st, h = O.decompose(0.0, 10.0, 64, 10.0 / (64 * 64))
    nodes = O.cheb_nodes(17, 0.0, 1.25)
    ends = O.logistic_rk4_ensemble(st, h, nodes, 1.0, 1.0)
    width = 10.0 / 64
    for m, y0 in enumerate(nodes):
        assert ends[3, m] == pytest.approx(logistic_exact(y0, width), abs=1e-11)


def test_logistic_rk4_is_fourth_order():
    errs = []
    for S in (4, 8, 16):
        _, _, st, h = O.decompose(0.0, 1.0, 1, 1.0 / S)
        e = O.logistic_rk4_ensemble(st, h, [0.1], 1.0, 1.0)[0, 0]
        errs.append(abs(e - logistic_exact(0.1, 1.0)))
    p1 = math.log2(errs[0] / errs[1])
    p2 = math.log2(errs[1] / errs[2])
    assert 3.7 < p1 < 4.3 and 3.7 < p2 < 4.3


def test_logistic_f32_tracks_f64():
    _, _, st, h = O.decompose(0.0, 10.0, 8, 10.0 / (8 * 32))
    nodes = O.cheb_nodes(33, 0.0, 1.25)
    e64 = O.logistic_rk4_ensemble(st, h, nodes, 1.0, 1.0)
    e32 = O.logistic_rk4_ensemble_f32(st, h, nodes.astype(np.float32), 1.0, 1.0)
    assert np.max(np.abs(e32 - e64) / np.maximum(1e-30, np.abs(e64))) < 1e-5


def test_lv_rk4_conserves_first_integral():
    a, b, d, g = 1.5, 1.0, 1.0, 3.0
    V = lambda u, v: d * u - g * math.log(u) + b * v - a * math.log(v)
    _, _, st, h = O.decompose(0.0, 10.0, 16, 10.0 / (16 * 256))
    un = O.uniform_nodes(5, 0.5, 3.0)
    vn = O.uniform_nodes(4, 0.5, 2.0)
    out = O.lv_rk4_ensemble(st, h, un, vn, [a, b, d, g])
    for iu in range(5):
        for iv in range(4):
            assert V(out[2, 0, iu, iv], out[2, 1, iu, iv]) == pytest.approx(V(un[iu], vn[iv]), rel=1e-7)
    sub = O.lv_rk4_subset(2 * 20 + 7, 2 * 20 + 9, st, h, un, vn, [a, b, d, g])
    assert np.array_equal(sub[0], out[2, :, 1, 3])
    assert np.array_equal(sub[1], out[2, :, 2, 0])


def test_bracket_semantics():
    x = np.array([0.0, 1.0, 2.0, 3.0])
    assert [O.bracket(x, q) for q in (-1.0, 0.0, 0.5, 1.0, 2.999, 3.0, 7.0)] == [0, 0, 0, 1, 2, 2, 2]
    xs = np.sort(np.random.default_rng(1304).uniform(0, 10, 100))
    for q in np.random.default_rng(7).uniform(-1, 11, 500):
        expect = min(max(int(np.searchsorted(xs, q, side="right")) - 1, 0), 98)
        assert O.bracket(xs, q) == expect


def test_bilinear_exact_on_bilinear_maps():
    un = O.uniform_nodes(9, 0.1, 8.0)
    vn = O.uniform_nodes(7, 0.1, 8.0)
    U, V = np.meshgrid(un, vn, indexing="ij")
    N = 3
    tables = np.empty((N, 2, 9, 7))
    # each slice map: u -> 0.9u + 0.01uv + 0.3, v -> 0.8v + 0.2  (bilinear in (u, v))
    for j in range(N):
        tables[j, 0] = 0.9 * U + 0.01 * U * V + 0.3
        tables[j, 1] = 0.8 * V + 0.2
    lam, br, ext = O.bilinear_sweep(un, vn, tables, 1.3, 2.2)
    u, v = 1.3, 2.2
    for j in range(N):
        u, v = 0.9 * u + 0.01 * u * v + 0.3, 0.8 * v + 0.2
        assert lam[j, 0] == pytest.approx(u, rel=1e-13)
        assert lam[j, 1] == pytest.approx(v, rel=1e-13)
    assert ext == 0
    assert br[0, 0] == O.bracket(un, 1.3) and br[0, 1] == O.bracket(vn, 2.2)


def test_closed_form_weights_agree_with_product_form_up_to_scale():
    for M in (5, 33, 512):
        x = O.cheb_nodes(M, 0.0, 2.0)
        wp = O.bary_weights(x)
        wc = O.bary_weights_closed2(M)
        ratio = wp / wc
        assert np.max(np.abs(ratio / ratio[0] - 1.0)) < 1e-11
    # M = 1024: product form overflows (reference gives inf/NaN), closed form stays usable
    x = O.cheb_nodes(1024, 0.0, 2.0)
    wc = O.bary_weights_closed2(1024)
    v = np.exp(0.3 * x)
    assert O.interp_eval(x, wc, v, 0.777) == pytest.approx(math.exp(0.3 * 0.777), rel=1e-13)


def test_tree_matches_chain():
    rng = np.random.default_rng(1304)
    N, n = 13, 6
    G = rng.uniform(-0.4, 0.4, (N, n, n))
    c = rng.uniform(-1, 1, (N, n))
    y0 = rng.uniform(-1, 1, n)
    chain = O.affine_chain(G, c, y0)
    _, _, tree = O.affine_tree(G, c, y0)
    assert np.max(np.abs(tree - chain)) <= 1e-13 * max(1.0, np.max(np.abs(chain)))
