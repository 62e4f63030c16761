"""Pins for the fp64 CPU oracle (CPU only, no GPU).

Each test checks the oracle against something other than itself: hand values
(tests/golden/, cited), closed forms, an independent library routine used as a
special case (numpy.linalg.eigh / norm / matmul), brute force on tiny inputs,
or an exact invariant stated in the paper.  See DESIGN.md "Oracle pins".
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rand_sym(rng, d, scale=1.0):
    A = rng.standard_normal((d, d)) * scale
    return 0.5 * (A + A.T)


# ---------------------------------------------------------------- step 1: sigma
def test_sigma_golden():
    g = _gold("spec_hand_examples.json")
    for key in ("sigma_all_ones_4x3", "sigma_single_row"):
        Qw = np.array(g[key]["Qw"], dtype=float)[None, None]          # [U=1, G=1, W, d]
        np.testing.assert_array_equal(orc.query_sigma(Qw)[0], g[key]["sigma"])


def test_sigma_pooled_gqa_matches_norm_of_concatenation():
    rng = np.random.default_rng(0)
    Qw = rng.standard_normal((3, 7, 32, 16))
    ref = np.linalg.norm(Qw.transpose(0, 3, 1, 2).reshape(3, 16, -1), axis=2)   # reading Q4
    np.testing.assert_allclose(orc.query_sigma(Qw), ref, rtol=1e-14)


def test_sigma_w0_is_ones():
    Qw = np.zeros((2, 1, 0, 8))
    np.testing.assert_array_equal(orc.query_sigma(Qw), np.ones((2, 8)))


# ---------------------------------------------------------------- step 2: mu, C
def test_cov_golden():
    g = _gold("spec_hand_examples.json")
    mu, C = orc.mean_cov(np.array(g["cov_two_keys"]["K"], float)[None])
    np.testing.assert_array_equal(mu[0], g["cov_two_keys"]["mu"])
    np.testing.assert_array_equal(C[0], g["cov_two_keys"]["C"])
    _, C1 = orc.mean_cov(np.array(g["cov_single_key"]["K"], float)[None])
    np.testing.assert_array_equal(C1[0], g["cov_single_key"]["C"])


def test_cov_two_pass_equals_one_pass_and_psd():
    rng = np.random.default_rng(1)
    K = rng.standard_normal((2, 64, 16)) + 3.0
    mu, C = orc.mean_cov(K)
    # different algorithm: one-pass K^T K - N mu mu^T with numpy's mean
    m = K.mean(axis=1)
    one = np.einsum("uni,unj->uij", K, K) - 64 * np.einsum("ui,uj->uij", m, m)
    np.testing.assert_allclose(mu, m, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(C, one, rtol=1e-10, atol=1e-10)
    for u in range(2):
        assert np.linalg.eigvalsh(C[u]).min() > -1e-10
        np.testing.assert_array_equal(C[u], C[u].T)


def test_cov_uncentered_is_KtK():
    rng = np.random.default_rng(2)
    K = rng.standard_normal((1, 40, 8))
    mu, C = orc.mean_cov(K, center=False)
    np.testing.assert_array_equal(mu, 0.0)
    np.testing.assert_allclose(C[0], K[0].T @ K[0], rtol=1e-13)


# ---------------------------------------------------------------- step 3: Hadamard
def test_hadamard_identity_equals_gram_of_weighted_keys():
    """(sigma sigma^T) (.) C == K_q^T K_q with K_q = (K - mu) diag(sigma)."""
    rng = np.random.default_rng(3)
    K = rng.standard_normal((2, 50, 12)) + 1.0
    Qw = rng.standard_normal((2, 3, 5, 12))
    sig = orc.query_sigma(Qw)
    mu, C = orc.mean_cov(K)
    Cq = orc.hadamard(C, sig)
    Kq = (K - K.mean(axis=1, keepdims=True)) * sig[:, None, :]
    np.testing.assert_allclose(Cq, np.einsum("uni,unj->uij", Kq, Kq), rtol=1e-11, atol=1e-11)


# ---------------------------------------------------------------- step 4: Jacobi
def test_jacobi_golden():
    g = _gold("spec_hand_examples.json")
    lam, V, sw = orc.jacobi(np.array(g["eig_diag"]["A"], float))
    np.testing.assert_array_equal(lam, g["eig_diag"]["lam"])
    np.testing.assert_array_equal(V, np.eye(2))
    assert sw == 0
    lam, V, sw = orc.jacobi(np.array(g["eig_2x2"]["A"], float))
    order = np.argsort(-lam)
    np.testing.assert_allclose(lam[order], g["eig_2x2"]["lam_desc"], rtol=1e-15)
    ref = np.array(g["eig_2x2"]["vecs_desc_up_to_sign"])
    for k, j in enumerate(order):
        assert abs(abs(V[:, j] @ ref[k]) - 1.0) < 1e-15


@pytest.mark.parametrize("d", [2, 5, 16, 64, 128])
def test_jacobi_invariants_and_numpy_eigh(d):
    rng = np.random.default_rng(d)
    A = _rand_sym(rng, d)
    lam, V, sw = orc.jacobi(A)
    assert sw > 0
    np.testing.assert_allclose(V.T @ V, np.eye(d), atol=1e-13)
    np.testing.assert_allclose(V @ np.diag(lam) @ V.T, A, atol=1e-12 * np.linalg.norm(A))
    assert abs(lam.sum() - np.trace(A)) <= 1e-12 * np.abs(A).sum()
    np.testing.assert_allclose(np.sort(lam), np.linalg.eigvalsh(A), atol=1e-12 * np.linalg.norm(A))
    # sign convention: largest-|entry| positive
    for j in range(d):
        assert V[np.argmax(np.abs(V[:, j])), j] > 0


def test_jacobi_projector_matches_eigh_on_gap_matrix():
    rng = np.random.default_rng(7)
    d, r = 32, 6
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    s = np.concatenate([np.linspace(9, 4, r), np.linspace(0.5, 0.01, d - r)])
    A = (Q * s) @ Q.T
    lam, V, _ = orc.jacobi(A)
    top = np.argsort(-lam)[:r]
    P = V[:, top] @ V[:, top].T
    w, E = np.linalg.eigh(A)
    Pref = E[:, -r:] @ E[:, -r:].T
    assert np.linalg.norm(P - Pref) < 1e-12


def test_jacobi_nonfinite():
    A = np.eye(4)
    A[1, 2] = A[2, 1] = np.nan
    _, _, sw = orc.jacobi(A)
    assert sw == -1000000


# ---------------------------------------------------------------- step 5: select
def _brute_select(lam, r):
    order = sorted(range(len(lam)), key=lambda i: (-lam[i], i))
    keep = sorted(order[:r])
    return keep


@pytest.mark.parametrize("case", ["random", "ties", "all_equal", "zeros_signed", "denorm"])
def test_select_brute_force(case):
    rng = np.random.default_rng(11)
    d = 40
    if case == "random":
        lam = rng.standard_normal(d)
    elif case == "ties":
        lam = rng.integers(0, 5, d).astype(float)
    elif case == "all_equal":
        lam = np.full(d, 2.5)
    elif case == "zeros_signed":
        lam = np.where(rng.random(d) < 0.5, 0.0, -0.0)
        lam[::7] = 1.0
    else:
        lam = rng.integers(0, 3, d) * 5e-324
    for r in (1, 3, 16, 39, 40):
        mask, idx = orc.select_topr(lam, r)
        keep = _brute_select(list(lam), r)
        assert list(idx) == keep
        bits = [i for i in range(d) if mask[i // 32] >> (i % 32) & 1]
        assert bits == keep


def test_select_nan():
    lam = np.array([1.0, np.nan, 0.5])
    assert orc.select_topr(lam, 1) is None


# ---------------------------------------------------------------- step 6: R_r, dmu
def test_rotation_orthonormal_and_residual_orthogonal():
    rng = np.random.default_rng(12)
    d, r = 24, 7
    lam, V, _ = orc.jacobi(_rand_sym(rng, d))
    _, idx = orc.select_topr(lam, r)
    mu = rng.standard_normal(d)
    R, dmu = orc.rotation(V, idx, mu)
    np.testing.assert_array_equal(R, V[:, idx])
    np.testing.assert_allclose(R.T @ R, np.eye(r), atol=1e-13)
    np.testing.assert_allclose(R.T @ dmu, 0.0, atol=1e-13)
    np.testing.assert_allclose(R @ (R.T @ mu) + dmu, mu, atol=1e-13)
    # r = d: P = I so dmu = 0
    _, idx_all = orc.select_topr(lam, d)
    _, dmu_all = orc.rotation(V, idx_all, mu)
    np.testing.assert_allclose(dmu_all, 0.0, atol=1e-13)


def test_dmu_from_R_invariants():
    """orc_dmu_from_R (Alg. 1 l.15: delta_mu = mu - R R^T mu for a given, e.g. stored
    fp32, R) pinned by what the projection must satisfy, not by retyping it:
      * orthonormal R: delta_mu is orthogonal to range(R) and Pythagoras holds;
      * mu in range(R) gives 0, mu orthogonal to range(R) gives mu itself;
      * non-orthonormal stored-fp32 R (what the GPU holds): R^T delta_mu = (I - R^T R) R^T mu,
        i.e. of the size of R's rounding, and the decomposition R(R^T mu) + delta_mu = mu;
      * linear in mu, batched per unit (a unit/row mix-up fails the per-unit checks)."""
    rng = np.random.default_rng(31)
    U, d, r = 3, 24, 7
    Q = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(U)])
    R = np.ascontiguousarray(Q[:, :, :r])
    mu = rng.standard_normal((U, d)) * np.array([1.0, 10.0, 0.1])[:, None]
    dmu = orc.dmu_from_R(R, mu)
    for u in range(U):
        assert np.abs(R[u].T @ dmu[u]).max() <= 1e-13 * np.abs(mu[u]).max() * d
        proj2 = float(np.sum((R[u].T @ mu[u]) ** 2))
        assert abs(np.sum(dmu[u] ** 2) - (np.sum(mu[u] ** 2) - proj2)) <= 1e-12 * np.sum(mu[u] ** 2)
    inside = np.einsum("udr,ur->ud", R, rng.standard_normal((U, r)))
    np.testing.assert_allclose(orc.dmu_from_R(R, inside), 0.0, atol=1e-13)
    outside = np.einsum("udk,uk->ud", Q[:, :, r:], rng.standard_normal((U, d - r)))
    np.testing.assert_allclose(orc.dmu_from_R(R, outside), outside, atol=1e-13)
    # stored fp32 R: not exactly orthonormal; the residual's component in range(R) is exactly
    # (I - R^T R) R^T mu, which is of the order of R's rounding
    R32 = R.astype(np.float32).astype(np.float64)
    d32 = orc.dmu_from_R(R32, mu)
    for u in range(U):
        got = R32[u].T @ d32[u]
        want = (np.eye(r) - R32[u].T @ R32[u]) @ (R32[u].T @ mu[u])
        np.testing.assert_allclose(got, want, atol=1e-12 * np.abs(mu[u]).max())
        assert np.abs(got).max() <= 1e-6 * np.abs(mu[u]).max()
    # linearity
    np.testing.assert_allclose(orc.dmu_from_R(R32, 3.0 * mu - 2.0 * inside),
                               3.0 * d32 - 2.0 * orc.dmu_from_R(R32, inside), atol=1e-12 * np.abs(mu).max())


def test_eckart_young_brute_force():
    """Captured variance tr(R_r^T C_q R_r) = sum of the top-r eigenvalues and is
    >= the variance of every coordinate subset of size r (the `\\iffalse`
    proposition)."""
    rng = np.random.default_rng(13)
    d, r = 10, 3
    K = rng.standard_normal((1, 30, d)) @ rng.standard_normal((d, d))
    Qw = rng.standard_normal((1, 1, 8, d))
    cal = orc.calibrate(K, Qw, r)
    Cq, R = cal["Cq"][0], cal["R"][0]
    cap = np.trace(R.T @ Cq @ R)
    np.testing.assert_allclose(cap, np.sort(cal["lam"][0])[-r:].sum(), rtol=1e-12)
    best_subset = max(sum(Cq[i, i] for i in s) for s in itertools.combinations(range(d), r))
    assert cap >= best_subset - 1e-9


# ---------------------------------------------------------------- step 7: K~ and rounding
def test_compress_full_rank_is_lossless():
    """r = d: K~ R^T = K R R^T = K (Eq. rotation-lossless)."""
    rng = np.random.default_rng(14)
    K = rng.standard_normal((2, 20, 8))
    Qw = rng.standard_normal((2, 1, 4, 8))
    cal = orc.calibrate(K, Qw, 8)
    Kt = orc.compress(K, cal["R"])
    np.testing.assert_allclose(np.einsum("unr,uir->uni", Kt, cal["R"]), K, atol=1e-13)


def test_round_bf16_hand_cases():
    rb = orc.round_bf16_scalar
    assert rb(1.0 + 2.0 ** -8) == 1.0                       # tie -> even
    assert rb(1.0 + 3 * 2.0 ** -8) == 1.0 + 2.0 ** -6          # tie -> even (up)
    assert rb(1.0 + 2.0 ** -8 + 2.0 ** -40) == 1.0 + 2.0 ** -7  # no double rounding
    assert rb(-(1.0 + 2.0 ** -8 + 2.0 ** -40)) == -(1.0 + 2.0 ** -7)
    assert rb(2.0 ** -130) == 2.0 ** -130                      # subnormal, exact
    assert rb(2.0 ** -134) == 0.0                               # half quantum -> even (0)
    assert rb(3 * 2.0 ** -134) == 2.0 ** -132                   # 1.5 quanta -> 2
    bmax = (2 - 2.0 ** -7) * 2.0 ** 127
    assert rb(bmax) == bmax
    assert rb((2 - 2.0 ** -8) * 2.0 ** 127) == math.inf        # tie beyond max -> inf
    assert rb(0.0) == 0.0 and math.copysign(1, rb(-0.0)) == -1


def test_round_bf16_matches_torch_on_f32_values():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(15)
    x = (rng.standard_normal(20000) * np.exp(rng.uniform(-20, 20, 20000))).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(orc.quantize(x.astype(np.float64), "bf16"), ref)
    np.testing.assert_array_equal(orc.quantize(x.astype(np.float64) * (1 + 1e-12), "f32"),
                                  x.astype(np.float64) * 0 + (x.astype(np.float64) * (1 + 1e-12)).astype(np.float32))


# ---------------------------------------------------------------- step 8: decode
def _attn(q, K, V, scale):
    s = (K @ q) * scale
    p = np.exp(s - s.max())
    return p @ V / p.sum()


def test_decode_full_rank_equals_standard_attention():
    """r = d with an orthogonal R reproduces unrotated attention (Eq. 1)."""
    rng = np.random.default_rng(16)
    U, G, d, N, M = 2, 3, 16, 37, 5
    K = rng.standard_normal((U, N, d)) + 0.5
    V = rng.standard_normal((U, N, d))
    Kx, Vx = rng.standard_normal((U, M, d)), rng.standard_normal((U, M, d))
    q = rng.standard_normal((U, G, d))
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(U)])
    dmu = np.zeros((U, d))
    out = orc.decode(q, orc.compress(K, R), V, R, dmu, Kx, Vx)
    for u in range(U):
        for g in range(G):
            ref = _attn(q[u, g], np.vstack([K[u], Kx[u]]), np.vstack([V[u], Vx[u]]), 1 / math.sqrt(d))
            np.testing.assert_allclose(out[u, g], ref, atol=1e-12)


def test_partial_states_merge_to_brute_force_attention():
    """Token-shard states (App. C online-softmax state) merged over any split
    equal brute-force softmax attention over the whole cache (r = d, orthogonal R so that
    the scores are standard attention; pins decode_partial / merge_partials independently
    of orc.decode), and a single shard's state has l = sum 2^(z - max z) with m the max."""
    rng = np.random.default_rng(23)
    U, G, d, N, M = 2, 2, 8, 29, 4
    K = rng.standard_normal((U, N, d))
    V = rng.standard_normal((U, N, d))
    Kx, Vx = rng.standard_normal((U, M, d)), rng.standard_normal((U, M, d))
    q = rng.standard_normal((U, G, d))
    R = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(U)])
    Kt = orc.compress(K, R)
    for cuts, xcuts in [([0, 29], [0, 4]), ([0, 1, 29], [0, 4, 4]), ([0, 10, 11, 29], [0, 0, 1, 4])]:
        parts = np.stack([orc.decode_partial(q, Kt[:, a:b], V[:, a:b], R, None,
                                             Kx[:, xa:xb], Vx[:, xa:xb])
                          for a, b, xa, xb in zip(cuts, cuts[1:], xcuts, xcuts[1:])])
        out = orc.merge_partials(parts)
        for u in range(U):
            for g in range(G):
                ref = _attn(q[u, g], np.vstack([K[u], Kx[u]]), np.vstack([V[u], Vx[u]]),
                            1 / math.sqrt(d))
                np.testing.assert_allclose(out[u, g], ref, atol=1e-12)
    one = orc.decode_partial(q, Kt, V, R, None, Kx, Vx)
    z = np.concatenate([np.einsum("gd,nd->gn", q[0], K[0]), np.einsum("gd,nd->gn", q[0], Kx[0])],
                       axis=1) / math.sqrt(d) * math.log2(math.e)
    np.testing.assert_allclose(one[0, :, -2], z.max(axis=1), atol=1e-12)
    np.testing.assert_allclose(one[0, :, -1], np.exp2(z - z.max(axis=1, keepdims=True)).sum(axis=1),
                               rtol=1e-12)


def test_decode_single_token_and_zero_query():
    rng = np.random.default_rng(17)
    d, r = 8, 3
    R = np.linalg.qr(rng.standard_normal((d, d)))[0][:, :r][None]
    V1 = rng.standard_normal((1, 1, d))
    out = orc.decode(rng.standard_normal((1, 1, d)), rng.standard_normal((1, 1, r)), V1, R,
                     rng.standard_normal((1, d)))
    np.testing.assert_array_equal(out[0, 0], V1[0, 0])
    V = rng.standard_normal((1, 9, d))
    Vx = rng.standard_normal((1, 4, d))
    out = orc.decode(np.zeros((1, 1, d)), rng.standard_normal((1, 9, r)), V, R,
                     rng.standard_normal((1, d)), rng.standard_normal((1, 4, d)), Vx)
    np.testing.assert_allclose(out[0, 0], np.vstack([V[0], Vx[0]]).mean(axis=0), atol=1e-14)


def test_decode_bias_irrelevant_without_text():
    """M = 0: b_t is constant over all tokens, softmax is shift invariant."""
    rng = np.random.default_rng(18)
    U, G, d, r, N = 1, 2, 12, 4, 30
    args = (rng.standard_normal((U, G, d)), rng.standard_normal((U, N, r)),
            rng.standard_normal((U, N, d)), rng.standard_normal((U, d, r)))
    a = orc.decode(*args, rng.standard_normal((U, d)))
    b = orc.decode(*args, None)
    np.testing.assert_allclose(a, b, atol=1e-13)


def test_decode_scale_is_sqrt_d_not_sqrt_r():
    """Text-segment scores do not depend on r (Alg. 2 line 4, reading Q12)."""
    rng = np.random.default_rng(19)
    d, N, M = 16, 10, 6
    q = rng.standard_normal((1, 1, d))
    Kx = rng.standard_normal((1, M, d))
    s_a = orc.scores(q, rng.standard_normal((1, N, 2)), rng.standard_normal((1, d, 2)), None, Kx)
    s_b = orc.scores(q, rng.standard_normal((1, N, 9)), rng.standard_normal((1, d, 9)), None, Kx)
    np.testing.assert_array_equal(s_a[..., N:], s_b[..., N:])
    np.testing.assert_allclose(s_a[0, 0, N:], Kx[0] @ q[0, 0] / 4.0, rtol=1e-14)


def test_residual_identity():
    """exact - approx = q (I - P_r)(K - 1 mu^T)^T / sqrt(d) per visual token
    (Eq. approx-error P:158-162 plus the mean bias P:188)."""
    rng = np.random.default_rng(20)
    d, r, N = 16, 5, 50
    K = rng.standard_normal((1, N, d)) @ rng.standard_normal((d, d)) + 2.0
    Qw = rng.standard_normal((1, 1, 8, d))
    q = rng.standard_normal((1, 1, d))
    cal = orc.calibrate(K, Qw, r)
    R = cal["R"][0]
    approx = orc.scores(q, orc.compress(K, cal["R"]), cal["R"], cal["dmu"])[0, 0]
    exact = K[0] @ q[0, 0] / 4.0
    mu = K[0].mean(axis=0)
    resid = (K[0] - mu) @ (np.eye(d) - R @ R.T) @ q[0, 0] / 4.0
    np.testing.assert_allclose(exact - approx, resid, atol=1e-12)


def test_constant_keys_exact_for_any_r():
    rng = np.random.default_rng(21)
    d, N = 12, 20
    K = np.repeat(rng.standard_normal((1, 1, d)), N, axis=1)
    V = rng.standard_normal((1, N, d))
    q = rng.standard_normal((1, 1, d))
    for r in (1, 4, 12):
        cal = orc.calibrate(K, rng.standard_normal((1, 1, 8, d)), r)
        out = orc.decode(q, orc.compress(K, cal["R"]), V, cal["R"], cal["dmu"])
        np.testing.assert_allclose(out[0, 0], _attn(q[0, 0], K[0], V[0], d ** -0.5), atol=1e-12)


def test_low_rank_keys_exact_query_agnostic():
    """Centered keys of rank <= r are reproduced exactly by K-only PCA (W=0)."""
    rng = np.random.default_rng(22)
    d, r, N = 16, 4, 40
    K = (rng.standard_normal((1, N, r)) @ rng.standard_normal((r, d))) + rng.standard_normal(d)
    V = rng.standard_normal((1, N, d))
    q = rng.standard_normal((1, 1, d)) * 2
    cal = orc.calibrate(K, None, r)
    out = orc.decode(q, orc.compress(K, cal["R"]), V, cal["R"], cal["dmu"])
    np.testing.assert_allclose(out[0, 0], _attn(q[0, 0], K[0], V[0], d ** -0.5), atol=1e-11)


def test_pipeline_f32_full_rank_close_to_exact():
    """End to end with r = d: only the fp32 quantisation point separates the
    output from exact attention."""
    from workload import CONFIGS, make_workload
    cfg = CONFIGS["toy"].with_(rank=16, dtype="f32", n_text=3)
    w = make_workload(cfg)
    out = orc.pipeline(w["K"].f64(), w["V"].f64(), w["Qw"].f64(), w["q"].f64(), 16, "f32",
                       w["Ktext"].f64(), w["Vtext"].f64())["out"]
    K = np.concatenate([w["K"].f64(), w["Ktext"].f64()], axis=1)[0]
    V = np.concatenate([w["V"].f64(), w["Vtext"].f64()], axis=1)[0]
    ref = _attn(w["q"].f64()[0, 0], K, V, 0.25)
    np.testing.assert_allclose(out[0, 0], ref, atol=1e-5 * np.abs(ref).max())


# ---------------------------------------------------------------- budget arithmetic
def test_budget_matches_paper_tables():
    g = _gold("budget_tables.json")
    for row in g["rows"]:
        m = orc.budget(row["token"], row["channel"])
        assert round(m + 1e-12, 2) == row["printed"], row
    assert orc.budget(1.0, 1.0) == 1.0


def _planted(rng, U, N, d, r, mean=0.5):
    """Keys with a planted top-r subspace (gap >> 1) per unit."""
    out = np.empty((U, N, d))
    for u in range(U):
        Qo = np.linalg.qr(rng.standard_normal((d, d)))[0]
        s = np.concatenate([np.linspace(3, 1, r), np.full(d - r, 0.05)])
        out[u] = (rng.standard_normal((N, d)) * s) @ Qo.T + mean
    return out


def test_calib_state_pools_samples_and_token_shards():
    """NEXT-3 / token-sharded calibration: Alg. 1 from accumulated sums.
    (1) one unit per entry reproduces calibrate() (one-pass S - n mu mu^T vs two-pass C);
    (2) splitting a unit's tokens over samples b (entries u % H) or over shards (states
        added) reproduces calibrate() on the whole unit -- the window pooled once (Q4)."""
    rng = np.random.default_rng(31)
    H, n, d, r, G, W = 2, 50, 16, 4, 2, 3
    K = _planted(rng, H, 3 * n, d, r)
    Qw = rng.standard_normal((H, G, W, d))
    ref = orc.calibrate(K, Qw, r)
    one = orc.calibrate_from_state(orc.calib_state(K, Qw, H), r)
    for h in range(H):
        P = one["R"][h] @ one["R"][h].T
        Pr = ref["R"][h] @ ref["R"][h].T
        assert np.linalg.norm(P - Pr) <= 1e-9
        np.testing.assert_allclose(one["dmu"][h], ref["dmu"][h], atol=1e-9)
        np.testing.assert_allclose(one["lam"][h].sum(), np.trace(ref["Cq"][h]), rtol=1e-10)
    # samples: unit b*H + h holds tokens [b n, (b+1) n) of head h; the window only in b = 0
    Ks = np.concatenate([K[:, b * n:(b + 1) * n] for b in range(3)], axis=0)
    Qs = np.concatenate([Qw] + [np.zeros_like(Qw)] * 2, axis=0)
    pooled = orc.calibrate_from_state(orc.calib_state(Ks, Qs, H), r)
    # token shards: two states added (an all-reduce), window in shard 0 only
    st = orc.calib_state(K[:, :70], Qw, H)
    st = orc.calib_state(K[:, 70:], None, H, state=st)
    shard = orc.calibrate_from_state(st, r)
    for res in (pooled, shard):
        for h in range(H):
            P = res["R"][h] @ res["R"][h].T
            Pr = ref["R"][h] @ ref["R"][h].T
            assert np.linalg.norm(P - Pr) <= 1e-9
            np.testing.assert_allclose(res["dmu"][h], ref["dmu"][h], atol=1e-9)
