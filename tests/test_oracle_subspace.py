"""Pins for the oracle's Cholesky-QR subspace iteration (NEXT-1; Alg. 1 lines 6-13)."""
import math

import numpy as np

from oracle import oracle as orc


def test_rank1_closed_form():
    """C = diag(4, 1), k = 1, V0 = (1, 1): after T steps V = (4^T, 1) / sqrt((16^T + 1)(1 + eps))
    (each step multiplies by C, then divides by sqrt((1 + eps) G) -- the k = 1 Cholesky)."""
    C = np.diag([4.0, 1.0])
    for T in (1, 2, 5):
        for eps in (0.0, 1e-6, 0.5):
            V = orc.subspace(C, np.array([[1.0], [1.0]]), T=T, eps=eps)
            # the ridge shrinks the norm by 1/sqrt(1+eps) each step, but the next C V then
            # Cholesky normalises again, so only the last step's factor survives
            ref = np.array([4.0 ** T, 1.0]) / math.sqrt(16.0 ** T + 1.0) / math.sqrt(1.0 + eps)
            np.testing.assert_allclose(V[:, 0], ref, rtol=1e-14)


def test_cholesky_qr_orthonormal_without_ridge():
    """eps = 0: V L^{-T} with L L^T = V^T V is exactly orthonormal."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((24, 24))
    C = A @ A.T
    V = orc.subspace(C, rng.standard_normal((24, 5)), T=3, eps=0.0)
    np.testing.assert_allclose(V.T @ V, np.eye(5), atol=1e-12)


def test_ridge_shrinks_gram_as_stated():
    """With the trace-scaled ridge, one step gives V^T V = L^{-1} G L^{-T} where
    L L^T = G + rho I, i.e. V^T V = I - rho (L^T L)^{-1}, whose eigenvalues are g / (g + rho)
    for the eigenvalues g of G (checked with numpy on W = C V0, G = W^T W, rho = eps tr(G)/k)."""
    rng = np.random.default_rng(1)
    A = rng.standard_normal((16, 16))
    C = A @ A.T
    V0 = rng.standard_normal((16, 4))
    eps = 1e-3
    V = orc.subspace(C, V0, T=1, eps=eps)
    W = C @ V0
    G = W.T @ W
    rho = eps * np.trace(G) / 4
    g = np.linalg.eigvalsh(G)
    np.testing.assert_allclose(np.linalg.eigvalsh(V.T @ V), np.sort(g / (g + rho)), atol=1e-12)
    # and span(V) = span(C V0)
    P = V @ np.linalg.pinv(V)
    np.testing.assert_allclose(P @ W, W, atol=1e-9 * np.abs(W).max())


def test_converges_to_eigh_projector_on_gap_matrix():
    """On a matrix with lambda_k / lambda_{k+1} = 5 the subspace converges to the top-k
    eigenspace of numpy.linalg.eigh (App. D solver parity) at rate (1/5)^T."""
    rng = np.random.default_rng(2)
    d, k = 32, 6
    Q, _ = np.linalg.qr(rng.standard_normal((d, d)))
    s = np.concatenate([np.linspace(50, 25, k), np.linspace(5, 0.1, d - k)])
    C = (Q * s) @ Q.T
    V = orc.subspace(C, rng.standard_normal((d, k)), T=5, eps=1e-6)
    P = V @ np.linalg.solve(V.T @ V, V.T)
    w, E = np.linalg.eigh(C)
    Pref = E[:, -k:] @ E[:, -k:].T
    e5 = np.linalg.norm(P - Pref)
    assert e5 < 50 * 0.2 ** 5
    V = orc.subspace(C, rng.standard_normal((d, k)), T=30, eps=1e-9)
    P = V @ V.T
    assert np.linalg.norm(P - Pref) < 1e-8


def test_calibrate_subspace_pipeline_bias():
    rng = np.random.default_rng(3)
    K = rng.standard_normal((2, 80, 16)) @ rng.standard_normal((16, 16)) + 1.5
    Qw = rng.standard_normal((2, 1, 8, 16))
    V0 = rng.standard_normal((2, 16, 4))
    cal = orc.calibrate_subspace(K, Qw, V0)
    for u in range(2):
        R = cal["R"][u]
        np.testing.assert_allclose(cal["dmu"][u], cal["mu"][u] - R @ (R.T @ cal["mu"][u]), atol=1e-12)
