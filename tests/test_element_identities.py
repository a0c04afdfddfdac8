"""CPU checks of the two algebraic identities the round-2 kernels rest on
(exact arithmetic identities, checked here in float64 on random data):

* K3, ZW form (n1_common.cuh element_zw): for the lowest-order Nedelec
  element with alpha, beta in P1 and exact integration,
      A_e x = antisym(B' X g),   B' = Btilde + t g,  t = sum(alpha) * 7200 / vol,
  where Btilde_pq = int beta lambda_p lambda_q * 120 / vol (S + beta_p + beta_q,
  2S + 4 beta_p on the diagonal), g = vol/120 grad lambda . grad lambda and
  X the antisymmetric matrix of the edge values. The reference assembles A_e
  from quadrature (forms.cpp:69-131, 133-193); here A_e is built from the
  element integrals directly (mass: exact monomial integration; curl-curl:
  constant curls).
* P2V closed-form moments (p2v_common.cuh p2v_exact_moments): K_rs =
  int k lambda_r lambda_s / vol for k in P2 against monomial integration.
"""
import itertools
import math

import numpy as np

EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]


def _tet(rng):
    P = rng.standard_normal((4, 3))
    J = (P[1:] - P[0]).T
    vol = abs(np.linalg.det(J)) / 6
    Ji = np.linalg.inv(J)
    grad = np.vstack([-Ji.sum(0), Ji])  # rows: grad lambda_p
    return vol, grad


def _int_monomial(alpha, vol):
    """int over the tet of prod lambda_i^alpha_i = 6 vol alpha! / (|alpha| + 3)!"""
    return 6 * vol * np.prod([math.factorial(a) for a in alpha]) / math.factorial(sum(alpha) + 3)


def _nd1_element_matrix(vol, grad, alpha, beta):
    """A_ij = int (sum alpha_m lambda_m) curl phi_i . curl phi_j + int (sum beta_m lambda_m) phi_i . phi_j,
    phi_(a,b) = lambda_a grad lambda_b - lambda_b grad lambda_a, by exact integration."""
    D = grad @ grad.T
    A = np.zeros((6, 6))
    for i, (a, b) in enumerate(EDGES):
        ci = 2 * np.cross(grad[a], grad[b])
        for j, (c, d) in enumerate(EDGES):
            cj = 2 * np.cross(grad[c], grad[d])
            A[i, j] += alpha.sum() * vol / 4 * (ci @ cj)
            # phi_i . phi_j = l_a l_c D_bd - l_a l_d D_bc - l_b l_c D_ad + l_b l_d D_ac
            for (p, q, s, coef) in ((a, c, 1, D[b, d]), (a, d, -1, D[b, c]), (b, c, -1, D[a, d]), (b, d, 1, D[a, c])):
                for m in range(4):
                    e = [0, 0, 0, 0]
                    e[m] += 1
                    e[p] += 1
                    e[q] += 1
                    A[i, j] += s * coef * beta[m] * _int_monomial(e, vol)
    return A


def test_zw_form_equals_element_matrix():
    rng = np.random.default_rng(7)
    for _ in range(20):
        vol, grad = _tet(rng)
        alpha, beta, x = rng.uniform(0.5, 2.0, 4), rng.uniform(0.5, 2.0, 4), rng.uniform(-1, 1, 6)
        y_ref = _nd1_element_matrix(vol, grad, alpha, beta) @ x
        g = vol / 120 * (grad @ grad.T)
        S = beta.sum()
        Bt = np.array([[S + beta[p] + beta[q] if p != q else 2 * S + 4 * beta[p] for q in range(4)] for p in range(4)])
        Bp = Bt + alpha.sum() * 7200 / vol * g
        X = np.zeros((4, 4))
        for i, (a, b) in enumerate(EDGES):
            X[a, b], X[b, a] = x[i], -x[i]
        Z = X @ g
        assert np.allclose(Z.sum(1), 0, atol=1e-12 * np.abs(Z).max())  # rows of Z sum to zero
        W = Bp @ Z
        y_zw = np.array([W[a, b] - W[b, a] for a, b in EDGES])
        assert np.abs(y_zw - y_ref).max() <= 1e-12 * np.abs(y_ref).max()


def test_p2v_closed_form_moments():
    rng = np.random.default_rng(3)
    for _ in range(20):
        kv = rng.uniform(-1, 2, 10)  # 4 vertex values, 6 edge-midpoint values
        kap = np.zeros((4, 4))
        for a in range(4):
            kap[a, a] = kv[a]
        for e, (a, b) in enumerate(EDGES):
            kap[a, b] = kap[b, a] = 4 * kv[4 + e] - kv[a] - kv[b]
        # monomial integration: K_rs = sum_{a<=b} kap_ab int l_a l_b l_r l_s / vol
        Kx = np.zeros((4, 4))
        for r, s in itertools.product(range(4), repeat=2):
            for a in range(4):
                for b in range(a, 4):
                    e = [0, 0, 0, 0]
                    for v in (a, b, r, s):
                        e[v] += 1
                    Kx[r, s] += kap[a, b] * _int_monomial(e, 1.0)
        # closed form (p2v_exact_moments)
        R = np.array([kap[r, r] + 0.5 * sum(kap[r, s] for s in range(4) if s != r) for r in range(4)])
        base = R.sum() + np.trace(kap)
        Q = R + np.diag(kap)
        Kc = np.array([[(base + 2 * (Q[r] + Q[s]) + kap[r, s]) if r != s else (2 * base + 8 * R[r] + 12 * kap[r, r])
                        for s in range(4)] for r in range(4)]) / 840
        assert np.abs(Kc - Kx).max() <= 1e-14 * np.abs(Kx).max()
        # and the nodal representation k = sum_{a<=b} kap_ab l_a l_b: k at the
        # vertices and the edge midpoints
        def k_at(lam):
            return sum(kap[a, b] * lam[a] * lam[b] for a in range(4) for b in range(a, 4))
        for a in range(4):
            lam = np.zeros(4)
            lam[a] = 1
            assert abs(k_at(lam) - kv[a]) <= 1e-14
        for e, (a, b) in enumerate(EDGES):
            lam = np.zeros(4)
            lam[a] = lam[b] = 0.5
            assert abs(k_at(lam) - kv[4 + e]) <= 1e-13
