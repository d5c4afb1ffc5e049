"""NumPy prototype of the two-stage tridiagonalisation used by the GPU eigensolver.

Design check only (tools/, not shipped): stage 1 reduces a dense symmetric A to
bandwidth b with blocked Householder panels (QR of the sub-panel + a two-sided
rank-2b update), stage 2 chases the band down to tridiagonal form (one
Householder of length ≤ b per task: type 1 starts a sweep, types 2+3 push the
bulge one block down), and the stage-2 reflectors are applied to a matrix in
blocks G(I, t) = {H(i, t): i in sweep block I} — sweep blocks last-to-first,
tasks t ascending inside a block.

Run: python tools/twostage_proto.py
"""
import numpy as np


def house(x):
    """dlarfg: H = I − τ v vᵀ, v[0] = 1, H x = β e0."""
    alpha = x[0]
    xn2 = float(np.dot(x[1:], x[1:]))
    v = np.zeros_like(x)
    v[0] = 1.0
    if xn2 == 0.0:
        return v, 0.0, alpha
    beta = -np.copysign(np.hypot(alpha, np.sqrt(xn2)), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def larft(V, taus):
    """Forward columnwise T: H_0 H_1 … = I − V T Vᵀ."""
    k = V.shape[1]
    T = np.zeros((k, k))
    for i in range(k):
        T[i, i] = taus[i]
        if i:
            T[:i, i] = -taus[i] * (T[:i, :i] @ (V[:, :i].T @ V[:, i]))
    return T


def sy2sb(A, b):
    A = A.copy()
    n = A.shape[0]
    panels = []
    for j in range(0, n, b):
        m = n - j - b
        if m <= 1:
            break
        P = A[j + b:, j:j + b].copy()
        kb = min(b, m)
        V = np.zeros((m, kb))
        taus = np.zeros(kb)
        for k in range(kb):
            v, tau, beta = house(P[k:, k])
            V[k:, k] = v
            taus[k] = tau
            P[k, k] = beta
            P[k + 1:, k] = 0.0
            if k + 1 < b:
                w = v @ P[k:, k + 1:]
                P[k:, k + 1:] -= tau * np.outer(v, w)
        T = larft(V, taus)
        A[j + b:, j:j + b] = P
        A[j:j + b, j + b:] = P.T
        A22 = A[j + b:, j + b:]
        X = A22 @ V @ T
        W = X - 0.5 * V @ (T.T @ (V.T @ X))
        A[j + b:, j + b:] = A22 - V @ W.T - W @ V.T
        panels.append((j, V, T))
    return A, panels


def apply_q1(panels, Z, b):
    """Z ← Q1 Z, Q1 = Π_k (I − V_k T_k V_kᵀ) on rows j+b: (last panel first)."""
    Z = Z.copy()
    for j, V, T in reversed(panels):
        Z[j + b:] -= V @ (T @ (V.T @ Z[j + b:]))
    return Z


def sb2st(B, b):
    """Bulge chasing on a dense copy. Returns d, e, reflectors {(i, t): (row0, v, tau)}."""
    A = B.copy()
    n = A.shape[0]
    refl = {}
    for i in range(n - 2):
        st, ed = i + 1, min(i + b, n - 1)
        v, tau, beta = house(A[st:ed + 1, i].copy())
        A[st, i] = A[i, st] = beta
        A[st + 1:ed + 1, i] = A[i, st + 1:ed + 1] = 0.0
        D = A[st:ed + 1, st:ed + 1]
        H = np.eye(len(v)) - tau * np.outer(v, v)
        A[st:ed + 1, st:ed + 1] = H @ D @ H
        refl[(i, 0)] = (st, v, tau)
        t = 0
        while True:
            st2, ed2 = ed + 1, min(ed + b, n - 1)
            if st2 > n - 1:
                break
            t += 1
            C = A[st2:ed2 + 1, st:ed + 1] @ H           # type 2: right-apply the previous reflector
            v2, tau2, beta2 = house(C[:, 0].copy())
            H2 = np.eye(len(v2)) - tau2 * np.outer(v2, v2)
            C[:, 0] = 0.0
            C[0, 0] = beta2
            C[:, 1:] = H2 @ C[:, 1:]
            A[st2:ed2 + 1, st:ed + 1] = C
            A[st:ed + 1, st2:ed2 + 1] = C.T
            A[st2:ed2 + 1, st2:ed2 + 1] = H2 @ A[st2:ed2 + 1, st2:ed2 + 1] @ H2   # type 3
            refl[(i, t)] = (st2, v2, tau2)
            st, ed, H = st2, ed2, H2
    return np.diag(A).copy(), np.diag(A, -1).copy(), refl, A


def apply_q2_sequential(refl, Z):
    Z = Z.copy()
    for (i, t) in sorted(refl, reverse=True):
        r0, v, tau = refl[(i, t)]
        Z[r0:r0 + len(v)] -= tau * np.outer(v, v @ Z[r0:r0 + len(v)])
    return Z


def apply_q2_grouped(refl, Z, n, b, gs):
    Z = Z.copy()
    nsweeps = max(i for i, _ in refl) + 1
    for I in reversed(range((nsweeps + gs - 1) // gs)):
        i_lo, i_hi = I * gs, min((I + 1) * gs, nsweeps) - 1
        tmax = max(t for (i, t) in refl if i_lo <= i <= i_hi)
        for t in range(tmax + 1):
            r0 = i_lo + 1 + t * b
            if r0 > n - 1:
                continue
            r1 = min(i_hi + (t + 1) * b, n - 1)
            V = np.zeros((r1 - r0 + 1, i_hi - i_lo + 1))
            taus = np.zeros(i_hi - i_lo + 1)
            for i in range(i_lo, i_hi + 1):
                if (i, t) in refl:
                    s, v, tau = refl[(i, t)]
                    V[s - r0:s - r0 + len(v), i - i_lo] = v
                    taus[i - i_lo] = tau
            T = larft(V, taus)
            Z[r0:r1 + 1] -= V @ (T @ (V.T @ Z[r0:r1 + 1]))
    return Z


def main():
    rng = np.random.default_rng(0)
    for n, b in ((40, 4), (67, 8), (130, 16), (33, 16), (18, 16)):
        a = rng.standard_normal((n, n))
        A = a + a.T
        B, panels = sy2sb(A, b)
        bandmask = np.abs(np.subtract.outer(np.arange(n), np.arange(n))) <= b
        assert np.abs(B[~bandmask]).max(initial=0) < 1e-12, "sy2sb left fill outside the band"
        Q1 = apply_q1(panels, np.eye(n), b)
        assert np.allclose(Q1.T @ A @ Q1, B, atol=1e-10)
        d, e, refl, Afin = sb2st(B, b)
        tri = np.diag(d) + np.diag(e, -1) + np.diag(e, 1)
        assert np.allclose(Afin, tri, atol=1e-10), np.abs(Afin - tri).max()
        Q2 = apply_q2_sequential(refl, np.eye(n))
        assert np.allclose(Q2.T @ B @ Q2, tri, atol=1e-10)
        for gs in (b, 2 * b, 3):
            Q2g = apply_q2_grouped(refl, np.eye(n), n, b, gs)
            assert np.allclose(Q2g, Q2, atol=1e-12), (n, b, gs, np.abs(Q2g - Q2).max())
        lam, S = np.linalg.eigh(tri)
        Zfull = apply_q1(panels, apply_q2_grouped(refl, S, n, b, b), b)
        assert np.allclose(Zfull @ np.diag(lam) @ Zfull.T, A, atol=1e-9)
        print(f"n={n} b={b}: ok ({len(refl)} stage-2 reflectors)")


if __name__ == "__main__":
    main()


def apply_q2_waves(refl, Z, n, b, gs):
    """Same groups, applied in waves w = t − I (groups of one wave are row-disjoint)."""
    Z = Z.copy()
    nsweeps = max(i for i, _ in refl) + 1
    NI = (nsweeps + gs - 1) // gs
    tmax = {I: max(t for (i, t) in refl if I * gs <= i < min((I + 1) * gs, nsweeps)) for I in range(NI)}
    wmin, wmax = -(NI - 1), max(tmax.values())
    for wv in range(wmin, wmax + 1):
        rows_used = set()
        for I in range(NI):
            t = wv + I
            if t < 0 or t > tmax[I]:
                continue
            i_lo, i_hi = I * gs, min((I + 1) * gs, nsweeps) - 1
            r0 = i_lo + 1 + t * b
            if r0 > n - 1:
                continue
            r1 = min(i_hi + (t + 1) * b, n - 1)
            assert not (set(range(r0, r1 + 1)) & rows_used), "wave groups overlap"
            rows_used |= set(range(r0, r1 + 1))
            V = np.zeros((r1 - r0 + 1, i_hi - i_lo + 1))
            taus = np.zeros(i_hi - i_lo + 1)
            for i in range(i_lo, i_hi + 1):
                if (i, t) in refl:
                    s, v, tau = refl[(i, t)]
                    V[s - r0:s - r0 + len(v), i - i_lo] = v
                    taus[i - i_lo] = tau
            T = larft(V, taus)
            Z[r0:r1 + 1] -= V @ (T @ (V.T @ Z[r0:r1 + 1]))
    return Z


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    for n, b, gs in ((130, 16, 32), (67, 8, 16), (200, 16, 64), (40, 4, 12)):
        a = rng.standard_normal((n, n))
        B, _ = sy2sb(a + a.T, b)
        _, _, refl, _ = sb2st(B, b)
        Q2 = apply_q2_sequential(refl, np.eye(n))
        assert np.allclose(apply_q2_waves(refl, np.eye(n), n, b, gs), Q2, atol=1e-12), (n, b, gs)
        print(f"waves n={n} b={b} gs={gs}: ok")
