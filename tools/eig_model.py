"""numpy model of eig.cu's eig_leading (same steps, fp64) for debugging the
control logic on CPU.  Development aid; not used by the product or the tests."""
import math
import sys

import numpy as np


def choose_block(J, d, p=0, kmax=116):
    p = p if p > 0 else max(8, min(J, 32))
    k = min(J + p, kmax, d)
    if k & 1:
        k = k + 1 if (k + 1 <= kmax and k + 1 <= d) else k - 1
    return max(k, J)


def chol_inv(G, shift=0.0):
    dsc = 1 / np.sqrt(np.maximum(np.diag(G), 1e-300))
    Gs = G * dsc[:, None] * dsc[None, :] + shift * np.eye(G.shape[0])
    R = np.linalg.cholesky(Gs).T
    return dsc[:, None] * np.linalg.inv(R)


def eig_leading(S, J, tol=1e-10, max_outer=60, verbose=True, Q0=None):
    d = S.shape[0]
    k = choose_block(J, d)
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (d, k)) if Q0 is None else Q0.copy()
    L = np.zeros((d, 0)); LT = np.zeros((d, 0)); thl = []
    th = np.zeros(k); res = np.zeros(k)
    nmat = 0

    def orth(A):
        if L.shape[1]:
            for _ in range(2):
                A = A - L @ (L.T @ A)
        ka = A.shape[1]
        shift = 11.0 * (d * ka + ka * (ka + 1)) * 1.1e-16 * ka
        for p in range(3):
            A = A @ chol_inv(A.T @ A, shift if p == 0 else 0.0)
        return A

    def op(Y):
        nonlocal nmat
        nmat += 1
        out = S @ Y
        if L.shape[1]:
            out = out - L @ (LT.T @ Y)
        return out

    def rr(A):
        SA = op(A)
        H = A.T @ SA
        w, V = np.linalg.eigh(0.5 * (H + H.T))
        o = np.argsort(-w, kind="stable")
        w, V = w[o], V[:, o]
        A = A @ V
        SA = SA @ V
        r = np.linalg.norm(SA - A * w, axis=0)
        return A, SA, w, r

    A = orth(A)
    A, SA, w, r = rr(A)
    nl0 = 0
    th[:] = w; res[:] = r
    def lock(A, SA):
        nonlocal L, LT
        nlock = L.shape[1]
        th1 = thl[0] if thl else th[0]
        nl = 0
        while nlock + nl < J and nl < A.shape[1] and res[nlock + nl] <= tol * th1:
            nl += 1
        if nl:
            L = np.hstack([L, A[:, :nl]]); LT = np.hstack([LT, SA[:, :nl]])
            thl.extend(th[nlock:nlock + nl])
            A, SA = A[:, nl:], SA[:, nl:]
        return A, SA
    A, SA = lock(A, SA)
    outer = 0
    while L.shape[1] < J and outer < max_outer:
        outer += 1
        nlock = L.shape[1]
        th1 = thl[0] if thl else th[0]
        thJ = th[J - 1]; thtop = th[nlock]; b = th[k - 1]
        if not b > 0:
            b = 1e-12 * th1
        if thJ <= b * (1 + 1e-12):
            b = thJ * (1 - 1e-3)
        a = 0.0; e = (b - a) / 2; c = (b + a) / 2
        xJ = max((thJ - c) / e, 1 + 1e-12); xt = max((thtop - c) / e, xJ)
        rJ, rt = math.acosh(xJ), math.acosh(xt)
        rmax = max(res[i] / th1 for i in range(nlock, J))
        m_need = math.ceil(math.log(max(rmax / tol, 4.0)) / max(rJ, 1e-6))
        m_amp = max(1, min(16, math.floor(math.log(2e7) / max(rt, 1e-6))))
        m = m_need = max(1, min(m_need, 64, (2 if m_amp < 6 else 8) * m_amp))
        done = 0
        while done < m_need:
            mseg = min(m_amp, m_need - done)
            sigma = e / (thtop - c); tau = 2 / sigma
            SA = op(A) if done > 0 else SA
            Y = (SA - c * A) * (sigma / e); X = A
            for _ in range(2, mseg + 1):
                s2 = 1 / (tau - sigma)
                T = (2 * s2 / e) * op(Y) - sigma * s2 * X - (2 * s2 * c / e) * Y
                X, Y = Y, T
                sigma = s2
            done += mseg
            A = Y
            if done < m_need:
                A = orth(A)
        Y = A
        A = orth(Y)
        A, SA, w, r = rr(A)
        th[nlock:] = w; res[nlock:] = r
        if not np.all(np.isfinite(w)):
            print("NON-FINITE at outer", outer); break
        A, SA = lock(A, SA)
        if verbose:
            print(f"outer {outer} m={m} (amp {m_amp}) nlock={L.shape[1]} rmax={rmax:.2e} thtop/thJ={thtop/thJ:.2f} b/thJ={b/thJ:.3f}")
    U = np.hstack([L, A])[:, :J]
    return U, outer, nmat


if __name__ == "__main__":
    d, J, gap = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (1000, 50, 3e-4)
    rng = np.random.default_rng(d + J)
    Q = np.linalg.qr(rng.standard_normal((d, d)))[0]
    w = np.sort(rng.uniform(0.1, 1.0, d))[::-1].copy()
    w[0] = 60.0
    w[J - 1] = w[J] * (1 + gap)
    w[:J] = np.maximum(w[:J], w[J - 1])
    S = (Q * w) @ Q.T
    U, outer, nmat = eig_leading(S, J)
    Uo = Q[:, np.argsort(-w)[:J]]
    a = U - Uo @ (Uo.T @ U); b = Uo - U @ (U.T @ Uo)
    print("outer", outer, "matvecs", nmat, "proj dist", math.sqrt((a * a).sum() + (b * b).sum()))
