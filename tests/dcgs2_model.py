"""numpy model of the device GMRES with DCGS2 Arnoldi (dg_runtime.cu:
dcgs2_cycle) -- test infrastructure: it documents the
algebra of the delayed re-orthogonalisation on the CPU, against the
reference's MGS + selective re-orthogonalisation (krylov.py:27-115,
restated in oracle/dg_oracle.py:gmres)."""

import numpy as np


def gmres_dcgs2(action, rhs, x0, tol_rel, restart=30, max_iter=1000):
    rhs = np.asarray(rhs, float).ravel()
    bn = np.linalg.norm(rhs)
    x = np.array(x0, float).ravel()
    r = rhs - action(x)
    target = tol_rel * bn
    m = restart
    its, hist, breakdown = 0, [], False
    while True:
        beta = np.linalg.norm(r)
        hist.append(beta / bn)
        if beta <= target or its >= max_iter or breakdown:
            break
        Qb = np.zeros((m + 1, r.size))
        Qb[0] = r / beta                      # slot j holds the lagged u_j
        Hb = np.zeros((m + 1, m))
        R = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        done = 0
        for j in range(m):
            u = Qb[j]
            z = action(u)
            Q = Qb[:j]
            t, s = Q @ z, Q @ u                # the fused dual dots (one read of Q)
            zz, uz, uu = z @ z, u @ z, u @ u
            alpha = 1.0
            if j > 0:
                alpha = np.sqrt(uu - s @ s)
                Hb[:j, j - 1] += s
                Hb[j, j - 1] = alpha
            gv = Hb[:j + 1, :j] @ s
            h = np.empty(j + 1)
            h[:j] = (t - gv[:j]) / alpha
            h[j] = ((uz - s @ t) / alpha - gv[j]) / alpha
            Hb[:j + 1, j] = h
            # one update pass: q_j in place, u_{j+1} = z/alpha - Q c - c_j q_j
            q = (u - s @ Q) / alpha
            c = gv / alpha + h
            un = z / alpha - c[:j] @ Q - c[j] * q
            Qb[j], Qb[j + 1] = q, un
            na = np.linalg.norm(un)
            Hb[j + 1, j] = na
            its += 1
            happy = na <= 1e-14 * max(bn, np.sqrt(zz) / alpha)
            R[:j + 2, j] = Hb[:j + 2, j]
            for i in range(j):
                tt = cs[i] * R[i, j] + sn[i] * R[i + 1, j]
                R[i + 1, j] = -sn[i] * R[i, j] + cs[i] * R[i + 1, j]
                R[i, j] = tt
            den = np.hypot(R[j, j], R[j + 1, j])
            cs[j] = R[j, j] / den if den else 1.0
            sn[j] = R[j + 1, j] / den if den else 0.0
            R[j, j], R[j + 1, j] = den, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            done = j + 1
            hist.append(abs(g[j + 1]) / bn)
            if happy:
                breakdown = True
                break
            if abs(g[j + 1]) <= target or its >= max_iter:
                break
        # least squares on the corrected Hbar: fresh Givens QR
        gg = np.zeros(done + 1)
        gg[0] = beta
        R2 = Hb[:done + 1, :done].copy()
        for j in range(done):
            for i in range(j):
                tt = cs[i] * R2[i, j] + sn[i] * R2[i + 1, j]
                R2[i + 1, j] = -sn[i] * R2[i, j] + cs[i] * R2[i + 1, j]
                R2[i, j] = tt
            den = np.hypot(R2[j, j], R2[j + 1, j])
            cs[j] = R2[j, j] / den if den else 1.0
            sn[j] = R2[j + 1, j] / den if den else 0.0
            R2[j, j], R2[j + 1, j] = den, 0.0
            gg[j + 1] = -sn[j] * gg[j]
            gg[j] = cs[j] * gg[j]
        y = np.linalg.solve(np.triu(R2[:done, :done]), gg[:done])
        x = x + y @ Qb[:done]
        r = rhs - action(x)
    return x, its, hist
