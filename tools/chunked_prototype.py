"""Numpy model of the chunk-parallel solve used by the CUDA kernels.

Design-validation tool (not product, not oracle): it runs, vectorised over the
batch, exactly the per-chunk passes and Hillis-Steele scans of
``paper_1701_03787_b200/csrc/shen_solve.cu`` so their numerics can be compared
with the sequential reference elimination at the hardest BASELINE corners
before touching the GPU.  Usage: ``python tools/chunked_prototype.py``.
"""

import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1701_03787_b200.matrices import assemble  # noqa: E402
from oracle import shen_oracle as O  # noqa: E402


def hs_scan(elems, combine, reverse=False):
    """Inclusive Hillis-Steele scan over a python list (log2 C rounds)."""
    c = len(elems)
    cur = list(elems)
    step = 1
    while step < c:
        nxt = list(cur)
        for i in range(c):
            j = i + step if reverse else i - step
            if 0 <= j < c:
                # reverse: cur[i] covers i..i+step-1, cur[j] covers j.. ; compose i after j
                nxt[i] = combine(cur[i], cur[j])
        cur = nxt
        step *= 2
    return cur


def helm_chunked(mats, nu, dt, z2, rhs, R):
    fac = O.helmholtz_factor(mats, nu, dt, z2)  # sequential build -> checkpoints
    ca, cb = O.helmholtz_coefficients(nu, dt, z2)
    cb = np.atleast_1d(cb).reshape(-1)
    nd = mats.n_dir
    sd = mats.stiff_dir.banded.diagonal(0)
    st = mats.stiff_dir.tail
    md = mats.mass_dir.diagonal(0)
    flat = rhs.reshape(nd, -1)
    out = np.empty_like(flat)
    sub = cb * (-np.pi / 2)
    for par in (0, 1):
        k = np.arange(par, nd, 2)
        n = k.size
        nsup = len(range(par, nd - 2, 2))
        C = -(-n // R)
        chunks = []
        for c in range(C):
            s, e_ = c * R, min(c * R + R, n)
            rows = []
            if s > 0:
                d_, e0, t_ = fac["d"][par][s - 1], fac["e"][par][s - 1], fac["tail"][par][s - 1]
                rdp = 1.0 / d_
            y0 = np.zeros_like(flat[0])
            h = np.ones_like(cb)
            for i in range(s, e_):
                kk = k[i]
                diag = ca * sd[kk] + cb * md[kk]
                tail = ca * st[kk] + 0.0 * cb
                sup = tail + sub if i < nsup else tail
                b = flat[par + 2 * i]
                if i == 0:
                    d_, e0, t_ = diag, sup, tail
                    y0 = b.copy()
                    h = np.zeros_like(cb)
                else:
                    low = sub * rdp
                    d_ = diag - low * e0
                    e0 = sup - low * t_
                    t_ = tail - low * t_
                    y0 = b - low * y0
                    h = -low * h
                rdp = 1.0 / d_
                rows.append(dict(rd=rdp, e=e0, t=t_, h=h, y0=y0))
            chunks.append(dict(rows=rows, M=h, Y=y0))
        # forward scan: exit_c = Y_c + M_c * exit_{c-1}
        comp = [(ch["M"], ch["Y"]) for ch in chunks]
        inc = hs_scan(comp, lambda a, b: (a[0] * b[0], a[1] + a[0] * b[1]))
        entry = [np.zeros_like(flat[0])] + [inc[c][1] for c in range(C - 1)]
        # pass 2: fix y, backward composite (P, tau): sigma_s = P sigma_{s+R} + tau
        bcomp = []
        for c, ch in enumerate(chunks):
            P = [np.ones_like(cb), np.zeros_like(cb), np.zeros_like(cb), np.ones_like(cb)]
            tau = [np.zeros_like(flat[0]), np.zeros_like(flat[0])]
            for r in ch["rows"]:
                r["y"] = r["y0"] + r["h"] * entry[c]
                al, be = -r["rd"] * r["e"], -r["rd"] * r["t"]
                cy = r["rd"] * r["y"]
                tau = [tau[0] + P[0] * cy, tau[1] + P[2] * cy]
                P = [P[0] * al + P[1], P[0] * be + P[1], P[2] * al + P[3], P[2] * be + P[3]]
            bcomp.append((P, tau))

        def comb(a, b):  # a after b  (a is left chunk)
            P, t = a
            Q, u = b
            return ([P[0] * Q[0] + P[1] * Q[2], P[0] * Q[1] + P[1] * Q[3],
                     P[2] * Q[0] + P[3] * Q[2], P[2] * Q[1] + P[3] * Q[3]],
                    [t[0] + P[0] * u[0] + P[1] * u[1], t[1] + P[2] * u[0] + P[3] * u[1]])
        suf = hs_scan(bcomp, comb, reverse=True)
        for c, ch in enumerate(chunks):
            if c + 1 < C:
                x1, S2 = suf[c + 1][1]
            else:
                x1, S2 = np.zeros_like(flat[0]), np.zeros_like(flat[0])
            s = c * R
            for j in range(len(ch["rows"]) - 1, -1, -1):
                r = ch["rows"][j]
                x = (r["y"] - r["e"] * x1 - r["t"] * S2) * r["rd"]
                S2 = x1 + S2
                x1 = x
                out[par + 2 * (s + j)] = x
    return out.reshape(rhs.shape)


def bih_chunked(mats, nu, dt, z2, rhs, R):
    fac = O.biharmonic_factor(mats, nu, dt, z2)
    xi0, xi1, xi2 = O.biharmonic_coefficients(nu, dt, z2)
    x1f = np.atleast_1d(xi1).reshape(-1)
    x2f = np.atleast_1d(xi2).reshape(-1)
    nb = mats.n_bih
    h, p, q, r_, s_ = O.biharmonic_bands(mats, xi0, x1f, x2f)
    flat = rhs.reshape(nb, -1)
    out = np.empty_like(flat)
    Z = np.zeros_like(flat[0])
    zb = np.zeros_like(x1f)
    for par in (0, 1):
        k = np.arange(par, nb, 2)
        n = k.size
        C = -(-n // R)

        def hb(name, i, off):
            kk = k[i]
            if off >= 0:
                return h[name][kk] if kk + 2 * off <= nb - 1 else zb
            return h[name][kk + 2 * off] if kk + 2 * off >= 0 else zb
        chunks = []
        for c in range(C):
            s, e_ = c * R, min(c * R + R, n)
            st = {}
            if s >= 1:
                st[1] = {key: fac[key][par][s - 1] for key in "defab"}
            if s >= 2:
                st[2] = {key: fac[key][par][s - 2] for key in "defab"}
            # y state: (y_{i-1}, y_{i-2}); particular + 2 homogeneous
            yp1, yp2 = Z, Z
            h11, h12 = np.ones_like(x1f), zb  # response of y_{i-1} to (E1,E2)
            h21, h22 = zb, np.ones_like(x1f)  # response of y_{i-2}
            rows = []
            for i in range(s, e_):
                kk = k[i]
                hd, hp2, hp4 = hb("d0", i, 0), hb("p2", i, 1), hb("p4", i, 2)
                hm2, hm4 = hb("m2", i, -1), hb("m4", i, -2)
                in2, in4 = kk + 2 <= nb - 1, kk + 4 <= nb - 1
                b = flat[par + 2 * i]
                if i == 0:
                    d_, e0, f0, a0, b0 = hd, hp2, hp4, p[kk] + zb, r_[kk] + zb
                    l2 = l4 = zb
                elif i == 1:
                    P1 = st[1]
                    l2 = hm2 * (1.0 / P1["d"])
                    l4 = zb
                    u24 = xi0 * (P1["a"] * q[kk + 4] + P1["b"] * s_[kk + 4]) if in4 else zb
                    d_ = hd - l2 * P1["e"]
                    e0 = hp2 - l2 * P1["f"]
                    f0 = hp4 - l2 * u24
                    a0 = p[kk] - l2 * P1["a"]
                    b0 = r_[kk] - l2 * P1["b"]
                else:
                    P1, P2 = st[1], st[2]
                    l4 = hm4 * (1.0 / P2["d"])
                    tmp = hm2 - l4 * P2["e"]
                    l2 = tmp * (1.0 / P1["d"])
                    u42 = xi0 * (P2["a"] * q[kk + 2] + P2["b"] * s_[kk + 2]) if in2 else zb
                    u44 = xi0 * (P2["a"] * q[kk + 4] + P2["b"] * s_[kk + 4]) if in4 else zb
                    u24 = xi0 * (P1["a"] * q[kk + 4] + P1["b"] * s_[kk + 4]) if in4 else zb
                    d_ = hd - l4 * P2["f"] - l2 * P1["e"]
                    e0 = hp2 - l4 * u42 - l2 * P1["f"]
                    f0 = hp4 - l4 * u44 - l2 * u24
                    a0 = p[kk] - l2 * P1["a"] - l4 * P2["a"]
                    b0 = r_[kk] - l2 * P1["b"] - l4 * P2["b"]
                st[2] = st.get(1)
                st[1] = dict(d=d_, e=e0, f=f0, a=a0, b=b0)
                # y particular and homogeneous
                y = b - l2 * yp1 - l4 * yp2
                g1 = -l2 * h11 - l4 * h21
                g2 = -l2 * h12 - l4 * h22
                yp2, yp1 = yp1, y
                h21, h22, h11, h12 = h11, h12, g1, g2
                rows.append(dict(rd=1.0 / d_, e=e0, f=f0, a=a0, b=b0, y0=y, h1=g1, h2=g2, kk=kk))
            # exit state (y_last, y_last-1) = Y + H (E1, E2)
            chunks.append(dict(rows=rows, H=(h11, h12, h21, h22), Y=(yp1, yp2)))

        def fcomb(a, b):  # a after b: a.H*(b.Y) + a.Y
            H, Y = a
            G, W = b
            return ((H[0] * G[0] + H[1] * G[2], H[0] * G[1] + H[1] * G[3],
                     H[2] * G[0] + H[3] * G[2], H[2] * G[1] + H[3] * G[3]),
                    (Y[0] + H[0] * W[0] + H[1] * W[1], Y[1] + H[2] * W[0] + H[3] * W[1]))
        inc = hs_scan([(ch["H"], ch["Y"]) for ch in chunks], fcomb)
        entries = [(Z, Z)] + [inc[c][1] for c in range(C - 1)]
        qq, ss = q[par::2], s_[par::2]
        bcomp = []
        for c, ch in enumerate(chunks):
            E1, E2 = entries[c]
            # sigma_i = (x_i, x_{i+1}, Q_{i+2}, S_{i+2}); sigma_s = P sigma_{s+R} + tau
            P = [[np.ones_like(x1f) if a == b else zb for b in range(4)] for a in range(4)]
            tau = [Z, Z, Z, Z]
            s = c * R
            for j, rw in enumerate(ch["rows"]):
                i = s + j
                rw["y"] = rw["y0"] + rw["h1"] * E1 + rw["h2"] * E2
                qn = qq[i + 2] if i + 2 < n else 0.0
                sn = ss[i + 2] if i + 2 < n else 0.0
                A0 = [-rw["rd"] * rw["e"], -rw["rd"] * rw["f"], -rw["rd"] * (xi0 * rw["a"]), -rw["rd"] * (xi0 * rw["b"])]
                cy = rw["rd"] * rw["y"]
                tau = [tau[a] + P[a][0] * cy for a in range(4)]
                newP = []
                for a in range(4):
                    pa = P[a]
                    newP.append([pa[0] * A0[0] + pa[1],
                                 pa[0] * A0[1] + pa[2] * qn + pa[3] * sn,
                                 pa[0] * A0[2] + pa[2],
                                 pa[0] * A0[3] + pa[3]])
                P = newP
            bcomp.append((P, tau))

        def bcomb(a, b):
            P, t = a
            Q, u = b
            R4 = [[sum(P[i][m] * Q[m][j] for m in range(4)) for j in range(4)] for i in range(4)]
            return (R4, [t[i] + sum(P[i][m] * u[m] for m in range(4)) for i in range(4)])
        suf = hs_scan(bcomp, bcomb, reverse=True)
        for c, ch in enumerate(chunks):
            sig = suf[c + 1][1] if c + 1 < C else [Z, Z, Z, Z]
            x1, x2, sq, sv = sig  # x_{i+1}, x_{i+2}, Q_{i+3}, S_{i+3} for i = last row
            s = c * R
            for j in range(len(ch["rows"]) - 1, -1, -1):
                rw = ch["rows"][j]
                i = s + j
                acc = rw["y"] - rw["e"] * x1 - rw["f"] * x2 - xi0 * (rw["a"] * sq + rw["b"] * sv)
                x = acc * rw["rd"]
                # new state for row i-1: Q_{i+2} = Q_{i+3} + q_{i+2} x_{i+2}
                if i + 2 < n:
                    sq = sq + qq[i + 2] * x2
                    sv = sv + ss[i + 2] * x2
                x2, x1 = x1, x
                out[par + 2 * i] = x
    return out.reshape(rhs.shape)


def main():
    rng = np.random.default_rng(0)
    cases = [
        ("cfg1-like H/B n_x=63", 63, 1e-3, 1e-3, np.linspace(0, 3000, 40)),
        ("test z=5400 n_x=256", 256, 1 / 5200, 1e-5, np.array([0, 10, 200, 1800, 5400.0]) ** 2),
        ("cfg4 corners n_x=1024", 1024, 1 / 2000, 1e-4,
         np.array([0.0, 1.0, 4.0, 1e4, 1e6, 1024.0 ** 2 + 2048.0 ** 2])),
    ]
    for name, n_x, nu, dt, z2 in cases:
        mats = assemble(n_x, 0)
        for R in (4, 8, 16):
            t0 = time.time()
            fh = rng.standard_normal((mats.n_dir, z2.size)) + 1j * rng.standard_normal((mats.n_dir, z2.size))
            want = O.helmholtz_solve(O.helmholtz_factor(mats, nu, dt, z2), fh)
            got = helm_chunked(mats, nu, dt, z2, fh, R)
            eh = O.max_rel_per_system(got, want).max()
            fb = rng.standard_normal((mats.n_bih, z2.size)) + 1j * rng.standard_normal((mats.n_bih, z2.size))
            wantb = O.biharmonic_solve(O.biharmonic_factor(mats, nu, dt, z2), fb)
            gotb = bih_chunked(mats, nu, dt, z2, fb, R)
            eb = O.max_rel_per_system(gotb, wantb).max()
            resg = max(O.residual_longdouble(O.dense_biharmonic(mats, nu, dt, zz), gotb[:, j], fb[:, j])
                       for j, zz in enumerate(z2))
            resr = max(O.residual_longdouble(O.dense_biharmonic(mats, nu, dt, zz), wantb[:, j], fb[:, j])
                       for j, zz in enumerate(z2))
            print(f"{name} R={R}: H maxrel {eh:.2e}  B maxrel {eb:.2e}  B resid chunked {resg:.2e} ref {resr:.2e}"
                  f"  ({time.time() - t0:.1f}s)")


if __name__ == "__main__":
    main()
