"""Mirror-pairing kernels (shen_pair_split / shen_pair_merge /
shen_cross_paired / shen_scale_rows) against numpy restatements: the pair
passes and the row-strided scaling are single IEEE operations per element,
so they are bit-identical; the paired cross product agrees with the plain
one on the unpaired fields to rounding."""

import ctypes

import numpy as np
import pytest

from paper_1701_03787_b200 import _lib

pytestmark = pytest.mark.gpu


def _split_np(x, P, Q):
    N = P + Q
    y = np.empty_like(x)
    j = np.arange(Q)
    y[:Q] = x[j] + x[N - 1 - j]
    if P > Q:
        y[Q] = x[Q]
    y[P:] = x[j] - x[N - 1 - j]
    return y


def _merge_np(y, P, Q):
    N = P + Q
    x = np.empty_like(y)
    j = np.arange(Q)
    x[j] = y[:Q] + y[P:]
    x[N - 1 - j] = y[:Q] - y[P:]
    if P > Q:
        x[Q] = y[Q]
    return x


@pytest.mark.parametrize("N", [9, 10, 257])
def test_pair_split_merge_bitwise(N):
    import torch

    P, Q = (N + 1) // 2, N // 2
    rng = np.random.default_rng(N)
    x = rng.standard_normal((N, 2 * 37))  # complex rows as doubles (M even)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    lib = _lib.lib()
    _lib.check(lib.shen_pair_split(P, Q, x.shape[1], xd.data_ptr(), yd.data_ptr(), None), "split")
    assert np.array_equal(yd.cpu().numpy(), _split_np(x, P, Q))
    zd = torch.empty_like(xd)
    _lib.check(lib.shen_pair_merge(P, Q, x.shape[1], yd.data_ptr(), zd.data_ptr(), None), "merge")
    assert np.array_equal(zd.cpu().numpy(), _merge_np(yd.cpu().numpy(), P, Q))


def test_pair_rejects_odd_rows_and_bad_sizes():
    import torch

    x = torch.zeros((5, 7), dtype=torch.float64, device="cuda")
    assert _lib.lib().shen_pair_split(3, 2, 7, x.data_ptr(), x.data_ptr(), None) != 0  # M odd
    assert _lib.lib().shen_pair_split(3, 1, 8, x.data_ptr(), x.data_ptr(), None) != 0  # P - Q > 1


def _cross_np(f):
    u, v, w, om_x, dv_dx, dw_dx, du_dy, du_dz = f
    om_y = du_dz - dw_dx
    om_z = dv_dx - du_dy
    return np.stack([v * om_z - w * om_y, w * om_x - u * om_z, u * om_y - v * om_x])


@pytest.mark.parametrize("N", [9, 10])
def test_cross_paired_vs_plain(N):
    import torch

    P, Q, M = (N + 1) // 2, N // 2, 48
    rng = np.random.default_rng(3 * N)
    f = rng.standard_normal((8, N, M))  # point values
    # paired form: f_j = e_j + o_j, f_{N-1-j} = e_j - o_j
    j = np.arange(Q)
    e = np.empty((8, P, M))
    o = (f[:, j] - f[:, N - 1 - j]) / 2
    e[:, :Q] = (f[:, j] + f[:, N - 1 - j]) / 2
    if P > Q:
        e[:, Q] = f[:, Q]
    fp = np.concatenate([e, o], axis=1)
    h = torch.empty((3, P + Q, M), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().shen_cross_paired(P, Q, M, torch.from_numpy(fp).cuda().data_ptr(), h.data_ptr(), None),
               "cross_paired")
    want = _split_np(_cross_np(f).transpose(1, 0, 2), P, Q).transpose(1, 0, 2)
    got = h.cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()


def test_scale_rows_interleaves_bitwise():
    import torch

    rows, L = 5, 33
    rng = np.random.default_rng(1)
    x = rng.standard_normal((rows, L)) + 1j * rng.standard_normal((rows, L))
    c = rng.standard_normal(L) + 1j * rng.standard_normal(L)
    out = torch.zeros((2 * rows, L), dtype=torch.complex128, device="cuda")
    xd = torch.from_numpy(x).cuda()
    cre, cim = torch.from_numpy(c.real.copy()).cuda(), torch.from_numpy(c.imag.copy()).cuda()
    _lib.check(_lib.lib().shen_scale_rows(rows, L, xd.data_ptr(), L, cre.data_ptr(), cim.data_ptr(),
                                          out[1:].data_ptr(), 2 * L, None), "scale_rows")
    got = out.cpu().numpy()
    # the kernel's order: (c.re x.re - c.im x.im, c.re x.im + c.im x.re), every
    # product rounded (numpy's own complex multiply may fuse them on this host)
    want = (c.real * x.real - c.imag * x.imag) + 1j * (c.real * x.imag + c.imag * x.real)
    assert np.array_equal(got[1::2], want)
    assert not got[0::2].any()
