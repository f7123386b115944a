"""Host-side mirror-pair tables (no GPU): the (m, n) / (-m, n) pairing of a
channel z2 grid that the pair kernels consume, in plain and warp-aligned form."""

import numpy as np
import pytest

from paper_1701_03787_b200.mesh import channel_z2
from paper_1701_03787_b200.solvers import mirror_pairs, mirror_pairs_grid


@pytest.mark.parametrize("ny,nz", [(16, 16), (64, 30), (12, 66), (2048, 64)])
def test_mirror_pairs_cover_every_system_once(ny, nz):
    z2 = channel_z2(ny, nz)
    pr = mirror_pairs(z2)
    assert pr is not None and pr.dtype == np.int64
    a, b = pr
    flat = z2.reshape(-1)
    assert np.array_equal(flat[a].view(np.int64), flat[b].view(np.int64))  # bitwise-identical z2
    systems = np.concatenate([a, b[a != b]])
    assert np.array_equal(np.sort(systems), np.arange(z2.size))  # each system exactly once
    assert (a == b).sum() == 2 * z2.shape[1]  # the self-paired rows m = 0 and m = ny / 2


@pytest.mark.parametrize("ny,nz", [(16, 16), (64, 30), (12, 66), (2048, 64)])
def test_mirror_pairs_grid_is_warp_aligned(ny, nz):
    z2 = channel_z2(ny, nz)
    pg, (gy, gz) = mirror_pairs_grid(z2)
    assert (gy, gz) == z2.shape and pg.shape[1] % 32 == 0
    a, b = pg
    pr = mirror_pairs(z2)
    # the padded table lists the same pairs in the same order, -1 on padding
    assert np.array_equal(a[a >= 0], pr[0]) and np.array_equal(b[b >= 0], pr[1])
    assert np.array_equal(a < 0, b < 0)
    # every run of 32 items: 32 consecutive kz columns of one row pair
    for w in range(pg.shape[1] // 32):
        wa, wb = a[32 * w:32 * w + 32], b[32 * w:32 * w + 32]
        ok = wa >= 0
        assert ok[0]
        ra, ca = np.divmod(wa[ok], gz)
        rb, cb = np.divmod(wb[ok], gz)
        assert len(set(ra)) == 1 and len(set(rb)) == 1
        assert np.array_equal(ca, ca[0] + np.arange(ok.sum())) and np.array_equal(ca, cb)


def test_mirror_pairs_none_without_mirror_rows():
    assert mirror_pairs(np.arange(12.0).reshape(3, 4)) is None
    assert mirror_pairs_grid(np.arange(12.0).reshape(3, 4)) is None
    assert mirror_pairs(np.zeros(5)) is None
