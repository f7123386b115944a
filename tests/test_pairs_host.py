"""Host-side mirror-pair tables (no GPU): the (m, n) / (-m, n) pairing of a
channel z2 grid that the biharmonic pair kernel consumes."""

import numpy as np
import pytest

from paper_1701_03787_b200.mesh import channel_z2
from paper_1701_03787_b200.solvers import mirror_pairs


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


def test_mirror_pairs_none_without_mirror_rows():
    assert mirror_pairs(np.arange(12.0).reshape(3, 4)) is None
    assert mirror_pairs(np.zeros(5)) is None
