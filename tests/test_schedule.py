"""Row-order schedules (paper_1507_06078_b200/schedule.py; eig_set_schedule):
host logic only — an exact cover of the rows by tiles of <= tile rows, in the
y-band order (Survey §7 hard part 1(a))."""
import numpy as np
import pytest

from paper_1507_06078_b200 import schedule


@pytest.mark.parametrize("N,by,tile", [(9, 2, 64), (9, 4, 16), (10, 3, 8), (7, 7, 64), (5, 1, 5)])
def test_yband_is_an_exact_cover_with_bounded_tiles(N, by, tile):
    r0, ln = schedule.yband_3d(N, N, N, by, tile)
    assert r0.dtype == np.int64 and ln.dtype == np.int32
    assert ln.min() >= 1 and ln.max() <= tile
    cover = np.zeros(N ** 3, dtype=np.int64)
    for a, l in zip(r0.tolist(), ln.tolist()):
        cover[a:a + l] += 1
    assert np.all(cover == 1)


def test_yband_order_is_band_major_then_z():
    N, by = 6, 2
    r0, ln = schedule.yband_3d(N, N, N, by, 64)
    # first tile: band 0 at z = 0 (rows 0 .. by*N-1); second: band 0 at z = 1
    assert r0[0] == 0 and ln[0] == by * N
    assert r0[1] == N * N and ln[1] == by * N
    # the band at y = by starts after all N z-planes of band 0
    assert r0[N] == by * N


def test_natural_and_auto_band():
    r0, ln = schedule.natural(130)
    assert list(r0) == [0, 64, 128] and list(ln) == [64, 64, 2]
    assert 1 <= schedule.auto_band(100, 100, 550) <= 100
    assert schedule.auto_band(256, 256, 282, l2_bytes=1e3) == 1
