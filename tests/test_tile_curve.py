"""Row f1 host logic: the tile numbering of option "tile_order" (bdm_tile_curve, no GPU).

Pins of the Hilbert variant against what defines a Hilbert curve rather than against
its own formula: it is a bijection of the 8^3 super-tile, every step moves to a
face-adjacent tile (continuity), it starts at the origin corner and ends at a corner
adjacent along one axis (the curve's end points), and every aligned 2^3 / 4^3 sub-cube
is visited in one contiguous run (the recursive structure).  Row-major is the identity."""
import pytest


def _xyz(l):
    return (l & 7, (l >> 3) & 7, l >> 6)


@pytest.fixture(scope="module")
def curves():
    from paper_2503_10796_b200 import tile_curve
    return {o: tile_curve(o) for o in (0, 1)}


def test_row_major_is_identity(curves):
    assert curves[0] == list(range(512))


def test_hilbert_is_a_continuous_bijection(curves):
    h = curves[1]
    assert sorted(h) == list(range(512))
    inv = [0] * 512
    for l, r in enumerate(h):
        inv[r] = l
    path = [_xyz(l) for l in inv]
    for a, b in zip(path, path[1:]):
        assert sum(abs(p - q) for p, q in zip(a, b)) == 1, (a, b)
    assert path[0] == (0, 0, 0)
    assert sum(1 for v in path[-1] if v == 7) == 1 and sum(path[-1]) == 7


@pytest.mark.parametrize("s", [2, 4])
def test_hilbert_visits_aligned_subcubes_contiguously(curves, s):
    h = curves[1]
    blocks = {}
    for l, r in enumerate(h):
        x, y, z = _xyz(l)
        blocks.setdefault((x // s, y // s, z // s), []).append(r)
    for ranks in blocks.values():
        ranks.sort()
        assert ranks[-1] - ranks[0] == s ** 3 - 1
        assert ranks[0] % (s ** 3) == 0


def test_bad_order_is_rejected():
    from paper_2503_10796_b200 import BdmError, tile_curve
    with pytest.raises(BdmError):
        tile_curve(2)
