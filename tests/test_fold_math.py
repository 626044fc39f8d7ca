"""CPU check of the stream-K piece arithmetic the deferred-fold GEMMs rely on
(csrc/device/gemm_decode.cu DecIter, device.cuh fold_pieces, attention.cu
decode_combine*): CTA c of G owns iterations [c I / G, (c + 1) I / G) of the
flattened (tile, k-block) space; a tile's pieces are the CTAs whose ranges
meet it, numbered from first = ((it0 + 1) G - 1) // I; the fold reads pieces
0 .. last - first. Every (tile, k-block) must be covered exactly once and
the piece indices a CTA writes must be exactly 0 .. pieces - 1."""
import random

import pytest


def pieces_formula(tile, num_kb, G, total):
    it0 = tile * num_kb
    first = ((it0 + 1) * G - 1) // total
    last = ((it0 + num_kb) * G - 1) // total
    return first, last - first + 1


def ranges(G, total):
    return [(total * c // G, total * (c + 1) // G) for c in range(G)]


@pytest.mark.parametrize("seed", range(40))
def test_streamk_pieces_cover_each_tile_once(seed):
    rng = random.Random(seed)
    tiles = rng.randint(1, 300)
    num_kb = rng.choice([8, 64, 224])
    total = tiles * num_kb
    G = rng.randint(1, min(148, total))
    seen = {}
    for c, (lo, hi) in enumerate(ranges(G, total)):
        it = lo
        while it < hi:
            tile, kb0 = divmod(it, num_kb)
            kb1 = min(num_kb, kb0 + (hi - it))
            first, n = pieces_formula(tile, num_kb, G, total)
            piece = c - first  # DecIter / WorkIter: blockIdx.x - first
            assert 0 <= piece < n
            for kb in range(kb0, kb1):
                assert (tile, kb) not in seen
                seen[(tile, kb)] = piece
            it += kb1 - kb0
    assert len(seen) == total
    for t in range(tiles):
        _, n = pieces_formula(t, num_kb, G, total)
        assert sorted({seen[(t, kb)] for kb in range(num_kb)}) == list(range(n))


def test_min_kblocks_cap_bounds_pieces():
    """gemm_decode caps the grid so each CTA streams >= 16 k-blocks; the plane
    budget (max_pieces) must bound every tile's piece count."""
    for rows, K in [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096)]:
        tiles, num_kb = (rows // 128 + 1) // 2, K // 64
        total = tiles * num_kb
        for sms in (8, 16, 32, 48, 64, 96, 148):
            G = min(sms, total, max(1, -(-total // 16)))
            per_min = total // G
            max_pieces = -(-num_kb // per_min) + 1
            for t in range(tiles):
                assert pieces_formula(t, num_kb, G, total)[1] <= max_pieces
