"""Host-side checks of the index arithmetic the sm_100a kernels rely on
(restated from paper_2204_05496_b200/csrc/ntt_fast.cuh; no GPU needed).

* swz(j + T r) = swz(j) + T r for j < T (pass-A exchange addresses as one
  swizzled base plus immediates);
* the warp-local cross-stage pass (x8_base / x8_ptr): every word of a warp's
  512-word block is read and written by exactly one lane, each lane's u/v
  chunks are the butterfly partners of stage 8 (x, x + 16 inside a 32-word
  group), and the eight lanes of a quarter-warp touch eight distinct 16-byte
  bank groups in every 128-bit access.
"""
import itertools


def swz(x: int) -> int:
    return x ^ (((x >> 5) & 7) << 2)


def x8_base(j: int) -> int:
    lane, qd = j & 31, (j & 31) >> 3
    gi, hh = (lane >> 1) & 3, lane & 1
    g = 2 * gi + (qd & 1) + 8 * (qd >> 1)
    return (j & ~31) * 16 + 32 * g + ((4 * hh) ^ ((g & 7) << 2))


def x8_chunk(b: int, c: int) -> int:
    return b ^ (8 if c & 1 else 0) ^ (16 if c & 2 else 0)


def test_pass_a_addresses_are_base_plus_immediate():
    for logn in (12, 13, 14):
        T = (1 << logn) // 16
        for j, r in itertools.product(range(T), range(16)):
            assert swz(j + T * r) == swz(j) + T * r


def test_cross_stage_pass_covers_the_block_and_pairs_partners():
    T = 512  # N = 8192
    for warp in range(T // 32):
        seen = {}
        for lane in range(32):
            j = 32 * warp + lane
            b = x8_base(j)
            chunks = [x8_chunk(b, c) for c in range(4)]
            # un-swizzle: physical word -> logical position (swz is an involution)
            logical = [[swz(p + i) for i in range(4)] for p in chunks]
            for c in range(4):
                assert chunks[c] % 4 == 0  # 128-bit aligned
                for i in range(4):
                    assert logical[c][i] not in seen
                    seen[logical[c][i]] = j
                    # a chunk stays inside one logical 4-word run (the swizzle permutes whole chunks)
                    assert logical[c][i] == logical[c][0] + i
            # u chunks c = 0, 1; their stage-8 partners 16 words up are c = 2, 3
            for c in range(2):
                assert logical[c + 2][0] == logical[c][0] + 16
                assert (logical[c][0] & 16) == 0
            # chunk 0 holds the next stage's u operands (offset bit 3 clear), chunk 1 its v operands
            assert (logical[0][0] & 8) == 0 and (logical[1][0] & 8) == 8
        assert sorted(seen) == list(range(512 * warp, 512 * warp + 512))


def test_cross_stage_pass_is_bank_conflict_free():
    for warp in range(16):
        for c in range(4):
            for qd in range(4):
                groups = set()
                for k in range(8):
                    j = 32 * warp + 8 * qd + k
                    word = x8_chunk(x8_base(j), c)
                    groups.add((word % 32) // 4)  # 16-byte bank group of a 128-byte row
                assert len(groups) == 8
