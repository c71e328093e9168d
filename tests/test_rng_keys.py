"""Counter RNG and k-means++ keys: independent pure-Python restatement of
rng.hpp:16-70 + published SplitMix64 vectors, checked against the oracle and
the product's host port (common.cuh, used by the synthetic generators)."""
import struct

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def mix64(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def bits(seed, stream, counter):
    h = mix64(seed ^ 0x2545F4914F6CDD1D)
    h = mix64((h + stream * GOLDEN) & M64)
    return mix64((h + counter * GOLDEN) & M64)


def hash_coords(vals):
    h = 0x6A09E667F3BCC909
    for v in vals:
        h = mix64(h ^ struct.unpack("<Q", struct.pack("<d", v))[0])
    return h


def test_splitmix64_published_vectors(orc):
    # SplitMix64 with state 0: outputs are mix64(k * golden), k = 1, 2, 3
    expected = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    for k, e in enumerate(expected, 1):
        assert mix64((k * GOLDEN) & M64) == e
        assert orc.load().orc_mix64((k * GOLDEN) & M64) == e


def test_bits_uniform_match_oracle(orc):
    lib = orc.load()
    for seed, stream, ctr in [(0, 0, 0), (1, 11, 8), (7, 12, 123456789), (2**63, 3, 2**40)]:
        assert lib.orc_bits(seed, stream, ctr) == bits(seed, stream, ctr)
        b = bits(seed, stream, ctr)
        assert lib.orc_uniform(seed, stream, ctr) == (b >> 11) * 2.0**-53
        assert lib.orc_uniform_pos(seed, stream, ctr) == ((b >> 11) + 1) * 2.0**-53


def test_keys_follow_column_major_quirk(orc, gm):
    """sogmm.cpp:210-213: key_i hashes 4 contiguous doubles of the
    column-major N x 4 buffer starting at x_i (wrapping into y at the end)."""
    p = gm.synthetic_frame_cloud(64, 48)
    flat = np.asfortranarray(p).ravel(order="F")
    n = len(p)
    import ctypes
    lib = orc.load()
    buf = np.ascontiguousarray(flat)
    ptr = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    for i in [0, 1, n // 2, n - 3, n - 2, n - 1]:
        want = hash_coords(flat[i:i + 4])
        got = lib.orc_hash_coords(ctypes.cast(ctypes.addressof(ptr.contents) + 8 * i,
                                              ctypes.POINTER(ctypes.c_double)), 4)
        assert got == want


def test_frame_keys_have_duplicates(gm):
    """on the cfg2 frame many keys coincide (back-wall x
    depends only on the pixel column), which makes exact clock ties common."""
    p = gm.synthetic_frame_cloud()
    flat = np.asfortranarray(p).ravel(order="F")
    n = len(p)
    keys = set()
    for i in range(0, n, 7):
        keys.add(tuple(flat[i:i + 4]))
    assert len(keys) < n // 7
