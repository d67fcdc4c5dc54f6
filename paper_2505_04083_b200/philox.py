"""Vectorised host Philox4x32-10 with random access (rng.hpp:17-104).

Draw t of stream `stream` under key `seed` is u64 = lo | hi << 32 of u32
slots 2*(t%2), 2*(t%2)+1 of block t//2, whose counter is
(block lo, block hi, stream lo, stream hi). Used for small host-side draws
(train mask, weight init); the large ones run on the GPU (csrc/philox.cuh).
"""

import numpy as np

_MA, _MB = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_WA, _WB = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
_M32 = np.uint64(0xFFFFFFFF)


def philox_blocks(seed, stream, blocks):
    """Philox blocks for counter indices `blocks` (u64 array) -> (n, 4) u32."""
    b = np.asarray(blocks, dtype=np.uint64)
    c0 = (b & _M32).astype(np.uint64)
    c1 = (b >> np.uint64(32)).astype(np.uint64)
    c2 = np.full_like(c0, np.uint64(stream) & _M32)
    c3 = np.full_like(c0, np.uint64(stream) >> np.uint64(32))
    k0 = np.uint64(np.uint64(seed) & _M32)
    k1 = np.uint64(np.uint64(seed) >> np.uint64(32))
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = _MA * c0
            p1 = _MB * c2
            hi0, lo0 = p0 >> np.uint64(32), p0 & _M32
            hi1, lo1 = p1 >> np.uint64(32), p1 & _M32
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint64((int(k0) + 0x9E3779B9) & 0xFFFFFFFF)
            k1 = np.uint64((int(k1) + 0xBB67AE85) & 0xFFFFFFFF)
    return np.stack([c0, c1, c2, c3], axis=1).astype(np.uint32)


def philox_u64(seed, stream, count, start=0):
    t = np.arange(start, start + count, dtype=np.uint64)
    blk = philox_blocks(seed, stream, t >> np.uint64(1)).astype(np.uint64)
    s = (t & np.uint64(1)).astype(np.int64) * 2
    rows = np.arange(count)
    return blk[rows, s] | (blk[rows, s + 1] << np.uint64(32))


def philox_doubles(seed, stream, count, start=0):
    return (philox_u64(seed, stream, count, start) >> np.uint64(11)).astype(np.float64) * 2.0**-53


def init_weights(dims, seed):
    """init_weights (model.hpp:17-33): Glorot U(+-sqrt(6/(fan_in+fan_out)))
    from Philox(seed, 100 + l), row-major, computed in double then cast."""
    out = []
    for l in range(len(dims) - 1):
        bound = np.sqrt(6.0 / float(dims[l] + dims[l + 1]))
        u = philox_doubles(seed, 100 + l, dims[l] * dims[l + 1])
        w = (-bound + (bound - -bound) * u).astype(np.float32)
        out.append(w.reshape(dims[l], dims[l + 1]))
    return out
