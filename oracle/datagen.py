"""TEST INFRASTRUCTURE -- the checker for the GPU data generator, never the
product path. numpy restatement of SPEC data_gen as defined
in include/hpsim_b200.h (hp_data_generate) / paper_1404_5997_b200/csrc/datagen.cu.

Parity unpinned by the reference: the reference specifies the module but ships
no code for it, so there are no golden vectors; the tests check the SPEC
properties (determinism, empty case, class balance, L < 2 error, learnability)
and this independent restatement of the generator's definition:
  Philox4x32-10 (Salmon et al., SC'11), key = seed (lo, hi), counter
  (a lo, a hi, m, stream); class(i) = perm(i) mod L with perm a balanced
  4-round Feistel network on [0, 2^bits) (bits even, 2^bits >= N) cycle-walked
  into [0, N), round function = Philox(counter (R lo, R hi, round, 3)) low
  `bits/2` bits; x_i[4m + j] = separation * BM_j(Philox(class, m, stream 1)) +
  BM_j(Philox(i, m, stream 2)), BM = Box-Muller on (c0, c1) for j = 0, 1 and
  (c2, c3) for j = 2, 3, u1 = (c + 1) 2^-32, u2 = c' 2^-32 (computed here in
  float64; the GPU uses float math, so values agree to ~1e-5 while the integer
  parts -- classes, one-hot targets -- are exact).
"""
import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox(c0, c1, c2, c3, seed):
    """Vectorised Philox4x32-10 over uint32 arrays; returns the 4 output words."""
    c = [np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3)]
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        h0, l0 = p0 >> np.uint64(32), p0 & MASK32
        h1, l1 = p1 >> np.uint64(32), p1 & MASK32
        c = [h1 ^ c[1] ^ np.uint64(k0), l1, h0 ^ c[3] ^ np.uint64(k1), l0]
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return c


def _bits(n):
    b = 1
    while (1 << b) < n:
        b += 1
    return b + (b % 2)


def permute(seed, n, i):
    """perm(i) for an array of indices."""
    h = _bits(n) // 2
    mask = np.uint64((1 << h) - 1)
    x = np.asarray(i, dtype=np.uint64).copy()
    todo = np.ones(x.shape, dtype=bool)
    while todo.any():
        xs = x[todo]
        L, R = xs >> np.uint64(h), xs & mask
        for rnd in range(4):
            c = philox(R & MASK32, R >> np.uint64(32), np.full_like(R, rnd), np.full_like(R, 3), seed)
            f = ((c[1] << np.uint64(32)) | c[0]) & mask
            L, R = R, L ^ f
        xs = (L << np.uint64(h)) | R
        x[todo] = xs
        todo = x >= np.uint64(n)
    return x.astype(np.int64)


def classes(seed, n, L, idx):
    return permute(seed, n, idx) % L


def _box_muller(c0, c1):
    u1 = (c0.astype(np.float64) + 1.0) * 2.0 ** -32
    u2 = c1.astype(np.float64) * 2.0 ** -32
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)


def normals(seed, stream, a, D):
    """The D values g(stream, a, 0..D-1): quad m = Box-Muller of (c0, c1) then (c2, c3)."""
    m = np.arange((D + 3) // 4, dtype=np.uint64)
    a = np.uint64(a)
    c = philox(np.full_like(m, a & MASK32), np.full_like(m, a >> np.uint64(32)), m, np.full_like(m, stream), seed)
    z0, z1 = _box_muller(c[0], c[1])
    z2, z3 = _box_muller(c[2], c[3])
    out = np.empty(4 * len(m))
    out[0::4], out[1::4], out[2::4], out[3::4] = z0, z1, z2, z3
    return out[:D]


def example(seed, n, L, separation, shape, i):
    """(x_i flattened, class) of example i."""
    D = int(np.prod(shape))
    cls = int(classes(seed, n, L, np.array([i]))[0])
    return separation * normals(seed, 1, cls, D) + normals(seed, 2, i, D), cls
