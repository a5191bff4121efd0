"""Pure-Python restatement of numpy's SeedSequence + PCG64 (XSL-RR) used by
the reference's per-env RNG streams (envs.py:129-133, randomize.py:125).
Test infrastructure: checks the device implementation (csrc/bsim_rng.cuh)."""

M32 = 0xFFFFFFFF
MULT128 = (2549297995355413924 << 64) + 4865540595714422341
M128 = (1 << 128) - 1


def seedseq_state(words, n_words=8, pool_size=4):
    hc = [0x43b0d7e5]

    def hashmix(v):
        v = (v ^ hc[0]) & M32
        hc[0] = (hc[0] * 0x931e8875) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (0xca01f9dd * x - 0x4973f715 * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(words[i] if i < len(words) else 0) for i in range(pool_size)]
    for s in range(pool_size):
        for d in range(pool_size):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(pool_size, len(words)):
        for d in range(pool_size):
            pool[d] = mix(pool[d], hashmix(words[s]))
    hb, out = 0x8b51f9dd, []
    for i in range(n_words):
        v = (pool[i % pool_size] ^ hb) & M32
        hb = (hb * 0x58f38ded) & M32
        v = (v * hb) & M32
        out.append(v ^ (v >> 16))
    return out


class PCG64:
    def __init__(self, words):
        st = seedseq_state(list(words), 8)
        u = [st[2 * i] | (st[2 * i + 1] << 32) for i in range(4)]
        self.inc = (((u[2] << 64) | u[3]) << 1 | 1) & M128
        self.state = (0 * MULT128 + self.inc) & M128
        self.state = (self.state + ((u[0] << 64) | u[1])) & M128
        self.state = (self.state * MULT128 + self.inc) & M128

    def next64(self):
        self.state = (self.state * MULT128 + self.inc) & M128
        hi, lo = self.state >> 64, self.state & ((1 << 64) - 1)
        x, rot = hi ^ lo, hi >> 58
        return ((x >> rot) | (x << ((64 - rot) & 63))) & ((1 << 64) - 1)

    def double(self):
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform(self, lo, hi):
        return lo + (hi - lo) * self.double()
