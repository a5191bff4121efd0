// bsim_rng.cuh -- numpy-compatible counter-keyed RNG on the device.
//
// The reference draws every reset / command / randomisation value from
// `np.random.default_rng([seed, env, count, ...])` (envs.py:129-133,
// 512-515; randomize.py:125): numpy's SeedSequence hash -> PCG64 (XSL-RR
// 128/64) -> 53-bit doubles.  This restates those published algorithms so a
// GPU thread reproduces, bit for bit, the doubles numpy would produce for
// its env -- resets stay identical to the reference with no host round trip,
// and results are independent of how envs are sharded across GPUs.
#pragma once

#include <cstdint>

#include "bsim_math.cuh"

namespace bsim {

struct NpRng {
    unsigned __int128 state, inc;
};

// SeedSequence(entropy=words).generate_state(8, uint32) with pool_size 4
// (numpy/random/bit_generator.pyx: hashmix / mix / mix_entropy / generate_state)
BS_HD void seedseq_state8(const uint32_t *words, int n, uint32_t out[8]) {
    const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
    const uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
    uint32_t hc = INIT_A;
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= MULT_A;
        v *= hc;
        v ^= v >> 16;
        return v;
    };
    auto mix = [](uint32_t x, uint32_t y) {
        uint32_t r = MIX_L * x - MIX_R * y;
        r ^= r >> 16;
        return r;
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? words[i] : 0u);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (int s = 4; s < n; ++s)
        for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(words[s]));
    uint32_t hb = INIT_B;
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i & 3];
        v ^= hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        out[i] = v;
    }
}

BS_HD unsigned __int128 pcg_mult() {
    return ((unsigned __int128)2549297995355413924ull << 64) | (unsigned __int128)4865540595714422341ull;
}

// PCG64(SeedSequence(words)) -- pcg_setseq_128_srandom_r
BS_HD NpRng np_rng(const uint32_t *words, int n) {
    uint32_t st[8];
    seedseq_state8(words, n, st);
    uint64_t u[4];
    for (int i = 0; i < 4; ++i) u[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
    unsigned __int128 initstate = ((unsigned __int128)u[0] << 64) | u[1];
    unsigned __int128 initseq = ((unsigned __int128)u[2] << 64) | u[3];
    NpRng r;
    r.inc = (initseq << 1) | 1u;
    r.state = 0;
    r.state = r.state * pcg_mult() + r.inc;
    r.state += initstate;
    r.state = r.state * pcg_mult() + r.inc;
    return r;
}

BS_HD uint64_t np_next64(NpRng &r) {  // XSL-RR output of the advanced state
    r.state = r.state * pcg_mult() + r.inc;
    uint64_t hi = (uint64_t)(r.state >> 64), lo = (uint64_t)r.state;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

// Jump the stream `delta` draws ahead (pcg_advance_lcg_128: the LCG's
// affine map squared log2(delta) times), so lane k of an env's reset group
// can take draw k of the env's stream without the k - 1 draws before it.
BS_HD void np_advance(NpRng &r, uint64_t delta) {
    unsigned __int128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = r.inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    r.state = acc_mult * r.state + acc_plus;
}

// Generator.uniform(lo, hi) = lo + (hi - lo) * next_double
BS_HD double np_uniform(NpRng &r, double lo, double hi) {
    double u = (double)(np_next64(r) >> 11) * (1.0 / 9007199254740992.0);
    return lo + (hi - lo) * u;
}

}  // namespace bsim
