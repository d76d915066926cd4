// rng.cuh -- numpy-exact random streams on device (and host).
//
// The reference draws every random variate from per-env numpy Generators
// (PCG64) spawned by SeedSequence(seed).spawn(n) (levelgen/env.py:591-594),
// and the draw order is part of its observable behaviour: maps, pinpoints,
// control targets and the binary diameter start all come from it
// (grid.py:124-125,186,215; problems.py:88,154; env.py:303). Bit-exact parity
// therefore means running numpy's algorithms here:
//   * SeedSequence pool mixing + generate_state (numpy bit_generator.pyx)
//   * PCG64 (XSL-RR 128/64) with the Generator's buffered 32-bit half-word
//   * Generator.integers -> random_bounded_uint64 (Lemire, 32- and 64-bit)
//   * Generator.random -> (next_u64 >> 11) * 2^-53
//   * Generator.choice(p=...) -> cdf searchsorted('right') over random()
//   * Generator.choice(replace=False) -> Floyd + bounded Fisher-Yates
// One env's generator lives in registers while its team steps it; all lanes
// of a team hold identical copies and draw in lockstep (uniform control flow).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define LG_HD __host__ __device__ __forceinline__
#else
#define LG_HD inline
#endif

namespace lg {

typedef unsigned __int128 u128;

struct Pcg {
    u128 s, inc;
    uint32_t has, u;  // Generator's buffered upper half (has_uint32, uinteger)
};

LG_HD u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

LG_HD void pcg_step(Pcg &g) { g.s = g.s * pcg_mult() + g.inc; }

LG_HD uint64_t pcg_next64(Pcg &g) {
    pcg_step(g);
    uint64_t hi = (uint64_t)(g.s >> 64), lo = (uint64_t)g.s;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

LG_HD uint32_t pcg_next32(Pcg &g) {
    if (g.has) {
        g.has = 0;
        return g.u;
    }
    uint64_t v = pcg_next64(g);
    g.has = 1;
    g.u = (uint32_t)(v >> 32);
    return (uint32_t)v;
}

LG_HD double pcg_double(Pcg &g) {
    return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

// random_bounded_uint64(off=0, rng, use_masked=False): uniform on [0, rng].
LG_HD uint64_t pcg_bounded(Pcg &g, uint64_t rng) {
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFULL) {
        if (rng == 0xFFFFFFFFULL) return pcg_next32(g);
        uint32_t ex = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)pcg_next32(g) * ex;
        uint32_t left = (uint32_t)m;
        if (left < ex) {
            uint32_t th = (0xFFFFFFFFu - (uint32_t)rng) % ex;
            while (left < th) {
                m = (uint64_t)pcg_next32(g) * ex;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
    if (rng == 0xFFFFFFFFFFFFFFFFULL) return pcg_next64(g);
    uint64_t ex = rng + 1;
    u128 m = (u128)pcg_next64(g) * ex;
    uint64_t left = (uint64_t)m;
    if (left < ex) {
        uint64_t th = (0xFFFFFFFFFFFFFFFFULL - rng) % ex;
        while (left < th) {
            m = (u128)pcg_next64(g) * ex;
            left = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

// Generator.integers(lo, hi) with exclusive hi.
LG_HD int64_t pcg_integers(Pcg &g, int64_t lo, int64_t hi) {
    return lo + (int64_t)pcg_bounded(g, (uint64_t)(hi - lo - 1));
}

// Jump the LCG ahead by `delta` steps (PCG's advance: O(log delta)).
// Used to let every row-lane of a team draw its slice of a row-major
// choice() block independently; double draws never touch the u32 buffer.
LG_HD void pcg_advance(Pcg &g, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = g.inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    g.s = acc_mult * g.s + acc_plus;
}

// SeedSequence(entropy, spawn_key=(key,) if has_key) -> PCG64 seeding.
LG_HD uint32_t ss_words(uint64_t v, uint32_t *w) {
    if (v == 0) {
        w[0] = 0;
        return 1;
    }
    uint32_t n = 0;
    while (v) {
        w[n++] = (uint32_t)v;
        v >>= 32;
    }
    return n;
}

LG_HD void seedseq_pcg(uint64_t entropy, bool has_key, uint64_t key, Pcg &g) {
    const uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu,
                   MULT_B = 0x58f38dedu, MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
    uint32_t ent[8];
    uint32_t n = ss_words(entropy, ent);
    if (has_key) {
        while (n < 4) ent[n++] = 0;
        n += ss_words(key, ent + n);
    }
    uint32_t hc = INIT_A;
    uint32_t pool[4];
    auto hashmix = [&](uint32_t v) {
        v ^= hc;
        hc *= MULT_A;
        v *= hc;
        v ^= v >> 16;
        return v;
    };
    auto mix = [&](uint32_t x, uint32_t y) {
        uint32_t r = MIX_L * x - MIX_R * y;
        return r ^ (r >> 16);
    };
    for (uint32_t i = 0; i < 4; i++) pool[i] = hashmix(i < n ? ent[i] : 0u);
    for (int s = 0; s < 4; s++)
        for (int d = 0; d < 4; d++)
            if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (uint32_t s = 4; s < n; s++)
        for (int d = 0; d < 4; d++) pool[d] = mix(pool[d], hashmix(ent[s]));
    uint32_t hb = INIT_B, w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i & 3] ^ hb;
        hb *= MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    u128 initstate = ((u128)((uint64_t)w[0] | ((uint64_t)w[1] << 32)) << 64) |
                     (u128)((uint64_t)w[2] | ((uint64_t)w[3] << 32));
    u128 initseq = ((u128)((uint64_t)w[4] | ((uint64_t)w[5] << 32)) << 64) |
                   (u128)((uint64_t)w[6] | ((uint64_t)w[7] << 32));
    g.inc = (initseq << 1) | 1;
    g.s = 0;
    pcg_step(g);
    g.s += initstate;
    pcg_step(g);
    g.has = 0;
    g.u = 0;
}

}  // namespace lg
