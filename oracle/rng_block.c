/* rng_block.c — TEST INFRASTRUCTURE ONLY: the inner loop of
 * mtfm_oracle.Rng.uniform_block (xoshiro256** of rng.hpp:35-46 and the
 * uniform draw of rng.hpp:55-57) in C, so the init port regenerates the
 * fixtures' multi-million-parameter stores in milliseconds. The Python loop in
 * mtfm_oracle.py is the restatement; this is its accelerator, checked against
 * it by tests/test_oracle_golden.py. Built on first use into oracle/_ref/. */
#include <stdint.h>

static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void rng_uniform_block(uint64_t* s, int64_t n, double lo, double hi, double* out) {
    const double span = hi - lo;
    uint64_t s0 = s[0], s1 = s[1], s2 = s[2], s3 = s[3];
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t r = rotl(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl(s3, 45);
        out[i] = lo + span * ((double)(r >> 11) * 0x1.0p-53);
    }
    s[0] = s0;
    s[1] = s1;
    s[2] = s2;
    s[3] = s3;
}
