/* div_check.c — TEST INFRASTRUCTURE: empirical check of the ramp division
 * identity the engine relies on:
 *     RN(a / N) == fma(a, y, RN(a * y_lo)),  y = RN(1/N), y_lo = RN((1 - y*N) / N)
 * for dividends a with |a| in [2^-700, 2^701) and divisors whose odd part is
 * below 2^50.  Counts mismatches over `n` dividends drawn with a SplitMix64
 * stream: random significands at random exponents, plus significands near
 * the quotient's rounding boundaries (a = m*N for midpoints m, nudged by a
 * few ulps), the only places a wrong rounding could hide. */
#include <math.h>
#include <stdint.h>
#include <string.h>

static uint64_t sm64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double from_bits(uint64_t b) {
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

static uint64_t to_bits(double d) {
    uint64_t b;
    memcpy(&b, &d, sizeof b);
    return b;
}

/* naive != 0 checks the one-multiply RN(a*y) instead — it must fail, which
 * shows the sample reaches the rounding boundaries. */
uint64_t oracle_div2_mismatches(double N, uint64_t n, uint64_t seed, int naive) {
    const double y = 1.0 / N;
    const double y_lo = fma(-y, N, 1.0) / N;
    uint64_t s = seed, bad = 0;
    for (uint64_t k = 0; k < n; ++k) {
        double a;
        const uint64_t r = sm64(&s);
        if (k & 1) {
            /* random significand, exponent in [-690, 690] */
            const int e = (int)(r % 1381) - 690;
            a = ldexp(1.0 + (double)(sm64(&s) >> 12) * 0x1.0p-52, e);
        } else {
            /* near a quotient midpoint: m = (54-bit odd) * 2^(e-54) lies halfway
             * between two doubles; a = RN(m*N), nudged by up to 4 ulps */
            const int e = (int)(r % 301) - 150;
            const uint64_t odd = (sm64(&s) >> 10) | 1ULL | (1ULL << 53);
            a = ldexp((double)(odd >> 1), e - 53) * N + ldexp(1.0, e - 54) * N;
            const int64_t nudge = (int64_t)(sm64(&s) % 9) - 4;
            a = from_bits(to_bits(a) + (uint64_t)nudge);
        }
        if (sm64(&s) & 1) a = -a;
        const double want = a / N;
        const double got = naive ? a * y : fma(a, y, a * y_lo);
        if (to_bits(want) != to_bits(got)) ++bad;
    }
    return bad;
}
