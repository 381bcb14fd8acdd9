/* recip_check.c -- exhaustive check of the quantizers' division-free rounding
 * (csrc/common.cuh quant_rne): for a scale s with r = RN(1/s),
 *     y = RN(x*r);  t = RN(x - y*s) (one FMA, exact);  q = RN(t*r + y) (one FMA)
 * must give sat(rint(q)) == sat(rint(RN(x/s))) -- the oracle's IEEE division
 * (oracle/cpu_ref.c) -- for EVERY float x whose quotient can round to a
 * nonzero grid point (|x| in [s/4, 256 s]; beyond that both saturate or give 0).
 * The device then rounds through the grid float t = RN(clamp(q) + 1.5*2^23)
 * (no conversion instructions): t's bits - 0x4B400000 is the integer, t's low
 * byte the int8 byte and t - 1.5*2^23 the grid value -- checked here for the
 * same x, and over every float quotient pattern once (argv "grid").
 * Scales: the argv list (hex bit patterns) -- edge significands (all ones,
 * 1.0, 1 + ulp) and seeded random ones.  Prints "mismatches N"; exit 1 if N > 0.
 * Built and run by tests/test_quant_recip.py (CPU). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static float bits_f(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t f_bits(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

static int sat_rint(float v) {
    float r = rintf(v);
    r = fminf(fmaxf(r, -127.0f), 127.0f);
    return (int)r;
}

/* csrc/common.cuh quant_rne_f: the grid float of a quotient v; returns the
 * integer and checks the byte / grid-value views agree with it (-1000 if not). */
static int grid(float v) {
    const float t = fminf(fmaxf(v, -127.0f), 127.0f) + 12582912.0f;
    const int q = (int)f_bits(t) - 0x4B400000;
    if ((int8_t)(f_bits(t) & 0xffu) != q || t - 12582912.0f != (float)q) return -1000;
    return q;
}

static int fast(float x, float s, float r) {
    const float y = x * r;
    const float t = fmaf(-y, s, x);
    const float v = fabsf(y) < 256.0f ? fmaf(t, r, y) : y;
    return grid(v);
}

int main(int argc, char** argv) {
    long long bad = 0, checked = 0;
    if (argc > 1 && strcmp(argv[1], "grid") == 0) {
        /* every non-NaN float quotient (+-inf included); a NaN quotient clamps to
         * -127 on the device (FMNMX returns the non-NaN operand) on both paths,
         * but x86 vector min/max order NaN operands differently, so it is not a
         * CPU-checkable identity */
#pragma omp parallel for reduction(+ : bad, checked) schedule(static)
        for (long long b = 0; b <= 0xffffffffLL; ++b) {
            const float v = bits_f((uint32_t)b);
            if (v != v) continue;
            if (grid(v) != sat_rint(v)) ++bad;
            ++checked;
        }
        printf("checked %lld mismatches %lld\n", checked, bad);
        return bad ? 1 : 0;
    }
    for (int a = 1; a < argc; ++a) {
        const float s = bits_f((uint32_t)strtoul(argv[a], NULL, 16));
        const float r = 1.0f / s;
        const uint32_t lo = f_bits(s * 0.25f), hi = f_bits(s * 256.0f);
        long long bad_s = 0;
#pragma omp parallel for reduction(+ : bad_s, checked) schedule(static)
        for (long long b = lo; b <= (long long)hi; ++b) {
            for (int sign = 0; sign < 2; ++sign) {
                const float x = bits_f((uint32_t)b | (sign ? 0x80000000u : 0u));
                const int want = sat_rint(x / s);
                const int got = fast(x, s, r);
                if (want != got) ++bad_s;
                ++checked;
            }
        }
        if (bad_s) printf("scale %a: %lld mismatches\n", s, bad_s);
        bad += bad_s;
    }
    printf("checked %lld mismatches %lld\n", checked, bad);
    return bad ? 1 : 0;
}
