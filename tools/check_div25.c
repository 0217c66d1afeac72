/* Exhaustive check (all 2^31 non-negative finite float32 x; negatives follow by symmetry):
 * q = RN(x * RN(1/25)); r = fma(-q, 25, x); q1 = fma(r, RN(1/25), q) equals the IEEE quotient
 * x / 25.  Used by the box smoothing in libsf.  gcc -O2 -mfma -ffp-contract=off */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
int main(int argc, char** argv) {
    const uint32_t stride = argc > 1 ? (uint32_t)atoi(argv[1]) : 1u; /* 1 = exhaustive */
    const float y = 1.0f / 25.0f;  /* RN(1/25) */
    uint64_t bad = 0, first_bad = 0, bad_normal = 0;
    for (uint32_t u = 0; u < 0x7f800000u; u += stride) {  /* all non-negative finite floats */
        float x; memcpy(&x, &u, 4);
        float q = x * y;
        float r = fmaf(-q, 25.0f, x);
        float q1 = fmaf(r, y, q);
        float ref = x / 25.0f;
        if (q1 != ref) {
            if (!bad) first_bad = u;
            ++bad;
            if (x >= 1.17549435e-38f * 64) ++bad_normal;
        }
    }
    printf("mismatches %llu (with x >= 2^-120: %llu), first bad bits 0x%08llx\n", (unsigned long long)bad,
           (unsigned long long)bad_normal, (unsigned long long)first_bad);
    return bad != 0;
}
