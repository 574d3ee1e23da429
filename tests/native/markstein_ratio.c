/* Exhaustive check of the K2 ratio() fast path (csrc/pbas.cu): for every
 * len in [1, 255] and tot in [0, 65535], one Markstein correction step with
 * rcp = RN(1/len) reproduces the IEEE quotient RN(tot/len) bit for bit:
 *   q0 = tot * rcp;  r = fma(-q0, len, tot);  q = fma(r, rcp, q0).
 * (glibc fma() is correctly rounded with or without hardware FMA.)
 * Prints the number of mismatches; exit status 1 if any. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

int main(void) {
    long bad = 0, cases = 0;
    for (int len = 1; len <= 255; ++len) {
        volatile double dl = (double)len;
        const double rcp = 1.0 / dl;
        for (int tot = 0; tot < 65536; ++tot) {
            const double t = (double)tot;
            const double q0 = t * rcp;
            const double q = fma(fma(-q0, dl, t), rcp, q0);
            const double ref = t / dl;
            uint64_t a, b;
            memcpy(&a, &q, 8);
            memcpy(&b, &ref, 8);
            if (a != b) {
                if (bad < 5) printf("len %d tot %d: %.17g != %.17g\n", len, tot, q, ref);
                ++bad;
            }
            ++cases;
        }
    }
    printf("cases %ld mismatches %ld\n", cases, bad);
    return bad != 0;
}
