/* Driver for tests/jit/heat.c: fills the fields, runs steps, prints the bits. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
void heat(double t[130][131], double tn[130][131], double src[130][131], double kappa, double dt, int jbeg,
          int jend, int nx);
static double a[130][131], b[130][131], s[130][131];
int main(void) {
    uint64_t x = 88172645463325252ull;
    for (int j = 0; j < 130; ++j)
        for (int i = 0; i < 131; ++i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            a[j][i] = (double)(x >> 11) * (1.0 / 9007199254740992.0);
            b[j][i] = a[j][i];
            s[j][i] = 0.01 * a[j][i];
        }
    for (int step = 0; step < 4; ++step) {
        if (step % 2 == 0) heat(a, b, s, 0.2, 0.5, 1, 129, 131);
        else heat(b, a, s, 0.2, 0.5, 1, 129, 131);
    }
    uint64_t h = 1469598103934665603ull;
    for (int j = 0; j < 130; ++j)
        for (int i = 0; i < 131; ++i) {
            uint64_t u;
            memcpy(&u, &a[j][i], 8);
            h = (h ^ u) * 1099511628211ull;
        }
    printf("%016llx %.17g\n", (unsigned long long)h, a[64][64]);
    return 0;
}
