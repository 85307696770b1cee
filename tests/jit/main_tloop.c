/* Driver for tests/jit/tloop.c: fills the fields, runs 5 time steps in one call, prints the bits. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
void relax(double a[66][71], double b[66][71], double c, int nt, int ny, int nx);
static double a[66][71], b[66][71];
int main(void) {
    uint64_t x = 88172645463325252ull;
    for (int j = 0; j < 66; ++j)
        for (int i = 0; i < 71; ++i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            a[j][i] = (double)(x >> 11) * (1.0 / 9007199254740992.0);
            b[j][i] = 0.0;
        }
    relax(a, b, 0.8, 5, 66, 71);
    uint64_t h = 1469598103934665603ull;
    for (int j = 0; j < 66; ++j)
        for (int i = 0; i < 71; ++i) {
            uint64_t u;
            memcpy(&u, &a[j][i], 8);
            h = (h ^ u) * 1099511628211ull;
        }
    printf("%016llx %.17g\n", (unsigned long long)h, a[33][35]);
    return 0;
}
