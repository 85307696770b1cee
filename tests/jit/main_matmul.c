/* Driver for tests/jit/matmul_g.c: fills the globals, runs, prints the bits. */
#include <stdio.h>
#include <stdint.h>
#include <string.h>
extern double A[48][40], B[40][56], C[48][56], alpha;
void matmul(void);
int main(void) {
    uint64_t x = 2463534242ull;
    for (int i = 0; i < 48; ++i)
        for (int l = 0; l < 40; ++l) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; A[i][l] = (double)(x >> 11) * 0x1p-53; }
    for (int l = 0; l < 40; ++l)
        for (int j = 0; j < 56; ++j) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; B[l][j] = (double)(x >> 11) * 0x1p-52; }
    alpha = 0.75;
    matmul();
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < 48; ++i)
        for (int j = 0; j < 56; ++j) { uint64_t u; memcpy(&u, &C[i][j], 8); h = (h ^ u) * 1099511628211ull; }
    printf("%016llx %.17g\n", (unsigned long long)h, C[20][30]);
    return 0;
}
