/* K1 jacobi7 — Parboil/SPEC-ACCEL ostencil-style 7-point Jacobi sweep, in the
 * satcc kernel subset (proj/src/parser.cpp:60-125).  Array-parameter form so a
 * harness can ping-pong A0/Anext and hand each worker a [kbeg, kend) slab.
 * ny, nx are the full array extents; the interior is 1 .. n-2.
 * BASELINE config: 258^3 fp64 (interior 256^3), c0 = 1/6, c1 = 1/36. */
void jacobi7(double A0[258][258][258], double Anext[258][258][258], double c0, double c1, int kbeg, int kend, int ny, int nx) {
    int i, j, k;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop worker
        for (j = 1; j < ny - 1; j++) {
            #pragma acc loop vector
            for (i = 1; i < nx - 1; i++) {
                Anext[k][j][i] = (A0[k + 1][j][i] + A0[k - 1][j][i] + A0[k][j + 1][i] + A0[k][j - 1][i] + A0[k][j][i + 1] + A0[k][j][i - 1]) * c1 - A0[k][j][i] * c0;
            }
        }
    }
}
