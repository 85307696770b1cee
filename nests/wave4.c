/* K5 wave4 — seismic 3-D 4th-order acoustic wave step (leapfrog, 3-level
 * rotation up -> u -> un), in the satcc kernel subset.  The subset has no
 * float (proj/include/satcc/ast.hpp:84), so the text is double; the fp32
 * BASELINE config (1028^3 with a 2-plane halo, interior 1024^3) runs a
 * textual double->float copy.  ny, nx are full extents; interior 2 .. n-3. */
void wave4(double u[1028][1028][1028], double up[1028][1028][1028], double un[1028][1028][1028], double vel2[1028][1028][1028], double c0, double c1, double c2, int kbeg, int kend, int ny, int nx) {
    int i, j, k;
    double lap;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop worker
        for (j = 2; j < ny - 2; j++) {
            #pragma acc loop vector
            for (i = 2; i < nx - 2; i++) {
                lap = c0 * u[k][j][i] + c1 * (u[k][j][i + 1] + u[k][j][i - 1] + u[k][j + 1][i] + u[k][j - 1][i] + u[k + 1][j][i] + u[k - 1][j][i]) + c2 * (u[k][j][i + 2] + u[k][j][i - 2] + u[k][j + 2][i] + u[k][j - 2][i] + u[k + 2][j][i] + u[k - 2][j][i]);
                un[k][j][i] = 2.0 * u[k][j][i] - up[k][j][i] + vel2[k][j][i] * lap;
            }
        }
    }
}
