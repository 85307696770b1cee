/* Nest file for the wrapper hand-off tests: an unmarked time loop ENCLOSING
 * two parallel regions, a live-in local (w, computed before the loop), the
 * enclosing loop index read inside a region (t), and a region temporary (r).
 * The hand-off keeps the time loop on the host and launches each region in
 * place (paper_2306_13002_b200/jit.py offload_regions). */
void relax(double a[66][71], double b[66][71], double c, int nt, int ny, int nx) {
    int t, j, i;
    double w;
    double r;
    w = 0.25 * c;
    for (t = 0; t < nt; t++) {
        #pragma acc parallel loop gang
        for (j = 1; j < ny - 1; j++) {
            #pragma acc loop vector
            for (i = 1; i < nx - 1; i++) {
                r = a[j][i - 1] + a[j][i + 1] + a[j - 1][i] + a[j + 1][i];
                b[j][i] = a[j][i] + w * (r - 4.0 * a[j][i]) + 0.001 * t;
            }
        }
        #pragma acc parallel loop gang
        for (j = 1; j < ny - 1; j++) {
            #pragma acc loop vector
            for (i = 1; i < nx - 1; i++) {
                a[j][i] = 0.5 * b[j][i] + 0.5 * a[j][i];
            }
        }
    }
}
