/* A user nest file for the B200 hand-off test (not a benchmark nest): a 2-D
 * heat-equation step with a nonlinear source, in the satcc kernel subset. */
void heat(double t[130][131], double tn[130][131], double src[130][131], double kappa, double dt, int jbeg,
          int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 1; i < nx - 1; i++) {
            tn[j][i] = t[j][i] + dt * (kappa * (t[j][i + 1] + t[j][i - 1] + t[j + 1][i] + t[j - 1][i] - 4.0 * t[j][i])
                       + src[j][i] * t[j][i] * t[j][i]);
        }
    }
}
