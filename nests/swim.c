/* K3 swim — SPEC swim shallow-water calc1/calc2/calc3 nests (one region each),
 * in the satcc kernel subset.  Arrays are [nx][nx] = [N+1][N+1]; the update
 * covers j, i in 0 .. N-1 with one-sided +1 neighbours.  [jbeg, jend) is the
 * row slab handed to one worker.  BASELINE config: N = 8192 fp64. */
void calc1(double u[8193][8193], double v[8193][8193], double p[8193][8193], double cu[8193][8193], double cv[8193][8193], double z[8193][8193], double h[8193][8193], double fsdx, double fsdy, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            cu[j][i + 1] = 0.5 * (p[j][i + 1] + p[j][i]) * u[j][i + 1];
            cv[j + 1][i] = 0.5 * (p[j + 1][i] + p[j][i]) * v[j + 1][i];
            z[j + 1][i + 1] = (fsdx * (v[j + 1][i + 1] - v[j + 1][i]) - fsdy * (u[j + 1][i + 1] - u[j][i + 1])) / (p[j][i] + p[j][i + 1] + p[j + 1][i + 1] + p[j + 1][i]);
            h[j][i] = p[j][i] + 0.25 * (u[j][i + 1] * u[j][i + 1] + u[j][i] * u[j][i] + v[j + 1][i] * v[j + 1][i] + v[j][i] * v[j][i]);
        }
    }
}

void calc2(double uold[8193][8193], double vold[8193][8193], double pold[8193][8193], double unew[8193][8193], double vnew[8193][8193], double pnew[8193][8193], double cu[8193][8193], double cv[8193][8193], double z[8193][8193], double h[8193][8193], double tdts8, double tdtsdx, double tdtsdy, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            unew[j][i + 1] = uold[j][i + 1] + tdts8 * (z[j + 1][i + 1] + z[j][i + 1]) * (cv[j + 1][i + 1] + cv[j + 1][i] + cv[j][i] + cv[j][i + 1]) - tdtsdx * (h[j][i + 1] - h[j][i]);
            vnew[j + 1][i] = vold[j + 1][i] - tdts8 * (z[j + 1][i + 1] + z[j + 1][i]) * (cu[j + 1][i + 1] + cu[j + 1][i] + cu[j][i] + cu[j][i + 1]) - tdtsdy * (h[j + 1][i] - h[j][i]);
            pnew[j][i] = pold[j][i] - tdtsdx * (cu[j][i + 1] - cu[j][i]) - tdtsdy * (cv[j + 1][i] - cv[j][i]);
        }
    }
}

void calc3(double u[8193][8193], double v[8193][8193], double p[8193][8193], double uold[8193][8193], double vold[8193][8193], double pold[8193][8193], double unew[8193][8193], double vnew[8193][8193], double pnew[8193][8193], double alpha, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            uold[j][i] = u[j][i] + alpha * (unew[j][i] - 2.0 * u[j][i] + uold[j][i]);
            vold[j][i] = v[j][i] + alpha * (vnew[j][i] - 2.0 * v[j][i] + vold[j][i]);
            pold[j][i] = p[j][i] + alpha * (pnew[j][i] - 2.0 * p[j][i] + pold[j][i]);
            u[j][i] = unew[j][i];
            v[j][i] = vnew[j][i];
            p[j][i] = pnew[j][i];
        }
    }
}
