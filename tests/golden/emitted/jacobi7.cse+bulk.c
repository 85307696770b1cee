void jacobi7(double A0[258][258][258], double Anext[258][258][258], double c0, double c1, int kbeg, int kend, int ny, int nx) {
    int i, j, k;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop worker
        for (j = 1; j < ny - 1; j++) {
            #pragma acc loop vector
            for (i = 1; i < nx - 1; i++) {
                int _v4, _v6, _v9, _v12, _v15, _v18;
                double _v5, _v7, _v13, _v10, _v16, _v19, _v23, _v8, _v11, _v14, _v17, _v20, _v22, _v25, _v26;
                _v4 = k + 1;
                _v6 = k - 1;
                _v9 = j + 1;
                _v12 = j - 1;
                _v15 = i + 1;
                _v18 = i - 1;
                _v5 = A0[_v4][j][i];
                _v7 = A0[_v6][j][i];
                _v13 = A0[k][_v12][i];
                _v10 = A0[k][_v9][i];
                _v16 = A0[k][j][_v15];
                _v19 = A0[k][j][_v18];
                _v23 = A0[k][j][i];
                _v8 = _v5 + _v7;
                _v11 = _v8 + _v10;
                _v14 = _v11 + _v13;
                _v17 = _v14 + _v16;
                _v20 = _v17 + _v19;
                _v22 = _v20 * c1;
                _v25 = _v23 * c0;
                _v26 = _v22 - _v25;
                Anext[k][j][i] = _v26;
            }
        }
    }
}
