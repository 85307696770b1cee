void wave4(double u[1028][1028][1028], double up[1028][1028][1028], double un[1028][1028][1028], double vel2[1028][1028][1028], double c0, double c1, double c2, int kbeg, int kend, int ny, int nx) {
    int i, j, k;
    double lap;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop worker
        for (j = 2; j < ny - 2; j++) {
            #pragma acc loop vector
            for (i = 2; i < nx - 2; i++) {
                int _v8, _v10, _v13, _v16, _v19, _v22, _v29, _v31, _v34, _v37, _v40, _v43;
                double _v20, _v23, _v41, _v44, _v14, _v17, _v35, _v38, _v11, _v30, _v32, _v9, _v4, _v50, _v52, _v5, _v12, _v15, _v18, _v21, _v24, _v25, _v26, _v33, _v36, _v39, _v42, _v45, _v46, _v47;
                _v8 = i + 1;
                _v10 = i - 1;
                _v13 = j + 1;
                _v16 = j - 1;
                _v19 = k + 1;
                _v22 = k - 1;
                _v29 = i + 2;
                _v31 = i - 2;
                _v34 = j + 2;
                _v37 = j - 2;
                _v40 = k + 2;
                _v43 = k - 2;
                _v20 = u[_v19][j][i];
                _v23 = u[_v22][j][i];
                _v41 = u[_v40][j][i];
                _v44 = u[_v43][j][i];
                _v14 = u[k][_v13][i];
                _v17 = u[k][_v16][i];
                _v35 = u[k][_v34][i];
                _v38 = u[k][_v37][i];
                _v11 = u[k][j][_v10];
                _v30 = u[k][j][_v29];
                _v32 = u[k][j][_v31];
                _v9 = u[k][j][_v8];
                _v4 = u[k][j][i];
                _v50 = up[k][j][i];
                _v52 = vel2[k][j][i];
                _v5 = c0 * _v4;
                _v12 = _v9 + _v11;
                _v15 = _v12 + _v14;
                _v18 = _v15 + _v17;
                _v21 = _v18 + _v20;
                _v24 = _v21 + _v23;
                _v25 = c1 * _v24;
                _v26 = _v5 + _v25;
                _v33 = _v30 + _v32;
                _v36 = _v33 + _v35;
                _v39 = _v36 + _v38;
                _v42 = _v39 + _v41;
                _v45 = _v42 + _v44;
                _v46 = c2 * _v45;
                _v47 = _v26 + _v46;
                lap = _v47;
                {
                    double _v49, _v51, _v53, _v54;
                    _v49 = 2.0 * _v4;
                    _v51 = _v49 - _v50;
                    _v53 = _v52 * _v47;
                    _v54 = _v51 + _v53;
                    un[k][j][i] = _v54;
                }
            }
        }
    }
}
