void calc1(double u[8193][8193], double v[8193][8193], double p[8193][8193], double cu[8193][8193], double cv[8193][8193], double z[8193][8193], double h[8193][8193], double fsdx, double fsdy, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            int _v3, _v11;
            double _v27, _v12, _v5, _v6, _v22, _v9, _v33, _v18, _v15, _v38, _v7, _v8, _v10;
            _v3 = i + 1;
            _v11 = j + 1;
            _v27 = p[_v11][_v3];
            _v12 = p[_v11][i];
            _v5 = p[j][_v3];
            _v6 = p[j][i];
            _v22 = u[_v11][_v3];
            _v9 = u[j][_v3];
            _v33 = u[j][i];
            _v18 = v[_v11][_v3];
            _v15 = v[_v11][i];
            _v38 = v[j][i];
            _v7 = _v5 + _v6;
            _v8 = 0.5 * _v7;
            _v10 = _v8 * _v9;
            cu[j][i + 1] = _v10;
            {
                double _v13, _v14, _v16;
                _v13 = _v12 + _v6;
                _v14 = 0.5 * _v13;
                _v16 = _v14 * _v15;
                cv[j + 1][i] = _v16;
                {
                    double _v19, _v20, _v23, _v24, _v25, _v28, _v29, _v30;
                    _v19 = _v18 - _v15;
                    _v20 = fsdx * _v19;
                    _v23 = _v22 - _v9;
                    _v24 = fsdy * _v23;
                    _v25 = _v20 - _v24;
                    _v28 = _v7 + _v27;
                    _v29 = _v28 + _v12;
                    _v30 = _v25 / _v29;
                    z[j + 1][i + 1] = _v30;
                    {
                        double _v32, _v35, _v37, _v40, _v42;
                        _v32 = _v9 * _v9;
                        _v35 = _v32 + _v33 * _v33;
                        _v37 = _v35 + _v15 * _v15;
                        _v40 = _v37 + _v38 * _v38;
                        _v42 = _v6 + 0.25 * _v40;
                        h[j][i] = _v42;
                    }
                }
            }
        }
    }
}

void calc2(double uold[8193][8193], double vold[8193][8193], double pold[8193][8193], double unew[8193][8193], double vnew[8193][8193], double pnew[8193][8193], double cu[8193][8193], double cv[8193][8193], double z[8193][8193], double h[8193][8193], double tdts8, double tdtsdx, double tdtsdy, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            int _v3, _v6;
            double _v30, _v31, _v35, _v33, _v11, _v12, _v16, _v14, _v40, _v21, _v22, _v44, _v4, _v26, _v7, _v27, _v8, _v9, _v10, _v13, _v15, _v17, _v19, _v23, _v24, _v25;
            _v3 = i + 1;
            _v6 = j + 1;
            _v30 = cu[_v6][_v3];
            _v31 = cu[_v6][i];
            _v35 = cu[j][_v3];
            _v33 = cu[j][i];
            _v11 = cv[_v6][_v3];
            _v12 = cv[_v6][i];
            _v16 = cv[j][_v3];
            _v14 = cv[j][i];
            _v40 = h[_v6][i];
            _v21 = h[j][_v3];
            _v22 = h[j][i];
            _v44 = pold[j][i];
            _v4 = uold[j][_v3];
            _v26 = vold[_v6][i];
            _v7 = z[_v6][_v3];
            _v27 = z[_v6][i];
            _v8 = z[j][_v3];
            _v9 = _v7 + _v8;
            _v10 = tdts8 * _v9;
            _v13 = _v11 + _v12;
            _v15 = _v13 + _v14;
            _v17 = _v15 + _v16;
            _v19 = _v4 + _v10 * _v17;
            _v23 = _v21 - _v22;
            _v24 = tdtsdx * _v23;
            _v25 = _v19 - _v24;
            unew[j][i + 1] = _v25;
            {
                double _v28, _v29, _v32, _v34, _v36, _v37, _v38, _v41, _v42, _v43;
                _v28 = _v7 + _v27;
                _v29 = tdts8 * _v28;
                _v32 = _v30 + _v31;
                _v34 = _v32 + _v33;
                _v36 = _v34 + _v35;
                _v37 = _v29 * _v36;
                _v38 = _v26 - _v37;
                _v41 = _v40 - _v22;
                _v42 = tdtsdy * _v41;
                _v43 = _v38 - _v42;
                vnew[j + 1][i] = _v43;
                {
                    double _v45, _v46, _v47, _v48, _v49, _v50;
                    _v45 = _v35 - _v33;
                    _v46 = tdtsdx * _v45;
                    _v47 = _v44 - _v46;
                    _v48 = _v12 - _v14;
                    _v49 = tdtsdy * _v48;
                    _v50 = _v47 - _v49;
                    pnew[j][i] = _v50;
                }
            }
        }
    }
}

void calc3(double u[8193][8193], double v[8193][8193], double p[8193][8193], double uold[8193][8193], double vold[8193][8193], double pold[8193][8193], double unew[8193][8193], double vnew[8193][8193], double pnew[8193][8193], double alpha, int jbeg, int jend, int nx) {
    int i, j;
    #pragma acc parallel loop gang
    for (j = jbeg; j < jend; j++) {
        #pragma acc loop vector
        for (i = 0; i < nx - 1; i++) {
            double _v20, _v21, _v24, _v2, _v4, _v8, _v12, _v13, _v16, _v7, _v9, _v11;
            _v20 = p[j][i];
            _v21 = pnew[j][i];
            _v24 = pold[j][i];
            _v2 = u[j][i];
            _v4 = unew[j][i];
            _v8 = uold[j][i];
            _v12 = v[j][i];
            _v13 = vnew[j][i];
            _v16 = vold[j][i];
            _v7 = _v4 + -2.0 * _v2;
            _v9 = _v7 + _v8;
            _v11 = _v2 + alpha * _v9;
            uold[j][i] = _v11;
            {
                double _v15, _v17, _v19;
                _v15 = _v13 + -2.0 * _v12;
                _v17 = _v15 + _v16;
                _v19 = _v12 + alpha * _v17;
                vold[j][i] = _v19;
                {
                    double _v23, _v25, _v27;
                    _v23 = _v21 + -2.0 * _v20;
                    _v25 = _v23 + _v24;
                    _v27 = _v20 + alpha * _v25;
                    pold[j][i] = _v27;
                    u[j][i] = _v4;
                    v[j][i] = _v13;
                    p[j][i] = _v21;
                }
            }
        }
    }
}
