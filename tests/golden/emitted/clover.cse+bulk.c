void ideal_gas(double density[7684][7684], double energy[7684][7684], double pressure[7684][7684], double soundspeed[7684][7684], int kbeg, int kend, int nx) {
    int j, k;
    double v, pressurebyenergy, pressurebyvolume, sound_speed_squared;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop vector
        for (j = 2; j < nx - 2; j++) {
            double _v3, _v8, _v4;
            _v3 = density[k][j];
            _v8 = energy[k][j];
            _v4 = 1.0 / _v3;
            v = _v4;
            {
                double _v6, _v7, _v9;
                _v6 = 1.4 - 1.0;
                _v7 = _v6 * _v3;
                _v9 = _v7 * _v8;
                pressure[k][j] = _v9;
                pressurebyenergy = _v7;
                {
                    double _v10, _v11;
                    _v10 = -_v3;
                    _v11 = _v10 * _v9;
                    pressurebyvolume = _v11;
                    {
                        double _v12, _v13, _v14, _v15;
                        _v12 = _v4 * _v4;
                        _v13 = _v9 * _v7;
                        _v14 = _v13 - _v11;
                        _v15 = _v12 * _v14;
                        sound_speed_squared = _v15;
                        {
                            double _v16;
                            _v16 = sqrt(_v15);
                            soundspeed[k][j] = _v16;
                        }
                    }
                }
            }
        }
    }
}

void pdv_predict(double xarea[7684][7684], double yarea[7684][7684], double volume[7684][7684], double density0[7684][7684], double density1[7684][7684], double energy0[7684][7684], double energy1[7684][7684], double pressure[7684][7684], double viscosity[7684][7684], double xvel0[7684][7684], double yvel0[7684][7684], double volume_change[7684][7684], double dt, int kbeg, int kend, int nx) {
    int j, k;
    double left_flux, right_flux, bottom_flux, top_flux, total_flux, recip_volume, energy_change, min_cell_volume;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop vector
        for (j = 2; j < nx - 2; j++) {
            int _v5, _v17;
            double _v65, _v72, _v64, _v67, _v51, _v18, _v2, _v20, _v6, _v19, _v3, _v38, _v28, _v40, _v39, _v30, _v29, _v7, _v8, _v9, _v10, _v12, _v14, _v16;
            _v5 = k + 1;
            _v17 = j + 1;
            _v65 = density0[k][j];
            _v72 = energy0[k][j];
            _v64 = pressure[k][j];
            _v67 = viscosity[k][j];
            _v51 = volume[k][j];
            _v18 = xarea[k][_v17];
            _v2 = xarea[k][j];
            _v20 = xvel0[_v5][_v17];
            _v6 = xvel0[_v5][j];
            _v19 = xvel0[k][_v17];
            _v3 = xvel0[k][j];
            _v38 = yarea[_v5][j];
            _v28 = yarea[k][j];
            _v40 = yvel0[_v5][_v17];
            _v39 = yvel0[_v5][j];
            _v30 = yvel0[k][_v17];
            _v29 = yvel0[k][j];
            _v7 = _v3 + _v6;
            _v8 = _v7 + _v3;
            _v9 = _v8 + _v6;
            _v10 = _v2 * _v9;
            _v12 = _v10 * 0.25;
            _v14 = _v12 * dt;
            _v16 = _v14 * 0.5;
            left_flux = _v16;
            {
                double _v21, _v22, _v23, _v24, _v25, _v26, _v27;
                _v21 = _v19 + _v20;
                _v22 = _v21 + _v19;
                _v23 = _v22 + _v20;
                _v24 = _v18 * _v23;
                _v25 = _v24 * 0.25;
                _v26 = _v25 * dt;
                _v27 = _v26 * 0.5;
                right_flux = _v27;
                {
                    double _v31, _v32, _v33, _v34, _v35, _v36, _v37;
                    _v31 = _v29 + _v30;
                    _v32 = _v31 + _v29;
                    _v33 = _v32 + _v30;
                    _v34 = _v28 * _v33;
                    _v35 = _v34 * 0.25;
                    _v36 = _v35 * dt;
                    _v37 = _v36 * 0.5;
                    bottom_flux = _v37;
                    {
                        double _v41, _v42, _v43, _v44, _v45, _v46, _v47;
                        _v41 = _v39 + _v40;
                        _v42 = _v41 + _v39;
                        _v43 = _v42 + _v40;
                        _v44 = _v38 * _v43;
                        _v45 = _v44 * 0.25;
                        _v46 = _v45 * dt;
                        _v47 = _v46 * 0.5;
                        top_flux = _v47;
                        {
                            double _v48, _v49, _v50;
                            _v48 = _v27 - _v16;
                            _v49 = _v48 + _v47;
                            _v50 = _v49 - _v37;
                            total_flux = _v50;
                            {
                                double _v52, _v53;
                                _v52 = _v51 + _v50;
                                _v53 = _v51 / _v52;
                                volume_change[k][j] = _v53;
                                {
                                    double _v54, _v55, _v56, _v57, _v58, _v59, _v60, _v61;
                                    _v54 = _v51 + _v27;
                                    _v55 = _v54 - _v16;
                                    _v56 = _v55 + _v47;
                                    _v57 = _v56 - _v37;
                                    _v58 = fmin(_v57, _v55);
                                    _v59 = _v51 + _v47;
                                    _v60 = _v59 - _v37;
                                    _v61 = fmin(_v58, _v60);
                                    min_cell_volume = _v61;
                                    {
                                        double _v63;
                                        _v63 = 1.0 / _v51;
                                        recip_volume = _v63;
                                        {
                                            double _v66, _v68, _v69, _v70, _v71;
                                            _v66 = _v64 / _v65;
                                            _v68 = _v67 / _v65;
                                            _v69 = _v66 + _v68;
                                            _v70 = _v69 * _v50;
                                            _v71 = _v70 * _v63;
                                            energy_change = _v71;
                                            {
                                                double _v73;
                                                _v73 = _v72 - _v71;
                                                energy1[k][j] = _v73;
                                                {
                                                    double _v74;
                                                    _v74 = _v65 * _v53;
                                                    density1[k][j] = _v74;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
    }
}

void advec_cell_x(double vol_flux_x[7684][7684], double pre_vol[7684][7684], double density1[7684][7684], double energy1[7684][7684], double mass_flux_x[7684][7684], double ener_flux[7684][7684], double vertexdx[7684], double one_by_six, int kbeg, int kend, int nx) {
    int j, k, upwind, donor, downwind, dif;
    double sigmat, sigma3, sigma4, sigmav, sigmam, diffuw, diffdw, wind, limiter;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop vector
        for (j = 2; j < nx - 2; j++) {
            int _v4;
            double _v23, _v11;
            _v23 = vertexdx[j];
            _v11 = vol_flux_x[k][j];
            _v4 = j - 1;
            if (vol_flux_x[k][j] > 0.0) {
                int _v2;
                _v2 = j - 2;
                upwind = _v2;
                donor = _v4;
                downwind = j;
                dif = _v4;
            } else {
                int _v5;
                _v5 = j + 1;
                upwind = _v5;
                if (upwind > nx - 1) {
                    int _v7;
                    _v7 = nx - 1;
                    upwind = _v7;
                }
                donor = j;
                downwind = _v4;
                dif = upwind;
            }
            {
                double _v29, _v32, _v30, _v57, _v60, _v58, _v19, _v24, _v18, _v20;
                _v29 = density1[k][donor];
                _v32 = density1[k][downwind];
                _v30 = density1[k][upwind];
                _v57 = energy1[k][donor];
                _v60 = energy1[k][downwind];
                _v58 = energy1[k][upwind];
                _v19 = pre_vol[k][donor];
                _v24 = vertexdx[dif];
                _v18 = fabs(_v11);
                _v20 = _v18 / _v19;
                sigmat = _v20;
                {
                    double _v22, _v25, _v26;
                    _v22 = 1.0 + _v20;
                    _v25 = _v23 / _v24;
                    _v26 = _v22 * _v25;
                    sigma3 = _v26;
                    {
                        double _v28;
                        _v28 = 2.0 - _v20;
                        sigma4 = _v28;
                        sigmav = _v20;
                        {
                            double _v31;
                            _v31 = _v29 - _v30;
                            diffuw = _v31;
                            {
                                double _v33;
                                _v33 = _v32 - _v29;
                                diffdw = _v33;
                                wind = 1.0;
                                {
                                    double _v34;
                                    _v34 = -1.0;
                                    if (diffdw <= 0.0)
                                        wind = _v34;
                                    if (diffuw * diffdw > 0.0) {
                                        double _v37, _v38, _v39, _v40, _v41, _v43, _v44, _v45, _v46, _v47, _v48;
                                        _v37 = 1.0 - _v20;
                                        _v38 = _v37 * wind;
                                        _v39 = fabs(_v31);
                                        _v40 = fabs(_v33);
                                        _v41 = fmin(_v39, _v40);
                                        _v43 = _v26 * _v39;
                                        _v44 = _v28 * _v40;
                                        _v45 = _v43 + _v44;
                                        _v46 = one_by_six * _v45;
                                        _v47 = fmin(_v41, _v46);
                                        _v48 = _v38 * _v47;
                                        limiter = _v48;
                                    } else {
                                        limiter = 0.0;
                                    }
                                    {
                                        double _v52, _v53;
                                        _v52 = _v29 + limiter;
                                        _v53 = _v11 * _v52;
                                        mass_flux_x[k][j] = _v53;
                                        {
                                            double _v54, _v55, _v56;
                                            _v54 = fabs(_v53);
                                            _v55 = _v29 * _v19;
                                            _v56 = _v54 / _v55;
                                            sigmam = _v56;
                                            {
                                                double _v59;
                                                _v59 = _v57 - _v58;
                                                diffuw = _v59;
                                                {
                                                    double _v61;
                                                    _v61 = _v60 - _v57;
                                                    diffdw = _v61;
                                                    wind = 1.0;
                                                    if (diffdw <= 0.0)
                                                        wind = _v34;
                                                    if (diffuw * diffdw > 0.0) {
                                                        double _v64, _v65, _v66, _v67, _v68, _v69, _v70, _v71, _v72, _v73, _v74;
                                                        _v64 = 1.0 - _v56;
                                                        _v65 = _v64 * wind;
                                                        _v66 = fabs(_v59);
                                                        _v67 = fabs(_v61);
                                                        _v68 = fmin(_v66, _v67);
                                                        _v69 = _v26 * _v66;
                                                        _v70 = _v28 * _v67;
                                                        _v71 = _v69 + _v70;
                                                        _v72 = one_by_six * _v71;
                                                        _v73 = fmin(_v68, _v72);
                                                        _v74 = _v65 * _v73;
                                                        limiter = _v74;
                                                    } else {
                                                        limiter = 0.0;
                                                    }
                                                    {
                                                        double _v78, _v79;
                                                        _v78 = _v57 + limiter;
                                                        _v79 = _v53 * _v78;
                                                        ener_flux[k][j] = _v79;
                                                    }
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    }
                }
            }
        }
    }
}
