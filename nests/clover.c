/* K4 clover — CloverLeaf-style 2-D hydro nests ideal_gas, PdV (predict) and
 * advec_cell (x sweep), in the satcc kernel subset.  Arrays are [nx][nx] =
 * [N+4][N+4] with a 2-cell halo; the update covers k, j in 2 .. N+1.  The
 * upwind clamp is CloverLeaf's MIN(j+1, x_max+2) = nx - 1.
 * BASELINE config: N = 7680 fp64. */
void ideal_gas(double density[7684][7684], double energy[7684][7684], double pressure[7684][7684], double soundspeed[7684][7684], int kbeg, int kend, int nx) {
    int j, k;
    double v, pressurebyenergy, pressurebyvolume, sound_speed_squared;
    #pragma acc parallel loop gang
    for (k = kbeg; k < kend; k++) {
        #pragma acc loop vector
        for (j = 2; j < nx - 2; j++) {
            v = 1.0 / density[k][j];
            pressure[k][j] = (1.4 - 1.0) * density[k][j] * energy[k][j];
            pressurebyenergy = (1.4 - 1.0) * density[k][j];
            pressurebyvolume = -density[k][j] * pressure[k][j];
            sound_speed_squared = v * v * (pressure[k][j] * pressurebyenergy - pressurebyvolume);
            soundspeed[k][j] = sqrt(sound_speed_squared);
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
            left_flux = (xarea[k][j] * (xvel0[k][j] + xvel0[k + 1][j] + xvel0[k][j] + xvel0[k + 1][j])) * 0.25 * dt * 0.5;
            right_flux = (xarea[k][j + 1] * (xvel0[k][j + 1] + xvel0[k + 1][j + 1] + xvel0[k][j + 1] + xvel0[k + 1][j + 1])) * 0.25 * dt * 0.5;
            bottom_flux = (yarea[k][j] * (yvel0[k][j] + yvel0[k][j + 1] + yvel0[k][j] + yvel0[k][j + 1])) * 0.25 * dt * 0.5;
            top_flux = (yarea[k + 1][j] * (yvel0[k + 1][j] + yvel0[k + 1][j + 1] + yvel0[k + 1][j] + yvel0[k + 1][j + 1])) * 0.25 * dt * 0.5;
            total_flux = right_flux - left_flux + top_flux - bottom_flux;
            volume_change[k][j] = volume[k][j] / (volume[k][j] + total_flux);
            min_cell_volume = fmin(fmin(volume[k][j] + right_flux - left_flux + top_flux - bottom_flux, volume[k][j] + right_flux - left_flux), volume[k][j] + top_flux - bottom_flux);
            recip_volume = 1.0 / volume[k][j];
            energy_change = (pressure[k][j] / density0[k][j] + viscosity[k][j] / density0[k][j]) * total_flux * recip_volume;
            energy1[k][j] = energy0[k][j] - energy_change;
            density1[k][j] = density0[k][j] * volume_change[k][j];
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
            if (vol_flux_x[k][j] > 0.0) {
                upwind = j - 2;
                donor = j - 1;
                downwind = j;
                dif = donor;
            } else {
                upwind = j + 1;
                if (upwind > nx - 1) upwind = nx - 1;
                donor = j;
                downwind = j - 1;
                dif = upwind;
            }
            sigmat = fabs(vol_flux_x[k][j]) / pre_vol[k][donor];
            sigma3 = (1.0 + sigmat) * (vertexdx[j] / vertexdx[dif]);
            sigma4 = 2.0 - sigmat;
            sigmav = sigmat;
            diffuw = density1[k][donor] - density1[k][upwind];
            diffdw = density1[k][downwind] - density1[k][donor];
            wind = 1.0;
            if (diffdw <= 0.0) wind = -1.0;
            if (diffuw * diffdw > 0.0) {
                limiter = (1.0 - sigmav) * wind * fmin(fmin(fabs(diffuw), fabs(diffdw)), one_by_six * (sigma3 * fabs(diffuw) + sigma4 * fabs(diffdw)));
            } else {
                limiter = 0.0;
            }
            mass_flux_x[k][j] = vol_flux_x[k][j] * (density1[k][donor] + limiter);
            sigmam = fabs(mass_flux_x[k][j]) / (density1[k][donor] * pre_vol[k][donor]);
            diffuw = energy1[k][donor] - energy1[k][upwind];
            diffdw = energy1[k][downwind] - energy1[k][donor];
            wind = 1.0;
            if (diffdw <= 0.0) wind = -1.0;
            if (diffuw * diffdw > 0.0) {
                limiter = (1.0 - sigmam) * wind * fmin(fmin(fabs(diffuw), fabs(diffdw)), one_by_six * (sigma3 * fabs(diffuw) + sigma4 * fabs(diffdw)));
            } else {
                limiter = 0.0;
            }
            ener_flux[k][j] = mass_flux_x[k][j] * (energy1[k][donor] + limiter);
        }
    }
}
