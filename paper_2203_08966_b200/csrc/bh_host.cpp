// bh_host.cpp -- host-side helpers of libbh.so for initial conditions (not the
// hot path).  They restate the reference's scalar generators operation for
// operation so that ICs are bit-identical to nbsim.initcond for a given seed:
// the Philox stream itself is drawn by numpy (the caller passes the doubles),
// and libm's pow/sqrt/sin/cos are the ones numpy's scalar paths call.
// Compiled with -ffp-contract=off (the reference never fuses multiply-adds).
#include <math.h>
#include <stdint.h>

extern "C" {

// initcond.py:62-77 plummer_cluster, consuming pre-drawn uniforms.
// Generates up to n bodies; stops early (returning the bodies completed) if
// the draw buffer runs out mid-body.  *used = draws consumed by the completed
// bodies.  pos/vel are [n][3].
int64_t bh_ic_plummer(const double *u, int64_t nu, int64_t n, double total_mass,
                      double *pos, double *vel, int64_t *used) {
  int64_t k = 0, done = 0;
  const double kPi2 = 2.0 * M_PI;
  const double vscale = sqrt(2.0 * total_mass);
  for (int64_t i = 0; i < n; ++i) {
    int64_t k0 = k;
    double r;
    // _radius (initcond.py:42-50)
    for (;;) {
      if (k >= nu) goto out;
      double a = u[k++];
      if (a == 0.0) continue;
      r = 1.0 / sqrt(pow(a, -2.0 / 3.0) - 1.0);
      if (r < 10.0) break;
    }
    {
      // _unit_vector (initcond.py:32-37)
      if (k + 2 > nu) { k = k0; goto out; }
      double z = 2.0 * u[k++] - 1.0;
      double phi = kPi2 * u[k++];
      double t = 1.0 - z * z;
      double s = sqrt(t > 0.0 ? t : 0.0);
      double ux = s * cos(phi), uy = s * sin(phi), uz = z;
      double v_esc = vscale * pow(1.0 + r * r, -0.25);
      // _speed_fraction (initcond.py:53-59)
      double q;
      for (;;) {
        if (k + 2 > nu) { k = k0; goto out; }
        q = u[k++];
        double g = 0.1 * u[k++];
        if (g < q * q * pow(1.0 - q * q, 3.5)) break;
      }
      double qv = q * v_esc;
      if (k + 2 > nu) { k = k0; goto out; }
      double z2 = 2.0 * u[k++] - 1.0;
      double phi2 = kPi2 * u[k++];
      double t2 = 1.0 - z2 * z2;
      double s2 = sqrt(t2 > 0.0 ? t2 : 0.0);
      pos[3 * i] = r * ux; pos[3 * i + 1] = r * uy; pos[3 * i + 2] = r * uz;
      vel[3 * i] = qv * (s2 * cos(phi2));
      vel[3 * i + 1] = qv * (s2 * sin(phi2));
      vel[3 * i + 2] = qv * z2;
      done = i + 1;
    }
  }
out:
  *used = k;
  return done;
}

// physics.py:273-285 _potential_pairs in its sequential pair order (used by
// initcond.standardize so that standardised ICs match the reference bitwise).
double bh_host_potential_pairs(const double *mass, const double *pos, int64_t n, double eps) {
  const double e2 = eps * eps;
  double pot = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      double dx = pos[3 * i] - pos[3 * j], dy = pos[3 * i + 1] - pos[3 * j + 1],
             dz = pos[3 * i + 2] - pos[3 * j + 2];
      double r2 = dx * dx + dy * dy + dz * dz;
      pot -= mass[i] * mass[j] / sqrt(r2 + e2);
    }
  return pot;
}
}
