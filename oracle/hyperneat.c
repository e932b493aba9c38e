/*
 * hyperneat.c -- TEST INFRASTRUCTURE ONLY (see flatneat_oracle.h).
 *
 * FP64 restatement of BASELINE config 4 (HyperNEAT on a synthetic
 * linear-dynamics rollout).  The reference has no HyperNEAT
 * code (SPEC.md:8 lists it out of scope), so these semantics are this
 * repo's definition, written down once here and in DESIGN.md section 9 and
 * restated by the CUDA path (csrc/hyper.cu): "parity unpinned" for the
 * substrate / rollout rules themselves.  The CPPN evaluation that feeds them
 * is the reference's own forward (network.hpp:238-330), checked by the tests
 * through oracle/_ref.
 *
 *   substrate   input i in [0, n_obs] at (x = -1 + 2 i / n_obs, y = -1)
 *               (i = n_obs is the bias input, value 1); output j in
 *               [0, n_act) at (x = -1 + 2 j / max(1, n_act - 1), y = +1)
 *   query q     = j * (n_obs + 1) + i, CPPN inputs (x_i, y_i, x_j, y_j, 1)
 *   weight      y' = clamp(cppn_out, -1, 1); |y'| < threshold -> 0, else
 *               sign(y') (|y'| - threshold) / (1 - threshold) * max_weight
 *   policy      a_j = tanh(sum_i W[j][i] s_i + W[j][n_obs])
 *   dynamics    s' = A s + B a                (A: n_obs x n_obs, B: n_obs x n_act)
 *   reward      r = -(sum_i s'_i^2) / n_obs - act_cost * (sum_j a_j^2) / n_act
 *   fitness     mean of r over `steps` steps, from s0
 */
#include <math.h>

#include "flatneat_oracle.h"

void fo_hyper_queries(const fo_hyper_cfg* c, double* q) {
  const int ni = c->n_obs + 1;
  for (int j = 0; j < c->n_act; ++j)
    for (int i = 0; i < ni; ++i) {
      double* r = q + 5 * (j * ni + i);
      r[0] = -1.0 + 2.0 * i / c->n_obs;
      r[1] = -1.0;
      r[2] = -1.0 + 2.0 * j / (c->n_act > 1 ? c->n_act - 1 : 1);
      r[3] = 1.0;
      r[4] = 1.0;
    }
}

double fo_hyper_weight(const fo_hyper_cfg* c, double y) {
  const double v = y < -1.0 ? -1.0 : (y > 1.0 ? 1.0 : y);
  const double m = fabs(v);
  if (m < c->weight_threshold) return 0.0;
  const double w = (m - c->weight_threshold) / (1.0 - c->weight_threshold) * c->max_weight;
  return v < 0.0 ? -w : w;
}

void fo_hyper_substrate(const fo_hyper_cfg* c, const double* cppn_out, double* W) {
  const int Q = (c->n_obs + 1) * c->n_act;
  for (int q = 0; q < Q; ++q) W[q] = fo_hyper_weight(c, cppn_out[q]);
}

double fo_hyper_rollout(const fo_hyper_cfg* c, const double* W, const double* A, const double* B,
                        const double* s0) {
  const int no = c->n_obs, na = c->n_act, ni = no + 1;
  double s[64], sn[64], a[64];
  if (no > 64 || na > 64) return NAN;
  for (int i = 0; i < no; ++i) s[i] = s0[i];
  double total = 0.0;
  for (int t = 0; t < c->steps; ++t) {
    double act_sq = 0.0;
    for (int j = 0; j < na; ++j) {
      double z = W[j * ni + no];
      for (int i = 0; i < no; ++i) z += W[j * ni + i] * s[i];
      a[j] = tanh(z);
      act_sq += a[j] * a[j];
    }
    double st_sq = 0.0;
    for (int i = 0; i < no; ++i) {
      double v = 0.0;
      for (int k = 0; k < no; ++k) v += A[i * no + k] * s[k];
      for (int j = 0; j < na; ++j) v += B[i * na + j] * a[j];
      sn[i] = v;
      st_sq += v * v;
    }
    total += -(st_sq / no) - c->act_cost * (act_sq / na);
    for (int i = 0; i < no; ++i) s[i] = sn[i];
  }
  return total / c->steps;
}
