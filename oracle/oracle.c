/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the COMMET
 * hot path (arXiv 2510.00884): NCM constitutive update + FE residual/stiffness
 * assembly into a global vector and a CSR matrix.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA library under
 * paper_2510_00884_b200/ and never includes or links it.
 *
 * What it computes: with W(F) = N(k(F)) + kappa (J-1)^2
 * - s0 (J-1), k = (I1-3, I2-3, J-1), and Pi(u) = sum_e sum_q w_eq W(F_eq(u)),
 *   r = dPi/du  (Eq. apprx-r / r-quad, no traction)
 *   K = d2Pi/du du (Eq. apprx-k / k-quad, incl. the
 *       geometric delta_ij tau_kl term)
 * organised exactly as Alg. 1, in MATERIAL form
 * (App. A.1): P = F S, A_iJkL = d_ik S_JL + F_iI C_IJKL F_kK.
 * The inner network follows Alg. 4 literally.
 * No blocking, no fusion, no reordering beyond Alg. 1 / Alg. 4; full 3x3x3x3
 * arrays (no Voigt).  Readings of the paper: DESIGN.md "Readings".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int32_t n_hidden;          /* number of hidden layers (n-1 in Eq. icnn), >= 1 */
  int32_t width;             /* neurons per hidden layer */
  const double* W1;          /* [w][3]  A^(1) (+B^(1)) of Eq. icnn-mid-1 */
  const double* W;           /* [L-1][w][w]  A^(k), k = 2..L, row-major (out,in) */
  const double* b;           /* [L][w]  c^(k) */
  const double* a;           /* [w]     A^(n) (output layer, Eq. icnn-output) */
  const double* skip_out;    /* [3] or NULL: B^(n) */
  const double* skip_hidden; /* [L-1][w][3] or NULL: B^(k), k = 2..L */
  double kappa;              /* volumetric penalty kappa (J-1)^2 */
  double ref_shift;          /* s0: W -= s0 (J-1) (off when 0) */
  int32_t kinematics;        /* 0: K = (I1-3, I2-3, J-1); 1: isochoric (Ibar1-3, Ibar2-3, J-1) (App. A.2.2);
                                2: anisotropic (App. A.2.1); 3: isochoric anisotropic (App. A.2.2 with Ibar4/5,ij) */
  int32_t network;           /* 0: ICNN (Eq. icnn, Alg. 4); 1: CANN (Eq. cann-def); 2: Gent-Thomas (App. C) */
  int32_t cann_n;            /* CANN: branches per kinematic input */
  const int32_t* cann_f;     /* CANN [3][n][3]: f0 (0 id, 1 Macaulay, 2 abs), f1 power (1..3),
                                f2 (0: w1 x, 1: exp(w1 x) - 1, 2: -ln(1 - w1 x))  (Eq. cann-fs) */
  const double* cann_w1;     /* CANN [3][n] */
  const double* cann_w2;     /* CANN [3][n] */
  double gt[3];              /* Gent-Thomas: N = gt0 K1 + gt1 ln(1 + K2/3) + gt2 K3^2 */
  int32_t kan_layers;        /* ICKAN (App. B.3): R layers */
  const int32_t* kan_width;  /* [R+1], n_0 = 3, n_R = 1 */
  int32_t kan_nb, kan_k;     /* control points per edge, spline order */
  const double* kan_grid;    /* [R][2] xmin, xmax */
  const double* kan_w;       /* [edges] */
  const double* kan_c;       /* [edges][nb] */
  double a0[3];              /* anisotropic kinematics (kinematics = 2, 3): structural vector A0 (reference) */
  int32_t n_sv;              /* anisotropic: number of structural vectors, 1 (0 = 1) or 2 (a0, a1) */
  double a1[3];              /* anisotropic, n_sv = 2: the second structural vector */
} oracle_ncm;

/* ---------------------------------------------------------------------- */
/* activation F = softplus (BASELINE configs), F' = sigmoid, F'' = s(1-s)  */
/* ---------------------------------------------------------------------- */
static double softplus(double y) { return (y > 0 ? y : 0.0) + log1p(exp(-fabs(y))); }
static double sigmoid(double y) {
  double e = exp(-fabs(y));
  return y >= 0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

/*
 * Alg. 4: one pass giving N, dN/dK, d2N/dKdK.
 *   z <- K;  dz <- I;  d2z <- 0
 *   for k = 1..n-1:  y = A z + B K + c;  dy = A dz + B;  d2y = A d2z
 *                    d2z = F'(y) (.) d2y + F''(y) (.) dy (x) dy
 *                    dz  = F'(y) (.) dy;   z = F(y)
 *   N = A^(n) z + B^(n) K;  dN = A^(n) dz + B^(n);  d2N = A^(n) d2z
 * Layer 1 uses A^(1) = W1 (B^(1) folded in, SURVEY s8(c) reading 7); layers
 * k >= 2 use A^(k) = W[k-2], B^(k) = skip_hidden[k-2] (reading 6: B is the
 * current layer's B^(k)).
 */
static int icnn_eval(const oracle_ncm* m, int nk, const double* K, double* N_out, double* g_out,
                     double* H_out) {
  /* nk inputs (3; 5 for anisotropic kinematics): W1 is [w][nk]; hidden skips B^(k) [w][3] act on
   * the first three inputs only and are refused for nk != 3 */
  const int w = m->width, L = m->n_hidden, n2 = nk * nk;
  if (w < 1 || L < 1 || (nk != 3 && m->skip_hidden)) return 1;
  const int nmax = w > nk ? w : nk;
  double* z = (double*)calloc(nmax, sizeof(double));
  double* dz = (double*)calloc((size_t)nmax * nk, sizeof(double));
  double* d2z = (double*)calloc((size_t)nmax * n2, sizeof(double));
  double* y = (double*)calloc(nmax, sizeof(double));
  double* dy = (double*)calloc((size_t)nmax * nk, sizeof(double));
  double* d2y = (double*)calloc((size_t)nmax * n2, sizeof(double));
  if (!z || !dz || !d2z || !y || !dy || !d2y) {
    free(z); free(dz); free(d2z); free(y); free(dy); free(d2y);
    return 2;
  }
  int nin = nk;
  for (int i = 0; i < nk; i++) {
    z[i] = K[i];
    for (int j = 0; j < nk; j++) dz[i * nk + j] = (i == j) ? 1.0 : 0.0;
    for (int j = 0; j < n2; j++) d2z[i * n2 + j] = 0.0;
  }
  for (int k = 1; k <= L; k++) {
    const double* A = (k == 1) ? m->W1 : m->W + (size_t)(k - 2) * w * w;
    const double* B = (k >= 2 && m->skip_hidden) ? m->skip_hidden + (size_t)(k - 2) * w * 3 : NULL;
    const double* c = m->b + (size_t)(k - 1) * w;
    for (int j = 0; j < w; j++) {
      double s = c[j];
      for (int i = 0; i < nin; i++) s += A[(size_t)j * nin + i] * z[i];
      if (B)
        for (int i = 0; i < 3; i++) s += B[j * 3 + i] * K[i];
      y[j] = s;
      for (int p = 0; p < nk; p++) {
        double t = 0.0;
        for (int i = 0; i < nin; i++) t += A[(size_t)j * nin + i] * dz[i * nk + p];
        if (B) t += B[j * 3 + p];
        dy[j * nk + p] = t;
      }
      for (int pq = 0; pq < n2; pq++) {
        double t = 0.0;
        for (int i = 0; i < nin; i++) t += A[(size_t)j * nin + i] * d2z[i * n2 + pq];
        d2y[j * n2 + pq] = t;
      }
    }
    for (int j = 0; j < w; j++) {
      double f1 = sigmoid(y[j]);
      double f2 = f1 * (1.0 - f1);
      for (int p = 0; p < nk; p++)
        for (int q = 0; q < nk; q++)
          d2z[j * n2 + p * nk + q] = f1 * d2y[j * n2 + p * nk + q] + f2 * dy[j * nk + p] * dy[j * nk + q];
      for (int p = 0; p < nk; p++) dz[j * nk + p] = f1 * dy[j * nk + p];
      z[j] = softplus(y[j]);
    }
    nin = w;
  }
  double N = 0.0;
  for (int p = 0; p < nk; p++) g_out[p] = 0.0;
  for (int pq = 0; pq < n2; pq++) H_out[pq] = 0.0;
  for (int j = 0; j < w; j++) {
    N += m->a[j] * z[j];
    for (int p = 0; p < nk; p++) g_out[p] += m->a[j] * dz[j * nk + p];
    for (int pq = 0; pq < n2; pq++) H_out[pq] += m->a[j] * d2z[j * n2 + pq];
  }
  if (m->skip_out)
    for (int p = 0; p < 3; p++) {
      N += m->skip_out[p] * K[p];
      g_out[p] += m->skip_out[p];
    }
  *N_out = N;
  free(z); free(dz); free(d2z); free(y); free(dy); free(d2y);
  return 0;
}

/*
 * CANN (Eq. cann-def / cann-chain-rule):
 *   N = sum_m sum_k w2_km f2(f1(f0(K_m)); w1_km)
 *   dN/dK_m   = sum_k w2 f2' f1' f0'
 *   d2N/dK_m2 = sum_k w2 ((f2'' f1'^2 + f2' f1'') f0'^2 + f2' f1' f0''),  d2N/dK_m dK_n = 0 (m != n)
 * f0 in {x, <x>, |x|} with f0' = {1, (1 + sign x)/2, sign x}, f0'' = 0; f1 = x^p;
 * f2 in {w1 x, exp(w1 x) - 1, -ln(1 - w1 x)} with f2'' = {0, w1^2 exp(w1 x),
 * +w1^2/(1 - w1 x)^2} (reading R22: the paper prints a minus sign on the last).
 */
static double sgn(double x) { return (x > 0) - (x < 0); }
static int cann_eval(const oracle_ncm* m, int nin, const double* K, double* N_out, double* g, double* H) {
  const int n = m->cann_n;
  double N = 0.0;
  for (int p = 0; p < nin * nin; p++) H[p] = 0.0;
  for (int mm = 0; mm < nin; mm++) {
    g[mm] = 0.0;
    for (int k = 0; k < n; k++) {
      const int32_t* f = m->cann_f + ((size_t)mm * n + k) * 3;
      const double w1 = m->cann_w1[mm * n + k], w2 = m->cann_w2[mm * n + k];
      const double x = K[mm];
      double v0, d0;
      if (f[0] == 0) { v0 = x; d0 = 1.0; }
      else if (f[0] == 1) { v0 = x > 0 ? x : 0.0; d0 = 0.5 * (1.0 + sgn(x)); }
      else { v0 = fabs(x); d0 = sgn(x); }
      const int pw = f[1];
      const double v1 = pow(v0, pw), d1 = pw * pow(v0, pw - 1), dd1 = pw * (pw - 1) * (pw >= 2 ? pow(v0, pw - 2) : 0.0);
      double v2, d2, dd2;
      if (f[2] == 0) { v2 = w1 * v1; d2 = w1; dd2 = 0.0; }
      else if (f[2] == 1) { v2 = exp(w1 * v1) - 1.0; d2 = w1 * exp(w1 * v1); dd2 = w1 * w1 * exp(w1 * v1); }
      else { v2 = -log(1.0 - w1 * v1); d2 = w1 / (1.0 - w1 * v1); dd2 = w1 * w1 / ((1.0 - w1 * v1) * (1.0 - w1 * v1)); }
      N += w2 * v2;
      g[mm] += w2 * d2 * d1 * d0;
      H[mm * nin + mm] += w2 * ((dd2 * d1 * d1 + d2 * dd1) * d0 * d0 + d2 * d1 * 0.0);
    }
  }
  if (m->skip_out)
    for (int p = 0; p < 3; p++) {
      N += m->skip_out[p] * K[p];
      g[p] += m->skip_out[p];
    }
  *N_out = N;
  return 0;
}

/* Gent-Thomas (App. C): Psi = 0.5 (Ibar1 - 3) + ln(Ibar2 / 3) + (J - 1)^2,
 * i.e. N(K) = gt0 K1 + gt1 ln((K2 + 3) / 3) + gt2 K3^2 with gt = (0.5, 1, 1). */
static int gt_eval(const oracle_ncm* m, const double K[3], double* N_out, double g[3], double H[9]) {
  for (int p = 0; p < 9; p++) H[p] = 0.0;
  *N_out = m->gt[0] * K[0] + m->gt[1] * log((K[1] + 3.0) / 3.0) + m->gt[2] * K[2] * K[2];
  g[0] = m->gt[0];
  g[1] = m->gt[1] / (K[1] + 3.0);
  g[2] = 2.0 * m->gt[2] * K[2];
  H[4] = -m->gt[1] / ((K[1] + 3.0) * (K[1] + 3.0));
  H[8] = 2.0 * m->gt[2];
  return 0;
}

/*
 * ICKAN (App. B.3).  B-spline psi(x) = sum_i c_i B_{i,k}(x) on the uniform knots
 * t_i = xmin + (i - k) h, h = (xmax - xmin) / (nb - k), i = 0..nb+k, by De Boor's recursion
 * (B_{i,0} = 1 on the knot span holding x, B_{i,k} = (x - t_i)/(t_{i+k} - t_i) B_{i,k-1}
 * + (t_{i+k+1} - x)/(t_{i+k+1} - t_{i+1}) B_{i+1,k-1}) and the textbook derivative
 * B'_{i,k} = k/(t_{i+k} - t_i) B_{i,k-1} - k/(t_{i+k+1} - t_{i+1}) B_{i+1,k-1}, applied twice for
 * psi''.  Outside [xmin, xmax]: linear continuation with the end slope (SPEC's reading).
 */
static void bspline_basis(const double* t, int nb, int k, int span, double x, double* B /* [k+1][nb+k] */) {
  const int nt = nb + k + 1;
  for (int p = 0; p <= k; p++)
    for (int i = 0; i < nt; i++) B[p * nt + i] = 0.0;
  B[span] = 1.0;
  for (int p = 1; p <= k; p++)
    for (int i = 0; i + p + 1 < nt; i++) {
      double v = 0.0;
      if (t[i + p] > t[i]) v += (x - t[i]) / (t[i + p] - t[i]) * B[(p - 1) * nt + i];
      if (t[i + p + 1] > t[i + 1]) v += (t[i + p + 1] - x) / (t[i + p + 1] - t[i + 1]) * B[(p - 1) * nt + i + 1];
      B[p * nt + i] = v;
    }
}
static void spline_eval(const double* c, int nb, int k, double xmin, double xmax, double x, double* v, double* d1,
                        double* d2) {
  double t[64], B[4 * 64];
  const int nt = nb + k + 1;
  const double h = (xmax - xmin) / (nb - k);
  for (int i = 0; i < nt; i++) t[i] = xmin + (i - k) * h;
  const double xe = x < xmin ? xmin : (x > xmax ? xmax : x);
  int span = k;
  while (span < nb - 1 && xe >= t[span + 1]) span++;
  bspline_basis(t, nb, k, span, xe, B);
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int i = 0; i < nb; i++) {
    s0 += c[i] * B[k * nt + i];
    /* B'_{i,k} */
    double b1 = 0.0;
    if (t[i + k] > t[i]) b1 += k / (t[i + k] - t[i]) * B[(k - 1) * nt + i];
    if (t[i + k + 1] > t[i + 1]) b1 -= k / (t[i + k + 1] - t[i + 1]) * B[(k - 1) * nt + i + 1];
    s1 += c[i] * b1;
    /* B''_{i,k} = k/(t_{i+k}-t_i) B'_{i,k-1} - k/(t_{i+k+1}-t_{i+1}) B'_{i+1,k-1} */
    double b2 = 0.0;
    for (int side = 0; side < 2; side++) {
      const int ii = i + side;
      const double den = side ? t[i + k + 1] - t[i + 1] : t[i + k] - t[i];
      if (!(den > 0)) continue;
      double bp = 0.0; /* B'_{ii,k-1} */
      if (t[ii + k - 1] > t[ii]) bp += (k - 1) / (t[ii + k - 1] - t[ii]) * B[(k - 2) * nt + ii];
      if (t[ii + k] > t[ii + 1]) bp -= (k - 1) / (t[ii + k] - t[ii + 1]) * B[(k - 2) * nt + ii + 1];
      b2 += (side ? -1.0 : 1.0) * k / den * bp;
    }
    s2 += c[i] * b2;
  }
  if (x != xe) { /* linear continuation */
    *v = s0 + s1 * (x - xe);
    *d1 = s1;
    *d2 = 0.0;
  } else {
    *v = s0;
    *d1 = s1;
    *d2 = s2;
  }
}
/* forward mode through the layers: z, dz/dK (3), d2z/dK2 (3x3) per node, as Alg. 4 does for the ICNN */
static int ickan_eval(const oracle_ncm* m, int nk, const double* K, double* N_out, double* g, double* H) {
  const int R = m->kan_layers, nb = m->kan_nb, k = m->kan_k;
  double z[32], dz[32][9], d2z[32][81], y[32], dy[32][9], d2y[32][81];
  int nin = m->kan_width[0];
  if (nin != nk || nk > 9) return 3;
  for (int j = 0; j < nin; j++) {
    z[j] = K[j];
    for (int p = 0; p < nk; p++) dz[j][p] = (p == j);
    for (int pq = 0; pq < nk * nk; pq++) d2z[j][pq] = 0.0;
  }
  size_t e = 0;
  for (int r = 0; r < R; r++) {
    const int nout = m->kan_width[r + 1];
    const double xmin = m->kan_grid[2 * r], xmax = m->kan_grid[2 * r + 1];
    for (int i = 0; i < nout; i++) {
      y[i] = 0.0;
      for (int p = 0; p < nk; p++) dy[i][p] = 0.0;
      for (int pq = 0; pq < nk * nk; pq++) d2y[i][pq] = 0.0;
      for (int j = 0; j < nin; j++, e++) {
        double v, d1, d2;
        spline_eval(m->kan_c + e * nb, nb, k, xmin, xmax, z[j], &v, &d1, &d2);
        const double w = m->kan_w[e];
        y[i] += w * v;
        for (int p = 0; p < nk; p++) dy[i][p] += w * d1 * dz[j][p];
        for (int p = 0; p < nk; p++)
          for (int q = 0; q < nk; q++) d2y[i][p * nk + q] += w * (d2 * dz[j][p] * dz[j][q] + d1 * d2z[j][p * nk + q]);
      }
    }
    for (int i = 0; i < nout; i++) {
      z[i] = y[i];
      for (int p = 0; p < nk; p++) dz[i][p] = dy[i][p];
      for (int pq = 0; pq < nk * nk; pq++) d2z[i][pq] = d2y[i][pq];
    }
    nin = nout;
  }
  *N_out = z[0];
  for (int p = 0; p < nk; p++) g[p] = dz[0][p];
  for (int pq = 0; pq < nk * nk; pq++) H[pq] = d2z[0][pq];
  if (m->skip_out)
    for (int p = 0; p < 3; p++) {
      *N_out += m->skip_out[p] * K[p];
      g[p] += m->skip_out[p];
    }
  return 0;
}

/* the inner network on nin = 3 inputs (standard / isochoric kinematics) or 5 (anisotropic:
 * ICNN, CANN and ICKAN); g [nin], H [nin][nin].  Returns 0, or a non-zero status for a
 * configuration the network cannot evaluate: 1 bad ICNN shape / skips on 5 inputs, 2 out of
 * memory, 3 ICKAN input count, 4 Gent-Thomas on 5 inputs, 5 unknown network. */
int oracle_ncm_eval_n(const oracle_ncm* m, int nin, const double* K, double* N_out, double* g_out, double* H_out) {
  if (m->network == 1) return cann_eval(m, nin, K, N_out, g_out, H_out);
  if (m->network == 3) return ickan_eval(m, nin, K, N_out, g_out, H_out);
  if (m->network == 0) return icnn_eval(m, nin, K, N_out, g_out, H_out);
  if (m->network != 2) return 5;
  if (nin != 3) return 4;
  return gt_eval(m, K, N_out, g_out, H_out);
}

int oracle_ncm_eval(const oracle_ncm* m, const double K[3], double* N_out, double g_out[3],
                    double H_out[9]) {
  return oracle_ncm_eval_n(m, 3, K, N_out, g_out, H_out);
}

/* ---------------------------------------------------------------------- */
/* kinematics + stress/tangent at one material point                       */
/* ---------------------------------------------------------------------- */
static double det3(const double M[9]) {
  /* cofactor expansion along the first row */
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}
static void inv3(const double M[9], double out[9]) {
  double d = det3(M);
  out[0] = (M[4] * M[8] - M[5] * M[7]) / d;
  out[1] = (M[2] * M[7] - M[1] * M[8]) / d;
  out[2] = (M[1] * M[5] - M[2] * M[4]) / d;
  out[3] = (M[5] * M[6] - M[3] * M[8]) / d;
  out[4] = (M[0] * M[8] - M[2] * M[6]) / d;
  out[5] = (M[2] * M[3] - M[0] * M[5]) / d;
  out[6] = (M[3] * M[7] - M[4] * M[6]) / d;
  out[7] = (M[1] * M[6] - M[0] * M[7]) / d;
  out[8] = (M[0] * M[4] - M[1] * M[3]) / d;
}
#define I4(i, j, k, l) ((((i) * 3 + (j)) * 3 + (k)) * 3 + (l))

/*
 * Isochoric kinematics (App. A.2.2) in the paper's SPATIAL form,
 * pulled back to S and CC for the material-form assembly:
 *   Fbar = J^-1/3 F, Bbar = Fbar Fbar^T, Ibar1 = tr Bbar, Ibar2 = (tr Bbar^2 - tr(Bbar^2))/2
 *   Gbar1 = Bbar, GGbar1 = O;  Gbar2 = Bbar tr Bbar - Bbar^2, GGbar2 = Bbar(x)Bbar - Bbar(x)_Bbar
 *   G^m = Gbar^m + e_m Ibar_m I,  e = (-1/3, -2/3)
 *   GG^m = GGbar^m + e_m (I(x)Gbar^m + Gbar^m(x)I + Ibar_m (e_m I(x)I - I(x)_I))
 *   J: G = J/2 I, GG = J/4 (I(x)I - 2 I(x)_I)
 *   tau = 2 sum_m g_m G^m;  c = 4 sum_mn H_mn G^m(x)G^n + 4 sum_m g_m GG^m   (Eq. stress-cgo)
 *   S = F^-1 tau F^-T;  CC_IJKL = F^-1_Ii F^-1_Jj F^-1_Kk F^-1_Ll c_ijkl  (App. A.1 pull-back)
 * with (A(x)_B)_ijkl = 1/2 (A_ik B_jl + A_il B_jk) (reading 5).
 */
static void spatial_to_material(const double F[9], int n, double G[][9], double GG[][81], const double* g,
                                const double* H, double S[9], double CC[81]);
static void isochoric_S_CC(const double F[9], double Jd, const double g[3], const double H[9], double S[9],
                           double CC[81]) {
  const double a = pow(Jd, -2.0 / 3.0);
  double Bb[9], Bb2[9], G[3][9], GG[3][81];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double t = 0.0;
      for (int K = 0; K < 3; K++) t += F[i * 3 + K] * F[j * 3 + K];
      Bb[i * 3 + j] = a * t;
    }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double t = 0.0;
      for (int k = 0; k < 3; k++) t += Bb[i * 3 + k] * Bb[k * 3 + j];
      Bb2[i * 3 + j] = t;
    }
  const double Ib1 = Bb[0] + Bb[4] + Bb[8];
  const double Ib2 = 0.5 * (Ib1 * Ib1 - (Bb2[0] + Bb2[4] + Bb2[8]));
  const double Ib[2] = {Ib1, Ib2}, e[2] = {-1.0 / 3.0, -2.0 / 3.0};
  double Gb[2][9], GGb[2][81];
  for (int ij = 0; ij < 9; ij++) {
    Gb[0][ij] = Bb[ij];
    Gb[1][ij] = Bb[ij] * Ib1 - Bb2[ij];
  }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      for (int k = 0; k < 3; k++)
        for (int l = 0; l < 3; l++) {
          GGb[0][I4(i, j, k, l)] = 0.0;
          GGb[1][I4(i, j, k, l)] = Bb[i * 3 + j] * Bb[k * 3 + l] -
                                   0.5 * (Bb[i * 3 + k] * Bb[j * 3 + l] + Bb[i * 3 + l] * Bb[j * 3 + k]);
        }
  for (int mm = 0; mm < 2; mm++)
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) {
        G[mm][i * 3 + j] = Gb[mm][i * 3 + j] + e[mm] * Ib[mm] * (i == j);
        for (int k = 0; k < 3; k++)
          for (int l = 0; l < 3; l++) {
            const double II = (double)((i == j) * (k == l));
            const double IsI = 0.5 * ((i == k) * (j == l) + (i == l) * (j == k));
            GG[mm][I4(i, j, k, l)] =
                GGb[mm][I4(i, j, k, l)] +
                e[mm] * ((i == j) * Gb[mm][k * 3 + l] + Gb[mm][i * 3 + j] * (k == l) + Ib[mm] * (e[mm] * II - IsI));
          }
      }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      G[2][i * 3 + j] = 0.5 * Jd * (i == j);
      for (int k = 0; k < 3; k++)
        for (int l = 0; l < 3; l++)
          GG[2][I4(i, j, k, l)] = 0.25 * Jd * ((double)((i == j) * (k == l)) -
                                                 ((i == k) * (j == l) + (i == l) * (j == k)));
    }
  spatial_to_material(F, 3, G, GG, g, H, S, CC);
}

/* tau = 2 sum_m g_m G^m, c = 4 sum_mn H_mn G^m (x) G^n + 4 sum_m g_m GG^m (Eq. stress-cgo /
 * stiffnes-cgo), pulled back: S = F^-1 tau F^-T, CC = F^-1 F^-1 F^-1 F^-1 c (App. A.1) */
static void spatial_to_material(const double F[9], int n, double G[][9], double GG[][81], const double* g,
                                const double* H, double S[9], double CC[81]) {
  double tau[9], c[81], Fi[9];
  for (int ij = 0; ij < 9; ij++) {
    double t = 0.0;
    for (int mm = 0; mm < n; mm++) t += g[mm] * G[mm][ij];
    tau[ij] = 2.0 * t;
  }
  for (int ij = 0; ij < 9; ij++)
    for (int kl = 0; kl < 9; kl++) {
      double t = 0.0;
      for (int mm = 0; mm < n; mm++)
        for (int nn = 0; nn < n; nn++) t += H[mm * n + nn] * G[mm][ij] * G[nn][kl];
      for (int mm = 0; mm < n; mm++) t += g[mm] * GG[mm][ij * 9 + kl];
      c[ij * 9 + kl] = 4.0 * t;
    }
  inv3(F, Fi);
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++) {
      double t = 0.0;
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) t += Fi[I * 3 + i] * tau[i * 3 + j] * Fi[J * 3 + j];
      S[I * 3 + J] = t;
    }
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++)
      for (int K = 0; K < 3; K++)
        for (int L = 0; L < 3; L++) {
          double t = 0.0;
          for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++)
              for (int k = 0; k < 3; k++)
                for (int l = 0; l < 3; l++)
                  t += Fi[I * 3 + i] * Fi[J * 3 + j] * Fi[K * 3 + k] * Fi[L * 3 + l] * c[I4(i, j, k, l)];
          CC[I4(I, J, K, L)] = t;
        }
}

/*
 * Anisotropic kinematics (App. A.2.1 table; Eq. standard-inv-II) with
 * n_sv = 1 or 2 structural vectors A_i (reference configuration), in the paper's spatial form,
 * a_i = F A_i:
 *   I1: G = B, GG = O;  I2: G = B tr B - B^2, GG = B(x)B - B(x)_B;  J: G = J/2 I, GG = J/4 (I(x)I - 2 I(x)_I)
 *   I4,ij = A_i.C A_j:   G = sym(a_i (x) a_j), GG = O
 *   I5,ij = A_i.C^2 A_j: G = sym(a_i (x) B a_j) + sym(a_j (x) B a_i)   (reading R28: the table's
 *                        2 sym(a_i (x) B a_j) holds for i = j only -- I5,ij is symmetric in i, j),
 *                        GG = B (x)_ sym(a_i (x) a_j) + sym(a_i (x) a_j) (x)_ B
 * for the pairs i <= j in the order (0,0), (0,1), (1,1); then tau, c and the pull-back as above.
 * Inputs K = (I1-3, I2-3, J-1, then per pair I4,ij - A_i.A_j, I5,ij - A_i.A_j): K = 0 at F = I
 * (for one unit vector: I4-1, I5-1).  nk = 3 + 2 n_pairs (5 or 9).
 */
static int aniso_pairs(const oracle_ncm* m, const double* A[2], int pi[3], int pj[3]) {
  const int nsv = m->n_sv > 1 ? 2 : 1;
  A[0] = m->a0;
  A[1] = m->a1;
  int np = 0;
  for (int i = 0; i < nsv; i++)
    for (int j = i; j < nsv; j++) {
      pi[np] = i;
      pj[np] = j;
      np++;
    }
  return np;
}

static void anisotropic_S_CC(const oracle_ncm* m, const double F[9], double Jd, const double* g, const double* H,
                             double S[9], double CC[81]) {
  const double* A[2];
  int pi[3], pj[3];
  const int np = aniso_pairs(m, A, pi, pj), nk = 3 + 2 * np;
  double B[9], B2[9], a[2][3], Ba[2][3], G[9][9], GG[9][81];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) B[i * 3 + j] = F[i * 3] * F[j * 3] + F[i * 3 + 1] * F[j * 3 + 1] + F[i * 3 + 2] * F[j * 3 + 2];
  for (int v = 0; v < 2; v++)
    for (int i = 0; i < 3; i++) a[v][i] = F[i * 3] * A[v][0] + F[i * 3 + 1] * A[v][1] + F[i * 3 + 2] * A[v][2];
  for (int v = 0; v < 2; v++)
    for (int i = 0; i < 3; i++) Ba[v][i] = B[i * 3] * a[v][0] + B[i * 3 + 1] * a[v][1] + B[i * 3 + 2] * a[v][2];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) B2[i * 3 + j] = B[i * 3] * B[j] + B[i * 3 + 1] * B[3 + j] + B[i * 3 + 2] * B[6 + j];
  const double trB = B[0] + B[4] + B[8];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      G[0][i * 3 + j] = B[i * 3 + j];
      G[1][i * 3 + j] = B[i * 3 + j] * trB - B2[i * 3 + j];
      G[2][i * 3 + j] = 0.5 * Jd * (i == j);
    }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      for (int k = 0; k < 3; k++)
        for (int l = 0; l < 3; l++) {
          const int x = I4(i, j, k, l);
          GG[0][x] = 0.0;
          GG[1][x] = B[i * 3 + j] * B[k * 3 + l] - 0.5 * (B[i * 3 + k] * B[j * 3 + l] + B[i * 3 + l] * B[j * 3 + k]);
          GG[2][x] = 0.25 * Jd * ((double)((i == j) * (k == l)) - ((i == k) * (j == l) + (i == l) * (j == k)));
        }
  for (int p = 0; p < np; p++) {
    const double *ai = a[pi[p]], *aj = a[pj[p]], *Bai = Ba[pi[p]], *Baj = Ba[pj[p]];
    double As[9];
    const int m4 = 3 + 2 * p, m5 = 4 + 2 * p;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) {
        As[i * 3 + j] = 0.5 * (ai[i] * aj[j] + aj[i] * ai[j]); /* sym(a_i (x) a_j) */
        G[m4][i * 3 + j] = As[i * 3 + j];
        G[m5][i * 3 + j] = 0.5 * (ai[i] * Baj[j] + Baj[i] * ai[j]) + 0.5 * (aj[i] * Bai[j] + Bai[i] * aj[j]);
      }
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++)
          for (int l = 0; l < 3; l++) {
            const int x = I4(i, j, k, l);
            GG[m4][x] = 0.0;
            GG[m5][x] = 0.5 * (B[i * 3 + k] * As[j * 3 + l] + B[i * 3 + l] * As[j * 3 + k]) +
                        0.5 * (As[i * 3 + k] * B[j * 3 + l] + As[i * 3 + l] * B[j * 3 + k]);
          }
  }
  spatial_to_material(F, nk, G, GG, g, H, S, CC);
}

/*
 * Isochoric anisotropic kinematics (App. A.2.2, the set
 * Ibar_m, m in {1, 2, (4,ij), (5,ij)}, with the App. A.2.1 table's I4,ij / I5,ij rows; reading R29):
 *   Fbar = J^-1/3 F, Bbar = Fbar Fbar^T, abar_i = Fbar A_i;  Ibar_m = I3^e_m I_m,
 *   e_m = -1/3 (m = 1, (4,ij)), -2/3 (m = 2, (5,ij))
 *   Ibar1 = tr Bbar, Ibar2 = (tr Bbar^2 - tr(Bbar^2))/2, Ibar4,ij = abar_i.abar_j, Ibar5,ij = abar_i.Bbar abar_j
 *   Gbar1 = Bbar, GGbar1 = O;  Gbar2 = Bbar tr Bbar - Bbar^2, GGbar2 = Bbar(x)Bbar - Bbar(x)_Bbar
 *   Gbar4,ij = sym(abar_i (x) abar_j), GGbar4,ij = O
 *   Gbar5,ij = sym(abar_i (x) Bbar abar_j) + sym(abar_j (x) Bbar abar_i)       (R28, R29: Bbar, not B)
 *   GGbar5,ij = Bbar (x)_ sym(abar_i (x) abar_j) + sym(abar_i (x) abar_j) (x)_ Bbar
 *   G^m = Gbar^m + e_m Ibar_m I
 *   GG^m = GGbar^m + e_m (I(x)Gbar^m + Gbar^m(x)I + Ibar_m (e_m I(x)I - I(x)_I))
 *   J: G = J/2 I, GG = J/4 (I(x)I - 2 I(x)_I)
 * inputs in the order (Ibar1, Ibar2, J, per pair Ibar4,ij, Ibar5,ij); then tau, c and the pull-back
 * (spatial_to_material).
 */
static void isochoric_anisotropic_S_CC(const oracle_ncm* m, const double F[9], double Jd, const double* g,
                                       const double* H, double S[9], double CC[81]) {
  const double* A[2];
  int pi[3], pj[3];
  const int np = aniso_pairs(m, A, pi, pj), nk = 3 + 2 * np;
  const double c13 = pow(Jd, -1.0 / 3.0);
  double Fb[9], Bb[9], Bb2[9], ab[2][3], Bab[2][3];
  for (int x = 0; x < 9; x++) Fb[x] = c13 * F[x];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      Bb[i * 3 + j] = Fb[i * 3] * Fb[j * 3] + Fb[i * 3 + 1] * Fb[j * 3 + 1] + Fb[i * 3 + 2] * Fb[j * 3 + 2];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) Bb2[i * 3 + j] = Bb[i * 3] * Bb[j] + Bb[i * 3 + 1] * Bb[3 + j] + Bb[i * 3 + 2] * Bb[6 + j];
  for (int v = 0; v < 2; v++)
    for (int i = 0; i < 3; i++) ab[v][i] = Fb[i * 3] * A[v][0] + Fb[i * 3 + 1] * A[v][1] + Fb[i * 3 + 2] * A[v][2];
  for (int v = 0; v < 2; v++)
    for (int i = 0; i < 3; i++) Bab[v][i] = Bb[i * 3] * ab[v][0] + Bb[i * 3 + 1] * ab[v][1] + Bb[i * 3 + 2] * ab[v][2];
  const double Ib1 = Bb[0] + Bb[4] + Bb[8];
  double Ib[9], e[9], Gb[9][9], GGb[9][81], G[9][9], GG[9][81];
  Ib[0] = Ib1;
  Ib[1] = 0.5 * (Ib1 * Ib1 - (Bb2[0] + Bb2[4] + Bb2[8]));
  e[0] = -1.0 / 3.0;
  e[1] = -2.0 / 3.0;
  for (int ij = 0; ij < 9; ij++) {
    Gb[0][ij] = Bb[ij];
    Gb[1][ij] = Bb[ij] * Ib1 - Bb2[ij];
  }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++)
      for (int k = 0; k < 3; k++)
        for (int l = 0; l < 3; l++) {
          GGb[0][I4(i, j, k, l)] = 0.0;
          GGb[1][I4(i, j, k, l)] = Bb[i * 3 + j] * Bb[k * 3 + l] -
                                   0.5 * (Bb[i * 3 + k] * Bb[j * 3 + l] + Bb[i * 3 + l] * Bb[j * 3 + k]);
        }
  for (int p = 0; p < np; p++) {
    const double *ai = ab[pi[p]], *aj = ab[pj[p]], *Bai = Bab[pi[p]], *Baj = Bab[pj[p]];
    const int m4 = 3 + 2 * p, m5 = 4 + 2 * p;
    double As[9];
    Ib[m4] = ai[0] * aj[0] + ai[1] * aj[1] + ai[2] * aj[2];
    Ib[m5] = ai[0] * Baj[0] + ai[1] * Baj[1] + ai[2] * Baj[2];
    e[m4] = -1.0 / 3.0;
    e[m5] = -2.0 / 3.0;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) {
        As[i * 3 + j] = 0.5 * (ai[i] * aj[j] + aj[i] * ai[j]);
        Gb[m4][i * 3 + j] = As[i * 3 + j];
        Gb[m5][i * 3 + j] = 0.5 * (ai[i] * Baj[j] + Baj[i] * ai[j]) + 0.5 * (aj[i] * Bai[j] + Bai[i] * aj[j]);
      }
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++)
        for (int k = 0; k < 3; k++)
          for (int l = 0; l < 3; l++) {
            const int x = I4(i, j, k, l);
            GGb[m4][x] = 0.0;
            GGb[m5][x] = 0.5 * (Bb[i * 3 + k] * As[j * 3 + l] + Bb[i * 3 + l] * As[j * 3 + k]) +
                         0.5 * (As[i * 3 + k] * Bb[j * 3 + l] + As[i * 3 + l] * Bb[j * 3 + k]);
          }
  }
  for (int mm = 0; mm < nk; mm++) {
    if (mm == 2) continue;
    for (int i = 0; i < 3; i++)
      for (int j = 0; j < 3; j++) {
        G[mm][i * 3 + j] = Gb[mm][i * 3 + j] + e[mm] * Ib[mm] * (i == j);
        for (int k = 0; k < 3; k++)
          for (int l = 0; l < 3; l++) {
            const double II = (double)((i == j) * (k == l));
            const double IsI = 0.5 * ((i == k) * (j == l) + (i == l) * (j == k));
            GG[mm][I4(i, j, k, l)] =
                GGb[mm][I4(i, j, k, l)] +
                e[mm] * ((i == j) * Gb[mm][k * 3 + l] + Gb[mm][i * 3 + j] * (k == l) + Ib[mm] * (e[mm] * II - IsI));
          }
      }
  }
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      G[2][i * 3 + j] = 0.5 * Jd * (i == j);
      for (int k = 0; k < 3; k++)
        for (int l = 0; l < 3; l++)
          GG[2][I4(i, j, k, l)] = 0.25 * Jd * ((double)((i == j) * (k == l)) -
                                                 ((i == k) * (j == l) + (i == l) * (j == k)));
    }
  spatial_to_material(F, nk, G, GG, g, H, S, CC);
}

/*
 * F (row-major F[i*3+J]) -> k, W, g, H (incl. penalty), S, CC, P, A.
 * Kinematic layer in material form:
 *   h1 = dI1/dC = I,  h2 = dI2/dC = I1 I - C,  h3 = dJ/dC = J/2 C^-1
 *   HH1 = 0,  HH2 = I(x)I - II,  HH3 = J/4 C^-1(x)C^-1 - J/2 II_{C^-1}
 *   (II_X)_IJKL = 1/2 (X_IK X_JL + X_IL X_JK)   (reading 5)
 * S = 2 sum_m g_m h_m;  CC = 4 sum_mn H_mn h_m (x) h_n + 4 sum_m g_m HH_m
 *   (Eq. stress-cgo / stiffnes-cgo, pulled back; reading 4)
 * P = F S;  A_iJkL = d_ik S_JL + F_iI CC_IJKL F_kK  (Eq. p-stiffness)
 * Returns J, or NaN (every output NaN) when the inner network rejects the configuration
 * (oracle_ncm_eval_n status != 0): the checker fails loudly instead of using garbage.
 */
static double ncm_failed(double* k_out, double* W_out, double* g_out, double* H_out, double S[9], double CC[81],
                         double P[9], double A[81]) {
  const double nan = NAN;
  if (k_out) for (int p = 0; p < 3; p++) k_out[p] = nan;
  if (W_out) *W_out = nan;
  if (g_out) for (int p = 0; p < 3; p++) g_out[p] = nan;
  if (H_out) for (int p = 0; p < 9; p++) H_out[p] = nan;
  for (int p = 0; p < 9; p++) S[p] = P[p] = nan;
  for (int p = 0; p < 81; p++) CC[p] = A[p] = nan;
  return nan;
}
double oracle_material_point(const oracle_ncm* m, const double F[9], double k_out[3],
                             double* W_out, double g_out[3], double H_out[9], double S[9],
                             double CC[81], double P[9], double A[81]) {
  double C[9], Ci[9];
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++) {
      double s = 0.0;
      for (int i = 0; i < 3; i++) s += F[i * 3 + I] * F[i * 3 + J];
      C[I * 3 + J] = s;
    }
  double I1 = C[0] + C[4] + C[8];
  double trC2 = 0.0;
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++) trC2 += C[I * 3 + J] * C[J * 3 + I];
  double I2 = 0.5 * (I1 * I1 - trC2);
  double Jd = det3(F);
  inv3(C, Ci);
  if (m->kinematics == 2 || m->kinematics == 3) {
    /* anisotropic: K = (I1-3, I2-3, J-1, per pair I4,ij - A_i.A_j, I5,ij - A_i.A_j);
     * isochoric anisotropic (3): K = (Ibar1-3, Ibar2-3, J-1, per pair Ibar4,ij - A_i.A_j, Ibar5,ij - A_i.A_j),
     * Ibar1 = J^-2/3 I1, Ibar2 = J^-4/3 I2, Ibar4,ij = J^-2/3 I4,ij, Ibar5,ij = J^-4/3 I5,ij (App. A.2.2) */
    const double a23 = m->kinematics == 3 ? pow(Jd, -2.0 / 3.0) : 1.0;
    const double* Av[2];
    int pi[3], pj[3];
    const int np = aniso_pairs(m, Av, pi, pj), nk = 3 + 2 * np;
    double CA[2][3];
    for (int v = 0; v < 2; v++)
      for (int I = 0; I < 3; I++) CA[v][I] = C[I * 3] * Av[v][0] + C[I * 3 + 1] * Av[v][1] + C[I * 3 + 2] * Av[v][2];
    double kN[9] = {a23 * I1 - 3.0, a23 * a23 * I2 - 3.0, Jd - 1.0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < np; p++) {
      const double *Ai = Av[pi[p]], *Aj = Av[pj[p]], *CAi = CA[pi[p]], *CAj = CA[pj[p]];
      double i4 = 0.0, i5 = 0.0, aa = 0.0;
      for (int I = 0; I < 3; I++) {
        i4 += Ai[I] * CAj[I];   /* A_i.C A_j */
        i5 += CAi[I] * CAj[I];  /* A_i.C^2 A_j = (C A_i).(C A_j) */
        aa += Ai[I] * Aj[I];
      }
      kN[3 + 2 * p] = a23 * i4 - aa;
      kN[4 + 2 * p] = a23 * a23 * i5 - aa;
    }
    double NN, gN[9], HN[81];
    if (oracle_ncm_eval_n(m, nk, kN, &NN, gN, HN) != 0) return ncm_failed(k_out, W_out, g_out, H_out, S, CC, P, A);
    const double WN = NN + m->kappa * (Jd - 1.0) * (Jd - 1.0) - m->ref_shift * (Jd - 1.0);
    gN[2] += 2.0 * m->kappa * (Jd - 1.0) - m->ref_shift;
    HN[2 * nk + 2] += 2.0 * m->kappa;
    if (m->kinematics == 3)
      isochoric_anisotropic_S_CC(m, F, Jd, gN, HN, S, CC);
    else
      anisotropic_S_CC(m, F, Jd, gN, HN, S, CC);
    for (int i = 0; i < 3; i++)
      for (int J = 0; J < 3; J++) {
        double t = 0.0;
        for (int I = 0; I < 3; I++) t += F[i * 3 + I] * S[I * 3 + J];
        P[i * 3 + J] = t;
      }
    for (int i = 0; i < 3; i++)
      for (int J = 0; J < 3; J++)
        for (int kk = 0; kk < 3; kk++)
          for (int L = 0; L < 3; L++) {
            double t = (i == kk) ? S[J * 3 + L] : 0.0;
            for (int I = 0; I < 3; I++)
              for (int K = 0; K < 3; K++) t += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[kk * 3 + K];
            A[I4(i, J, kk, L)] = t;
          }
    if (k_out)
      for (int p = 0; p < 3; p++) k_out[p] = kN[p];
    if (W_out) *W_out = WN;
    if (g_out)
      for (int p = 0; p < 3; p++) g_out[p] = gN[p];
    if (H_out)
      for (int p = 0; p < 3; p++)
        for (int q = 0; q < 3; q++) H_out[p * 3 + q] = HN[p * nk + q];
    return Jd;
  }
  double k[3] = {I1 - 3.0, I2 - 3.0, Jd - 1.0};
  if (m->kinematics == 1) {  /* isochoric invariants (App. A.2.2): Ibar1 = J^-2/3 I1, Ibar2 = J^-4/3 I2 */
    const double a = pow(Jd, -2.0 / 3.0);
    k[0] = a * I1 - 3.0;
    k[1] = a * a * I2 - 3.0;
  }
  double N, g[3], H[9];
  if (oracle_ncm_eval(m, k, &N, g, H) != 0) return ncm_failed(k_out, W_out, g_out, H_out, S, CC, P, A);
  /* volumetric penalty (a5) and optional reference shift (reading 11) */
  double W = N + m->kappa * (Jd - 1.0) * (Jd - 1.0) - m->ref_shift * (Jd - 1.0);
  g[2] += 2.0 * m->kappa * (Jd - 1.0) - m->ref_shift;
  H[8] += 2.0 * m->kappa;
  if (m->kinematics == 1) {
    isochoric_S_CC(F, Jd, g, H, S, CC);
    goto push;
  }

  double h[3][9];
  double HHl[3][81];
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++) {
      double d = (I == J) ? 1.0 : 0.0;
      h[0][I * 3 + J] = d;
      h[1][I * 3 + J] = I1 * d - C[I * 3 + J];
      h[2][I * 3 + J] = 0.5 * Jd * Ci[I * 3 + J];
    }
  for (int I = 0; I < 3; I++)
    for (int J = 0; J < 3; J++)
      for (int K = 0; K < 3; K++)
        for (int L = 0; L < 3; L++) {
          double dIJ = (I == J), dKL = (K == L), dIK = (I == K), dJL = (J == L), dIL = (I == L),
                 dJK = (J == K);
          HHl[0][I4(I, J, K, L)] = 0.0;
          HHl[1][I4(I, J, K, L)] = dIJ * dKL - 0.5 * (dIK * dJL + dIL * dJK);
          HHl[2][I4(I, J, K, L)] =
              0.25 * Jd * Ci[I * 3 + J] * Ci[K * 3 + L] -
              0.5 * Jd * 0.5 * (Ci[I * 3 + K] * Ci[J * 3 + L] + Ci[I * 3 + L] * Ci[J * 3 + K]);
        }
  for (int IJ = 0; IJ < 9; IJ++) {
    double s = 0.0;
    for (int mm = 0; mm < 3; mm++) s += g[mm] * h[mm][IJ];
    S[IJ] = 2.0 * s;
  }
  for (int IJ = 0; IJ < 9; IJ++)
    for (int KL = 0; KL < 9; KL++) {
      double s = 0.0;
      for (int mm = 0; mm < 3; mm++)
        for (int nn = 0; nn < 3; nn++) s += H[mm * 3 + nn] * h[mm][IJ] * h[nn][KL];
      double t = 0.0;
      for (int mm = 0; mm < 3; mm++) t += g[mm] * HHl[mm][IJ * 9 + KL];
      CC[IJ * 9 + KL] = 4.0 * s + 4.0 * t;
    }
push:
  for (int i = 0; i < 3; i++)
    for (int J = 0; J < 3; J++) {
      double s = 0.0;
      for (int I = 0; I < 3; I++) s += F[i * 3 + I] * S[I * 3 + J];
      P[i * 3 + J] = s;
    }
  for (int i = 0; i < 3; i++)
    for (int J = 0; J < 3; J++)
      for (int kk = 0; kk < 3; kk++)
        for (int L = 0; L < 3; L++) {
          double s = (i == kk) ? S[J * 3 + L] : 0.0;
          for (int I = 0; I < 3; I++)
            for (int K = 0; K < 3; K++)
              s += F[i * 3 + I] * CC[I4(I, J, K, L)] * F[kk * 3 + K];
          A[I4(i, J, kk, L)] = s;
        }
  if (k_out)
    for (int p = 0; p < 3; p++) k_out[p] = k[p];
  if (W_out) *W_out = W;
  if (g_out)
    for (int p = 0; p < 3; p++) g_out[p] = g[p];
  if (H_out)
    for (int p = 0; p < 9; p++) H_out[p] = H[p];
  return Jd;
}

/* F at one quadrature point: F = I + sum_a u_a (x) GradN_a (Alg. 1 line 3) */
static void qp_F(int n_en, const int32_t* conn_e, const double* gN, const double* u, double F[9]) {
  for (int i = 0; i < 3; i++)
    for (int J = 0; J < 3; J++) F[i * 3 + J] = (i == J) ? 1.0 : 0.0;
  for (int a = 0; a < n_en; a++) {
    int64_t node = conn_e[a];
    for (int i = 0; i < 3; i++)
      for (int J = 0; J < 3; J++) F[i * 3 + J] += u[3 * node + i] * gN[a * 3 + J];
  }
}

/* all F's, row-major [n_el][n_q][9] (test helper: patch tests, min J) */
void oracle_qp_F(int64_t n_el, int n_en, int n_q, const int32_t* conn, const double* gradN,
                 const double* u, double* F_out) {
  for (int64_t e = 0; e < n_el; e++)
    for (int q = 0; q < n_q; q++)
      qp_F(n_en, conn + e * n_en, gradN + ((size_t)e * n_q + q) * n_en * 3, u,
           F_out + ((size_t)e * n_q + q) * 9);
}

/* Pi(u) = sum_e sum_q w W(F) */
double oracle_energy(const oracle_ncm* m, int64_t n_el, int n_en, int n_q, const int32_t* conn,
                     const double* gradN, const double* qp_w, const double* u) {
  double Pi = 0.0;
  double S[9], CC[81], P[9], A[81], W;
  for (int64_t e = 0; e < n_el; e++)
    for (int q = 0; q < n_q; q++) {
      double F[9];
      qp_F(n_en, conn + e * n_en, gradN + ((size_t)e * n_q + q) * n_en * 3, u, F);
      oracle_material_point(m, F, NULL, &W, NULL, NULL, S, CC, P, A);
      Pi += qp_w[e * n_q + q] * W;
    }
  return Pi;
}

/* ---------------------------------------------------------------------- */
/* sparsity pattern                                  */
/* ---------------------------------------------------------------------- */
static int cmp_i64(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

/* Node adjacency: adj(a) = sorted unique nodes of all elements containing a.
 * Outputs (malloc'd): adj_ptr [n_nodes+1], adj [adj_ptr[n_nodes]]. */
static int node_adjacency(int64_t n_nodes, int64_t n_el, int n_en, const int32_t* conn,
                          int64_t** adj_ptr_out, int64_t** adj_out) {
  int64_t* cnt = (int64_t*)calloc(n_nodes + 1, sizeof(int64_t));
  for (int64_t e = 0; e < n_el; e++)
    for (int a = 0; a < n_en; a++) cnt[conn[e * n_en + a] + 1]++;
  for (int64_t v = 0; v < n_nodes; v++) cnt[v + 1] += cnt[v];
  int64_t* inc = (int64_t*)malloc(sizeof(int64_t) * (cnt[n_nodes] + 1));
  int64_t* fill = (int64_t*)calloc(n_nodes, sizeof(int64_t));
  for (int64_t e = 0; e < n_el; e++)
    for (int a = 0; a < n_en; a++) {
      int64_t v = conn[e * n_en + a];
      inc[cnt[v] + fill[v]++] = e;
    }
  int64_t* adj_ptr = (int64_t*)calloc(n_nodes + 1, sizeof(int64_t));
  /* pass 1: degree of each node */
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n_nodes; v++) {
    int64_t ne = cnt[v + 1] - cnt[v];
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (ne * n_en + 1));
    int64_t t = 0;
    for (int64_t p = cnt[v]; p < cnt[v + 1]; p++)
      for (int b = 0; b < n_en; b++) tmp[t++] = conn[inc[p] * n_en + b];
    qsort(tmp, t, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t s = 0; s < t; s++)
      if (s == 0 || tmp[s] != tmp[s - 1]) u++;
    adj_ptr[v + 1] = u;
    free(tmp);
  }
  for (int64_t v = 0; v < n_nodes; v++) adj_ptr[v + 1] += adj_ptr[v];
  int64_t* adj = (int64_t*)malloc(sizeof(int64_t) * (adj_ptr[n_nodes] + 1));
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n_nodes; v++) {
    int64_t ne = cnt[v + 1] - cnt[v];
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (ne * n_en + 1));
    int64_t t = 0;
    for (int64_t p = cnt[v]; p < cnt[v + 1]; p++)
      for (int b = 0; b < n_en; b++) tmp[t++] = conn[inc[p] * n_en + b];
    qsort(tmp, t, sizeof(int64_t), cmp_i64);
    int64_t o = adj_ptr[v];
    for (int64_t s = 0; s < t; s++)
      if (s == 0 || tmp[s] != tmp[s - 1]) adj[o++] = tmp[s];
    free(tmp);
  }
  free(cnt); free(inc); free(fill);
  *adj_ptr_out = adj_ptr;
  *adj_out = adj;
  return 0;
}

/* Rows [3*node_begin, 3*node_end): row 3a+i has columns {3b+k : b in adj(a)
 * ascending, k = 0..2}.  Call with row_ptr != NULL, col_idx == NULL to get
 * row_ptr (and *nnz); then again with col_idx to fill it. */
int oracle_pattern(int64_t n_nodes, int64_t n_el, int n_en, const int32_t* conn,
                   int64_t node_begin, int64_t node_end, int64_t* row_ptr, int32_t* col_idx,
                   int64_t* nnz) {
  int64_t *adj_ptr, *adj;
  node_adjacency(n_nodes, n_el, n_en, conn, &adj_ptr, &adj);
  int64_t nr = 3 * (node_end - node_begin);
  row_ptr[0] = 0;
  for (int64_t a = node_begin; a < node_end; a++)
    for (int i = 0; i < 3; i++) {
      int64_t row = 3 * (a - node_begin) + i;
      row_ptr[row + 1] = row_ptr[row] + 3 * (adj_ptr[a + 1] - adj_ptr[a]);
    }
  *nnz = row_ptr[nr];
  if (col_idx) {
#pragma omp parallel for schedule(static)
    for (int64_t a = node_begin; a < node_end; a++)
      for (int i = 0; i < 3; i++) {
        int64_t o = row_ptr[3 * (a - node_begin) + i];
        for (int64_t p = adj_ptr[a]; p < adj_ptr[a + 1]; p++)
          for (int kk = 0; kk < 3; kk++) col_idx[o++] = (int32_t)(3 * adj[p] + kk);
      }
  }
  free(adj_ptr); free(adj);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* assembly: Alg. 1                                            */
/* ---------------------------------------------------------------------- */
static int64_t find_col(const int64_t* row_ptr, const int32_t* col_idx, int64_t row, int64_t col) {
  int64_t lo = row_ptr[row], hi = row_ptr[row + 1] - 1;
  while (lo <= hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (col_idx[mid] == col) return mid;
    if (col_idx[mid] < col) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* One element: loops q, I, J of Alg. 1; accumulates K_e then scatters.
 * Rows outside [node_begin, node_end) are skipped (multi-rank ownership). */
static void assemble_element(const oracle_ncm* m, int64_t e, int n_en, int n_q,
                             const int32_t* conn, const double* gradN, const double* qp_w,
                             const double* u, int64_t node_begin, int64_t node_end,
                             const int64_t* row_ptr, const int32_t* col_idx, double* r,
                             double* vals, int64_t* bad, int64_t* missing, int64_t* ncm_err) {
  const int nd = 3 * n_en;
  double* Ke = (double*)calloc((size_t)nd * nd, sizeof(double));
  const int32_t* ce = conn + e * n_en;
  for (int q = 0; q < n_q; q++) {
    const double* gN = gradN + ((size_t)e * n_q + q) * n_en * 3;
    const double wq = qp_w[e * n_q + q];
    double F[9], S[9], CC[81], P[9], A[81];
    qp_F(n_en, ce, gN, u, F);
    double Jd = oracle_material_point(m, F, NULL, NULL, NULL, NULL, S, CC, P, A);
    if (isnan(Jd)) (*ncm_err)++;
    if (Jd <= 0.0) {
      int64_t flat = e * n_q + q;
#pragma omp critical(oracle_bad)
      { if (*bad < 0 || flat < *bad) *bad = flat; }
    }
    for (int a = 0; a < n_en; a++) {
      int64_t node = ce[a];
      for (int i = 0; i < 3; i++) {
        double s = 0.0;
        for (int J = 0; J < 3; J++) s += P[i * 3 + J] * gN[a * 3 + J];
        if (node >= node_begin && node < node_end) r[3 * (node - node_begin) + i] += wq * s;
      }
      for (int b = 0; b < n_en; b++)
        for (int i = 0; i < 3; i++)
          for (int kk = 0; kk < 3; kk++) {
            double s = 0.0;
            for (int J = 0; J < 3; J++)
              for (int L = 0; L < 3; L++) s += gN[a * 3 + J] * A[I4(i, J, kk, L)] * gN[b * 3 + L];
            Ke[(a * 3 + i) * nd + b * 3 + kk] += wq * s;
          }
    }
  }
  for (int a = 0; a < n_en; a++) {
    int64_t na = ce[a];
    if (na < node_begin || na >= node_end) continue;
    for (int i = 0; i < 3; i++) {
      int64_t row = 3 * (na - node_begin) + i;
      for (int b = 0; b < n_en; b++)
        for (int kk = 0; kk < 3; kk++) {
          int64_t pos = find_col(row_ptr, col_idx, row, 3 * (int64_t)ce[b] + kk);
          if (pos < 0) { (*missing)++; continue; }
          vals[pos] += Ke[(a * 3 + i) * nd + b * 3 + kk];
        }
    }
  }
  free(Ke);
}

/* Greedy element colouring (first colour not used by any element sharing a
 * node), elements in index order.  Returns the number of colours. */
static int colour_elements(int64_t n_nodes, int64_t n_el, int n_en, const int32_t* conn,
                           int32_t* colour) {
  /* node -> bitmask of colours already used by elements touching it (<= 64) */
  uint64_t* used = (uint64_t*)calloc(n_nodes, sizeof(uint64_t));
  int ncol = 0;
  for (int64_t e = 0; e < n_el; e++) {
    uint64_t mask = 0;
    for (int a = 0; a < n_en; a++) mask |= used[conn[e * n_en + a]];
    int c = 0;
    while (c < 64 && (mask >> c) & 1ULL) c++;
    if (c >= 64) { free(used); return -1; }
    colour[e] = c;
    if (c + 1 > ncol) ncol = c + 1;
    for (int a = 0; a < n_en; a++) used[conn[e * n_en + a]] |= (1ULL << c);
  }
  free(used);
  return ncol;
}

/* r and vals are OVERWRITTEN.  mode 0: serial, element order (Alg. 1 as
 * written).  mode 1: OpenMP over the elements of one colour at a time
 * (deterministic for any thread count).  Returns #missing pattern entries
 * (0 expected), -1 on colouring failure, or -2 if the inner network could not
 * be evaluated (unsupported network / kinematics combination: the outputs are
 * then meaningless and the caller must fail). */
int64_t oracle_assemble(const oracle_ncm* m, int64_t n_nodes, int64_t n_el, int n_en, int n_q,
                        const int32_t* conn, const double* gradN, const double* qp_w,
                        const double* u, int64_t node_begin, int64_t node_end,
                        const int64_t* row_ptr, const int32_t* col_idx, double* r, double* vals,
                        int64_t* bad, int mode, int n_threads) {
  int64_t nr = 3 * (node_end - node_begin);
  memset(r, 0, sizeof(double) * nr);
  memset(vals, 0, sizeof(double) * row_ptr[nr]);
  *bad = -1;
  int64_t missing = 0, ncm_err = 0;
  if (mode == 0) {
    for (int64_t e = 0; e < n_el; e++)
      assemble_element(m, e, n_en, n_q, conn, gradN, qp_w, u, node_begin, node_end, row_ptr,
                       col_idx, r, vals, bad, &missing, &ncm_err);
    return ncm_err ? -2 : missing;
  }
  int32_t* colour = (int32_t*)malloc(sizeof(int32_t) * (n_el + 1));
  int ncol = colour_elements(n_nodes, n_el, n_en, conn, colour);
  if (ncol < 0) { free(colour); return -1; }
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
  for (int c = 0; c < ncol; c++) {
    int64_t miss_c = 0, err_c = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : miss_c, err_c)
    for (int64_t e = 0; e < n_el; e++)
      if (colour[e] == c)
        assemble_element(m, e, n_en, n_q, conn, gradN, qp_w, u, node_begin, node_end, row_ptr,
                         col_idx, r, vals, bad, &miss_c, &err_c);
    missing += miss_c;
    ncm_err += err_c;
  }
  free(colour);
  return ncm_err ? -2 : missing;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
