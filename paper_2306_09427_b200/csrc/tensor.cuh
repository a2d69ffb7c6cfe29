// Small-tensor math of the constitutive pre/post-processing, run on the device once per
// point (prep_kernel / post_kernel).  Same IEEE operation sequences as the reference
// (proj/src/tensor.cpp, stiffness.cpp) -- the library is compiled with --fmad=false so no
// a*b+c is contracted.  Layouts: Def3 row-major [9]; SymTensor3 {xx,yy,zz,yz,xz,xy};
// Mandel66 row-major [36].
#pragma once

#include <cfloat>
#include <cmath>

#define FB_HD __host__ __device__ __forceinline__

namespace fibra_b200 {

constexpr double kSqrt2 = 1.4142135623730951;  // tensor.cpp:11

FB_HD double smax(double a, double b) { return (a < b) ? b : a; }  // std::max
FB_HD double smin(double a, double b) { return (b < a) ? b : a; }  // std::min

FB_HD double det3(const double* m) {  // Def3::det tensor.cpp:29-33
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

FB_HD bool inverse3(const double* m, double* r) {  // Def3::inverse tensor.cpp:35-49
  const double d = det3(m);
  if (d == 0.0) return false;
  r[0] = (m[4] * m[8] - m[5] * m[7]) / d;
  r[1] = (m[2] * m[7] - m[1] * m[8]) / d;
  r[2] = (m[1] * m[5] - m[2] * m[4]) / d;
  r[3] = (m[5] * m[6] - m[3] * m[8]) / d;
  r[4] = (m[0] * m[8] - m[2] * m[6]) / d;
  r[5] = (m[2] * m[3] - m[0] * m[5]) / d;
  r[6] = (m[3] * m[7] - m[4] * m[6]) / d;
  r[7] = (m[1] * m[6] - m[0] * m[7]) / d;
  r[8] = (m[0] * m[4] - m[1] * m[3]) / d;
  return true;
}

FB_HD void transpose3(const double* m, double* r) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[3 * i + j] = m[3 * j + i];
}

FB_HD void matmul3(const double* a, const double* b, double* r) {  // tensor.cpp:64-73
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += a[3 * i + k] * b[3 * k + j];
      r[3 * i + j] = s;
    }
}

FB_HD double sym_at(const double* s, int i, int j) {  // SymTensor3::operator() :75-79
  if (i == j) return i == 0 ? s[0] : (i == 1 ? s[1] : s[2]);
  const int k = i + j;
  return k == 1 ? s[5] : (k == 2 ? s[4] : s[3]);
}

FB_HD void sym_full(const double* s, double* a) {  // SymTensor3::full :90-99
  a[0] = s[0];
  a[4] = s[1];
  a[8] = s[2];
  a[5] = a[7] = s[3];
  a[2] = a[6] = s[4];
  a[1] = a[3] = s[5];
}

FB_HD void sym_from_full(const double* a, double* s) {  // :101-110 (symmetrizes)
  s[0] = a[0];
  s[1] = a[4];
  s[2] = a[8];
  s[3] = 0.5 * (a[5] + a[7]);
  s[4] = 0.5 * (a[2] + a[6]);
  s[5] = 0.5 * (a[1] + a[3]);
}

FB_HD double sym_frobenius(const double* a) {  // tensor.hpp:53, ddot :112-115
  return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2] +
              2.0 * (a[3] * a[3] + a[4] * a[4] + a[5] * a[5]));
}

FB_HD void mandel6(const double* s, double* v) {  // tensor.cpp:127-136
  v[0] = s[0];
  v[1] = s[1];
  v[2] = s[2];
  v[3] = kSqrt2 * s[3];
  v[4] = kSqrt2 * s[4];
  v[5] = kSqrt2 * s[5];
}

FB_HD void unmandel6(const double* v, double* s) {  // :138-147
  s[0] = v[0];
  s[1] = v[1];
  s[2] = v[2];
  s[3] = v[3] / kSqrt2;
  s[4] = v[4] / kSqrt2;
  s[5] = v[5] / kSqrt2;
}

FB_HD void matmul6(const double* a, const double* b, double* r) {  // Mandel66::matmul :159-168
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0;
      for (int k = 0; k < 6; ++k) s += a[6 * i + k] * b[6 * k + j];
      r[6 * i + j] = s;
    }
}

FB_HD void probing_matrix(double* t) {  // tensor.cpp:258-273
  const double h = 0.5;
  const double s = 0.5 * kSqrt2;
  for (int i = 0; i < 36; ++i) t[i] = 0.0;
  t[0] = h; t[4] = s; t[5] = s;
  t[7] = h; t[9] = s; t[11] = s;
  t[14] = h; t[15] = s; t[16] = s;
  t[21] = 1; t[28] = 1; t[35] = 1;
}

FB_HD void probing_direction(int q, double* dir) {  // tensor.cpp:275-284
  double t[36], col[6];
  probing_matrix(t);
  for (int i = 0; i < 6; ++i) col[i] = t[6 * i + q];
  unmandel6(col, dir);
}

FB_HD void mandel_M_of_U(const double* u, double* m) {  // tensor.cpp:238-256
  const int MI[6] = {0, 1, 2, 1, 0, 0};
  const int MJ[6] = {0, 1, 2, 2, 2, 1};
  for (int p = 0; p < 6; ++p) {
    const int k = MI[p], l = MJ[p];
    const double wp = p < 3 ? 1.0 : kSqrt2;
    for (int q = 0; q < 6; ++q) {
      const int r = MI[q], s = MJ[q];
      const double wq = q < 3 ? 1.0 : kSqrt2;
      double v = 0.0;
      v += (k == s ? sym_at(u, r, l) : 0.0);
      v += (l == s ? sym_at(u, r, k) : 0.0);
      v += (k == r ? sym_at(u, s, l) : 0.0);
      v += (l == r ? sym_at(u, s, k) : 0.0);
      m[6 * p + q] = 0.25 * wp * wq * v;
    }
  }
}

// C = (1/J) B A B^T with B the Mandel matrix of S -> F S F^T (tensor.cpp:286-300)
FB_HD bool push_forward_stiffness(const double* a, const double* f, double* c) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  double b[36], ft[9];
  transpose3(f, ft);
  for (int q = 0; q < 6; ++q) {
    double e[6] = {0, 0, 0, 0, 0, 0}, s[6], sf[9], t1[9], fs[9], sym[6], col[6];
    e[q] = 1.0;
    unmandel6(e, s);
    sym_full(s, sf);
    matmul3(f, sf, t1);
    matmul3(t1, ft, fs);
    sym_from_full(fs, sym);
    mandel6(sym, col);
    for (int p = 0; p < 6; ++p) b[6 * p + q] = col[p];
  }
  double bt[36], ba[36], bab[36];
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < 6; ++k) bt[6 * i + k] = b[6 * k + i];
  matmul6(b, a, ba);
  matmul6(ba, bt, bab);
  const double inv = 1.0 / j;
  for (int i = 0; i < 36; ++i) c[i] = bab[i] * inv;
  return true;
}

// Pi = J F^-1 sigma F^-T (tensor.cpp:309-315)
FB_HD bool pull_back_stress(const double* sig, const double* f, double* out) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  double finv[9], finvt[9], sf[9], t1[9], s[9], sym[6];
  if (!inverse3(f, finv)) return false;
  transpose3(finv, finvt);
  sym_full(sig, sf);
  matmul3(finv, sf, t1);
  matmul3(t1, finvt, s);
  sym_from_full(s, sym);
  for (int i = 0; i < 6; ++i) out[i] = sym[i] * j;
  return true;
}

// sigma = R sigma_U R^T, symmetrized (stiffness.cpp:171-173)
FB_HD void rotate_stress(const double* rot, const double* su6, double* out) {
  double su[9], rt[9], t1[9], s9[9];
  sym_full(su6, su);
  transpose3(rot, rt);
  matmul3(rot, su, t1);
  matmul3(t1, rt, s9);
  sym_from_full(s9, out);
}

// ---- Eigen 3.4.0 on the reference's hot path, restated (oracle/fibra_oracle.c carries
// the derivation: SSE2 Packet2d build, no FMA).  Same IEEE sequence as the oracle.

// Matrix3d product assignment (SliceVectorizedTraversal): rows 0-1 of each column as one
// packet, ((l0 r0 + l1 r1) + l2 r2); row 2 through coeff(), l0 r0 + (l1 r1 + l2 r2).
FB_HD void eig_prod3_slice(const double* l, const double* r, double* out) {
  for (int j = 0; j < 3; ++j) {
    for (int i = 0; i < 2; ++i)
      out[3 * i + j] = (l[3 * i] * r[j] + l[3 * i + 1] * r[3 + j]) + l[3 * i + 2] * r[6 + j];
    out[6 + j] = l[6] * r[j] + (l[7] * r[3 + j] + l[8] * r[6 + j]);
  }
}

FB_HD double eig_hypot(double x, double y) {  // positive_real_hypot (MathFunctionsImpl.h)
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  const double p = smax(x, y);
  if (p == 0.0) return 0.0;
  const double qp = smin(y, x) / p;
  return p * sqrt(1.0 + qp * qp);
}

FB_HD void eig_make_givens(double p, double q, double& c, double& s) {  // Jacobi.h
  if (q == 0.0) {
    c = p < 0.0 ? -1.0 : 1.0;
    s = 0.0;
  } else if (p == 0.0) {
    c = 0.0;
    s = q < 0.0 ? 1.0 : -1.0;
  } else if (fabs(p) > fabs(q)) {
    const double t = q / p;
    double u = sqrt(1.0 + t * t);
    if (p < 0.0) u = -u;
    c = 1.0 / u;
    s = -t * c;
  } else {
    const double t = p / q;
    double u = sqrt(1.0 + t * t);
    if (q < 0.0) u = -u;
    s = -1.0 / u;
    c = -t * s;
  }
}

FB_HD void eig_qr_step(double* diag, double* sub, int start, int end, double* q) {
  // tridiagonal_qr_step (SelfAdjointEigenSolver.h), Wilkinson shift
  const double td = (diag[end - 1] - diag[end]) * 0.5;
  const double e = sub[end - 1];
  double mu = diag[end];
  if (td == 0.0) {
    mu -= fabs(e);
  } else if (e != 0.0) {
    const double e2 = e * e;
    const double h = eig_hypot(td, e);
    if (e2 == 0.0)
      mu -= e / ((td + (td > 0.0 ? h : -h)) / e);
    else
      mu -= e2 / (td + (td > 0.0 ? h : -h));
  }
  double x = diag[start] - mu;
  double z = sub[start];
  for (int k = start; k < end && z != 0.0; ++k) {
    double c, s;
    eig_make_givens(x, z, c, s);
    const double sdk = s * diag[k] + c * sub[k];
    const double dkp1 = s * sub[k] + c * diag[k + 1];
    diag[k] = c * (c * diag[k] - s * sub[k]) - s * (c * sub[k] - s * diag[k + 1]);
    diag[k + 1] = s * sdk + c * dkp1;
    sub[k] = c * sdk - s * dkp1;
    if (k > start) sub[k - 1] = c * sub[k - 1] - s * z;
    x = sub[k];
    if (k < end - 1) {
      z = -s * sub[k + 1];
      sub[k + 1] = c * sub[k + 1];
    }
    if (!(c == 1.0 && -s == 0.0))  // Q.applyOnTheRight(k, k+1, rot): rotation (c, -s)
      for (int i = 0; i < 3; ++i) {
        const double xi = q[3 * i + k], yi = q[3 * i + k + 1];
        q[3 * i + k] = c * xi + (-s) * yi;
        q[3 * i + k + 1] = s * xi + c * yi;
      }
  }
}

// SelfAdjointEigenSolver<Matrix3d>::compute(a, ComputeEigenvectors); false = NoConvergence
FB_HD bool eigen_sym3(const double* a, double* lam, double* q) {
  double m[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = (j <= i) ? a[3 * i + j] : 0.0;
  double scale = 0.0;
  for (int k = 0; k < 9; ++k) scale = smax(scale, fabs(m[k]));
  if (scale == 0.0) scale = 1.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j <= i; ++j) m[3 * i + j] /= scale;
  double diag[3], sub[2];  // tridiagonalization_inplace_selector<MatrixType, 3, false>
  diag[0] = m[0];
  const double v1norm2 = m[6] * m[6];
  if (v1norm2 <= DBL_MIN) {
    diag[1] = m[4];
    diag[2] = m[8];
    sub[0] = m[3];
    sub[1] = m[7];
    for (int k = 0; k < 9; ++k) q[k] = (k % 4 == 0) ? 1.0 : 0.0;
  } else {
    const double beta = sqrt(m[3] * m[3] + v1norm2);
    const double inv_beta = 1.0 / beta;
    const double m01 = m[3] * inv_beta;
    const double m02 = m[6] * inv_beta;
    const double qq = 2.0 * m01 * m[7] + m02 * (m[8] - m[4]);
    diag[1] = m[4] + m02 * qq;
    diag[2] = m[8] - m02 * qq;
    sub[0] = beta;
    sub[1] = m[7] - m01 * qq;
    q[0] = 1; q[1] = 0; q[2] = 0;
    q[3] = 0; q[4] = m01; q[5] = m02;
    q[6] = 0; q[7] = m02; q[8] = -m01;
  }
  const double precision_inv = 1.0 / DBL_EPSILON;  // computeFromTridiagonal_impl
  int end = 2, start = 0, iter = 0;
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (fabs(sub[i]) < DBL_MIN) {
        sub[i] = 0.0;
      } else {
        const double scaled = precision_inv * sub[i];
        if (scaled * scaled <= (fabs(diag[i]) + fabs(diag[i + 1]))) sub[i] = 0.0;
      }
    }
    while (end > 0 && sub[end - 1] == 0.0) end--;
    if (end <= 0) break;
    iter++;
    if (iter > 30 * 3) break;
    start = end - 1;
    while (start > 0 && sub[start - 1] != 0.0) start--;
    eig_qr_step(diag, sub, start, end, q);
  }
  if (iter > 30 * 3) return false;
  for (int i = 0; i < 2; ++i) {  // ascending sort, first minimum, columns follow
    int k = 0;
    for (int t = 1; t < 3 - i; ++t)
      if (diag[i + t] < diag[i + k]) k = t;
    if (k > 0) {
      const double d = diag[i];
      diag[i] = diag[k + i];
      diag[k + i] = d;
      for (int r = 0; r < 3; ++r) {
        const double v = q[3 * r + i];
        q[3 * r + i] = q[3 * r + k + i];
        q[3 * r + k + i] = v;
      }
    }
  }
  for (int k = 0; k < 3; ++k) lam[k] = diag[k] * scale;
  return true;
}

// F = R U via the eigendecomposition of F^T F (tensor.cpp:203-224)
FB_HD bool polar_decompose(const double* f, double* rot, double* u6) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  double c[9];
  for (int i = 0; i < 3; ++i)  // fe.transpose() * fe (vectorized redux per coefficient)
    for (int jj = 0; jj < 3; ++jj)
      c[3 * i + jj] = (f[i] * f[jj] + f[3 + i] * f[3 + jj]) + f[6 + i] * f[6 + jj];
  double lam[3], q[9];
  if (!eigen_sym3(c, lam, q)) return false;
  if (smin(smin(lam[0], lam[1]), lam[2]) <= 0.0) return false;
  double sq[3], isq[3];
  for (int k = 0; k < 3; ++k) sq[k] = sqrt(lam[k]);
  for (int k = 0; k < 3; ++k) isq[k] = 1.0 / sq[k];
  double qd[9], qdi[9], qt[9], u[9], uinv[9];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      qd[3 * i + k] = q[3 * i + k] * sq[k];
      qdi[3 * i + k] = q[3 * i + k] * isq[k];
      qt[3 * k + i] = q[3 * i + k];
    }
  eig_prod3_slice(qd, qt, u);
  eig_prod3_slice(qdi, qt, uinv);
  eig_prod3_slice(f, uinv, rot);
  sym_from_full(u, u6);
  return true;
}

// ([M][T])^T A^T = P^T by Eigen::FullPivLU (stiffness.cpp:26-39); false when
// rank-deficient (isInvertible() == false).  Solve order = Eigen's blocked TRSM on the
// row-major rhs copy (see the oracle).
FB_HD bool fullpiv_solve6(const double* a_in, const double* rhs, double* x) {
  double lu[36], c[36];
  int rt[6], ct[6];
  for (int i = 0; i < 36; ++i) lu[i] = a_in[i];
  double maxpivot = 0;
  int nonzero = 6;
  for (int k = 0; k < 6; ++k) {
    double big = -1.0;
    int br = k, bc = k;
    for (int jj = k; jj < 6; ++jj)
      for (int i = k; i < 6; ++i) {
        const double v = fabs(lu[6 * i + jj]);
        if (v > big) { big = v; br = i; bc = jj; }
      }
    if (big == 0.0) {
      nonzero = k;
      for (int i = k; i < 6; ++i) rt[i] = ct[i] = i;
      break;
    }
    if (big > maxpivot) maxpivot = big;
    rt[k] = br;
    ct[k] = bc;
    if (br != k)
      for (int jj = 0; jj < 6; ++jj) { const double t = lu[6 * k + jj]; lu[6 * k + jj] = lu[6 * br + jj]; lu[6 * br + jj] = t; }
    if (bc != k)
      for (int i = 0; i < 6; ++i) { const double t = lu[6 * i + k]; lu[6 * i + k] = lu[6 * i + bc]; lu[6 * i + bc] = t; }
    if (k < 5) {
      const double piv = lu[6 * k + k];
      for (int i = k + 1; i < 6; ++i) lu[6 * i + k] /= piv;
      for (int jj = k + 1; jj < 6; ++jj)
        for (int i = k + 1; i < 6; ++i) lu[6 * i + jj] -= lu[6 * i + k] * lu[6 * k + jj];
    }
  }
  const double thr = maxpivot * (DBL_EPSILON * 6.0);
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += fabs(lu[6 * i + i]) > thr;
  if (rank != 6) return false;
  for (int i = 0; i < 36; ++i) c[i] = rhs[i];
  for (int k = 0; k < 6; ++k)
    if (rt[k] != k)
      for (int jj = 0; jj < 6; ++jj) { const double t = c[6 * k + jj]; c[6 * k + jj] = c[6 * rt[k] + jj]; c[6 * rt[k] + jj] = t; }
  for (int jj = 0; jj < 6; ++jj) {
    double* y = c + jj;
    for (int i = 1; i < 4; ++i)  // unit lower: 4-row panel, gebp rows 4-5, 2-row panel
      for (int k = 0; k < i; ++k) y[6 * i] -= y[6 * k] * lu[6 * i + k];
    for (int i = 4; i < 6; ++i) {
      double acc = 0.0;
      for (int k = 0; k < 4; ++k) acc = acc + y[6 * k] * lu[6 * i + k];
      y[6 * i] = y[6 * i] + (-1.0) * acc;
    }
    y[6 * 5] -= y[6 * 4] * lu[6 * 5 + 4];
    y[6 * 5] *= 1.0 / lu[6 * 5 + 5];  // upper: 2-row panel, gebp rows 0-3, 4-row panel
    y[6 * 4] -= y[6 * 5] * lu[6 * 4 + 5];
    y[6 * 4] *= 1.0 / lu[6 * 4 + 4];
    for (int i = 0; i < 4; ++i) {
      double acc = 0.0;
      for (int k = 4; k < 6; ++k) acc = acc + y[6 * k] * lu[6 * i + k];
      y[6 * i] = y[6 * i] + (-1.0) * acc;
    }
    for (int i = 3; i >= 0; --i) {
      for (int k = i + 1; k < 4; ++k) y[6 * i] -= y[6 * k] * lu[6 * i + k];
      y[6 * i] *= 1.0 / lu[6 * i + i];
    }
  }
  for (int k = 5; k >= 0; --k)
    if (ct[k] != k)
      for (int jj = 0; jj < 6; ++jj) { const double t = c[6 * k + jj]; c[6 * k + jj] = c[6 * ct[k] + jj]; c[6 * ct[k] + jj] = t; }
  for (int i = 0; i < 36; ++i) x[i] = c[i];
  return true;
}

// A from the six probe Pi's (stiffness.cpp:15-41)
FB_HD bool material_stiffness_from_probes(const double* u, const double* base_pk2,
                                          const double* probe_pk2, double h, double* a) {
  double base[6], p[36], m[36], t[36], mt[36], mtt[36], pt[36], at[36];
  mandel6(base_pk2, base);
  for (int q = 0; q < 6; ++q) {
    double col[6];
    mandel6(probe_pk2 + 6 * q, col);
    for (int i = 0; i < 6; ++i) p[6 * i + q] = (col[i] - base[i]) / h;
  }
  mandel_M_of_U(u, m);
  probing_matrix(t);
  matmul6(m, t, mt);
  for (int i = 0; i < 6; ++i)
    for (int jj = 0; jj < 6; ++jj) {
      mtt[6 * i + jj] = mt[6 * jj + i];
      pt[6 * i + jj] = p[6 * jj + i];
    }
  if (!fullpiv_solve6(mtt, pt, at)) return false;
  for (int i = 0; i < 6; ++i)
    for (int jj = 0; jj < 6; ++jj) a[6 * i + jj] = at[6 * jj + i];
  return true;
}

}  // namespace fibra_b200
