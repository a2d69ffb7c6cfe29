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

// Cyclic Jacobi eigensolver for the symmetric 3x3 F^T F (stands in for Eigen's
// SelfAdjointEigenSolver, tensor.cpp:208-215).  Identical IEEE sequence in the oracle.
FB_HD void jacobi3(double* a, double* q) {
  for (int i = 0; i < 9; ++i) q[i] = (i % 4 == 0) ? 1.0 : 0.0;
  const int P[3] = {0, 0, 1}, Q[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 64; ++sweep) {
    bool rotated = false;
    for (int r = 0; r < 3; ++r) {
      const int p = P[r], qq = Q[r];
      const double apq = a[3 * p + qq];
      const double app = a[3 * p + p], aqq = a[3 * qq + qq];
      if (fabs(apq) <= 1e-18 * (fabs(app) + fabs(aqq))) {
        a[3 * p + qq] = a[3 * qq + p] = 0.0;
        continue;
      }
      rotated = true;
      const double tau = (aqq - app) / (2.0 * apq);
      const double t = tau >= 0.0 ? 1.0 / (tau + sqrt(1.0 + tau * tau))
                                  : -1.0 / (-tau + sqrt(1.0 + tau * tau));
      const double c = 1.0 / sqrt(1.0 + t * t);
      const double s = t * c;
      a[3 * p + p] = app - t * apq;
      a[3 * qq + qq] = aqq + t * apq;
      a[3 * p + qq] = a[3 * qq + p] = 0.0;
      const int o = 3 - p - qq;
      const double arp = a[3 * o + p], arq = a[3 * o + qq];
      a[3 * o + p] = a[3 * p + o] = c * arp - s * arq;
      a[3 * o + qq] = a[3 * qq + o] = s * arp + c * arq;
      for (int k = 0; k < 3; ++k) {
        const double qkp = q[3 * k + p], qkq = q[3 * k + qq];
        q[3 * k + p] = c * qkp - s * qkq;
        q[3 * k + qq] = s * qkp + c * qkq;
      }
    }
    if (!rotated) break;
  }
}

// F = R U via the eigendecomposition of F^T F (tensor.cpp:203-224)
FB_HD bool polar_decompose(const double* f, double* rot, double* u6) {
  const double j = det3(f);
  if (!(j > 0.0)) return false;
  double ft[9], c[9], q[9];
  transpose3(f, ft);
  matmul3(ft, f, c);
  jacobi3(c, q);
  const double lam[3] = {c[0], c[4], c[8]};
  if (lam[0] <= 0.0 || lam[1] <= 0.0 || lam[2] <= 0.0) return false;
  double sq[3], isq[3];
  for (int k = 0; k < 3; ++k) {
    sq[k] = sqrt(lam[k]);
    isq[k] = 1.0 / sq[k];
  }
  double u[9], uinv[9];
  for (int i = 0; i < 3; ++i)
    for (int jj = 0; jj < 3; ++jj) {
      double s = 0, si = 0;
      for (int k = 0; k < 3; ++k) {
        s += (q[3 * i + k] * sq[k]) * q[3 * jj + k];
        si += (q[3 * i + k] * isq[k]) * q[3 * jj + k];
      }
      u[3 * i + jj] = s;
      uinv[3 * i + jj] = si;
    }
  matmul3(f, uinv, rot);
  sym_from_full(u, u6);
  return true;
}

// ([M][T])^T A^T = P^T by full-pivot LU (stands in for Eigen::FullPivLU,
// stiffness.cpp:26-39); returns false when rank-deficient (isInvertible() == false).
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
    for (int k = 0; k < 6; ++k)
      for (int i = k + 1; i < 6; ++i) c[6 * i + jj] -= lu[6 * i + k] * c[6 * k + jj];
    for (int k = 5; k >= 0; --k) {
      c[6 * k + jj] /= lu[6 * k + k];
      for (int i = 0; i < k; ++i) c[6 * i + jj] -= lu[6 * i + k] * c[6 * k + jj];
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
