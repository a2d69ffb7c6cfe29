/*
 * fibra_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE:
 * the parity checker for the B200 solver, never shipped or measured as the product.
 * Build with -ffp-contract=off (proj/CMakeLists.txt:14-16) so every a*b+c rounds twice,
 * exactly as the reference does.  See fibra_oracle.h for the pinning story.
 *
 * Every function cites the reference function it restates (paths under
 * /root/reference/proj).  Floating-point expressions keep the reference's evaluation
 * order (C evaluates a+b+c as (a+b)+c, like C++).
 */
#include "fibra_oracle.h"

#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double kSqrt2 = 1.4142135623730951; /* tensor.cpp:11 */

/* std::max / std::min semantics (first argument wins ties and NaN compares) */
static inline double smax(double a, double b) { return (a < b) ? b : a; }
static inline double smin(double a, double b) { return (b < a) ? b : a; }

/* ------------------------------------------------------------------------- */
/* FiberLaw  network.cpp:16-59                                               */
/* ------------------------------------------------------------------------- */
static double law_force(const or_law* law, double ea, double stretch) { /* :16-26 */
  const double s = law->ea_scale * ea;
  if (law->buckling_off && stretch < 1.0) return 0.0;
  if (law->kind == 0) return s * (stretch - 1.0);
  return s / law->nonlinearity * expm1(law->nonlinearity * (stretch - 1.0));
}

static double law_tangent(const or_law* law, double ea, double stretch) { /* :28-38 */
  const double s = law->ea_scale * ea;
  if (law->buckling_off && stretch < 1.0) return 0.0;
  if (law->kind == 0) return s;
  return s * exp(law->nonlinearity * (stretch - 1.0));
}

static double law_energy(const or_law* law, double ea, double stretch, double rl) { /* :40-53 */
  const double s = law->ea_scale * ea;
  if (law->buckling_off && stretch < 1.0) return 0.0;
  const double e = stretch - 1.0;
  if (law->kind == 0) return 0.5 * s * rl * e * e;
  const double b = law->nonlinearity;
  return rl * s / b * (expm1(b * e) / b - e);
}

static int law_validate(const or_law* law) { /* :55-59 */
  if (!(law->ea_scale > 0)) return OR_CONFIG;
  if (law->kind == 1 && !(law->nonlinearity > 0)) return OR_CONFIG;
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* FiberNetwork constructor  network.cpp:67-157                               */
/* ------------------------------------------------------------------------- */
static int cmp_pair(const void* x, const void* y) {
  const int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  return (a > b) - (a < b);
}

int or_network_build(const double* coords, int nn, const int32_t* fa, const int32_t* fb,
                     const double* area, const double* modulus, int nf, double h,
                     double tol, or_network* net) {
  memset(net, 0, sizeof *net);
  if (nn <= 0) return OR_CONFIG;                         /* :71 */
  if (!(h > 0)) return OR_CONFIG;                        /* :72 */
  for (int i = 0; i < nn; ++i)                           /* :74-83 */
    for (int k = 0; k < 3; ++k) {
      const double c = coords[3 * i + k];
      if (!isfinite(c)) return OR_CONFIG;
      if (fabs(c) > h + tol) return OR_CONFIG;
    }
  net->n_nodes = nn;
  net->n_fibers = nf;
  net->box_half = h;
  net->tol_bnd = tol;
  net->coords = malloc(sizeof(double) * 3 * nn);
  memcpy(net->coords, coords, sizeof(double) * 3 * nn);
  net->fib_a = malloc(sizeof(int32_t) * (nf ? nf : 1));
  net->fib_b = malloc(sizeof(int32_t) * (nf ? nf : 1));
  net->area = malloc(sizeof(double) * (nf ? nf : 1));
  net->modulus = malloc(sizeof(double) * (nf ? nf : 1));
  net->rest_length = malloc(sizeof(double) * (nf ? nf : 1));
  int64_t* keys = malloc(sizeof(int64_t) * (nf ? nf : 1));
  double max_ea = 0;
  for (int f = 0; f < nf; ++f) {                         /* :85-107 */
    const int32_t a = fa[f], b = fb[f];
    if (a < 0 || b < 0 || a >= nn || b >= nn || a == b) { free(keys); or_network_free(net); return OR_CONFIG; }
    if (!(area[f] > 0) || !(modulus[f] > 0)) { free(keys); or_network_free(net); return OR_CONFIG; }
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    keys[f] = ((int64_t)lo << 32) | (int64_t)hi;
    const double* xa = coords + 3 * a;
    const double* xb = coords + 3 * b;
    const double d0 = xb[0] - xa[0], d1 = xb[1] - xa[1], d2 = xb[2] - xa[2];
    const double l0 = sqrt(d0 * d0 + d1 * d1 + d2 * d2); /* norm3, tensor.hpp:11-14 */
    if (!(l0 > 0)) { free(keys); or_network_free(net); return OR_CONFIG; }
    net->fib_a[f] = a;
    net->fib_b[f] = b;
    net->area[f] = area[f];
    net->modulus[f] = modulus[f];
    net->rest_length[f] = l0;
    max_ea = smax(max_ea, area[f] * modulus[f]);
  }
  qsort(keys, nf, sizeof(int64_t), cmp_pair);            /* duplicate-fiber check :98-101 */
  for (int f = 1; f < nf; ++f)
    if (keys[f] == keys[f - 1]) { free(keys); or_network_free(net); return OR_CONFIG; }
  free(keys);
  net->max_ea = max_ea;

  net->boundary_mask = calloc(nn, 1);                    /* :109-117 */
  net->boundary_nodes = malloc(sizeof(int32_t) * nn);
  int nb = 0;
  for (int i = 0; i < nn; ++i) {
    for (int k = 0; k < 3; ++k)
      if (fabs(fabs(coords[3 * i + k]) - h) <= tol) net->boundary_mask[i] = 1;
    if (net->boundary_mask[i]) net->boundary_nodes[nb++] = i;
  }
  net->n_boundary = nb;
  if (nb == 0) { or_network_free(net); return OR_CONFIG; }

  net->packed_of_dof = malloc(sizeof(int32_t) * 3 * nn); /* free-first packing :120-138 */
  net->dof_of_packed = malloc(sizeof(int32_t) * 3 * nn);
  int slot = 0;
  for (int i = 0; i < nn; ++i)
    if (!net->boundary_mask[i])
      for (int k = 0; k < 3; ++k) {
        net->packed_of_dof[3 * i + k] = slot;
        net->dof_of_packed[slot] = 3 * i + k;
        ++slot;
      }
  net->n_free = slot;
  for (int i = 0; i < nn; ++i)
    if (net->boundary_mask[i])
      for (int k = 0; k < 3; ++k) {
        net->packed_of_dof[3 * i + k] = slot;
        net->dof_of_packed[slot] = 3 * i + k;
        ++slot;
      }
  net->packed_ref = malloc(sizeof(double) * 3 * nn);     /* :140-143 */
  for (int i = 0; i < nn; ++i)
    for (int k = 0; k < 3; ++k) net->packed_ref[net->packed_of_dof[3 * i + k]] = coords[3 * i + k];
  net->fiber_dofs = malloc(sizeof(int32_t) * 6 * (nf ? nf : 1)); /* :145-149 */
  for (int f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      net->fiber_dofs[6 * f + k] = net->packed_of_dof[3 * net->fib_a[f] + k];
      net->fiber_dofs[6 * f + 3 + k] = net->packed_of_dof[3 * net->fib_b[f] + k];
    }
  net->node_lump = calloc(nn, sizeof(double));           /* :151-156 */
  for (int f = 0; f < nf; ++f) {
    const double half_seg = 0.5 * net->rest_length[f] * net->area[f];
    net->node_lump[net->fib_a[f]] += half_seg;
    net->node_lump[net->fib_b[f]] += half_seg;
  }
  return OR_OK;
}

void or_network_free(or_network* n) {
  free(n->coords); free(n->fib_a); free(n->fib_b); free(n->area); free(n->modulus);
  free(n->rest_length); free(n->boundary_mask); free(n->boundary_nodes);
  free(n->packed_of_dof); free(n->dof_of_packed); free(n->packed_ref);
  free(n->fiber_dofs); free(n->node_lump);
  memset(n, 0, sizeof *n);
}

/* ------------------------------------------------------------------------- */
/* small tensors  tensor.cpp                                                  */
/* row-major 3x3 (Def3::m), SymTensor3 as {xx,yy,zz,yz,xz,xy}, Mandel66 row-major */
/* ------------------------------------------------------------------------- */
double or_det(const double m[9]) { /* Def3::det tensor.cpp:29-33 */
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

int or_inverse(const double m[9], double r[9]) { /* Def3::inverse tensor.cpp:35-49 */
  const double d = or_det(m);
  if (d == 0.0) return OR_KINEMATICS;
  r[0] = (m[4] * m[8] - m[5] * m[7]) / d;
  r[1] = (m[2] * m[7] - m[1] * m[8]) / d;
  r[2] = (m[1] * m[5] - m[2] * m[4]) / d;
  r[3] = (m[5] * m[6] - m[3] * m[8]) / d;
  r[4] = (m[0] * m[8] - m[2] * m[6]) / d;
  r[5] = (m[2] * m[3] - m[0] * m[5]) / d;
  r[6] = (m[3] * m[7] - m[4] * m[6]) / d;
  r[7] = (m[1] * m[6] - m[0] * m[7]) / d;
  r[8] = (m[0] * m[4] - m[1] * m[3]) / d;
  return OR_OK;
}

static void transpose3(const double m[9], double r[9]) { /* tensor.cpp:51-56 */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r[3 * i + j] = m[3 * j + i];
}

static void apply3(const double m[9], const double x[3], double y[3]) { /* tensor.cpp:58-62 */
  y[0] = m[0] * x[0] + m[1] * x[1] + m[2] * x[2];
  y[1] = m[3] * x[0] + m[4] * x[1] + m[5] * x[2];
  y[2] = m[6] * x[0] + m[7] * x[1] + m[8] * x[2];
}

void or_matmul(const double a[9], const double b[9], double r[9]) { /* tensor.cpp:64-73 */
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += a[3 * i + k] * b[3 * k + j];
      r[3 * i + j] = s;
    }
}

static double sym_get(const double s[6], int i, int j) { /* SymTensor3::operator() tensor.cpp:75-79 */
  if (i == j) return i == 0 ? s[0] : (i == 1 ? s[1] : s[2]);
  const int k = i + j;
  return k == 1 ? s[5] : (k == 2 ? s[4] : s[3]);
}

void or_sym_full(const double s[6], double a[9]) { /* SymTensor3::full tensor.cpp:90-99 */
  a[0] = s[0]; a[4] = s[1]; a[8] = s[2];
  a[5] = a[7] = s[3];
  a[2] = a[6] = s[4];
  a[1] = a[3] = s[5];
}

void or_sym_from_full(const double a[9], double s[6]) { /* tensor.cpp:101-110 */
  s[0] = a[0];
  s[1] = a[4];
  s[2] = a[8];
  s[3] = 0.5 * (a[5] + a[7]);
  s[4] = 0.5 * (a[2] + a[6]);
  s[5] = 0.5 * (a[1] + a[3]);
}

static double sym_frobenius(const double a[6]) { /* tensor.hpp:53 + ddot tensor.cpp:112-115 */
  return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2] +
              2.0 * (a[3] * a[3] + a[4] * a[4] + a[5] * a[5]));
}

void or_mandel(const double s[6], double v[6]) { /* tensor.cpp:127-136 */
  v[0] = s[0];
  v[1] = s[1];
  v[2] = s[2];
  v[3] = kSqrt2 * s[3];
  v[4] = kSqrt2 * s[4];
  v[5] = kSqrt2 * s[5];
}

static void unmandel(const double v[6], double s[6]) { /* tensor.cpp:138-147 */
  s[0] = v[0];
  s[1] = v[1];
  s[2] = v[2];
  s[3] = v[3] / kSqrt2;
  s[4] = v[4] / kSqrt2;
  s[5] = v[5] / kSqrt2;
}

static void m66_matmul(const double a[36], const double b[36], double r[36]) { /* tensor.cpp:159-168 */
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      double s = 0;
      for (int k = 0; k < 6; ++k) s += a[6 * i + k] * b[6 * k + j];
      r[6 * i + j] = s;
    }
}

static const int kMI[6] = {0, 1, 2, 1, 0, 0}; /* tensor.hpp:104-105 */
static const int kMJ[6] = {0, 1, 2, 2, 2, 1};

void or_mandel_M_of_U(const double u[6], double m[36]) { /* tensor.cpp:238-256 */
  for (int p = 0; p < 6; ++p) {
    const int k = kMI[p], l = kMJ[p];
    const double wp = p < 3 ? 1.0 : kSqrt2;
    for (int q = 0; q < 6; ++q) {
      const int r = kMI[q], s = kMJ[q];
      const double wq = q < 3 ? 1.0 : kSqrt2;
      double v = 0.0;
      v += (k == s ? sym_get(u, r, l) : 0.0);
      v += (l == s ? sym_get(u, r, k) : 0.0);
      v += (k == r ? sym_get(u, s, l) : 0.0);
      v += (l == r ? sym_get(u, s, k) : 0.0);
      m[6 * p + q] = 0.25 * wp * wq * v;
    }
  }
}

void or_probing_matrix(double t[36]) { /* tensor.cpp:258-273 */
  const double h = 0.5;
  const double s = 0.5 * kSqrt2;
  const double rows[36] = {h, 0, 0, 0, s, s,  0, h, 0, s, 0, s,  0, 0, h, s, s, 0,
                           0, 0, 0, 1, 0, 0,  0, 0, 0, 0, 1, 0,  0, 0, 0, 0, 0, 1};
  memcpy(t, rows, sizeof rows);
}

void or_probing_direction(int q, double dir[6]) { /* tensor.cpp:275-284 */
  double t[36], col[6];
  or_probing_matrix(t);
  for (int i = 0; i < 6; ++i) col[i] = t[6 * i + q];
  unmandel(col, dir);
}

int or_push_forward_stiffness(const double a[36], const double f[9], double c[36]) {
  /* tensor.cpp:286-300 */
  const double j = or_det(f);
  if (!(j > 0.0)) return OR_KINEMATICS;
  double b[36], ft[9];
  transpose3(f, ft);
  for (int q = 0; q < 6; ++q) {
    double e[6] = {0, 0, 0, 0, 0, 0}, s[6], sf[9], t1[9], fs[9], sym[6], col[6];
    e[q] = 1.0;
    unmandel(e, s);
    or_sym_full(s, sf);
    or_matmul(f, sf, t1);
    or_matmul(t1, ft, fs);
    or_sym_from_full(fs, sym);
    or_mandel(sym, col);
    for (int p = 0; p < 6; ++p) b[6 * p + q] = col[p];
  }
  double bt[36], ba[36], bab[36];
  for (int i = 0; i < 6; ++i)
    for (int k = 0; k < 6; ++k) bt[6 * i + k] = b[6 * k + i];
  m66_matmul(b, a, ba);
  m66_matmul(ba, bt, bab);
  const double inv = 1.0 / j;
  for (int i = 0; i < 36; ++i) c[i] = bab[i] * inv;
  return OR_OK;
}

int or_pull_back_stress(const double sig[6], const double f[9], double out[6]) {
  /* tensor.cpp:309-315 */
  const double j = or_det(f);
  if (!(j > 0.0)) return OR_KINEMATICS;
  double finv[9], finvt[9], sf[9], t1[9], s[9], sym[6];
  if (or_inverse(f, finv)) return OR_KINEMATICS;
  transpose3(finv, finvt);
  or_sym_full(sig, sf);
  or_matmul(finv, sf, t1);
  or_matmul(t1, finvt, s);
  or_sym_from_full(s, sym);
  for (int i = 0; i < 6; ++i) out[i] = sym[i] * j;
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Eigen 3.4.0 pieces on the hot path (RESTATEMENT of the published library)  */
/* ------------------------------------------------------------------------- */
/* The reference builds tensor.cpp / stiffness.cpp against the system Eigen
 * (CMakeLists.txt:34, /usr/include/eigen3), which is absent here.  We pin Eigen 3.4.0
 * (the Ubuntu 24.04 libeigen3-dev package this image's toolchain matches) at the
 * reference's compile flags: -O3 -ffp-contract=off, no -march, so x86-64 SSE2 only
 * (Packet2d, EIGEN_UNALIGNED_VECTORIZE=1, no FMA), and restate, operation by
 * operation, what that build executes:
 *   - Matrix3d products (CoeffBasedProductMode, lazy product evaluator,
 *     Eigen/src/Core/ProductEvaluators.h + AssignEvaluator.h): a column-major 3x3
 *     result whose product evaluator has packet access (column-major lhs) is assigned
 *     by SliceVectorizedTraversal with InnerUnrolling: rows 0-1 of every column as one
 *     Packet2d, accumulated ((l0*r0 + l1*r1) + l2*r2) (etor_product_packet_impl), row 2
 *     through coeff() = (lhs.row(2)' .* rhs.col(j)).sum(), whose strided operands give a
 *     non-vectorized redux, redux_novec_unroller's halving order l0*r0 + (l1*r1 + l2*r2).
 *     Without packet access (F^T F: row-major lhs, column-major rhs) every coefficient
 *     goes through coeff(), and there the operands are contiguous, so the redux is
 *     LinearVectorized: predux(packet(0,1)) + x2 = (x0 + x1) + x2.
 *   - SelfAdjointEigenSolver<Matrix3d>::compute (Eigenvalues/SelfAdjointEigenSolver.h):
 *     lower triangle scaled by its max |entry|; tridiagonalization_inplace_selector<...,3,
 *     false> (Eigenvalues/Tridiagonalization.h, closed-form Householder);
 *     computeFromTridiagonal_impl (deflation |s| < DBL_MIN or (s/eps)^2 <= |d_i|+|d_i+1|,
 *     30*n iteration cap) with tridiagonal_qr_step (Wilkinson shift via numext::hypot,
 *     JacobiRotation::makeGivens, Q.applyOnTheRight(k, k+1, G)), then the selection sort
 *     of the eigenvalues (first minimum) with their columns; eigenvalues *= scale.
 *   - FullPivLU<Matrix<double,6,6>> (LU/FullPivLU.h): computeInPlace as in the previous
 *     restatement; _solve_impl with c = RhsType::PlainObject, which for the reference's
 *     rhs pe.transpose() is ROW-major, so both triangular solves go through
 *     triangular_solve_matrix<..., RowMajor other> = the OnTheRight kernel on the
 *     transposed problem (Core/products/TriangularSolverMatrix.h) with SmallPanelWidth =
 *     max(mr, nr) = 4 (gebp_traits<double,double>, SSE2: nr = 4, mr = 2*2) and one
 *     kc = 6 block: panels of 4 and 2 columns, the off-panel part through gebp (an
 *     accumulator started at +0.0, depth in ascending order, then r + (-1)*acc), the
 *     in-panel part left-looking (r -= x_k * t_kj, k ascending), the non-unit diagonal
 *     applied as r *= 1/t_jj.
 * Nothing in the reference's tests pins Eigen's bits, so this is "parity by
 * restatement"; csrc/tensor.cuh executes the identical sequence on the device. */

/* R = L * Rh for 3x3 (row-major storage of the math matrices) as the reference's
 * Matrix3d product assignment evaluates it (see above): rows 0-1 left fold, row 2
 * l0 + (l1 + l2). */
static void eig_prod3_slice(const double l[9], const double r[9], double out[9]) {
  for (int j = 0; j < 3; ++j) {
    for (int i = 0; i < 2; ++i)
      out[3 * i + j] = (l[3 * i] * r[j] + l[3 * i + 1] * r[3 + j]) + l[3 * i + 2] * r[6 + j];
    out[6 + j] = l[6] * r[j] + (l[7] * r[3 + j] + l[8] * r[6 + j]);
  }
}

static double eig_hypot(double x, double y) { /* MathFunctionsImpl.h positive_real_hypot */
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return INFINITY;
  if (isnan(x) || isnan(y)) return NAN;
  const double p = smax(x, y);
  if (p == 0.0) return 0.0;
  const double qp = smin(y, x) / p;
  return p * sqrt(1.0 + qp * qp);
}

/* JacobiRotation<double>::makeGivens(p, q) (Jacobi/Jacobi.h, real case) */
static void eig_make_givens(double p, double q, double* c, double* s) {
  if (q == 0.0) {
    *c = p < 0.0 ? -1.0 : 1.0;
    *s = 0.0;
  } else if (p == 0.0) {
    *c = 0.0;
    *s = q < 0.0 ? 1.0 : -1.0;
  } else if (fabs(p) > fabs(q)) {
    const double t = q / p;
    double u = sqrt(1.0 + t * t);
    if (p < 0.0) u = -u;
    *c = 1.0 / u;
    *s = -t * *c;
  } else {
    const double t = p / q;
    double u = sqrt(1.0 + t * t);
    if (q < 0.0) u = -u;
    *s = -1.0 / u;
    *c = -t * *s;
  }
}

/* tridiagonal_qr_step<ColMajor> (Eigenvalues/SelfAdjointEigenSolver.h) on n = 3 */
static void eig_qr_step(double diag[3], double sub[2], int start, int end, double q[9]) {
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
    eig_make_givens(x, z, &c, &s);
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
    /* q.applyOnTheRight(k, k+1, rot): apply_rotation_in_the_plane(col k, col k+1,
     * rot.transpose() = (c, -s)): x' = c*x + (-s)*y, y' = s*x + c*y */
    if (!(c == 1.0 && -s == 0.0))
      for (int i = 0; i < 3; ++i) {
        const double xi = q[3 * i + k], yi = q[3 * i + k + 1];
        q[3 * i + k] = c * xi + (-s) * yi;
        q[3 * i + k + 1] = s * xi + c * yi;
      }
  }
}

/* SelfAdjointEigenSolver<Matrix3d>(a, ComputeEigenvectors): eigenvalues ascending in
 * lam, eigenvectors as the columns of q.  Returns 0 on Success, 1 on NoConvergence. */
int or_eigen_sym3(const double a[9], double lam[3], double q[9]) {
  double m[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = (j <= i) ? a[3 * i + j] : 0.0;
  double scale = 0.0;
  for (int k = 0; k < 9; ++k) scale = smax(scale, fabs(m[k])); /* cwiseAbs().maxCoeff() */
  if (scale == 0.0) scale = 1.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j <= i; ++j) m[3 * i + j] /= scale;
  /* tridiagonalization_inplace_selector<MatrixType, 3, false>::run */
  double diag[3], sub[2];
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
    const double qm[9] = {1, 0, 0, 0, m01, m02, 0, m02, -m01};
    memcpy(q, qm, sizeof qm);
  }
  /* computeFromTridiagonal_impl(diag, subdiag, m_maxIterations = 30, true, eivec) */
  const double consider_as_zero = DBL_MIN;
  const double precision_inv = 1.0 / DBL_EPSILON;
  int end = 2, start = 0, iter = 0;
  while (end > 0) {
    for (int i = start; i < end; ++i) {
      if (fabs(sub[i]) < consider_as_zero) {
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
  if (iter > 30 * 3) return 1; /* NoConvergence */
  for (int i = 0; i < 2; ++i) { /* sort: diag.segment(i, n-i).minCoeff(&k) */
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
  return 0;
}

int or_polar_decompose(const double f[9], double rot[9], double u6[6]) {
  /* tensor.cpp:203-224 */
  const double j = or_det(f);
  if (!(j > 0.0)) return OR_KINEMATICS;
  double c[9];
  for (int i = 0; i < 3; ++i) /* fe.transpose() * fe: every coefficient via coeff() */
    for (int jj = 0; jj < 3; ++jj)
      c[3 * i + jj] = (f[i] * f[jj] + f[3 + i] * f[3 + jj]) + f[6 + i] * f[6 + jj];
  double lam[3], q[9];
  if (or_eigen_sym3(c, lam, q)) return OR_KINEMATICS; /* es.info() != Success */
  if (smin(smin(lam[0], lam[1]), lam[2]) <= 0.0) return OR_KINEMATICS;
  double sq[3], isq[3];
  for (int k = 0; k < 3; ++k) sq[k] = sqrt(lam[k]);
  for (int k = 0; k < 3; ++k) isq[k] = 1.0 / sq[k]; /* sq.cwiseInverse() */
  double qd[9], qdi[9], qt[9], u[9], uinv[9];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) {
      qd[3 * i + k] = q[3 * i + k] * sq[k]; /* q * sq.asDiagonal() */
      qdi[3 * i + k] = q[3 * i + k] * isq[k];
      qt[3 * k + i] = q[3 * i + k];
    }
  eig_prod3_slice(qd, qt, u);
  eig_prod3_slice(qdi, qt, uinv);
  eig_prod3_slice(f, uinv, rot); /* fe * uinv */
  or_sym_from_full(u, u6);
  return OR_OK;
}

/* 6x6 full-pivot LU solve of ([M][T])^T [A]^T = [P]^T: Eigen::FullPivLU (stiffness.cpp:
 * 26-39), computeInPlace + _solve_impl as described above. */
static int fullpiv_solve6(const double a_in[36], const double rhs[36], double x[36]) {
  double lu[36], c[36];
  int rt[6], ct[6];
  memcpy(lu, a_in, sizeof lu);
  double maxpivot = 0;
  int nonzero = 6;
  for (int k = 0; k < 6; ++k) {
    double big = -1.0;
    int br = k, bc = k;
    for (int jj = k; jj < 6; ++jj) /* maxCoeff(&row, &col): column-major scan, first max */
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
      for (int jj = 0; jj < 6; ++jj) { double t = lu[6 * k + jj]; lu[6 * k + jj] = lu[6 * br + jj]; lu[6 * br + jj] = t; }
    if (bc != k)
      for (int i = 0; i < 6; ++i) { double t = lu[6 * i + k]; lu[6 * i + k] = lu[6 * i + bc]; lu[6 * i + bc] = t; }
    if (k < 5) {
      const double piv = lu[6 * k + k];
      for (int i = k + 1; i < 6; ++i) lu[6 * i + k] /= piv;
      for (int jj = k + 1; jj < 6; ++jj) /* outer product, column by column */
        for (int i = k + 1; i < 6; ++i) lu[6 * i + jj] -= lu[6 * i + k] * lu[6 * k + jj];
    }
  }
  const double thr = maxpivot * (DBL_EPSILON * 6.0);
  int rank = 0;
  for (int i = 0; i < nonzero; ++i) rank += fabs(lu[6 * i + i]) > thr;
  if (rank != 6) return OR_SINGULAR;
  memcpy(c, rhs, sizeof c);
  for (int k = 0; k < 6; ++k) /* c = P * rhs */
    if (rt[k] != k)
      for (int jj = 0; jj < 6; ++jj) { double t = c[6 * k + jj]; c[6 * k + jj] = c[6 * rt[k] + jj]; c[6 * rt[k] + jj] = t; }
  for (int jj = 0; jj < 6; ++jj) { /* every rhs column independently (one "row" of c^T) */
    double* y = c + jj; /* y[6 * i] = c(i, jj) */
    /* L y = c, unit lower: panel rows 0-3 left-looking, rows 4-5 = gebp over 0-3, then
     * the 2-row panel */
    for (int i = 1; i < 4; ++i)
      for (int k = 0; k < i; ++k) y[6 * i] -= y[6 * k] * lu[6 * i + k];
    for (int i = 4; i < 6; ++i) {
      double acc = 0.0;
      for (int k = 0; k < 4; ++k) acc = acc + y[6 * k] * lu[6 * i + k];
      y[6 * i] = y[6 * i] + (-1.0) * acc;
    }
    y[6 * 5] -= y[6 * 4] * lu[6 * 5 + 4];
    /* U x = y: panel rows 4-5 first (5, then 4), rows 0-3 = gebp over 4-5, then the
     * 4-row panel bottom up, left-looking over the rows already solved in it */
    y[6 * 5] *= 1.0 / lu[6 * 5 + 5];
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
  for (int k = 5; k >= 0; --k) /* dst.row(Q.indices(i)) = c.row(i) */
    if (ct[k] != k)
      for (int jj = 0; jj < 6; ++jj) { double t = c[6 * k + jj]; c[6 * k + jj] = c[6 * ct[k] + jj]; c[6 * ct[k] + jj] = t; }
  memcpy(x, c, sizeof c);
  return OR_OK;
}

int or_material_stiffness_from_probes(const double u[6], const double base_pk2[6],
                                      const double probe_pk2[36], double h, double a[36]) {
  /* stiffness.cpp:15-41 */
  double base[6], p[36], m[36], t[36], mt[36], mtt[36], pt[36], at[36];
  or_mandel(base_pk2, base);
  for (int q = 0; q < 6; ++q) {
    double col[6];
    or_mandel(probe_pk2 + 6 * q, col);
    for (int i = 0; i < 6; ++i) p[6 * i + q] = (col[i] - base[i]) / h;
  }
  or_mandel_M_of_U(u, m);
  or_probing_matrix(t);
  m66_matmul(m, t, mt);
  for (int i = 0; i < 6; ++i)
    for (int jj = 0; jj < 6; ++jj) {
      mtt[6 * i + jj] = mt[6 * jj + i];
      pt[6 * i + jj] = p[6 * jj + i];
    }
  const int st = fullpiv_solve6(mtt, pt, at);
  if (st) return st;
  for (int i = 0; i < 6; ++i)
    for (int jj = 0; jj < 6; ++jj) a[6 * i + jj] = at[6 * jj + i];
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* BLAS-1 contract  kernels_scalar.cpp:7-65 (4 interleaved partials)          */
/* ------------------------------------------------------------------------- */
double or_norm2_sq(int64_t n, const double* x) { /* kernels_scalar.cpp:20-33 */
  double s[4] = {0, 0, 0, 0};
  for (int64_t i = 0; i < n; ++i) s[i & 3] += x[i] * x[i];
  return (s[0] + s[1]) + (s[2] + s[3]);
}

double or_weighted_sq(int64_t n, const double* w, const double* x) { /* :35-48 */
  double s[4] = {0, 0, 0, 0};
  for (int64_t i = 0; i < n; ++i) s[i & 3] += w[i] * (x[i] * x[i]);
  return (s[0] + s[1]) + (s[2] + s[3]);
}

/* ------------------------------------------------------------------------- */
/* forces, BC, stress  network.cpp                                            */
/* ------------------------------------------------------------------------- */
int or_apply_affine_bc(const or_network* net, const double F[9], or_state st) {
  /* network.cpp:254-269 */
  const double j = or_det(F);
  if (!(j > 0)) return OR_KINEMATICS;
  for (int b = 0; b < net->n_boundary; ++b) {
    const int node = net->boundary_nodes[b];
    const double* x = net->coords + 3 * node;
    double fx[3];
    apply3(F, x, fx);
    for (int k = 0; k < 3; ++k) {
      const int p = net->packed_of_dof[3 * node + k];
      st.u[p] = fx[k] - x[k];
      st.v[p] = 0.0;
      st.a[p] = 0.0;
    }
  }
  if (st.converged) *st.converged = 0;
  return OR_OK;
}

int or_internal_forces_cfl(const or_network* net, const or_law* law, const double* u,
                           double* f_int, const double* mred_l0, double* min_dtsq_out) {
  /* force_loop<WithCfl> network.cpp:275-311 */
  const int nd = 3 * net->n_nodes;
  for (int i = 0; i < nd; ++i) f_int[i] = 0.0;
  const double* ref = net->packed_ref;
  double min_dtsq = INFINITY;
  for (int f = 0; f < net->n_fibers; ++f) {
    const int32_t* p = net->fiber_dofs + 6 * f;
    const double dx = (ref[p[3]] + u[p[3]]) - (ref[p[0]] + u[p[0]]);
    const double dy = (ref[p[4]] + u[p[4]]) - (ref[p[1]] + u[p[1]]);
    const double dz = (ref[p[5]] + u[p[5]]) - (ref[p[2]] + u[p[2]]);
    const double len = sqrt(dx * dx + dy * dy + dz * dz);
    const double l0 = net->rest_length[f];
    if (len <= 1e-8 * l0) return OR_COLLAPSE;
    const double stretch = len / l0;
    const double ea = net->area[f] * net->modulus[f];
    const double n_ax = law_force(law, ea, stretch);
    const double g = n_ax / len;
    f_int[p[0]] -= g * dx;
    f_int[p[1]] -= g * dy;
    f_int[p[2]] -= g * dz;
    f_int[p[3]] += g * dx;
    f_int[p[4]] += g * dy;
    f_int[p[5]] += g * dz;
    if (mred_l0) {
      const double kt = smax(fabs(law_tangent(law, ea, stretch)), law->ea_scale * ea);
      min_dtsq = smin(min_dtsq, mred_l0[f] / kt);
    }
  }
  if (min_dtsq_out) *min_dtsq_out = min_dtsq;
  return OR_OK;
}

double or_strain_energy(const or_network* net, const or_law* law, const double* u) {
  /* relax.cpp:57-72 */
  const double* ref = net->packed_ref;
  double e = 0;
  for (int f = 0; f < net->n_fibers; ++f) {
    const int32_t* p = net->fiber_dofs + 6 * f;
    const double dx = (ref[p[3]] + u[p[3]]) - (ref[p[0]] + u[p[0]]);
    const double dy = (ref[p[4]] + u[p[4]]) - (ref[p[1]] + u[p[1]]);
    const double dz = (ref[p[5]] + u[p[5]]) - (ref[p[2]] + u[p[2]]);
    const double len = sqrt(dx * dx + dy * dy + dz * dz);
    const double l0 = net->rest_length[f];
    e += law_energy(law, net->area[f] * net->modulus[f], len / l0, l0);
  }
  return e;
}

double or_orientation_p2(const or_network* net, const double* u, const double ref_dir[3]) {
  /* network.cpp:398-415, same expression order */
  const double* ref = net->packed_ref;
  double wsum = 0, acc = 0;
  for (int f = 0; f < net->n_fibers; ++f) {
    const int32_t* p = net->fiber_dofs + 6 * f;
    const double d0 = (ref[p[3]] + u[p[3]]) - (ref[p[0]] + u[p[0]]);
    const double d1 = (ref[p[4]] + u[p[4]]) - (ref[p[1]] + u[p[1]]);
    const double d2 = (ref[p[5]] + u[p[5]]) - (ref[p[2]] + u[p[2]]);
    const double len = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (!(len > 0)) continue;
    const double c = (d0 * ref_dir[0] + d1 * ref_dir[1] + d2 * ref_dir[2]) / len;
    acc += len * 0.5 * (3.0 * c * c - 1.0);
    wsum += len;
  }
  return wsum > 0 ? acc / wsum : 0.0;
}

int or_homogenized_stress(const or_network* net, const or_state* st, const double F[9],
                          double sigma[6], double* asym_out) {
  /* network.cpp:341-372 */
  if (!st->converged || !*st->converged) return OR_NOT_CONVERGED_STATE;
  const double h = net->box_half;
  const double vol = or_det(F) * (8.0 * h * h * h);
  const double* ref = net->packed_ref;
  double s[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  for (int b = 0; b < net->n_boundary; ++b) {
    const int node = net->boundary_nodes[b];
    double r[3], x[3];
    for (int k = 0; k < 3; ++k) {
      const int p = net->packed_of_dof[3 * node + k];
      r[k] = st->f_int[p];
      x[k] = ref[p] + st->u[p];
    }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) s[i][j] += r[i] * x[j];
  }
  double raw[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) raw[3 * i + j] = s[i][j] / vol;
  double asym = 0, mag = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      asym += (raw[3 * i + j] - raw[3 * j + i]) * (raw[3 * i + j] - raw[3 * j + i]);
      mag += raw[3 * i + j] * raw[3 * i + j];
    }
  or_sym_from_full(raw, sigma);
  *asym_out = mag > 0 ? sqrt(asym / mag) : 0.0;
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* relax_solve  relax.cpp:93-191                                              */
/* ------------------------------------------------------------------------- */
static int relax_validate(const or_relax_cfg* c) { /* relax.cpp:12-19 */
  if (!(c->damping >= 0)) return OR_CONFIG;
  if (!(c->tolerance > 0)) return OR_CONFIG;
  if (c->max_iterations < 1) return OR_CONFIG;
  if (!(c->dt_safety > 0) || c->dt_safety > 1) return OR_CONFIG;
  if (!(c->density_scale > 0)) return OR_CONFIG;
  return OR_OK;
}

int or_relax_solve(const or_network* net, const or_law* law, const double F[9],
                   const or_relax_cfg* cfg, or_state st, int warm_reuse,
                   or_relax_report* rep) {
  memset(rep, 0, sizeof *rep);
  int rc = relax_validate(cfg);
  if (rc) return rc;
  if ((rc = law_validate(law))) return rc;
  const int n_dof = st.n_dof, n_free = st.n_free;
  if (n_dof != 3 * net->n_nodes || n_free != net->n_free) return OR_CONFIG;

  /* setup_mass relax.cpp:25-44 */
  double max_lump = 0;
  for (int i = 0; i < net->n_nodes; ++i) {
    if (!(net->node_lump[i] > 0)) return OR_CONFIG;
    max_lump = smax(max_lump, net->node_lump[i]);
  }
  const double scale = cfg->density_scale / max_lump;
  for (int i = 0; i < net->n_nodes; ++i) {
    const double m = net->node_lump[i] * scale;
    for (int k = 0; k < 3; ++k) {
      const int p = net->packed_of_dof[3 * i + k];
      st.mass[p] = m;
      st.inv_mass[p] = 1.0 / m;
    }
  }
  if (!warm_reuse)                                       /* relax.cpp:104-105 */
    for (int i = 0; i < n_free; ++i) st.u[i] = 0.0;
  for (int i = 0; i < n_dof; ++i) st.v[i] = st.a[i] = st.f_damp[i] = 0.0; /* :106-108 */
  if ((rc = or_apply_affine_bc(net, F, st))) return rc;   /* :109 */

  double* mred = malloc(sizeof(double) * (net->n_fibers ? net->n_fibers : 1)); /* :46-55 */
  for (int f = 0; f < net->n_fibers; ++f) {
    const double ma = st.mass[net->fiber_dofs[6 * f]];
    const double mb = st.mass[net->fiber_dofs[6 * f + 3]];
    mred[f] = ma * mb / (ma + mb) * net->rest_length[f];
  }
  const double force_floor = law->ea_scale * net->max_ea * 1e-12; /* :112 */
  double* u = st.u;
  double* v = st.v;
  double* a = st.a;
  double* fi = st.f_int;
  double* fdmp = st.f_damp;
  const int64_t nf = n_free, nfix = n_dof - n_free;
  const double c = cfg->damping;

  double min_dtsq = 0;
  if ((rc = or_internal_forces_cfl(net, law, u, fi, mred, &min_dtsq))) { free(mred); return rc; }
  double residual = sqrt(or_norm2_sq(nf, fi));
  double react = sqrt(or_norm2_sq(nfix, fi + n_free));
  double eps_eff = cfg->tolerance * smax(react, force_floor);
  rep->eps_eff = eps_eff;
  rep->residual = residual;
  if (residual <= eps_eff) {                             /* :138-143 */
    rep->converged = 1;
    if (st.converged) *st.converged = 1;
    rep->kinetic_fraction = 0.0;
    free(mred);
    return OR_OK;
  }
  for (int64_t i = 0; i < nf; ++i) {                     /* accel :145 */
    const double d = c * st.mass[i] * v[i];
    fdmp[i] = d;
    a[i] = -(fi[i] + d) * st.inv_mass[i];
  }
  int64_t n = 0;
  while (n < cfg->max_iterations) {                      /* hot loop :148-179 */
    ++n;
    const double dt = cfg->dt_safety * sqrt(min_dtsq);
    if (!isfinite(dt) || !(dt > 0)) { free(mred); return OR_BAD_DT; }
    if (st.t) *st.t += dt;
    const double hdt = 0.5 * dt;
    for (int64_t i = 0; i < nf; ++i) v[i] += hdt * a[i];
    for (int64_t i = 0; i < nf; ++i) u[i] += dt * v[i];
    if ((rc = or_internal_forces_cfl(net, law, u, fi, mred, &min_dtsq))) { free(mred); return rc; }
    residual = sqrt(or_norm2_sq(nf, fi));
    if (!isfinite(residual)) { free(mred); return OR_DIVERGED; }
    react = sqrt(or_norm2_sq(nfix, fi + n_free));
    eps_eff = cfg->tolerance * smax(react, force_floor);
    for (int64_t i = 0; i < nf; ++i) {
      const double d = c * st.mass[i] * v[i];
      fdmp[i] = d;
      a[i] = -(fi[i] + d) * st.inv_mass[i];
    }
    for (int64_t i = 0; i < nf; ++i) v[i] += hdt * a[i];
    rep->dt = dt;
    if (residual <= eps_eff) {
      rep->converged = 1;
      break;
    }
  }
  rep->iterations = n;                                   /* exit :181-190 */
  rep->residual = residual;
  rep->eps_eff = eps_eff;
  rep->energy_drift = 0;
  const double ke = 0.5 * or_weighted_sq(nf, st.mass, v);
  const double se = or_strain_energy(net, law, u);
  rep->kinetic_fraction = (ke + se) > 0 ? ke / (ke + se) : 0.0;
  if (st.iters) *st.iters += n;
  if (st.converged) *st.converged = rep->converged ? 1 : 0;
  free(mred);
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* constitutive_response  stiffness.cpp:66-175                                 */
/* ------------------------------------------------------------------------- */
int or_constitutive_response(const or_network* net, const or_law* law, const double F[9],
                             const or_relax_cfg* rcfg, double fd_rel_step, int reuse_warm,
                             int want_tangent, or_state st, or_response* out) {
  memset(out, 0, sizeof *out);
  out->failed_probe = -1;
  if (!(fd_rel_step > 0) || fd_rel_step >= 1e-2) return OR_CONFIG; /* :10-13 */
  /* solve_base :66-83 */
  double R[9], U[6], fu[9];
  int rc = or_polar_decompose(F, R, U);
  if (rc) return rc;
  or_sym_full(U, fu);
  or_relax_report rep;
  rc = or_relax_solve(net, law, fu, rcfg, st, 1, &rep);
  if (rc) return rc;
  if (!rep.converged) return OR_NOT_CONVERGED;
  double sigma_u[6], asym, pk2[6];
  if ((rc = or_homogenized_stress(net, &st, fu, sigma_u, &asym))) return rc;
  if ((rc = or_pull_back_stress(sigma_u, fu, pk2))) return rc;
  out->solves = 1;
  out->relax_iterations = rep.iterations;
  out->base_report = rep;
  memcpy(out->pk2, pk2, sizeof pk2);
  out->stress_asymmetry = asym;

  if (want_tangent) {
    const double h = fd_rel_step * sym_frobenius(U); /* probe_step :125-127 */
    const int nd = st.n_dof;
    double* buf = calloc((size_t)7 * nd, sizeof(double));
    double tsc = 0;
    int64_t isc = 0;
    uint8_t csc = 0;
    or_state sc = {buf, buf + nd, buf + 2 * nd, buf + 3 * nd, buf + 4 * nd, buf + 5 * nd,
                   buf + 6 * nd, &tsc, &isc, &csc, st.n_free, nd};
    double probes[36];
    for (int q = 0; q < 6; ++q) { /* probe_pk2s :86-123 */
      double dir[6], up[6], fq[9];
      or_probing_direction(q, dir);
      for (int i = 0; i < 6; ++i) up[i] = U[i] + dir[i] * h;
      or_sym_full(up, fq);
      if (!(or_det(fq) > 0)) { free(buf); return OR_PROBE_FAILED; }
      if (reuse_warm) memcpy(sc.u, st.u, sizeof(double) * nd);
      or_relax_report pr;
      rc = or_relax_solve(net, law, fq, rcfg, sc, reuse_warm, &pr);
      if (rc) {
        out->failed_probe = q;
        free(buf);
        return rc == OR_CONFIG ? rc : OR_PROBE_FAILED;
      }
      ++out->solves;
      out->relax_iterations += pr.iterations;
      if (!pr.converged) { out->failed_probe = q; free(buf); return OR_PROBE_FAILED; }
      double sq[6], aq;
      if ((rc = or_homogenized_stress(net, &sc, fq, sq, &aq))) { free(buf); return rc; }
      if ((rc = or_pull_back_stress(sq, fq, probes + 6 * q))) { free(buf); return rc; }
    }
    free(buf);
    if ((rc = or_material_stiffness_from_probes(U, pk2, probes, h, out->material_a))) return rc;
    if ((rc = or_push_forward_stiffness(out->material_a, F, out->spatial_c))) return rc;
  }
  double su[9], rt[9], t1[9], s9[9];
  or_sym_full(sigma_u, su);
  transpose3(R, rt);
  or_matmul(R, su, t1);
  or_matmul(t1, rt, s9);
  or_sym_from_full(s9, out->sigma);
  return OR_OK;
}

/* ------------------------------------------------------------------------- */
/* batch_response  batch.cpp:155-187                                          */
/* ------------------------------------------------------------------------- */
typedef struct {
  const or_network* const* entries;
  const int32_t* entry_of_point;
  int n_points;
  const int64_t* offsets;
  double *u, *v, *a, *f_int, *f_damp, *mass, *inv_mass, *t;
  int64_t* iters;
  uint8_t* converged;
  const int32_t* n_free;
  const or_law* law;
  const double* F;
  const or_relax_cfg* rcfg;
  double fd;
  int reuse, tangent;
  or_response* out;
  int32_t* status;
  int next;
  int config_error;
  pthread_mutex_t mu;
} batch_job;

static void solve_point(batch_job* j, int p) {
  const or_network* net = j->entries[j->entry_of_point[p]];
  const int64_t lo = j->offsets[p];
  const int nd = (int)(j->offsets[p + 1] - lo);
  or_state st = {j->u + lo, j->v + lo, j->a + lo, j->f_int + lo, j->f_damp + lo,
                 j->mass + lo, j->inv_mass + lo, j->t + p, j->iters + p, j->converged + p,
                 j->n_free[p], nd};
  or_response r;
  const int rc = or_constitutive_response(net, j->law, j->F + 9 * p, j->rcfg, j->fd, j->reuse,
                                          j->tangent, st, &r);
  if (rc == OR_CONFIG) {
    pthread_mutex_lock(&j->mu);
    j->config_error = 1;
    pthread_mutex_unlock(&j->mu);
  }
  if (rc) {
    memset(&j->out[p], 0, sizeof(or_response)); /* value-initialized slot */
    j->out[p].failed_probe = -1;
  } else {
    j->out[p] = r;
  }
  j->status[p] = rc;
}

static void* batch_worker(void* arg) {
  batch_job* j = arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    const int p = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (p >= j->n_points) return NULL;
    solve_point(j, p);
  }
}

int or_batch_response(const or_network* const* entries, const int32_t* entry_of_point,
                      int n_points, const int64_t* offsets, double* u, double* v, double* a,
                      double* f_int, double* f_damp, double* mass, double* inv_mass, double* t,
                      int64_t* iters, uint8_t* converged, const int32_t* n_free,
                      const or_law* law, const double* F, const or_relax_cfg* rcfg,
                      double fd_rel_step, int reuse_warm, int want_tangent, int n_threads,
                      or_response* out, int32_t* status) {
  batch_job j = {entries, entry_of_point, n_points, offsets, u, v, a, f_int, f_damp, mass,
                 inv_mass, t, iters, converged, n_free, law, F, rcfg, fd_rel_step, reuse_warm,
                 want_tangent, out, status, 0, 0};
  pthread_mutex_init(&j.mu, NULL);
  if (n_threads <= 1) {
    for (int p = 0; p < n_points; ++p) solve_point(&j, p);
  } else {
    pthread_t* th = malloc(sizeof(pthread_t) * n_threads);
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, batch_worker, &j);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  pthread_mutex_destroy(&j.mu);
  return j.config_error ? OR_CONFIG : OR_OK;
}

/* ------------------------------------------------------------------------- */
/* Macro assembly  macrofem.cpp:41-60 (b_matrix), :64-86 (mandel_b),          */
/* :104-187 (assemble).  The 3x3 determinant / inverse are Eigen's fixed-size */
/* paths (Eigen is absent here: restated from Eigen 3.4 Determinant.h         */
/* determinant_impl<3> and InverseImpl.h compute_inverse<3>), and the         */
/* SparseMatrix::setFromTriplets duplicate folding (SparseMatrix.h             */
/* set_from_triplets: first value, then acc = acc + next in triplet order,     */
/* transposed copy sorts rows within each column).                            */
/* ------------------------------------------------------------------------- */
static inline double eig_cof3(const double* m, int i, int j) { /* InverseImpl.h cofactor_3x3 */
  const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
  return m[3 * i1 + j1] * m[3 * i2 + j2] - m[3 * i1 + j2] * m[3 * i2 + j1];
}

/* b_matrix (macrofem.cpp:41-60): grad[4][3], volume; OR_KINEMATICS on det <= 0 */
int or_tet_geom(const double* coords, const int32_t n[4], double grad[12], double* volume) {
  double jac[9]; /* row-major; columns are edge vectors (:43-47) */
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) jac[3 * r + c] = coords[3 * n[c + 1] + r] - coords[3 * n[0] + r];
  /* Eigen determinant_impl<3>: bruteforce_det3_helper(m,0,1,2) - (m,1,0,2) + (m,2,0,1) */
  const double det = jac[0] * (jac[4] * jac[8] - jac[5] * jac[7]) -
                     jac[1] * (jac[3] * jac[8] - jac[5] * jac[6]) +
                     jac[2] * (jac[3] * jac[7] - jac[4] * jac[6]);
  if (!(det > 0)) return OR_KINEMATICS;
  /* Eigen compute_inverse<3>: cofactors of column 0, det as (c0*m00 + c1*m10) + c2*m20 */
  const double c0 = eig_cof3(jac, 0, 0), c1 = eig_cof3(jac, 1, 0), c2 = eig_cof3(jac, 2, 0);
  const double idet = 1.0 / ((c0 * jac[0] + c1 * jac[3]) + c2 * jac[6]);
  double inv[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) inv[3 * r + c] = eig_cof3(jac, c, r) * idet;
  *volume = det / 6.0;
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 3; ++k) grad[3 * (a + 1) + k] = inv[3 * a + k];
  for (int k = 0; k < 3; ++k) grad[k] = -grad[3 + k] - grad[6 + k] - grad[9 + k];
  return OR_OK;
}

/* mandel_b (macrofem.cpp:64-86): b[6][12] accumulated onto zeros */
void or_mandel_b(const double grad[12], double b[72]) {
  static const int pair[3][2] = {{1, 2}, {0, 2}, {0, 1}};
  for (int i = 0; i < 72; ++i) b[i] = 0;
  for (int node = 0; node < 4; ++node) {
    const double* gn = grad + 3 * node;
    for (int ax = 0; ax < 3; ++ax) {
      const int col = 3 * node + ax;
      b[12 * ax + col] += gn[ax];
      for (int sh = 0; sh < 3; ++sh) {
        const int i = pair[sh][0], j = pair[sh][1];
        double v = 0;
        if (ax == i) v += 0.5 * gn[j];
        if (ax == j) v += 0.5 * gn[i];
        b[12 * (3 + sh) + col] += kSqrt2 * v;
      }
    }
  }
}

/* per-element work of assemble (macrofem.cpp:118-167): fe[12], ke[144] (row-major) */
int or_element_matrices(const double* coords, const int32_t n[4], const double sigma[6],
                        const double c66[36], double fe[12], double ke[144]) {
  double sig[6], grad[12], vol, b[72], cb[72], sf[9];
  or_mandel(sigma, sig);
  for (int i = 0; i < 6; ++i)
    if (!isfinite(sig[i])) return OR_ASM_STRESS; /* :122-125 */
  if (or_tet_geom(coords, n, grad, &vol)) return OR_KINEMATICS; /* :128-132 */
  or_mandel_b(grad, b);
  for (int c = 0; c < 12; ++c) { /* :137-142 */
    double s = 0;
    for (int p = 0; p < 6; ++p) s += b[12 * p + c] * sig[p];
    fe[c] = vol * s;
  }
  for (int p = 0; p < 6; ++p) /* :145-150 */
    for (int c = 0; c < 12; ++c) {
      double s = 0;
      for (int q = 0; q < 6; ++q) s += c66[6 * p + q] * b[12 * q + c];
      cb[12 * p + c] = s;
    }
  for (int r = 0; r < 12; ++r) /* :151-157 */
    for (int c = 0; c < 12; ++c) {
      double s = 0;
      for (int p = 0; p < 6; ++p) s += b[12 * p + r] * cb[12 * p + c];
      ke[12 * r + c] = vol * s;
    }
  or_sym_full(sigma, sf); /* :160-168 geometric part */
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) {
      double gsg = 0;
      for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) gsg += grad[3 * i + p] * sf[3 * p + q] * grad[3 * j + q];
      gsg *= vol;
      for (int ax = 0; ax < 3; ++ax) ke[12 * (3 * i + ax) + 3 * j + ax] += gsg;
    }
  return OR_OK;
}

typedef struct { int32_t r, c; int64_t ord; double v; } or_trip;

static int trip_cmp(const void* x, const void* y) { /* (col, row, triplet order) */
  const or_trip* a = (const or_trip*)x;
  const or_trip* b = (const or_trip*)y;
  if (a->c != b->c) return a->c < b->c ? -1 : 1;
  if (a->r != b->r) return a->r < b->r ? -1 : 1;
  return a->ord < b->ord ? -1 : (a->ord > b->ord);
}

/* assemble (macrofem.cpp:104-187).  tets[4 n_tets], coords[3 n_nodes] (current),
 * sigma[6 n_tets] (SymTensor3), c66[36 n_tets] (Mandel66 row-major), free_of_dof[3 n_nodes],
 * f_ext[n_free] (NULL = zero).  Out: residual[n_free]; the compressed column-major matrix
 * (col_ptr[n_free+1], row_idx/values with capacity cap >= 144 n_tets), *nnz.
 * On an element error *bad_element = the first failing element (element order). */
int or_assemble(const int32_t* tets, int32_t n_tets, const double* coords,
                const double* sigma, const double* c66, const int32_t* free_of_dof,
                int32_t n_free, const double* f_ext, double* residual, int64_t* col_ptr,
                int32_t* row_idx, double* values, int64_t cap, int64_t* nnz,
                int32_t* bad_element) {
  or_trip* trips = (or_trip*)malloc(sizeof(or_trip) * (size_t)(144 * (int64_t)n_tets + 1));
  if (!trips) return OR_CONFIG;
  int64_t nt = 0;
  *bad_element = -1;
  for (int32_t i = 0; i < n_free; ++i) residual[i] = 0.0; /* VectorXd::Zero */
  for (int32_t e = 0; e < n_tets; ++e) {
    const int32_t* n = tets + 4 * e;
    double fe[12], ke[144];
    const int rc = or_element_matrices(coords, n, sigma + 6 * e, c66 + 36 * e, fe, ke);
    if (rc) {
      *bad_element = e;
      free(trips);
      return rc;
    }
    for (int a = 0; a < 4; ++a) /* :170-183 */
      for (int ax = 0; ax < 3; ++ax) {
        const int32_t rf = free_of_dof[3 * n[a] + ax];
        if (rf < 0) continue;
        residual[rf] += fe[3 * a + ax];
        for (int bn = 0; bn < 4; ++bn)
          for (int bx = 0; bx < 3; ++bx) {
            const int32_t cf = free_of_dof[3 * n[bn] + bx];
            if (cf < 0) continue;
            trips[nt].r = rf;
            trips[nt].c = cf;
            trips[nt].ord = nt;
            trips[nt].v = ke[12 * (3 * a + ax) + 3 * bn + bx];
            ++nt;
          }
      }
  }
  for (int32_t i = 0; i < n_free; ++i) residual[i] -= f_ext ? f_ext[i] : 0.0; /* :185 */
  qsort(trips, (size_t)nt, sizeof(or_trip), trip_cmp);
  int64_t k = -1;
  for (int32_t c = 0; c <= n_free; ++c) col_ptr[c] = 0;
  for (int64_t t = 0; t < nt; ++t) {
    if (k >= 0 && trips[t].r == row_idx[k] && trips[t].c == trips[t - 1].c) {
      values[k] = values[k] + trips[t].v; /* collapseDuplicates: scalar_sum_op */
      continue;
    }
    if (++k >= cap) {
      free(trips);
      return OR_CONFIG;
    }
    row_idx[k] = trips[t].r;
    values[k] = trips[t].v;
    col_ptr[trips[t].c + 1]++;
  }
  *nnz = k + 1;
  for (int32_t c = 0; c < n_free; ++c) col_ptr[c + 1] += col_ptr[c];
  free(trips);
  for (int32_t i = 0; i < n_free; ++i)
    if (!isfinite(residual[i])) return OR_ASM_RESIDUAL; /* :186-187 */
  return OR_OK;
}

/* The host libm's exp / expm1 (what the reference's FiberLaw calls, network.cpp:16-53) over
 * an array: the checker of the device restatement (csrc/libm_glibc.cuh). */
void or_libm(int which, const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = which ? expm1(x[i]) : exp(x[i]);
}
