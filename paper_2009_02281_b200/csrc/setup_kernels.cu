// Device-side static setup of AIMx (S0), all in fp64 on the B200:
//   * per-RWG triangle geometry,
//   * projection weights Lambda (moment matching == Lagrange interpolation,
//     P:109-110) by collapsed Gauss-Legendre quadrature (exact for the
//     polynomial integrand),
//   * static near-region entries L_s,NR with G_s = 1/(4 pi r) (eq:Lmatdecomp2
//     P:267, change (a) P:297): analytic inner potential integrals, 7-point
//     outer rule, symmetrised (reading R9),
//   * precorrection L_s,P = W H_s,NR P (eq:aimLPs P:276) with H_s(0) = 0
//     (eq:Hsmm P:321), and C = L_s,NR - L_s,P,
//   * the linear-term modification's C_lin = L_lin - W H_lin P on overlapping
//     pairs (analytic inner integrals of R and (rho' - rho) R).
// The paper's own static fill is its "one-time static matrix-fill" (tab:prof
// P:715); here it runs once per context on the GPU.
#include <cmath>
#include <vector>

#include "aimx_internal.h"

namespace aimx {

namespace {

__constant__ double c_gl_x[8];
__constant__ double c_gl_w[8];
__constant__ double c_hs_tab[512];   // 1/(4 pi h sqrt(q)), q = |delta|^2; [0] = 0

// 7-point degree-5 rule (barycentric weights of v0, v1, v2; weights sum to 1)
__device__ __forceinline__ void radon7(int q, double& b0, double& b1, double& b2, double& w) {
  const double s15 = 3.872983346207417;  // sqrt(15)
  const double a1 = (6.0 - s15) / 21.0, a2 = (6.0 + s15) / 21.0;
  const double w1 = (155.0 - s15) / 1200.0, w2 = (155.0 + s15) / 1200.0;
  switch (q) {
    case 0: b0 = 1.0 / 3.0; b1 = 1.0 / 3.0; b2 = 1.0 / 3.0; w = 9.0 / 40.0; break;
    case 1: b0 = a1; b1 = a1; b2 = 1.0 - 2.0 * a1; w = w1; break;
    case 2: b0 = a1; b1 = 1.0 - 2.0 * a1; b2 = a1; w = w1; break;
    case 3: b0 = 1.0 - 2.0 * a1; b1 = a1; b2 = a1; w = w1; break;
    case 4: b0 = a2; b1 = a2; b2 = 1.0 - 2.0 * a2; w = w2; break;
    case 5: b0 = a2; b1 = 1.0 - 2.0 * a2; b2 = a2; w = w2; break;
    default: b0 = 1.0 - 2.0 * a2; b1 = a2; b2 = a2; w = w2; break;
  }
}

struct Vec3 { double x, y, z; };
__device__ __forceinline__ Vec3 v3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ Vec3 operator+(Vec3 a, Vec3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ Vec3 operator-(Vec3 a, Vec3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ Vec3 operator*(double s, Vec3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(Vec3 a, Vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ Vec3 cross(Vec3 a, Vec3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(Vec3 a) { return sqrt(dot(a, a)); }

// side record: v0 v1 v2 free (12), coef = sigma l/(2A), div = sigma l/A, area
__global__ void k_rwg_sides(int nb, const double* __restrict__ V, const int32_t* __restrict__ T,
                            const int32_t* __restrict__ ea, const int32_t* __restrict__ eb,
                            const int32_t* __restrict__ tp, const int32_t* __restrict__ tm,
                            const int32_t* __restrict__ pp, const int32_t* __restrict__ pm,
                            double* __restrict__ side) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 2 * (int64_t)nb) return;
  int e = (int)(i >> 1), sd = (int)(i & 1);
  int tri = sd ? tm[e] : tp[e];
  int fv = sd ? pm[e] : pp[e];
  double* o = side + i * kSideStride;
  Vec3 a = v3(V + 3 * (int64_t)T[3 * tri]), b = v3(V + 3 * (int64_t)T[3 * tri + 1]),
       c = v3(V + 3 * (int64_t)T[3 * tri + 2]);
  Vec3 f = v3(V + 3 * (int64_t)fv);
  double area = 0.5 * norm(cross(b - a, c - a));
  double len = norm(v3(V + 3 * (int64_t)eb[e]) - v3(V + 3 * (int64_t)ea[e]));
  double sg = sd ? -1.0 : 1.0;
  o[0] = a.x; o[1] = a.y; o[2] = a.z;
  o[3] = b.x; o[4] = b.y; o[5] = b.z;
  o[6] = c.x; o[7] = c.y; o[8] = c.z;
  o[9] = f.x; o[10] = f.y; o[11] = f.z;
  o[12] = sg * len / (2.0 * area);
  o[13] = sg * len / area;
  o[14] = area;
  o[15] = 0.0;
}

// Lagrange basis on nodes t = 0..n
__device__ __forceinline__ double lagrange(int order, int i, double t) {
  double v = 1.0;
  for (int j = 0; j <= order; ++j)
    if (j != i) v *= (t - (double)j) / (double)(i - j);
  return v;
}

// Thread per (rwg, slot s): Lambda^c_s = int f_c l_i l_j l_k dS, Lambda^rho_s = int div f (...)
__global__ void k_weights(int nb, int order, int q, const double* __restrict__ side,
                          const int32_t* __restrict__ anchor, double ox, double oy, double oz,
                          double h, double* __restrict__ lam, uint8_t* __restrict__ nzflag) {
  const int p = order + 1, p3 = p * p * p;
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nb * p3) return;
  int e = (int)(idx / p3), s = (int)(idx % p3);
  int si = s % p, sj = (s / p) % p, sk = s / (p * p);
  double Ax = anchor[3 * e], Ay = anchor[3 * e + 1], Az = anchor[3 * e + 2];
  double acc[4] = {0, 0, 0, 0};
  for (int sd = 0; sd < 2; ++sd) {
    const double* o = side + (2 * (int64_t)e + sd) * kSideStride;
    Vec3 a = v3(o), b = v3(o + 3), c = v3(o + 6), f = v3(o + 9);
    double coef = o[12], dv = o[13], area = o[14];
    double sx = 0, sy = 0, sz = 0, sr = 0;
    for (int iu = 0; iu < q; ++iu) {
      double u = c_gl_x[iu];
      for (int iv = 0; iv < q; ++iv) {
        double v = c_gl_x[iv];
        double l1 = u, l2 = v * (1.0 - u);
        double w = c_gl_w[iu] * c_gl_w[iv] * (1.0 - u) * 2.0;   // sums to 1 over the triangle
        Vec3 r = a + l1 * (b - a) + l2 * (c - a);
        double tx = (r.x - ox) / h - Ax, ty = (r.y - oy) / h - Ay, tz = (r.z - oz) / h - Az;
        double L = lagrange(order, si, tx) * lagrange(order, sj, ty) * lagrange(order, sk, tz) * w;
        sx += L * (r.x - f.x);
        sy += L * (r.y - f.y);
        sz += L * (r.z - f.z);
        sr += L;
      }
    }
    acc[0] += area * coef * sx;
    acc[1] += area * coef * sy;
    acc[2] += area * coef * sz;
    acc[3] += area * dv * sr;
  }
  double* out = lam + ((int64_t)e * p3 + s) * 4;
  out[0] = acc[0]; out[1] = acc[1]; out[2] = acc[2]; out[3] = acc[3];
  nzflag[idx] = (acc[0] != 0.0 || acc[1] != 0.0 || acc[2] != 0.0 || acc[3] != 0.0) ? 1 : 0;
}

// ln(R + s) without cancellation (s < 0: R + s = R0^2 / (R - s))
__device__ __forceinline__ double logsum(double R, double s, double R0sq) {
  return s >= 0.0 ? log(R + s) : log(R0sq / (R - s));
}

struct Frame {
  Vec3 v[3];
  Vec3 n;
  Vec3 sh[3], mh[3];
  double L[3];
};

__device__ __forceinline__ void make_frame(const double* o, Frame& F) {
  F.v[0] = v3(o); F.v[1] = v3(o + 3); F.v[2] = v3(o + 6);
  Vec3 nn = cross(F.v[1] - F.v[0], F.v[2] - F.v[0]);
  F.n = (1.0 / norm(nn)) * nn;
  for (int k = 0; k < 3; ++k) {
    Vec3 ev = F.v[(k + 1) % 3] - F.v[k];
    F.L[k] = norm(ev);
    F.sh[k] = (1.0 / F.L[k]) * ev;
    F.mh[k] = cross(F.sh[k], F.n);
  }
}

// Closed-form I0 = int 1/R dS', I1 = int (rho' - rho)/R dS' over the flat source
// triangle (Wilton et al. / Graglia form); same guards as the oracle's recipe.
__device__ __forceinline__ void potentials(const Frame& F, Vec3 r, double& I0, Vec3& I1, Vec3& rho) {
  double d = dot(r - F.v[0], F.n);
  rho = r - d * F.n;
  double ad = fabs(d);
  I0 = 0.0;
  I1 = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k) {
    Vec3 va = F.v[k], vb = F.v[(k + 1) % 3];
    double sm = dot(va - rho, F.sh[k]);
    double sp = dot(vb - rho, F.sh[k]);
    double t0 = dot(va - rho, F.mh[k]);
    double R0sq = t0 * t0 + d * d;
    double Rm = norm(r - va), Rp = norm(r - vb);
    double lim = 1e-14 * F.L[k];
    double f2 = 0.0;
    if (R0sq > lim * lim) f2 = logsum(Rp, sp, R0sq) - logsum(Rm, sm, R0sq);
    double beta = 0.0;
    if (ad > 0.0) beta = atan(t0 * sp / (R0sq + ad * Rp)) - atan(t0 * sm / (R0sq + ad * Rm));
    I0 += t0 * f2 - ad * beta;
    double g = 0.5 * (R0sq * f2 + sp * Rp - sm * Rm);
    I1 = I1 + g * F.mh[k];
  }
}

// Warp per row m; lanes over the row's entries: unsymmetrised static entries,
// outer integral over m's triangles, inner (analytic) over n's triangles.
__global__ void k_static_near(int nb, const int64_t* __restrict__ rowptr,
                              const int32_t* __restrict__ col, const double* __restrict__ side,
                              double* __restrict__ LA, double* __restrict__ YR) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp >= nb) return;
  const int m = (int)warp;
  const double inv4pi = 1.0 / (4.0 * kPi);
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const int n = col[k];
    double la = 0.0, yr = 0.0;
    for (int sm = 0; sm < 2; ++sm) {
      const double* om = side + (2 * (int64_t)m + sm) * kSideStride;
      Vec3 a = v3(om), b = v3(om + 3), c = v3(om + 6), pm = v3(om + 9);
      double coef_m = om[12], div_m = om[13], area_m = om[14];
      for (int sn = 0; sn < 2; ++sn) {
        const double* on = side + (2 * (int64_t)n + sn) * kSideStride;
        Frame F;
        make_frame(on, F);
        Vec3 pn = v3(on + 9);
        double coef_n = on[12], div_n = on[13];
        double sA = 0.0, sR = 0.0;
        for (int q = 0; q < 7; ++q) {
          double b0, b1, b2, w;
          radon7(q, b0, b1, b2, w);
          Vec3 r = b0 * a + b1 * b + b2 * c;
          double I0;
          Vec3 I1, rho;
          potentials(F, r, I0, I1, rho);
          Vec3 inner = coef_n * (I1 + I0 * (rho - pn));
          Vec3 fm = coef_m * (r - pm);
          sA += w * area_m * dot(fm, inner);
          sR += w * area_m * I0;
        }
        la += sA * inv4pi;
        yr += div_m * div_n * sR * inv4pi;
      }
    }
    LA[k] = la;
    YR[k] = yr;
  }
}

// Warp per row m: symmetrise (L + L^T)/2 via the transposed position, then the
// precorrection L_s,P[m,n] = sum_c Lambda^c_m^T B_D Lambda^c_n, B_D[s,s'] =
// H_s(s - s' - D), D = A_n - A_m, and C = L_s,NR - L_s,P.
__global__ void k_precorrect(int nb, int order, const int64_t* __restrict__ rowptr,
                             const int32_t* __restrict__ col, const int32_t* __restrict__ anchor,
                             const double* __restrict__ lam, const double* __restrict__ LAun,
                             const double* __restrict__ YRun, double* __restrict__ LA_NR,
                             double* __restrict__ YR_NR, double* __restrict__ LA_P,
                             double* __restrict__ YR_P, double* __restrict__ CA,
                             double* __restrict__ CR) {
  extern __shared__ double sh[];
  const int p = order + 1, p3 = p * p * p;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  double* hs_tab = sh;   // H_s table in shared memory (lanes read different offsets)
  for (int t = threadIdx.x; t < 512; t += blockDim.x) hs_tab[t] = c_hs_tab[t];
  double* lm = sh + 512 + wib * (p3 * 4);
  const bool active = warp < nb;
  const int m = active ? (int)warp : 0;
  for (int t = lane; t < p3 * 4; t += 32) lm[t] = active ? lam[(int64_t)m * p3 * 4 + t] : 0.0;
  __syncthreads();
  if (!active) return;
  const int Amx = anchor[3 * m], Amy = anchor[3 * m + 1], Amz = anchor[3 * m + 2];
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const int n = col[k];
    // transposed position: column m inside row n (columns ascending)
    int64_t lo = rowptr[n], hi = rowptr[n + 1] - 1;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (col[mid] < m) lo = mid + 1; else hi = mid;
    }
    const int64_t kt = lo;
    const double la_nr = 0.5 * (LAun[k] + LAun[kt]);
    const double yr_nr = 0.5 * (YRun[k] + YRun[kt]);
    const int Dx = anchor[3 * n] - Amx, Dy = anchor[3 * n + 1] - Amy, Dz = anchor[3 * n + 2] - Amz;
    // per-axis squared offsets (i - i' - D)^2 for i - i' in [-n, n]
    int sqx[7], sqy[7], sqz[7];
    for (int d = -order; d <= order; ++d) {
      sqx[d + order] = (d - Dx) * (d - Dx);
      sqy[d + order] = (d - Dy) * (d - Dy);
      sqz[d + order] = (d - Dz) * (d - Dz);
    }
    const double* ln = lam + (int64_t)n * p3 * 4;
    double acc[4] = {0, 0, 0, 0};
    for (int s2 = 0; s2 < p3; ++s2) {
      const int i2 = s2 % p, j2 = (s2 / p) % p, k2 = s2 / (p * p);
      double u0 = 0, u1 = 0, u2 = 0, u3 = 0;
      for (int s1 = 0; s1 < p3; ++s1) {
        const int i1 = s1 % p, j1 = (s1 / p) % p, k1 = s1 / (p * p);
        const int qq = sqx[i1 - i2 + order] + sqy[j1 - j2 + order] + sqz[k1 - k2 + order];
        const double hs = hs_tab[qq];
        u0 += lm[s1 * 4 + 0] * hs;
        u1 += lm[s1 * 4 + 1] * hs;
        u2 += lm[s1 * 4 + 2] * hs;
        u3 += lm[s1 * 4 + 3] * hs;
      }
      acc[0] += u0 * ln[s2 * 4 + 0];
      acc[1] += u1 * ln[s2 * 4 + 1];
      acc[2] += u2 * ln[s2 * 4 + 2];
      acc[3] += u3 * ln[s2 * 4 + 3];
    }
    const double la_p = acc[0] + acc[1] + acc[2];
    const double yr_p = acc[3];
    LA_NR[k] = la_nr;
    YR_NR[k] = yr_nr;
    LA_P[k] = la_p;
    YR_P[k] = yr_p;
    CA[k] = la_nr - la_p;
    CR[k] = yr_nr - yr_p;
  }
}

// ---- linear-term modification: kernel G_lin = -R/(8 pi)
// Closed forms over the flat source triangle (surface divergence theorem in
// its plane, u = rho' - rho, R0^2 = t0^2 + d^2 per edge):
//   J0 = int R dS'   = (d^2 I0 + sum_k t0_k int_k R ds) / 3
//   J1 = int u R dS' = (1/3) sum_k m_k int_k R^3 ds
//   int R ds   = [s R + R0^2 ln(s + R)] / 2
//   int R^3 ds = s R^3 / 4 + 3 R0^2 s R / 8 + 3 R0^4 ln(s + R) / 8
__device__ __forceinline__ void r_potentials(const Frame& F, Vec3 r, double& J0, Vec3& J1, Vec3& rho) {
  double d = dot(r - F.v[0], F.n);
  rho = r - d * F.n;
  double ad = fabs(d);
  double I0 = 0.0, S = 0.0;
  J1 = {0.0, 0.0, 0.0};
  for (int k = 0; k < 3; ++k) {
    Vec3 va = F.v[k], vb = F.v[(k + 1) % 3];
    double sm = dot(va - rho, F.sh[k]);
    double sp = dot(vb - rho, F.sh[k]);
    double t0 = dot(va - rho, F.mh[k]);
    double R0sq = t0 * t0 + d * d;
    double Rm = norm(r - va), Rp = norm(r - vb);
    double lim = 1e-14 * F.L[k];
    double f2 = 0.0;
    if (R0sq > lim * lim) f2 = logsum(Rp, sp, R0sq) - logsum(Rm, sm, R0sq);
    double beta = 0.0;
    if (ad > 0.0) beta = atan(t0 * sp / (R0sq + ad * Rp)) - atan(t0 * sm / (R0sq + ad * Rm));
    I0 += t0 * f2 - ad * beta;
    double lin = sp * Rp - sm * Rm;
    S += t0 * 0.5 * (lin + R0sq * f2);
    double k3 = 0.25 * (sp * Rp * Rp * Rp - sm * Rm * Rm * Rm) + 0.375 * R0sq * lin + 0.375 * R0sq * R0sq * f2;
    J1 = J1 + k3 * F.mh[k];
  }
  J0 = (d * d * I0 + S) / 3.0;
  J1 = (1.0 / 3.0) * J1;
}

// Unsymmetrised (L^A_lin, y^rho_lin)[m, n]: outer 7-point rule on m, analytic inner on n.
__device__ void lin_pair(const double* __restrict__ side, int m, int n, double& la, double& yr) {
  la = 0.0;
  yr = 0.0;
  for (int sm = 0; sm < 2; ++sm) {
    const double* om = side + (2 * (int64_t)m + sm) * kSideStride;
    Vec3 a = v3(om), b = v3(om + 3), c = v3(om + 6), pm = v3(om + 9);
    double coef_m = om[12], div_m = om[13], area_m = om[14];
    for (int sn = 0; sn < 2; ++sn) {
      const double* on = side + (2 * (int64_t)n + sn) * kSideStride;
      Frame F;
      make_frame(on, F);
      Vec3 pn = v3(on + 9);
      double coef_n = on[12], div_n = on[13];
      double sA = 0.0, sR = 0.0;
      for (int q = 0; q < 7; ++q) {
        double b0, b1, b2, w;
        radon7(q, b0, b1, b2, w);
        Vec3 r = b0 * a + b1 * b + b2 * c;
        double J0;
        Vec3 J1, rho;
        r_potentials(F, r, J0, J1, rho);
        Vec3 inner = coef_n * (J1 + J0 * (rho - pn));
        Vec3 fm = coef_m * (r - pm);
        sA += w * area_m * dot(fm, inner);
        sR += w * area_m * J0;
      }
      la += sA;
      yr += div_m * div_n * sR;
    }
  }
  const double g = -1.0 / (8.0 * kPi);
  la *= g;
  yr *= g;
}

// Thread per (row m, overlap slot j): symmetrised L_lin entry minus the grid's
// share W H_lin P, H_lin(delta) = -h |delta| / (8 pi) (H_lin(0) = 0).
template <typename T2>
__global__ void k_lin_entries(int nb, int order, double h, const int32_t* __restrict__ cols,
                              const int32_t* __restrict__ anchor, const double* __restrict__ side,
                              const double* __restrict__ lam, T2* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)nb * kLinW) return;
  const int m = (int)(i / kLinW), n = cols[i];
  if (n < 0) {
    out[i] = T2{0, 0};
    return;
  }
  double la1, yr1, la2, yr2;
  lin_pair(side, m, n, la1, yr1);
  lin_pair(side, n, m, la2, yr2);
  const int p = order + 1, p3 = p * p * p;
  const int Dx = anchor[3 * n] - anchor[3 * m], Dy = anchor[3 * n + 1] - anchor[3 * m + 1],
            Dz = anchor[3 * n + 2] - anchor[3 * m + 2];
  const double* lm = lam + (int64_t)m * p3 * 4;
  const double* ln = lam + (int64_t)n * p3 * 4;
  const double g = -h / (8.0 * kPi);
  double pa = 0.0, pr = 0.0;
  for (int s2 = 0; s2 < p3; ++s2) {
    const int i2 = s2 % p, j2 = (s2 / p) % p, k2 = s2 / (p * p);
    double u0 = 0, u1 = 0, u2 = 0, u3 = 0;
    for (int s1 = 0; s1 < p3; ++s1) {
      const int dx = s1 % p - i2 - Dx, dy = (s1 / p) % p - j2 - Dy, dz = s1 / (p * p) - k2 - Dz;
      const double hl = g * sqrt((double)(dx * dx + dy * dy + dz * dz));
      u0 += lm[s1 * 4 + 0] * hl;
      u1 += lm[s1 * 4 + 1] * hl;
      u2 += lm[s1 * 4 + 2] * hl;
      u3 += lm[s1 * 4 + 3] * hl;
    }
    pa += u0 * ln[s2 * 4 + 0] + u1 * ln[s2 * 4 + 1] + u2 * ln[s2 * 4 + 2];
    pr += u3 * ln[s2 * 4 + 3];
  }
  using R = decltype(T2{}.x);
  out[i] = T2{(R)(0.5 * (la1 + la2) - pa), (R)(0.5 * (yr1 + yr2) - pr)};
}

// ---- conventional AIM: per-frequency near correction
// D(k0) = L_d,NR(k0) - W H_d,NR(k0) P on the near pattern (reading R22).
__constant__ double2 c_hd_tab[512];   // H_d(delta) = G_d(k0, h sqrt(q)), [0] = -j k0/(4 pi)

// G_d(k0, R) = (e^{-j k0 R} - 1)/(4 pi R), cancellation-free; R = 0: -j k0/(4 pi)
__device__ __forceinline__ double2 green_d(double k0, double R) {
  if (R == 0.0) return make_double2(0.0, -k0 / (4.0 * kPi));
  double sh, ch, s, c;
  sincos(0.5 * k0 * R, &sh, &ch);
  s = 2.0 * sh * ch;
  (void)c;
  const double inv = 1.0 / (4.0 * kPi * R);
  return make_double2(-2.0 * sh * sh * inv, -s * inv);
}

// Warp per row m, lanes over its near entries: L_d by the 7 x 7 product rule
// over the 2 x 2 triangle combinations (the direct reference's recipe), minus
// sum_c Lambda^c_m^T B_D(k0) Lambda^c_n with B_D[s,s'] = H_d(s - s' - D).
template <typename T2>
__global__ void k_aim_fill(int nb, int order, double k0, const int64_t* __restrict__ rowptr,
                           const int32_t* __restrict__ col, const int32_t* __restrict__ anchor,
                           const double* __restrict__ side, const double* __restrict__ lam, T2* __restrict__ DA,
                           T2* __restrict__ DR) {
  extern __shared__ double sh[];
  const int p = order + 1, p3 = p * p * p;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  // H_d table in shared memory: the lanes of a warp read different offsets
  // (the constant bank would serialise them)
  double2* hd_tab = reinterpret_cast<double2*>(sh);
  for (int t = threadIdx.x; t < 512; t += blockDim.x) hd_tab[t] = c_hd_tab[t];
  double* lm = sh + 2 * 512 + wib * (p3 * 4);
  const bool active = warp < nb;
  const int m = active ? (int)warp : 0;
  for (int t = lane; t < p3 * 4; t += 32) lm[t] = active ? lam[(int64_t)m * p3 * 4 + t] : 0.0;
  __syncthreads();
  if (!active) return;
  const int Amx = anchor[3 * m], Amy = anchor[3 * m + 1], Amz = anchor[3 * m + 2];
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const int n = col[k];
    double2 la = make_double2(0, 0), yr = make_double2(0, 0);
    for (int sm = 0; sm < 2; ++sm) {
      const double* om = side + (2 * (int64_t)m + sm) * kSideStride;
      const Vec3 a = v3(om), b = v3(om + 3), c = v3(om + 6), pm = v3(om + 9);
      const double coef_m = om[12], div_m = om[13], area_m = om[14];
      for (int sn = 0; sn < 2; ++sn) {
        const double* on = side + (2 * (int64_t)n + sn) * kSideStride;
        const Vec3 a2 = v3(on), b2 = v3(on + 3), c2 = v3(on + 6), pn = v3(on + 9);
        const double coef_n = on[12], div_n = on[13], area_n = on[14];
        for (int q1 = 0; q1 < 7; ++q1) {
          double b0, b1, bb2, w1;
          radon7(q1, b0, b1, bb2, w1);
          const Vec3 r = b0 * a + b1 * b + bb2 * c;
          const Vec3 fm = coef_m * (r - pm);
          double2 sa = make_double2(0, 0), sr = make_double2(0, 0);
          for (int q2 = 0; q2 < 7; ++q2) {
            double e0, e1, e2, w2;
            radon7(q2, e0, e1, e2, w2);
            const Vec3 r2 = e0 * a2 + e1 * b2 + e2 * c2;
            const double2 g = green_d(k0, norm(r - r2));
            const double wf = w2 * dot(fm, coef_n * (r2 - pn));
            sa.x += wf * g.x; sa.y += wf * g.y;
            sr.x += w2 * g.x; sr.y += w2 * g.y;
          }
          const double wm = w1 * area_m * area_n;
          la.x += wm * sa.x; la.y += wm * sa.y;
          const double wr = wm * div_m * div_n;
          yr.x += wr * sr.x; yr.y += wr * sr.y;
        }
      }
    }
    const int Dx = anchor[3 * n] - Amx, Dy = anchor[3 * n + 1] - Amy, Dz = anchor[3 * n + 2] - Amz;
    int sqx[7], sqy[7], sqz[7];
    for (int d = -order; d <= order; ++d) {
      sqx[d + order] = (d - Dx) * (d - Dx);
      sqy[d + order] = (d - Dy) * (d - Dy);
      sqz[d + order] = (d - Dz) * (d - Dz);
    }
    const double* ln = lam + (int64_t)n * p3 * 4;
    double2 pa = make_double2(0, 0), pr = make_double2(0, 0);
    for (int s2 = 0; s2 < p3; ++s2) {
      const int i2 = s2 % p, j2 = (s2 / p) % p, k2 = s2 / (p * p);
      double2 u[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
      for (int s1 = 0; s1 < p3; ++s1) {
        const int i1 = s1 % p, j1 = (s1 / p) % p, k1 = s1 / (p * p);
        const double2 hd = hd_tab[sqx[i1 - i2 + order] + sqy[j1 - j2 + order] + sqz[k1 - k2 + order]];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          u[ch].x += lm[s1 * 4 + ch] * hd.x;
          u[ch].y += lm[s1 * 4 + ch] * hd.y;
        }
      }
      for (int ch = 0; ch < 3; ++ch) {
        pa.x += u[ch].x * ln[s2 * 4 + ch];
        pa.y += u[ch].y * ln[s2 * 4 + ch];
      }
      pr.x += u[3].x * ln[s2 * 4 + 3];
      pr.y += u[3].y * ln[s2 * 4 + 3];
    }
    using R = decltype(T2{}.x);
    DA[k] = T2{(R)(la.x - pa.x), (R)(la.y - pa.y)};
    DR[k] = T2{(R)(yr.x - pr.x), (R)(yr.y - pr.y)};
  }
}

// ---- the double-layer operator K, static near part (
// the oracle kop module, readings R23-R25): C_K = sym(K_s,PV) + residue - K_s,P.
// Q(r) = int_T (r - r')/R^3 dS' = sum_i m_i f2_i + n sgn(d) Omega (in-plane
// points up to rounding are in-plane: the +-2 pi jump is the residue's).
__device__ __forceinline__ Vec3 k_q(const Frame& F, Vec3 r) {
  double d = dot(r - F.v[0], F.n);
  if (fabs(d) <= 1e-12 * (F.L[0] + F.L[2])) d = 0.0;
  const Vec3 rho = r - d * F.n;
  const double ad = fabs(d);
  Vec3 Q = {0.0, 0.0, 0.0};
  double omega = 0.0;
  for (int k = 0; k < 3; ++k) {
    Vec3 va = F.v[k], vb = F.v[(k + 1) % 3];
    double sm = dot(va - rho, F.sh[k]);
    double sp = dot(vb - rho, F.sh[k]);
    double t0 = dot(va - rho, F.mh[k]);
    double R0sq = t0 * t0 + d * d;
    double Rm = norm(r - va), Rp = norm(r - vb);
    double lim = 1e-14 * F.L[k];
    double f2 = 0.0;
    if (R0sq > lim * lim) f2 = logsum(Rp, sp, R0sq) - logsum(Rm, sm, R0sq);
    if (ad > 0.0) omega += atan(t0 * sp / (R0sq + ad * Rp)) - atan(t0 * sm / (R0sq + ad * Rm));
    Q = Q + f2 * F.mh[k];
  }
  const double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
  return Q + (sg * omega) * F.n;
}

// barycentric point q of the 7-point rule on sub-triangle t of an nsub x nsub
// subdivision (t < nsub^2; weight = radon weight / nsub^2)
__device__ __forceinline__ void sub_point(int nsub, int t, int q, double& b0, double& b1, double& b2, double& w) {
  // sub-triangles enumerated as in oracle kop.subdivided_rule: for i, for j < nsub - i:
  // the "up" triangle, then (if i + j + 1 < nsub) the "down" one
  int i = 0, j = 0, down = 0, c = 0;
  for (i = 0; i < nsub; ++i) {
    for (j = 0; j < nsub - i; ++j) {
      if (c == t) { down = 0; goto found; }
      ++c;
      if (i + j + 1 < nsub) {
        if (c == t) { down = 1; goto found; }
        ++c;
      }
    }
  }
found:
  double u0, v0, u1, v1, u2, v2;
  if (!down) { u0 = i; v0 = j; u1 = i + 1; v1 = j; u2 = i; v2 = j + 1; }
  else { u0 = i + 1; v0 = j + 1; u1 = i; v1 = j + 1; u2 = i + 1; v2 = j; }
  double c0, c1, c2, wq;
  radon7(q, c0, c1, c2, wq);
  const double u = (c0 * u0 + c1 * u1 + c2 * u2) / nsub, v = (c0 * v0 + c1 * v1 + c2 * v2) / nsub;
  b0 = 1.0 - u - v;
  b1 = u;
  b2 = v;
  w = wq / ((double)nsub * nsub);
}

// Warp per row m, lanes over its near entries: the unsymmetrised PV part of
// K_s (outer rule subdivided 8 x 8 on touching triangle pairs) and the
// residue 1/2 int f_m . (n x f_n) on shared triangles.
__global__ void k_K_near_un(int nb, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const double* __restrict__ side, const int32_t* __restrict__ T,
                            const int32_t* __restrict__ tp, const int32_t* __restrict__ tm,
                            double* __restrict__ Kun, double* __restrict__ Res) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp >= nb) return;
  const int m = (int)warp;
  const double inv4pi = 1.0 / (4.0 * kPi);
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const int n = col[k];
    double kv = 0.0, rv = 0.0;
    for (int sm = 0; sm < 2; ++sm) {
      const double* om = side + (2 * (int64_t)m + sm) * kSideStride;
      const int trm = sm ? tm[m] : tp[m];
      const Vec3 a = v3(om), b = v3(om + 3), c = v3(om + 6), pm = v3(om + 9);
      const double coef_m = om[12], area_m = om[14];
      for (int sn = 0; sn < 2; ++sn) {
        const double* on = side + (2 * (int64_t)n + sn) * kSideStride;
        const int trn = sn ? tm[n] : tp[n];
        const Vec3 pn = v3(on + 9);
        const double coef_n = on[12];
        if (trm == trn) {   // residue on the shared triangle (7-point rule exact)
          Vec3 nn = cross(b - a, c - a);
          nn = (1.0 / norm(nn)) * nn;
          for (int q = 0; q < 7; ++q) {
            double b0, b1, b2, w;
            radon7(q, b0, b1, b2, w);
            const Vec3 r = b0 * a + b1 * b + b2 * c;
            rv += 0.5 * w * area_m * dot(coef_m * (r - pm), cross(nn, coef_n * (r - pn)));
          }
          continue;        // coinciding triangles: PV part 0
        }
        bool touch = false;
        for (int u = 0; u < 3; ++u)
          for (int v = 0; v < 3; ++v) touch = touch || (T[3 * trm + u] == T[3 * trn + v]);
        Frame F;
        make_frame(on, F);
        const int nsub = touch ? 8 : 1, nt = nsub * nsub;
        double acc = 0.0;
        for (int t = 0; t < nt; ++t)
          for (int q = 0; q < 7; ++q) {
            double b0, b1, b2, w;
            if (nsub == 1) radon7(q, b0, b1, b2, w);
            else sub_point(nsub, t, q, b0, b1, b2, w);
            const Vec3 r = b0 * a + b1 * b + b2 * c;
            const Vec3 Q = k_q(F, r);
            const Vec3 inner = (-coef_n * inv4pi) * cross(Q, r - pn);
            acc += w * dot(coef_m * (r - pm), inner);
          }
        kv -= area_m * acc;
      }
    }
    Kun[k] = kv;
    Res[k] = rv;
  }
}

__constant__ double c_gk_tab[3 * 2197];   // d_a G_s(h delta) for |delta_i| <= 6: [(dz+6)*169 + (dy+6)*13 + (dx+6)][a]

// Warp per row: C_K = (Kun + Kun^T)/2 + Res - K_s,P, K_s,P[m,n] = -sum_{c,a,b}
// eps_cab Lambda^c_m B^a_D Lambda^b_n, B^a_D[s,s'] = d_a G_s(h (s - s' - D)).
__global__ void k_K_combine(int nb, int order, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ anchor, const double* __restrict__ lam,
                            const double* __restrict__ Kun, const double* __restrict__ Res,
                            double* __restrict__ CK, double* __restrict__ CKpv) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (warp >= nb) return;
  const int m = (int)warp;
  const int p = order + 1, p3 = p * p * p;
  const double* lm = lam + (int64_t)m * p3 * 4;
  for (int64_t k = rowptr[m] + lane; k < rowptr[m + 1]; k += 32) {
    const int n = col[k];
    int64_t lo = rowptr[n], hi = rowptr[n + 1] - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (col[mid] < m) lo = mid + 1; else hi = mid;
    }
    const double ks = 0.5 * (Kun[k] + Kun[lo]);
    const int Dx = anchor[3 * n] - anchor[3 * m], Dy = anchor[3 * n + 1] - anchor[3 * m + 1],
              Dz = anchor[3 * n + 2] - anchor[3 * m + 2];
    const double* ln = lam + (int64_t)n * p3 * 4;
    double kp = 0.0;
    for (int s2 = 0; s2 < p3; ++s2) {
      const int i2 = s2 % p, j2 = (s2 / p) % p, k2 = s2 / (p * p);
      double u[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};   // u[a][c] = sum_s1 Lam^c_m[s1] B^a[s1, s2]
      for (int s1 = 0; s1 < p3; ++s1) {
        const int dx = s1 % p - i2 - Dx, dy = (s1 / p) % p - j2 - Dy, dz = s1 / (p * p) - k2 - Dz;
        const double* g = c_gk_tab + 3 * ((dz + 6) * 169 + (dy + 6) * 13 + (dx + 6));
        for (int a = 0; a < 3; ++a)
          for (int c = 0; c < 3; ++c) u[a][c] += lm[s1 * 4 + c] * g[a];
      }
      // sum_{c,a,b} eps_cab u[a][c] Lam^b_n[s2]
      const double l0 = ln[s2 * 4 + 0], l1 = ln[s2 * 4 + 1], l2 = ln[s2 * 4 + 2];
      kp += u[1][0] * l2 - u[2][0] * l1     // c = x: (a,b) = (y,z) +, (z,y) -
            + u[2][1] * l0 - u[0][1] * l2   // c = y: (z,x) +, (x,z) -
            + u[0][2] * l1 - u[1][2] * l0;  // c = z: (x,y) +, (y,x) -
    }
    CK[k] = ks + Res[k] + kp;   // - K_s,P = + sum eps ...
    if (CKpv) CKpv[k] = ks + kp;   // principal value only (PMCHWT: the residues cancel)
  }
}

void gauss_legendre(int q, double* x, double* w) {
  // nodes/weights on [0, 1]
  for (int i = 0; i < q; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (q + 0.5));
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= q; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      double dp = q * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) {
        // recompute derivative at the converged root
        p0 = 1.0; p1 = z;
        for (int k = 2; k <= q; ++k) {
          double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
          p0 = p1;
          p1 = p2;
        }
        dp = q * (z * p1 - p0) / (z * z - 1.0);
        x[i] = 0.5 * (1.0 - z);
        w[i] = 1.0 / ((1.0 - z * z) * dp * dp);   // (2/((1-z^2) dp^2)) * 1/2
        break;
      }
    }
  }
}

}  // namespace

void launch_rwg_sides(const Topology& t, SetupDev& d, cudaStream_t s) {
  int64_t n = 2 * t.nb;
  k_rwg_sides<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((int)t.nb, d.V, d.T, d.ea, d.eb, d.tp,
                                                          d.tm, d.pp, d.pm, d.side);
  AIMX_CHECK_LAUNCH();
}

void launch_weights(const Topology& t, SetupDev& d, cudaStream_t s, uint8_t* nzflag) {
  const int q = (3 * t.order + 4) / 2;   // exact for degree 3n+1 after the collapse
  double x[8], w[8];
  gauss_legendre(q, x, w);
  AIMX_CUDA(cudaMemcpyToSymbolAsync(c_gl_x, x, sizeof(double) * q, 0, cudaMemcpyHostToDevice, s));
  AIMX_CUDA(cudaMemcpyToSymbolAsync(c_gl_w, w, sizeof(double) * q, 0, cudaMemcpyHostToDevice, s));
  int64_t n = t.nb * (int64_t)t.p3;
  k_weights<<<(unsigned)((n + 127) / 128), 128, 0, s>>>((int)t.nb, t.order, q, d.side, d.anchor,
                                                        t.origin[0], t.origin[1], t.origin[2], t.h,
                                                        d.lam, nzflag);
  AIMX_CHECK_LAUNCH();
}

void launch_static_near(const Topology& t, SetupDev& d, cudaStream_t s) {
  const int threads = 128;
  int64_t blocks = (t.nb * 32 + threads - 1) / threads;
  k_static_near<<<(unsigned)blocks, threads, 0, s>>>((int)t.nb, d.rowptr, d.col, d.side, d.LA_un,
                                                     d.YR_un);
  AIMX_CHECK_LAUNCH();
}

void launch_lin_entries(const Topology& t, const SetupDev& d, const int32_t* cols, bool f32, void* out,
                        cudaStream_t s) {
  const int64_t n = t.nb * (int64_t)kLinW;
  const unsigned g = (unsigned)((n + 127) / 128);
  if (f32)
    k_lin_entries<float2><<<g, 128, 0, s>>>((int)t.nb, t.order, t.h, cols, d.anchor, d.side, d.lam, (float2*)out);
  else
    k_lin_entries<double2><<<g, 128, 0, s>>>((int)t.nb, t.order, t.h, cols, d.anchor, d.side, d.lam,
                                             (double2*)out);
  AIMX_CHECK_LAUNCH();
}

void launch_aim_fill(const Topology& t, const SetupDev& d, double k0, bool f32, void* DA, void* DR, cudaStream_t s) {
  std::vector<double2> tab(512);
  tab[0] = make_double2(0.0, -k0 / (4.0 * kPi));
  for (int q = 1; q < 512; ++q) {
    const double r = t.h * std::sqrt((double)q), sh = std::sin(0.5 * k0 * r);
    tab[q] = make_double2(-2.0 * sh * sh / (4.0 * kPi * r), -std::sin(k0 * r) / (4.0 * kPi * r));
  }
  const int R = 2 * t.order + t.near_cells;
  if (3 * R * R >= 512) throw Error(AIMX_E_GRID, "precorrection offset table too small");
  AIMX_CUDA(cudaMemcpyToSymbolAsync(c_hd_tab, tab.data(), sizeof(double2) * 512, 0, cudaMemcpyHostToDevice, s));
  const int threads = 128;
  const int64_t blocks = (t.nb * 32 + threads - 1) / threads;
  const size_t shm = (2 * 512 + (threads / 32) * t.p3 * 4) * sizeof(double);
  if (f32)
    k_aim_fill<float2><<<(unsigned)blocks, threads, shm, s>>>((int)t.nb, t.order, k0, d.rowptr, d.col, d.anchor,
                                                               d.side, d.lam, (float2*)DA, (float2*)DR);
  else
    k_aim_fill<double2><<<(unsigned)blocks, threads, shm, s>>>((int)t.nb, t.order, k0, d.rowptr, d.col, d.anchor,
                                                                d.side, d.lam, (double2*)DA, (double2*)DR);
  AIMX_CHECK_LAUNCH();
}

void launch_K_static(const Topology& t, const SetupDev& d, double* CK, cudaStream_t s, double* CKpv) {
  const int R = 2 * t.order + t.near_cells;
  if (R > 6) throw Error(AIMX_E_GRID, "K precorrection offset table too small");
  std::vector<double> tab(3 * 2197, 0.0);
  for (int dz = -6; dz <= 6; ++dz)
    for (int dy = -6; dy <= 6; ++dy)
      for (int dx = -6; dx <= 6; ++dx) {
        const double q = (double)(dx * dx + dy * dy + dz * dz);
        if (q == 0.0) continue;
        const double f = -1.0 / (4.0 * kPi * t.h * t.h * q * std::sqrt(q));   // d_a G_s = -delta_a / (4 pi h^2 |delta|^3)
        double* g = tab.data() + 3 * ((dz + 6) * 169 + (dy + 6) * 13 + (dx + 6));
        g[0] = f * dx; g[1] = f * dy; g[2] = f * dz;
      }
  AIMX_CUDA(cudaMemcpyToSymbolAsync(c_gk_tab, tab.data(), sizeof(double) * tab.size(), 0, cudaMemcpyHostToDevice, s));
  const int64_t nnz = t.rowptr[t.nb];
  double *Kun = nullptr, *Res = nullptr;
  AIMX_CUDA(cudaMallocAsync(&Kun, (size_t)std::max<int64_t>(nnz, 1) * sizeof(double), s));
  AIMX_CUDA(cudaMallocAsync(&Res, (size_t)std::max<int64_t>(nnz, 1) * sizeof(double), s));
  const int threads = 128;
  const int64_t blocks = (t.nb * 32 + threads - 1) / threads;
  k_K_near_un<<<(unsigned)blocks, threads, 0, s>>>((int)t.nb, d.rowptr, d.col, d.side, d.T, d.tp, d.tm, Kun, Res);
  AIMX_CHECK_LAUNCH();
  k_K_combine<<<(unsigned)blocks, threads, 0, s>>>((int)t.nb, t.order, d.rowptr, d.col, d.anchor, d.lam, Kun, Res, CK,
                                                    CKpv);
  AIMX_CHECK_LAUNCH();
  AIMX_CUDA(cudaFreeAsync(Kun, s));
  AIMX_CUDA(cudaFreeAsync(Res, s));
}

void launch_precorrect(const Topology& t, SetupDev& d, cudaStream_t s) {
  std::vector<double> tab(512, 0.0);
  for (int qq = 1; qq < 512; ++qq) tab[qq] = 1.0 / (4.0 * kPi * t.h * std::sqrt((double)qq));
  const int R = 2 * t.order + t.near_cells;
  if (3 * R * R >= 512) throw Error(AIMX_E_GRID, "precorrection offset table too small");
  AIMX_CUDA(cudaMemcpyToSymbolAsync(c_hs_tab, tab.data(), sizeof(double) * 512, 0,
                                    cudaMemcpyHostToDevice, s));
  const int threads = 128;
  int64_t blocks = (t.nb * 32 + threads - 1) / threads;
  size_t shm = (512 + (threads / 32) * t.p3 * 4) * sizeof(double);
  k_precorrect<<<(unsigned)blocks, threads, shm, s>>>((int)t.nb, t.order, d.rowptr, d.col, d.anchor,
                                                     d.lam, d.LA_un, d.YR_un, d.LA_NR, d.YR_NR,
                                                     d.LA_P, d.YR_P, d.CA, d.CR);
  AIMX_CHECK_LAUNCH();
}

}  // namespace aimx
