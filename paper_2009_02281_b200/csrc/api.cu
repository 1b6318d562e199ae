// C ABI of the AIMx B200 library (include/aimx.h): context lifecycle, setup
// orchestration (host topology -> device fp64 static fill -> hot-path data),
// frequency binding, matvec / sweep entry points and introspection.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "aimx_internal.h"

using namespace aimx;

struct aimx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  aimx_prec prec = AIMX_C64;
  Topology topo;
  NodeMap nodes;
  SetupDev sd;
  HotDev hot;
  SpectrumPlan sp;
  double2* Hs = nullptr;        // static spectrum octant, fp64, unnormalised
  void* Hs_T = nullptr;         // static spectrum in compute precision (c64 only)
  int64_t dev_bytes = 0;
  bool freq_set = false;
  double f = 0, k0 = 0, omega = 0;
  cudaEvent_t ev_spec = nullptr, ev_use = nullptr;
  void* stage = nullptr;        // sweep_host staging
  int64_t stage_bytes = 0;
  double setup_seconds = 0;
  int near_R = 0, near_order = 0;
  int64_t near_union = 0;
  Profiler prof;
  std::vector<void*> allocs;
  std::string last_error;
};

namespace aimx {
int64_t& launch_counter() {
  static thread_local int64_t n = 0;
  return n;
}
}  // namespace aimx

namespace {

thread_local std::string g_setup_error;

template <typename P>
P* dalloc(aimx_ctx* c, int64_t count) {
  void* p = nullptr;
  size_t bytes = (size_t)std::max<int64_t>(count, 1) * sizeof(P);
  AIMX_CUDA(cudaMalloc(&p, bytes));
  c->allocs.push_back(p);
  c->dev_bytes += (int64_t)bytes;
  return (P*)p;
}

template <typename P>
void dfree(aimx_ctx* c, P*& p, int64_t bytes) {
  for (auto& a : c->allocs)
    if (a == (void*)p) { a = nullptr; break; }
  AIMX_CUDA(cudaFree(p));
  c->dev_bytes -= bytes;
  p = nullptr;
}

template <typename P>
P* dupload(aimx_ctx* c, const std::vector<P>& v) {
  P* p = dalloc<P>(c, (int64_t)v.size());
  if (!v.empty())
    AIMX_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(P), cudaMemcpyHostToDevice, c->stream));
  return p;
}

// ---- small conversion kernels ------------------------------------------------------
// weight (rwg, slot) i -> its row-group slot (exactly-zero weights have none)
// weight (rwg, slot) i -> byte offset slot[i] of the near payload (exactly-zero weights have none)
template <typename T4>
__global__ void k_lam_to(int64_t n, const int64_t* __restrict__ slot, const double* __restrict__ lam, T4*,
                         unsigned char* __restrict__ payload) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || slot[i] < 0) return;
  T4 v;
  v.x = lam[4 * i]; v.y = lam[4 * i + 1]; v.z = lam[4 * i + 2]; v.w = lam[4 * i + 3];
  *reinterpret_cast<T4*>(payload + slot[i]) = v;
}
template <typename T4>
__global__ void k_ent_w(int64_t n, int p3, const int32_t* __restrict__ er, const int32_t* __restrict__ es,
                        const double* __restrict__ lam, T4* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* l = lam + ((int64_t)er[i] * p3 + es[i]) * 4;
  T4 v;
  v.x = l[0]; v.y = l[1]; v.z = l[2]; v.w = l[3];
  out[i] = v;
}
// CSR entry k of (C_A, C_rho) -> byte offset slot[k] of the near payload
template <typename T2>
__global__ void k_pack_c(int64_t n, const int64_t* __restrict__ slot, const double* __restrict__ CA,
                         const double* __restrict__ CR, T2*, unsigned char* __restrict__ payload) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  T2 v;
  v.x = CA[i];
  v.y = CR[i];
  *reinterpret_cast<T2*>(payload + slot[i]) = v;
}
__global__ void k_d2f(int64_t n, const double2* __restrict__ a, float2* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  b[i] = make_float2((float)a[i].x, (float)a[i].y);
}

unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

void* make_twiddles(aimx_ctx* c, int L) {
  // exp(-2 pi i m / L) with exact octant reduction, computed in fp64
  std::vector<double> re(L), im(L);
  for (int m = 0; m < L; ++m) {
    double a = 2.0 * kPi * (double)m / (double)L;
    re[m] = std::cos(a);
    im[m] = -std::sin(a);
    if (4 * m == L || 4 * m == 3 * L) re[m] = 0.0;
    if (2 * m == L || m == 0) im[m] = 0.0;
  }
  if (c->prec == AIMX_C64) {
    std::vector<float2> v(L);
    for (int m = 0; m < L; ++m) v[m] = make_float2((float)re[m], (float)im[m]);
    return dupload(c, v);
  }
  std::vector<double2> v(L);
  for (int m = 0; m < L; ++m) v[m] = make_double2(re[m], im[m]);
  return dupload(c, v);
}

void do_setup(aimx_ctx* c, const aimx_mesh_desc* mesh, const aimx_grid_desc* grid) {
  Topology& t = c->topo;
  build_topology(mesh, grid, t);
  for (int a = 0; a < 3; ++a)
    if (!fft_length_supported(2 * t.n[a]))
      throw Error(AIMX_E_UNSUPPORTED, "2*N_a must be a power of two in [8, 1024]");
  const int64_t nb = t.nb, nnz = t.rowptr[nb], p3 = t.p3;
  SetupDev& d = c->sd;
  // ---- upload topology
  d.V = dupload(c, t.V);
  d.T = dupload(c, t.T);
  d.ea = dupload(c, t.ea); d.eb = dupload(c, t.eb);
  d.tp = dupload(c, t.tp); d.tm = dupload(c, t.tm);
  d.pp = dupload(c, t.pp); d.pm = dupload(c, t.pm);
  d.anchor = dupload(c, t.anchor);
  d.rowptr = dupload(c, t.rowptr);
  d.col = dupload(c, t.col);
  d.side = dalloc<double>(c, 2 * nb * kSideStride);
  d.lam = dalloc<double>(c, nb * p3 * 4);
  uint8_t* nzf = dalloc<uint8_t>(c, nb * p3);
  launch_rwg_sides(t, d, c->stream);
  launch_weights(t, d, c->stream, nzf);
  std::vector<uint8_t> nz((size_t)(nb * p3));
  AIMX_CUDA(cudaMemcpyAsync(nz.data(), nzf, nz.size(), cudaMemcpyDeviceToHost, c->stream));
  // ---- static near fill + precorrection (fp64)
  d.LA_un = dalloc<double>(c, nnz);
  d.YR_un = dalloc<double>(c, nnz);
  d.LA_NR = dalloc<double>(c, nnz);
  d.YR_NR = dalloc<double>(c, nnz);
  d.LA_P = dalloc<double>(c, nnz);
  d.YR_P = dalloc<double>(c, nnz);
  d.CA = dalloc<double>(c, nnz);
  d.CR = dalloc<double>(c, nnz);
  launch_static_near(t, d, c->stream);
  launch_precorrect(t, d, c->stream);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  build_nodemap(t, nz, c->nodes);
  // ---- hot-path data
  HotDev& h = c->hot;
  NodeMap& m = c->nodes;
  h.Nx = t.n[0]; h.Ny = t.n[1]; h.Nz = t.n[2];
  h.p = t.p; h.p3 = t.p3;
  h.nb = (int)nb;
  h.nnz = nnz;
  h.nocc = (int)m.node_lin.size();
  h.nlines = (int)m.line_id.size();
  h.nzocc = (int)m.zplanes.size();
  std::vector<int32_t> base(nb);
  for (int64_t e = 0; e < nb; ++e)
    base[e] = t.anchor[3 * e] + t.n[0] * (t.anchor[3 * e + 1] + t.n[1] * t.anchor[3 * e + 2]);
  h.rwg_base = dupload(c, base);
  h.node_lin = dupload(c, m.node_lin);
  h.node_ptr = dupload(c, m.node_ptr);
  h.node_line = dupload(c, m.node_line);
  h.ent_rwg = dupload(c, m.ent_rwg);
  int32_t* ent_slot = dupload(c, m.ent_slot);
  h.line_id = dupload(c, m.line_id);
  h.zplanes = dupload(c, m.zplanes);
  h.line_occ = dupload(c, m.line_occ);
  {
    std::vector<uint8_t> zo(t.n[2], 0);
    for (int z : m.zplanes) zo[z] = 1;
    h.zocc = dupload(c, zo);
  }
  // near matrix in row-group form (host ordering and unions; values scattered on device)
  NearGroups grp;
  build_near_groups(t, nz, grp);
  if (grp.ptr.back() > (int64_t)INT32_MAX || grp.wptr.back() > (int64_t)INT32_MAX)
    throw Error(AIMX_E_GRID, "near matrix too large");
  h.R = grp.R;
  h.ngrp = (int)grp.ngrp;
  h.grp_rows = dupload(c, grp.rows);
  const int64_t nU = grp.ptr.back(), nUw = grp.wptr.back();
  int64_t* gslot = nullptr;
  int64_t* wslot = nullptr;
  {
    int nsm = 148;
    AIMX_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    NearChunks ck;
    const bool f32p = c->prec == AIMX_C64;
    const int cs = f32p ? 8 : 16;
    build_near_chunks(grp, f32p ? 32 : 16, f32p ? 128 : 64, cs, ck);
    // value slot (u R + r) -> payload byte offset
    for (auto& v : grp.slot) v = ck.uoff_c[v / grp.R] + (v % grp.R) * cs;
    for (auto& v : grp.wslot)
      if (v >= 0) v = ck.uoff_w[v / grp.R] + (v % grp.R) * 2 * cs;
    gslot = dupload(c, grp.slot);
    wslot = dupload(c, grp.wslot);
    h.payload = dupload(c, ck.payload);
    h.chunks = dupload(c, ck.chunks);
    std::vector<int32_t> cp = near_partition(ck, grp.ngrp, near_ctas_per_sm(f32p, false) * nsm);
    h.cta_ptr = dupload(c, cp);
    h.near_ctas = (int)cp.size() - 1;
    cp = near_partition(ck, grp.ngrp, near_ctas_per_sm(f32p, true) * nsm);
    h.cta_ptr1 = dupload(c, cp);
    h.near_ctas1 = (int)cp.size() - 1;
  }
  c->near_R = grp.R;
  c->near_order = grp.order_kind;
  c->near_union = nU;
  const int64_t nent = (int64_t)m.ent_rwg.size();
  const int64_t ng = (int64_t)h.Nx * h.Ny * h.Nz;
  const bool f32 = c->prec == AIMX_C64;
  const size_t cs = f32 ? sizeof(float2) : sizeof(double2);
  if (f32) {
    h.ent_w = dalloc<float4>(c, nent);
    k_lam_to<float4><<<nblk(nb * p3), 256, 0, c->stream>>>(nb * p3, wslot, d.lam, (float4*)nullptr, h.payload);
    k_ent_w<float4><<<nblk(nent), 256, 0, c->stream>>>(nent, (int)p3, h.ent_rwg, ent_slot, d.lam,
                                                      (float4*)h.ent_w);
    k_pack_c<float2><<<nblk(nnz), 256, 0, c->stream>>>(nnz, gslot, d.CA, d.CR, (float2*)nullptr, h.payload);
  } else {
    h.ent_w = dalloc<double4>(c, nent);
    k_lam_to<double4><<<nblk(nb * p3), 256, 0, c->stream>>>(nb * p3, wslot, d.lam, (double4*)nullptr, h.payload);
    k_ent_w<double4><<<nblk(nent), 256, 0, c->stream>>>(nent, (int)p3, h.ent_rwg, ent_slot, d.lam,
                                                       (double4*)h.ent_w);
    k_pack_c<double2><<<nblk(nnz), 256, 0, c->stream>>>(nnz, gslot, d.CA, d.CR, (double2*)nullptr, h.payload);
  }
  AIMX_CHECK_LAUNCH();
  // ---- batch slots and grid buffers
  const int64_t nS = (int64_t)h.nlines * h.Nx * 4;
  const int64_t nA = (int64_t)h.Nz * h.Ny * 2 * h.Nx * 4;
  const int64_t nB = (int64_t)h.Nz * 2 * h.Ny * 2 * h.Nx * 4;
  const int64_t nP = ng * 4;
  const int64_t noct = (int64_t)(h.Nx + 1) * (h.Ny + 1) * (h.Nz + 1);
  const int64_t per_freq = (int64_t)cs * (nS + 2 * nA + nB + nP + noct) + 2 * (int64_t)sizeof(double2) * noct;
  int slots = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxBatch, (int64_t)(1536ll << 20) / per_freq));
  if (const char* e = std::getenv("AIMX_BATCH")) slots = std::max(1, std::min(kMaxBatch, std::atoi(e)));
  while (slots & (slots - 1)) slots &= slots - 1;   // power of two (batch buckets never exceed it)
  h.batch = slots;
  h.sS = nS; h.sA = nA; h.sB = nB; h.sP = nP; h.sH = noct;
  h.S = dalloc<char>(c, nS * slots * (int64_t)cs);
  h.bufA = dalloc<char>(c, nA * slots * (int64_t)cs);
  h.bufB = dalloc<char>(c, nB * slots * (int64_t)cs);
  h.bufC = dalloc<char>(c, nA * slots * (int64_t)cs);
  h.phi = dalloc<char>(c, nP * slots * (int64_t)cs + 64);   // + 64: 16-byte row blocks may overhang
  AIMX_CUDA(cudaMemsetAsync(h.S, 0, nS * slots * cs, c->stream));
  AIMX_CUDA(cudaMemsetAsync(h.bufA, 0, nA * slots * cs, c->stream));
  AIMX_CUDA(cudaMemsetAsync(h.bufB, 0, nB * slots * cs, c->stream));
  AIMX_CUDA(cudaMemsetAsync(h.bufC, 0, nA * slots * cs, c->stream));
  AIMX_CUDA(cudaMemsetAsync(h.phi, 0, nP * slots * cs, c->stream));
  h.twx = make_twiddles(c, 2 * h.Nx);
  h.twy_tab = make_twiddles(c, 2 * h.Ny);
  h.twz_tab = make_twiddles(c, 2 * h.Nz);
  h.twy = pick_tile(2 * h.Ny, 8 * h.Nx, f32);
  h.twz = pick_tile(2 * h.Nz, 8 * h.Nx, f32);
  {
    const double avg = h.nocc > 0 ? (double)nent / h.nocc : 1.0;
    int G = 4;
    while (G < 32 && G < avg) G *= 2;
    h.G = G;
  }
  // ---- static spectrum
  c->sp.Nx = h.Nx; c->sp.Ny = h.Ny; c->sp.Nz = h.Nz; c->sp.h = t.h;
  spectrum_plan_init(c->sp, slots, c->stream);
  c->Hs = dalloc<double2>(c, noct);
  spectrum_static(c->sp, c->Hs, c->stream);
  if (f32) {
    c->Hs_T = dalloc<float2>(c, noct);
    k_d2f<<<nblk(noct), 256, 0, c->stream>>>(noct, c->Hs, (float2*)c->Hs_T);
    AIMX_CHECK_LAUNCH();
  } else {
    c->Hs_T = c->Hs;
  }
  h.Hoct = dalloc<char>(c, noct * slots * (int64_t)cs);
  h.xt = dalloc<char>(c, (int64_t)nb * kMaxBatch * (int64_t)cs + 64);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  dfree(c, gslot, nnz * (int64_t)sizeof(int64_t));
  dfree(c, wslot, nb * p3 * (int64_t)sizeof(int64_t));
  dfree(c, d.LA_un, nnz * sizeof(double));
  dfree(c, d.YR_un, nnz * sizeof(double));
  AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_spec, cudaEventDisableTiming));
  AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_use, cudaEventDisableTiming));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
}

// S1 for B frequency points into spectrum slots 0..B-1.
void spectra(aimx_ctx* c, int B, const double* f, cudaStream_t s) {
  double k0[kMaxBatch];
  for (int b = 0; b < B; ++b) {
    if (!(f[b] > 0.0) || !std::isfinite(f[b])) throw Error(AIMX_E_INVALID_ARG, "frequency must be finite and > 0");
    k0[b] = 2.0 * kPi * f[b] / kC0;
  }
  const HotDev& h = c->hot;
  const double M = 8.0 * (double)h.Nx * h.Ny * h.Nz;
  StageScope sc(&c->prof, 0, s);
  if (c->prec == AIMX_C64)
    spectrum_dynamic_f32(c->sp, B, k0, (const float2*)c->Hs_T, (float)(1.0 / M), (float2*)h.Hoct, s);
  else
    spectrum_dynamic_f64(c->sp, B, k0, c->Hs, 1.0 / M, (double2*)h.Hoct, s);
}

void bind_frequency(aimx_ctx* c, double f, cudaStream_t s) {
  spectra(c, 1, &f, s);
  c->f = f;
  c->k0 = 2.0 * kPi * f / kC0;
  c->omega = 2.0 * kPi * f;
  c->freq_set = true;
}

Combine make_combine(int B, const double* f, int mode, int64_t nb) {
  Combine cb;
  for (int b = 0; b < kMaxBatch; ++b) cb.alpha_im[b] = cb.beta[b] = 0.0;
  cb.B = B;
  cb.mode = mode;
  cb.xstride = nb;
  cb.ystride = nb;
  for (int b = 0; b < B; ++b) {
    const double k0 = 2.0 * kPi * f[b] / kC0;
    cb.alpha_im[b] = -2.0 * kPi * f[b] * kMu0;
    cb.beta[b] = 1.0 / (k0 * k0);
  }
  return cb;
}

void run_matvec(aimx_ctx* c, const void* x, void* y0, void* y1, int mode, cudaStream_t s) {
  Combine cb = make_combine(1, &c->f, mode, c->hot.nb);
  if (c->prec == AIMX_C64) hot_matvec_f32(c->hot, x, y0, y1, cb, s, &c->prof);
  else hot_matvec_f64(c->hot, x, y0, y1, cb, s, &c->prof);
}

// B frequency points: spectra into slots, then one batched matvec.
void run_batch(aimx_ctx* c, int B, const double* f, const void* X, void* Y, cudaStream_t s) {
  spectra(c, B, f, s);
  Combine cb = make_combine(B, f, 0, c->hot.nb);
  if (c->prec == AIMX_C64) hot_matvec_f32(c->hot, X, Y, nullptr, cb, s, &c->prof);
  else hot_matvec_f64(c->hot, X, Y, nullptr, cb, s, &c->prof);
}

aimx_status fail(aimx_ctx* c, const Error& e) {
  if (c) c->last_error = e.what();
  return e.code;
}

void check_sticky(aimx_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(AIMX_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
  (void)c;
}

cudaStream_t pick(aimx_ctx* c, void* s) { return s ? (cudaStream_t)s : c->stream; }

void destroy_impl(aimx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : c->allocs) if (p) cudaFree(p);
  spectrum_plan_free(c->sp);
  if (c->stage) cudaFree(c->stage);
  if (c->ev_spec) cudaEventDestroy(c->ev_spec);
  if (c->ev_use) cudaEventDestroy(c->ev_use);
  delete c;
}

}  // namespace

#define AIMX_API_BEGIN try {
#define AIMX_API_END(ctx)                                     \
  }                                                           \
  catch (const Error& e) { return fail(ctx, e); }             \
  catch (const std::bad_alloc&) {                             \
    if (ctx) (ctx)->last_error = "host allocation failed";    \
    return AIMX_E_OOM;                                        \
  }                                                           \
  catch (const std::exception& e) {                           \
    if (ctx) (ctx)->last_error = e.what();                    \
    return AIMX_E_INTERNAL;                                   \
  }                                                           \
  return AIMX_OK;

extern "C" {

aimx_status aimx_setup(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, aimx_prec prec,
                       int device, void* stream, aimx_ctx** out) {
  g_setup_error.clear();
  if (!out) { g_setup_error = "out is NULL"; return AIMX_E_INVALID_ARG; }
  *out = nullptr;
  if (prec != AIMX_C64 && prec != AIMX_C128) { g_setup_error = "bad precision"; return AIMX_E_INVALID_ARG; }
  aimx_ctx* c = nullptr;
  try {
    auto t0 = std::chrono::steady_clock::now();
    AIMX_CUDA(cudaSetDevice(device));
    c = new aimx_ctx;
    c->device = device;
    c->prec = prec;
    c->stream = (cudaStream_t)stream;
    do_setup(c, mesh, grid);
    c->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c;
    return AIMX_OK;
  } catch (const Error& e) {
    g_setup_error = e.what();
    destroy_impl(c);
    return e.code;
  } catch (const std::bad_alloc&) {
    g_setup_error = "host allocation failed";
    destroy_impl(c);
    return AIMX_E_OOM;
  } catch (const std::exception& e) {
    g_setup_error = e.what();
    destroy_impl(c);
    return AIMX_E_INTERNAL;
  }
}

aimx_status aimx_set_frequency(aimx_ctx* c, double f_hz) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  AIMX_CUDA(cudaStreamWaitEvent(c->stream, c->ev_use, 0));
  bind_frequency(c, f_hz, c->stream);
  AIMX_CUDA(cudaEventRecord(c->ev_spec, c->stream));
  AIMX_API_END(c)
}

static aimx_status matvec_common(aimx_ctx* c, const void* x, void* y0, void* y1, int mode, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (!x || (mode == 0 && !y0) || (mode == 1 && !y0 && !y1))
    throw Error(AIMX_E_INVALID_ARG, "null vector");
  if (x == y0 || x == y1) throw Error(AIMX_E_INVALID_ARG, "input and output alias");
  if (!c->freq_set) throw Error(AIMX_E_STATE, "aimx_set_frequency has not been called");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  if (s != c->stream) AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_spec, 0));
  run_matvec(c, x, y0, y1, mode, s);
  AIMX_CUDA(cudaEventRecord(c->ev_use, s));
  AIMX_API_END(c)
}

aimx_status aimx_matvec(aimx_ctx* c, const void* x, void* y, void* stream) {
  return matvec_common(c, x, y, nullptr, 0, stream);
}

aimx_status aimx_matvec_parts(aimx_ctx* c, const void* x, void* yA, void* yPhi, void* stream) {
  return matvec_common(c, x, yA, yPhi, 1, stream);
}

static void sweep_impl(aimx_ctx* c, int64_t nf, const double* f, const char* X, char* Y, int B,
                       cudaStream_t s) {
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  for (int64_t i = 0; i < nf; i += B) {
    const int nb_ = (int)std::min<int64_t>(B, nf - i);
    run_batch(c, nb_, f + i, X + i * vb, Y + i * vb, s);
  }
}

static int sweep_batch(const aimx_ctx* c, int32_t batch) {
  int B = batch > 0 ? batch : c->hot.batch;
  return std::max(1, std::min(B, c->hot.batch));
}

aimx_status aimx_sweep(aimx_ctx* c, int64_t nf, const double* f_hz, const void* X, void* Y,
                       int32_t batch, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (nf < 0 || (nf > 0 && (!f_hz || !X || !Y))) throw Error(AIMX_E_INVALID_ARG, "bad sweep arguments");
  for (int64_t i = 0; i < nf; ++i)
    if (!(f_hz[i] > 0.0) || !std::isfinite(f_hz[i])) throw Error(AIMX_E_INVALID_ARG, "bad frequency");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  const bool had = c->freq_set;
  const double f0 = c->f;
  if (s != c->stream) {
    AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_spec, 0));
    AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_use, 0));
  }
  sweep_impl(c, nf, f_hz, (const char*)X, (char*)Y, sweep_batch(c, batch), s);
  if (had) bind_frequency(c, f0, s);
  else c->freq_set = false;
  AIMX_CUDA(cudaEventRecord(c->ev_spec, s));
  AIMX_CUDA(cudaEventRecord(c->ev_use, s));
  if (s != c->stream) AIMX_CUDA(cudaStreamWaitEvent(c->stream, c->ev_use, 0));
  AIMX_API_END(c)
}

aimx_status aimx_sweep_host(aimx_ctx* c, int64_t nf, const double* f_hz, const void* X, void* Y,
                            int32_t batch, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (nf < 0 || (nf > 0 && (!f_hz || !X || !Y))) throw Error(AIMX_E_INVALID_ARG, "bad sweep arguments");
  for (int64_t i = 0; i < nf; ++i)
    if (!(f_hz[i] > 0.0) || !std::isfinite(f_hz[i])) throw Error(AIMX_E_INVALID_ARG, "bad frequency");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  const int64_t B = sweep_batch(c, batch);
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  const int64_t need = 2 * B * (int64_t)vb;
  if (c->stage_bytes < need) {
    if (c->stage) AIMX_CUDA(cudaFree(c->stage));
    c->stage = nullptr;
    AIMX_CUDA(cudaMalloc(&c->stage, need));
    c->stage_bytes = need;
  }
  char* dX = (char*)c->stage;
  char* dY = dX + B * vb;
  const bool had = c->freq_set;
  const double f0 = c->f;
  if (s != c->stream) {
    AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_spec, 0));
    AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_use, 0));
  }
  for (int64_t i0 = 0; i0 < nf; i0 += B) {
    const int64_t nb_ = std::min(B, nf - i0);
    AIMX_CUDA(cudaMemcpyAsync(dX, (const char*)X + i0 * vb, nb_ * vb, cudaMemcpyHostToDevice, s));
    sweep_impl(c, nb_, f_hz + i0, dX, dY, (int)B, s);
    AIMX_CUDA(cudaMemcpyAsync((char*)Y + i0 * vb, dY, nb_ * vb, cudaMemcpyDeviceToHost, s));
  }
  if (had) bind_frequency(c, f0, s);
  else c->freq_set = false;
  AIMX_CUDA(cudaEventRecord(c->ev_spec, s));
  AIMX_CUDA(cudaEventRecord(c->ev_use, s));
  AIMX_CUDA(cudaStreamSynchronize(s));
  AIMX_API_END(c)
}

int64_t aimx_num_unknowns(const aimx_ctx* c) { return c ? c->topo.nb : -1; }

aimx_status aimx_get_stats(const aimx_ctx* c, aimx_stats* o) {
  if (!c || !o) return AIMX_E_INVALID_ARG;
  o->num_unknowns = c->topo.nb;
  o->nnz = c->topo.rowptr.empty() ? 0 : c->topo.rowptr.back();
  o->occupied_nodes = (int64_t)c->nodes.node_lin.size();
  o->occupied_lines = (int64_t)c->nodes.line_id.size();
  o->occupied_planes = (int64_t)c->nodes.zplanes.size();
  o->projection_entries = (int64_t)c->nodes.ent_rwg.size();
  o->device_bytes = c->dev_bytes;
  o->batch_slots = c->hot.batch;
  o->setup_seconds = c->setup_seconds;
  for (int a = 0; a < 3; ++a) { o->n[a] = c->topo.n[a]; o->origin[a] = c->topo.origin[a]; }
  o->order = c->topo.order;
  o->h = c->topo.h;
  o->near_group_rows = c->near_R;
  o->near_row_order = c->near_order;
  o->near_union = c->near_union;
  return AIMX_OK;
}

aimx_status aimx_get_rwg(const aimx_ctx* c, int32_t* edge_ab, int32_t* tri_pm, int32_t* free_pm) {
  if (!c) return AIMX_E_INVALID_ARG;
  const Topology& t = c->topo;
  for (int64_t e = 0; e < t.nb; ++e) {
    if (edge_ab) { edge_ab[2 * e] = t.ea[e]; edge_ab[2 * e + 1] = t.eb[e]; }
    if (tri_pm) { tri_pm[2 * e] = t.tp[e]; tri_pm[2 * e + 1] = t.tm[e]; }
    if (free_pm) { free_pm[2 * e] = t.pp[e]; free_pm[2 * e + 1] = t.pm[e]; }
  }
  return AIMX_OK;
}

aimx_status aimx_get_anchors(const aimx_ctx* c, int32_t* a) {
  if (!c || !a) return AIMX_E_INVALID_ARG;
  std::memcpy(a, c->topo.anchor.data(), c->topo.anchor.size() * sizeof(int32_t));
  return AIMX_OK;
}

aimx_status aimx_get_near_csr(const aimx_ctx* c, int64_t* rowptr, int32_t* col, int64_t* nnz) {
  if (!c) return AIMX_E_INVALID_ARG;
  const Topology& t = c->topo;
  if (nnz) *nnz = t.rowptr.back();
  if (rowptr) std::memcpy(rowptr, t.rowptr.data(), t.rowptr.size() * sizeof(int64_t));
  if (col) std::memcpy(col, t.col.data(), t.col.size() * sizeof(int32_t));
  return AIMX_OK;
}

aimx_status aimx_get_static(const aimx_ctx* cc, double* CA, double* Crho, double* LA_NR,
                            double* Yrho_NR, double* LA_P, double* Yrho_P) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  const size_t n = (size_t)c->topo.rowptr.back() * sizeof(double);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  if (CA) AIMX_CUDA(cudaMemcpy(CA, c->sd.CA, n, cudaMemcpyDeviceToHost));
  if (Crho) AIMX_CUDA(cudaMemcpy(Crho, c->sd.CR, n, cudaMemcpyDeviceToHost));
  if (LA_NR) AIMX_CUDA(cudaMemcpy(LA_NR, c->sd.LA_NR, n, cudaMemcpyDeviceToHost));
  if (Yrho_NR) AIMX_CUDA(cudaMemcpy(Yrho_NR, c->sd.YR_NR, n, cudaMemcpyDeviceToHost));
  if (LA_P) AIMX_CUDA(cudaMemcpy(LA_P, c->sd.LA_P, n, cudaMemcpyDeviceToHost));
  if (Yrho_P) AIMX_CUDA(cudaMemcpy(Yrho_P, c->sd.YR_P, n, cudaMemcpyDeviceToHost));
  AIMX_API_END(c)
}

aimx_status aimx_get_weights(const aimx_ctx* cc, double* lam) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c || !lam) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  const int64_t nb = c->topo.nb, p3 = c->topo.p3;
  std::vector<double> tmp((size_t)(nb * p3 * 4));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  AIMX_CUDA(cudaMemcpy(tmp.data(), c->sd.lam, tmp.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int64_t e = 0; e < nb; ++e)
    for (int64_t s = 0; s < p3; ++s)
      for (int ch = 0; ch < 4; ++ch) lam[(e * 4 + ch) * p3 + s] = tmp[(e * p3 + s) * 4 + ch];
  AIMX_API_END(c)
}

aimx_status aimx_get_spectrum(const aimx_ctx* cc, int which, double* out) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c || !out || (which != 0 && which != 1)) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (which == 1 && !c->freq_set) throw Error(AIMX_E_STATE, "no frequency bound");
  AIMX_CUDA(cudaSetDevice(c->device));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t n = c->sp.noct;
  if (which == 0) {
    AIMX_CUDA(cudaMemcpy(out, c->Hs, n * sizeof(double2), cudaMemcpyDeviceToHost));
  } else {
    const double M = 8.0 * (double)c->hot.Nx * c->hot.Ny * c->hot.Nz;
    if (c->prec == AIMX_C64) {
      std::vector<float2> tmp(n);
      AIMX_CUDA(cudaMemcpy(tmp.data(), c->hot.Hoct, n * sizeof(float2), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i) { out[2 * i] = tmp[i].x * M; out[2 * i + 1] = tmp[i].y * M; }
    } else {
      AIMX_CUDA(cudaMemcpy(out, c->hot.Hoct, n * sizeof(double2), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < 2 * n; ++i) out[i] *= M;
    }
  }
  AIMX_API_END(c)
}

aimx_status aimx_profile_enable(aimx_ctx* c, int on) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  c->prof.collect();
  c->prof.on = on != 0;
  launch_counter() = 0;
  AIMX_API_END(c)
}

aimx_status aimx_profile_read(aimx_ctx* c, double* ms, int64_t* launches, int64_t* kernels) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  c->prof.collect();
  if (kernels) *kernels = launch_counter();
  launch_counter() = 0;
  for (int i = 0; i < AIMX_NUM_STAGES; ++i) {
    if (ms) ms[i] = c->prof.ms[i];
    if (launches) launches[i] = c->prof.n[i];
    c->prof.ms[i] = 0;
    c->prof.n[i] = 0;
  }
  AIMX_API_END(c)
}

void aimx_destroy(aimx_ctx* c) { destroy_impl(c); }

const char* aimx_status_string(aimx_status s) {
  switch (s) {
    case AIMX_OK: return "ok";
    case AIMX_E_INVALID_ARG: return "invalid argument";
    case AIMX_E_MESH: return "mesh error";
    case AIMX_E_GRID: return "grid error";
    case AIMX_E_STATE: return "invalid state";
    case AIMX_E_OOM: return "out of memory";
    case AIMX_E_CUDA: return "CUDA error";
    case AIMX_E_UNSUPPORTED: return "unsupported configuration";
    case AIMX_E_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* aimx_last_error(const aimx_ctx* c) { return c ? c->last_error.c_str() : ""; }
const char* aimx_last_setup_error(void) { return g_setup_error.c_str(); }
const char* aimx_version(void) { return "aimx-b200 0.1 (sm_100a)"; }

}  // extern "C"
