// C ABI of the AIMx B200 library (include/aimx.h): context lifecycle, setup
// orchestration (host topology -> device fp64 static fill -> hot-path data),
// frequency binding, matvec / sweep entry points and introspection.
#include <algorithm>
#include <array>
#include <complex>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda.h>
#include <dlfcn.h>
#include <memory>

#include <nccl.h>   // types only: NCCL is loaded at run time (dlopen), see NcclApi

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
  // sweep pipeline: side stream for the next batch's spectra, double buffer
  cudaStream_t s2 = nullptr;
  void* HB[2] = {nullptr, nullptr};
  void* XT[2] = {nullptr, nullptr};            // interleaved columns of batches i, i+1
  cudaStream_t sc[2] = {nullptr, nullptr};   // host sweep copy streams (H2D, D2H)
  std::vector<cudaEvent_t> ev_io;
  cudaEvent_t ev_start = nullptr, ev_sp[2] = {nullptr, nullptr}, ev_mv[2] = {nullptr, nullptr};
  cudaEvent_t ev_xt[2] = {nullptr, nullptr};   // the batch's interleaved columns are ready
  // sweep pipeline, S4+S5 of batch i on s3 while the grid part of batch i+1 runs:
  cudaStream_t s3 = nullptr;
  cudaEvent_t ev_grid[2] = {nullptr, nullptr};
  void* PHI[2] = {nullptr, nullptr};          // potentials of batches i, i+1
  void* stage = nullptr;        // sweep_host staging
  int64_t stage_bytes = 0;
  double setup_seconds = 0;
  int near_R = 0, near_order = 0;
  int64_t near_union = 0;
  Profiler prof;
  std::vector<uint8_t> nz;      // exactly-nonzero projection weights [N_b][p3]
  bool from_cache = false;      // S0 static matrices read from an aimx_save_static file
  // batched GMRES (aimx_solve): static self terms and lazily allocated workspace
  double* dA = nullptr;         // L^A_s,NR[m,m]
  double* dR = nullptr;         // y^rho_s,NR[m,m]
  void* gm_ws = nullptr;
  int64_t gm_ws_bytes = 0;
  void* gm_host = nullptr;      // pinned Arnoldi-step values
  cudaEvent_t ev_gm = nullptr;  // their copy has landed
  size_t gm_host_bytes = 0;
  // slab-decomposed FFT (aimx_setup_slab)
  bool slab = false;
  int world = 1, rank = 0;
  std::vector<std::array<int, 5>> plans;   // per rank: y0, y1, yh1, kx0, kx1
  std::vector<SlabRank> slabs;             // emulation: all ranks; NCCL: this rank
  std::unique_ptr<SlabExchange> xchg;
  void* comm = nullptr;                    // ncclComm_t
  bool nccl_dead = false;                  // the communicator was aborted (sticky AIMX_E_NCCL)
  int slots = 0;
  bool planar = false;          // one occupied z plane: the 2-D S3 path (HotDev::planar)
  void* Hoct = nullptr;         // bound spectra [slots][noct], compute precision, scaled 1/M
  // linear-term modification (aimx_set_linear_term), built on first use
  int32_t* lin_col = nullptr;   // [nb][kLinW] overlapping columns
  void* lin_c = nullptr;        // [nb][kLinW] (C^A_lin, C^rho_lin), compute precision
  bool lin_on = false;
  // CUDA graphs of single matvecs (run_matvec): keyed by buffers, mode and
  // frequency, captured when a key repeats (GMRES-style reuse), at most 8
  struct MvGraph {
    const void* x; void* y0; void* y1; int mode; double f;
    cudaGraphExec_t exec; int64_t launches;
  };
  std::vector<MvGraph> graphs;
  MvGraph last_mv{nullptr, nullptr, nullptr, -1, 0.0, nullptr, 0};
  cudaStream_t cap = nullptr;   // capture stream
  // double-layer operator K (aimx_set_kop, NEXT #1)
  bool kop_on = false;
  double2* HsF = nullptr;       // static spectra of K's grid part, fp64: the gradient form's
                                // d_a G_s (a = x, y, z; [3][noct]) or the radial F_s = 1/(4 pi r^3)
  void* HsF_T = nullptr;        // ... compute precision (c64)
  bool kgrad = false;           // K through the gradient-of-kernel spectra (else the radial form)
  void* HF = nullptr;           // F_hat of the bound frequency (slot 0), scaled 1/M
  void* kphi1 = nullptr;        // F (*) J and F (*) (s x J), phi layout
  void* kphi2 = nullptr;
  void* ck_T = nullptr;         // C_K (compute precision, CSR order)
  bool cfie_on = false;         // aimx_set_cfie: matvec / sweep / solve apply -j w mu0 L - eta0 K
  void* ktmp = nullptr;         // [nb] K x
  void* ckpv_T = nullptr;       // C_K without the residue (PMCHWT), compute precision
  void* pm_H1 = nullptr;        // PMCHWT: spectra of the interior medium (H_hat, F_hat)
  void* pm_HF1 = nullptr;
  void* pm_t = nullptr;         // [3][nb] temporaries
  // conventional AIM mode (aimx_set_conventional): D(k0) on the near pattern
  bool aim_on = false;
  void* aimDA = nullptr;        // [nnz] compute precision complex
  void* aimDR = nullptr;
  std::vector<void*> allocs;
  std::vector<std::unique_ptr<CUtensorMap>> tmaps;   // tensor maps referenced by HotDev::tmB
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
  if (i >= n || slot[i] < 0) return;   // entries of rows outside this context's groups
  T2 v;
  v.x = CA[i];
  v.y = CR[i];
  *reinterpret_cast<T2*>(payload + slot[i]) = v;
}
__global__ void k_d2f_real(int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = (float)a[i];
}

__global__ void k_d2f(int64_t n, const double2* __restrict__ a, float2* __restrict__ b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  b[i] = make_float2((float)a[i].x, (float)a[i].y);
}

unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

// flag[i] = 1 if column i of Y ([nf][n] complex, as reals) holds a non-finite value
template <typename R>
__global__ void k_nonfinite(int64_t n2, int64_t nf, const R* __restrict__ Y, int32_t* flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n2 * nf) return;
  if (!isfinite(Y[i])) flag[i / n2] = 1;   // benign race: every writer stores 1
}

// flag = 1 if any weight of channel c is non-zero (lam [n][4], fp64)
__global__ void k_chan_nonzero(int64_t n, const double* __restrict__ lam, int c, int* flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && lam[4 * i + c] != 0.0) atomicOr(flag, 1);
}

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

// ---- S0 common part: topology, fp64 static fill, weights, full node map
// ---- static-setup cache (the frequency-independent near matrix is
// stored and reused across sweeps).  Key: FNV-1a of the mesh arrays and the
// grid descriptor (h and origin after derivation); payload: the fp64 static
// matrices in CSR order, the projection weights and their exact-zero flags.
constexpr char kCacheMagic[8] = {'A', 'I', 'M', 'X', 'S', 'T', 'A', 'T'};
constexpr int64_t kCacheVersion = 1;

uint64_t static_key(const Topology& t) {
  uint64_t hsh = 1469598103934665603ull;
  auto mix = [&](const void* p, size_t n) {
    const unsigned char* b = (const unsigned char*)p;
    for (size_t i = 0; i < n; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
  };
  mix(t.V.data(), t.V.size() * sizeof(double));
  mix(t.T.data(), t.T.size() * sizeof(int32_t));
  mix(t.n, sizeof(t.n));
  mix(&t.order, sizeof(t.order));
  mix(&t.near_cells, sizeof(t.near_cells));
  mix(&t.h, sizeof(t.h));
  mix(t.origin, sizeof(t.origin));
  return hsh;
}

struct CacheHeader {
  char magic[8];
  int64_t version, key, nb, nnz, p3;
};

void setup_static(aimx_ctx* c, const aimx_mesh_desc* mesh, const aimx_grid_desc* grid,
                  const char* cache = nullptr) {
  Topology& t = c->topo;
  build_topology(mesh, grid, t);
  if (cache) {   // the topology is rebuilt (cheap, integer) and must match the file
    std::FILE* fp = std::fopen(cache, "rb");
    if (!fp) throw Error(AIMX_E_INVALID_ARG, std::string("cannot open static cache ") + cache);
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(fp, std::fclose);
    CacheHeader hd;
    if (std::fread(&hd, sizeof(hd), 1, fp) != 1 || std::memcmp(hd.magic, kCacheMagic, 8) != 0 ||
        hd.version != kCacheVersion)
      throw Error(AIMX_E_INVALID_ARG, "not an AIMx static cache (or another version)");
    if ((uint64_t)hd.key != static_key(t) || hd.nb != t.nb || hd.nnz != t.rowptr[t.nb] || hd.p3 != t.p3)
      throw Error(AIMX_E_INVALID_ARG, "static cache was written for another mesh or grid");
    for (int a = 0; a < 3; ++a)
      if (!fft_length_supported(2 * t.n[a]))
        throw Error(AIMX_E_UNSUPPORTED, "2*N_a must be a power of two in [8, 1024]");
    const int64_t nb = t.nb, nnz = t.rowptr[nb], p3 = t.p3;
    SetupDev& d = c->sd;
    d.anchor = dupload(c, t.anchor);
    d.rowptr = dupload(c, t.rowptr);
    d.col = dupload(c, t.col);
    std::vector<double> buf((size_t)std::max<int64_t>(nnz, nb * p3 * 4));
    auto read_up = [&](double*& dst, int64_t n) {
      if (std::fread(buf.data(), sizeof(double), (size_t)n, fp) != (size_t)n)
        throw Error(AIMX_E_INVALID_ARG, "static cache truncated");
      dst = dalloc<double>(c, n);
      AIMX_CUDA(cudaMemcpy(dst, buf.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    };
    read_up(d.CA, nnz);
    read_up(d.CR, nnz);
    read_up(d.LA_NR, nnz);
    read_up(d.YR_NR, nnz);
    read_up(d.LA_P, nnz);
    read_up(d.YR_P, nnz);
    read_up(d.lam, nb * p3 * 4);
    c->nz.resize((size_t)(nb * p3));
    if (std::fread(c->nz.data(), 1, c->nz.size(), fp) != c->nz.size())
      throw Error(AIMX_E_INVALID_ARG, "static cache truncated");
    d.LA_un = dalloc<double>(c, 1);
    d.YR_un = dalloc<double>(c, 1);
    build_nodemap(t, c->nz, c->nodes);
    c->slots = 0;
    c->from_cache = true;
    return;
  }
  for (int a = 0; a < 3; ++a)
    if (!fft_length_supported(2 * t.n[a]))
      throw Error(AIMX_E_UNSUPPORTED, "2*N_a must be a power of two in [8, 1024]");
  const int64_t nb = t.nb, nnz = t.rowptr[nb], p3 = t.p3;
  SetupDev& d = c->sd;
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
  c->nz.resize((size_t)(nb * p3));
  AIMX_CUDA(cudaMemcpyAsync(c->nz.data(), nzf, c->nz.size(), cudaMemcpyDeviceToHost, c->stream));
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
  build_nodemap(t, c->nz, c->nodes);
  c->slots = 0;
}

// geometry common to every HotDev of the context
void hot_common(aimx_ctx* c, HotDev& h) {
  const Topology& t = c->topo;
  h.Nx = t.n[0]; h.Ny = t.n[1]; h.Nz = t.n[2];
  h.W = 8 * h.Nx;
  h.p = t.p; h.p3 = t.p3;
  h.nb = (int)t.nb;
  h.nnz = t.rowptr[t.nb];
}

// S2 gather structures of a node map (node-major projection entries)
void build_gather(aimx_ctx* c, HotDev& h, const NodeMap& m) {
  const Topology& t = c->topo;
  h.nocc = (int)m.node_lin.size();
  h.nlines = (int)m.line_id.size();
  h.nzocc = (int)m.zplanes.size();
  h.node_lin = dupload(c, m.node_lin);
  h.node_ptr = dupload(c, m.node_ptr);
  h.node_line = dupload(c, m.node_line);
  h.ent_rwg = dupload(c, m.ent_rwg);
  if (h.planar) {   // bufA / bufC hold the one occupied plane: line id = y
    std::vector<int32_t> lid(m.line_id);
    for (auto& v : lid) v -= m.zplanes[0] * t.n[1];
    h.line_id = dupload(c, lid);
  } else {
    h.line_id = dupload(c, m.line_id);
  }
  h.zplanes = dupload(c, m.zplanes);
  h.zplane0 = m.zplanes.empty() ? 0 : m.zplanes[0];
  h.line_occ = dupload(c, m.line_occ);
  std::vector<uint8_t> zo(t.n[2], 0);
  for (int z : m.zplanes) zo[z] = 1;
  h.zocc = dupload(c, zo);
  const int64_t nent = (int64_t)m.ent_rwg.size();
  int32_t* ent_slot = dupload(c, m.ent_slot);
  if (nent == 0) {   // a slab rank whose rows hold no occupied node
    h.ent_w = dalloc<double4>(c, 1);
  } else if (c->prec == AIMX_C64) {
    h.ent_w = dalloc<float4>(c, nent);
    k_ent_w<float4><<<nblk(nent), 256, 0, c->stream>>>(nent, (int)t.p3, h.ent_rwg, ent_slot, c->sd.lam,
                                                      (float4*)h.ent_w);
  } else {
    h.ent_w = dalloc<double4>(c, nent);
    k_ent_w<double4><<<nblk(nent), 256, 0, c->stream>>>(nent, (int)t.p3, h.ent_rwg, ent_slot, c->sd.lam,
                                                       (double4*)h.ent_w);
  }
  if (nent > 0) AIMX_CHECK_LAUNCH();
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  dfree(c, ent_slot, nent * (int64_t)sizeof(int32_t));
  const double avg = h.nocc > 0 ? (double)nent / h.nocc : 1.0;
  int G = 4;
  // four to eight entries per lane: loads in flight per lane hide the gather
  // latency and the shuffle reduction stays a small share (measured: cfg3 G = 4
  // 69 us, 8 73, 16 81, 32 106 for gather + x fwd)
  // ... unless that leaves too few threads to fill the GPU (cfg2: 8448 nodes
  // want 32 lanes each)
  while (G < 32 && (8 * G <= avg || (int64_t)h.nocc * G < 148 * 2048)) G *= 2;
  if (const char* e = std::getenv("AIMX_GATHER_G")) G = std::max(4, std::min(32, std::atoi(e)));   // experiments
  h.G = G;
}

// S4+S5 structures for the testing functions `rows` (empty: all)
void build_near(aimx_ctx* c, HotDev& h, const std::vector<int32_t>& rows) {
  const Topology& t = c->topo;
  const int64_t nb = t.nb, nnz = t.rowptr[nb], p3 = t.p3;
  std::vector<int32_t> base(nb);
  for (int64_t e = 0; e < nb; ++e)
    base[e] = t.anchor[3 * e] + t.n[0] * (t.anchor[3 * e + 1] + t.n[1] * t.anchor[3 * e + 2]);
  h.rwg_base = dupload(c, base);
  NearGroups grp;
  build_near_groups(t, c->nz, grp, rows);
  if (h.planar)   // phi holds the occupied plane only
    for (auto& v : grp.wnode) v -= (int32_t)h.phi_off;
  if (grp.ptr.back() > (int64_t)INT32_MAX || grp.wptr.back() > (int64_t)INT32_MAX)
    throw Error(AIMX_E_GRID, "near matrix too large");
  h.R = grp.R;
  h.ngrp = (int)grp.ngrp;
  h.grp_rows = dupload(c, grp.rows);
  int nsm = 148;
  AIMX_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  NearChunks ck;
  const bool f32 = c->prec == AIMX_C64;
  const int cs = f32 ? 8 : 16;
  if (c->slots <= 0) throw Error(AIMX_E_INTERNAL, "batch slots not chosen before the near layout");
  std::vector<int64_t> cta_begin;
  // one wave of resident CTAs (AIMX_NEAR_SMS: spread over fewer SMs, experiments)
  int nsm_near = nsm;
  if (const char* e = std::getenv("AIMX_NEAR_SMS")) nsm_near = std::max(1, std::min(nsm, std::atoi(e)));
  // AIMX_NEAR_MMA=1: batched c64 launches on the legacy tensor path (measured
  // slower; the same chunk layout and 5 CTAs per SM)
  const char* mm = std::getenv("AIMX_NEAR_MMA");
  h.near_mma = (f32 && grp.R == 8 && mm && mm[0] == '1') ? 1 : 0;
  h.near_half = c->slots >= 32 ? 1 : 0;
  { const char* o1 = getenv("AIMX_NEAR1_OLD"); h.near1_old = (o1 && o1[0] == '1') ? 1 : 0; }
  int per_sm = near_ctas_per_sm(f32, false, grp.R);   // AIMX_NEAR_PER_SM: fewer (experiments)
  if (const char* e = std::getenv("AIMX_NEAR_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
  const int ncta = per_sm * nsm_near;
  const std::vector<int64_t> order = near_round_order(grp.ngrp, ncta, cta_begin);
  build_near_chunks(grp, near_chw(f32, c->slots), near_chc(f32, c->slots), cs, ck, order);
  // value slot (u R + r) -> payload byte offset
  for (auto& v : grp.slot)
    if (v >= 0) v = ck.uoff_c[v / grp.R] + (v % grp.R) * cs;
  for (auto& v : grp.wslot)
    if (v >= 0) v = ck.uoff_w[v / grp.R] + (v % grp.R) * 2 * cs;
  int64_t* gslot = dupload(c, grp.slot);
  int64_t* wslot = dupload(c, grp.wslot);
  h.payload = dupload(c, ck.payload);
  h.chunks = dupload(c, ck.chunks);
  // chunk range of each CTA (its groups are contiguous in `order`)
  std::vector<int32_t> cp(cta_begin.size());
  for (size_t k = 0; k + 1 < cta_begin.size(); ++k)
    cp[k] = cta_begin[k] < grp.ngrp ? (int32_t)ck.gfirst[order[cta_begin[k]]] : (int32_t)ck.nchunk;
  cp.back() = (int32_t)ck.nchunk;
  h.cta_ptr = dupload(c, cp);
  h.near_ctas = (int)cp.size() - 1;
  h.cta_ptr1 = h.cta_ptr;   // single-column launches: the same order and CTAs
  h.near_ctas1 = h.near_ctas;
  if (f32 && grp.R == 8 && h.near_half && !h.near1_old && !std::getenv("AIMX_NEAR_PER_SM")) {
    // k_interp_near1 keeps 8 CTAs per SM resident on half-length chunks: the
    // same chunk stream cut into that many contiguous ranges of whole groups
    // with equal chunk counts
    const int n1 = near1_ctas_per_sm(true) * nsm_near;
    std::vector<int32_t> gb((size_t)grp.ngrp + 1);   // first chunk of each group in payload order
    for (int64_t i = 0; i < grp.ngrp; ++i) gb[(size_t)i] = (int32_t)ck.gfirst[order[(size_t)i]];
    gb.back() = (int32_t)ck.nchunk;
    if (!std::is_sorted(gb.begin(), gb.end())) throw Error(AIMX_E_INTERNAL, "near chunks not in group order");
    std::vector<int32_t> cp1((size_t)n1 + 1);
    for (int j = 0; j <= n1; ++j) {
      const int32_t target = (int32_t)((int64_t)ck.nchunk * j / n1);
      cp1[(size_t)j] = *std::lower_bound(gb.begin(), gb.end(), target);
    }
    h.cta_ptr1 = dupload(c, cp1);
    h.near_ctas1 = n1;
    // k_interp_near1w: one range per warp, 4 CTAs of 4 warps per SM
    // (AIMX_NEAR1_WARP=0: keep the CTA-per-range kernel, A/B)
    const char* w1 = std::getenv("AIMX_NEAR1_WARP");
    if (!(w1 && w1[0] == '0')) {
      const int nw = 16 * nsm_near;
      std::vector<int32_t> wp((size_t)nw + 1);
      for (int j = 0; j <= nw; ++j) {
        const int32_t target = (int32_t)((int64_t)ck.nchunk * j / nw);
        wp[(size_t)j] = *std::lower_bound(gb.begin(), gb.end(), target);
      }
      h.warp_ptr1 = dupload(c, wp);
      h.near_warps1 = nw;
    }
  }
  const SetupDev& d = c->sd;
  if (f32) {
    k_lam_to<float4><<<nblk(nb * p3), 256, 0, c->stream>>>(nb * p3, wslot, d.lam, (float4*)nullptr, h.payload);
    k_pack_c<float2><<<nblk(nnz), 256, 0, c->stream>>>(nnz, gslot, d.CA, d.CR, (float2*)nullptr, h.payload);
  } else {
    k_lam_to<double4><<<nblk(nb * p3), 256, 0, c->stream>>>(nb * p3, wslot, d.lam, (double4*)nullptr, h.payload);
    k_pack_c<double2><<<nblk(nnz), 256, 0, c->stream>>>(nnz, gslot, d.CA, d.CR, (double2*)nullptr, h.payload);
  }
  AIMX_CHECK_LAUNCH();
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  dfree(c, gslot, nnz * (int64_t)sizeof(int64_t));
  dfree(c, wslot, nb * p3 * (int64_t)sizeof(int64_t));
  if (rows.empty() || c->near_R == 0) {
    c->near_R = grp.R;
    c->near_order = grp.order_kind;
  }
  c->near_union += grp.ptr.back();
}

// TMA tensor map of a HotDev's bufB for the z pass (AIMX_NO_TMA=1 disables)
void attach_z_map(aimx_ctx* c, HotDev& h) {
  if (std::getenv("AIMX_NO_TMA")) return;
  std::unique_ptr<CUtensorMap> m(new CUtensorMap);
  if (make_z_tensor_map(h, c->prec == AIMX_C64, m.get())) {
    h.tmB = m.get();
    c->tmaps.push_back(std::move(m));
  }
}

// static self terms for the diagonal preconditioner
void setup_self_terms(aimx_ctx* c) {
  const Topology& t = c->topo;
  std::vector<int64_t> di(t.nb);
  for (int64_t m = 0; m < t.nb; ++m) {
    di[m] = -1;
    for (int64_t k = t.rowptr[m]; k < t.rowptr[m + 1]; ++k)
      if (t.col[k] == m) di[m] = k;
    if (di[m] < 0) throw Error(AIMX_E_INTERNAL, "near row without its diagonal");
  }
  int64_t* d_di = dupload(c, di);
  c->dA = dalloc<double>(c, t.nb);
  c->dR = dalloc<double>(c, t.nb);
  gm_take(t.nb, d_di, c->sd.LA_NR, c->dA, c->stream);
  gm_take(t.nb, d_di, c->sd.YR_NR, c->dR, c->stream);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  dfree(c, d_di, t.nb * (int64_t)sizeof(int64_t));
}

// batch slots from the full-grid per-frequency footprint (<= 1.5 GB of buffers)
int choose_slots(aimx_ctx* c) {
  const Topology& t = c->topo;
  const size_t cs = c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2);
  const int64_t Nx = t.n[0], Ny = t.n[1], Nz = t.n[2];
  const int64_t nS = (int64_t)c->nodes.line_id.size() * Nx * 4;
  const int64_t nz = c->planar ? 1 : Nz;   // planes held by bufA / bufC / phi
  const int64_t nA = nz * Ny * 2 * Nx * 4, nB = c->planar ? 0 : Nz * 2 * Ny * 2 * Nx * 4, nP = Nx * Ny * nz * 4;
  const int64_t noct = (Nx + 1) * (Ny + 1) * (c->planar ? 1 : Nz + 1);
  // S, bufA, bufC, bufB, phi (double-buffered), the spectra (bound + 2 sweep
  // buffers) and the spectrum plan's two fp64 work octants
  const int64_t per_freq = (int64_t)cs * (nS + 2 * nA + nB + 2 * nP + 3 * noct) + 2 * (int64_t)sizeof(double2) * noct;
  // per-frequency grid buffers within 12 GB (of 180 GB): cfg3 gets 8 slots, its
  // 16-point sweep +17% over 2 slots (round 1: 1566 / 1691 / 1827 / 1730
  // freq-pts/s at 2 / 4 / 8 / 16); planar cfg5 32
  int slots = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxBatch, (int64_t)(12288ll << 20) / per_freq));
  if (const char* e = std::getenv("AIMX_BATCH")) slots = std::max(1, std::min(kMaxBatch, std::atoi(e)));
  while (slots & (slots - 1)) slots &= slots - 1;   // power of two (batch buckets never exceed it)
  return slots;
}

template <typename P> P* zalloc(aimx_ctx* c, int64_t bytes) {
  P* p = (P*)dalloc<char>(c, bytes);
  AIMX_CUDA(cudaMemsetAsync(p, 0, bytes, c->stream));
  return p;
}

// static spectrum (fp64, and its compute-precision copy) and the spectrum plan
void setup_spectrum(aimx_ctx* c) {
  const Topology& t = c->topo;
  c->sp.Nx = t.n[0]; c->sp.Ny = t.n[1]; c->sp.Nz = t.n[2]; c->sp.h = t.h;
  c->sp.nz1 = c->planar ? 1 : t.n[2] + 1;
  spectrum_plan_init(c->sp, c->slots, c->stream);
  const int64_t noct = c->sp.noct;
  c->Hs = dalloc<double2>(c, noct);
  spectrum_static(c->sp, c->Hs, c->stream);
  if (c->prec == AIMX_C64) {
    c->Hs_T = dalloc<float2>(c, noct);
    k_d2f<<<nblk(noct), 256, 0, c->stream>>>(noct, c->Hs, (float2*)c->Hs_T);
    AIMX_CHECK_LAUNCH();
  } else {
    c->Hs_T = c->Hs;
  }
  const size_t cs = c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2);
  c->Hoct = dalloc<char>(c, noct * c->slots * (int64_t)cs);
}

void finish_setup(aimx_ctx* c) {
  const Topology& t = c->topo;
  const int64_t nnz = c->from_cache ? 1 : t.rowptr[t.nb];
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  dfree(c, c->sd.LA_un, nnz * (int64_t)sizeof(double));
  dfree(c, c->sd.YR_un, nnz * (int64_t)sizeof(double));
  AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_spec, cudaEventDisableTiming));
  AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_use, cudaEventDisableTiming));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
}

void do_setup(aimx_ctx* c, const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, const char* cache = nullptr) {
  setup_static(c, mesh, grid, cache);
  const Topology& t = c->topo;
  HotDev& h = c->hot;
  hot_common(c, h);
  // planar grids (one occupied z plane): the exact 2-D form of S3 (SURVEY
  // 8(d) pruning); AIMX_NO_PLANAR=1 keeps the general 3-D path
  c->planar = c->nodes.zplanes.size() == 1 && !std::getenv("AIMX_NO_PLANAR");
  if (c->planar) {
    h.planar = 1;
    h.phi_off = (int64_t)c->nodes.zplanes[0] * h.Nx * h.Ny;
    // a mesh in a z plane has f_z = 0, so Lambda^z is exactly zero: the z
    // channel of the grid is never transformed (reading R12)
    int* flag = dalloc<int>(c, 1);
    AIMX_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), c->stream));
    const int64_t nw = (int64_t)t.nb * t.p3;
    k_chan_nonzero<<<nblk(nw), 256, 0, c->stream>>>(nw, c->sd.lam, 2, flag);
    AIMX_CHECK_LAUNCH();
    int hf = 1;
    AIMX_CUDA(cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    AIMX_CUDA(cudaStreamSynchronize(c->stream));
    dfree(c, flag, (int64_t)sizeof(int));
    // and the grid buffers store 3 channels (x, y, rho): a quarter less of
    // every grid pass and of the potential gathers
    if (hf == 0 && !std::getenv("AIMX_NO_ZSKIP")) {
      h.nc = 3;
      h.W = 2 * h.Nx * 3;
    }
  }
  const int slots = c->slots = choose_slots(c);
  build_gather(c, h, c->nodes);
  build_near(c, h, {});
  // ---- batch slots and grid buffers
  const size_t cs = c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2);
  const int64_t nzb = c->planar ? 1 : h.Nz;   // planes held by bufA / bufC / phi
  const int64_t nS = (int64_t)h.nlines * h.Nx * 4;
  const int64_t nA = nzb * h.Ny * 2 * h.Nx * 4;
  const int64_t nB = c->planar ? 0 : (int64_t)h.Nz * 2 * h.Ny * 2 * h.Nx * 4;
  const int64_t nP = (int64_t)h.Nx * h.Ny * nzb * 4;
  const int64_t noct = (int64_t)(h.Nx + 1) * (h.Ny + 1) * (c->planar ? 1 : h.Nz + 1);
  h.batch = slots;
  h.sS = nS; h.sA = nA; h.sB = nB; h.sP = nP; h.sH = noct;
  h.S = zalloc<char>(c, nS * slots * (int64_t)cs);
  h.bufA = zalloc<char>(c, nA * slots * (int64_t)cs);
  h.bufB = nB ? zalloc<char>(c, nB * slots * (int64_t)cs) : nullptr;
  h.bufC = zalloc<char>(c, nA * slots * (int64_t)cs);
  h.phi = zalloc<char>(c, nP * slots * (int64_t)cs + 64);
  h.twx = make_twiddles(c, 2 * h.Nx);
  h.twy_tab = make_twiddles(c, 2 * h.Ny);
  h.twz_tab = make_twiddles(c, 2 * h.Nz);
  if (!c->planar) attach_z_map(c, h);
  setup_spectrum(c);
  h.Hoct = c->Hoct;
  {
    for (int k = 0; k < 2; ++k) c->HB[k] = dalloc<char>(c, noct * slots * (int64_t)cs);
    for (int k = 0; k < 2; ++k) c->XT[k] = dalloc<char>(c, (int64_t)t.nb * kMaxBatch * (int64_t)cs + 64);
    // stream priorities (experiments: AIMX_PRIO_S2 / AIMX_PRIO_S3, 0 = default, 1 = high, -1 = low)
    int plo = 0, phi_ = 0;
    AIMX_CUDA(cudaDeviceGetStreamPriorityRange(&plo, &phi_));
    auto prio = [&](const char* env) {
      const char* e = std::getenv(env);
      const int v = e ? std::atoi(e) : 0;
      return v > 0 ? phi_ : (v < 0 ? plo : 0);
    };
    AIMX_CUDA(cudaStreamCreateWithPriority(&c->s2, cudaStreamNonBlocking, prio("AIMX_PRIO_S2")));
    AIMX_CUDA(cudaStreamCreateWithPriority(&c->s3, cudaStreamNonBlocking, prio("AIMX_PRIO_S3")));
    AIMX_CUDA(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));   // CUDA-graph capture (run_matvec)
    AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming));
    for (int k = 0; k < 2; ++k) {
      AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_sp[k], cudaEventDisableTiming));
      AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_xt[k], cudaEventDisableTiming));
      AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_mv[k], cudaEventDisableTiming));
      AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_grid[k], cudaEventDisableTiming));
    }
    c->PHI[0] = h.phi;
    c->PHI[1] = zalloc<char>(c, nP * slots * (int64_t)cs + 64);
  }
  h.xt = dalloc<char>(c, (int64_t)t.nb * kMaxBatch * (int64_t)cs + 64);
  setup_self_terms(c);
  finish_setup(c);
}

// ---- NCCL, loaded at run time (the library itself does not link it)
struct NcclApi {
  void* lib = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclCommGetAsyncError) getAsyncError = nullptr;
  decltype(&ncclCommAbort) commAbort = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char* n : names)
      if ((api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL)) != nullptr) break;
    if (!api.lib) return;
    api.getUniqueId = (decltype(api.getUniqueId))dlsym(api.lib, "ncclGetUniqueId");
    api.commInitRank = (decltype(api.commInitRank))dlsym(api.lib, "ncclCommInitRank");
    api.commDestroy = (decltype(api.commDestroy))dlsym(api.lib, "ncclCommDestroy");
    api.send = (decltype(api.send))dlsym(api.lib, "ncclSend");
    api.recv = (decltype(api.recv))dlsym(api.lib, "ncclRecv");
    api.groupStart = (decltype(api.groupStart))dlsym(api.lib, "ncclGroupStart");
    api.groupEnd = (decltype(api.groupEnd))dlsym(api.lib, "ncclGroupEnd");
    api.allReduce = (decltype(api.allReduce))dlsym(api.lib, "ncclAllReduce");
    api.errorString = (decltype(api.errorString))dlsym(api.lib, "ncclGetErrorString");
    api.getAsyncError = (decltype(api.getAsyncError))dlsym(api.lib, "ncclCommGetAsyncError");
    api.commAbort = (decltype(api.commAbort))dlsym(api.lib, "ncclCommAbort");
  });
  if (!api.lib || !api.getUniqueId || !api.commInitRank || !api.send || !api.recv || !api.groupStart ||
      !api.groupEnd || !api.allReduce)
    throw Error(AIMX_E_UNSUPPORTED, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}
#define AIMX_NCCL(call)                                                                        \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      throw Error(AIMX_E_NCCL, std::string("NCCL: ") + (nccl().errorString ? nccl().errorString(r_) : "error")); \
  } while (0)

// Exchange geometry.  Step 0 (rows -> kx slabs): rank p sends rank q the
// block [slot][z][y in p's rows][4 kx in q's slab] of its x-transformed rows;
// q stores it in rows y0_p.. of its column buffer.  Step 1 (kx slabs -> rows):
// rank q sends rank p the block [slot][z][y in [y0_p, yh1_p)][4 kx in q's slab]
// of its y-inverse buffer; p stores it at kx0_q of its row buffer.
struct XchgGeom {
  const aimx_ctx* c;
  int64_t Nz, Ny, Nx;
  int64_t rows(int p, int step) const { const auto& q = c->plans[p]; return step == 0 ? q[1] - q[0] : q[2] - q[0]; }
  int64_t W(int q) const { return 4 * (int64_t)(c->plans[q][4] - c->plans[q][3]); }
  // complex per block from src to dst for B slots
  int64_t block(int src, int dst, int step, int B) const {
    return step == 0 ? B * Nz * rows(src, 0) * W(dst) : B * Nz * rows(dst, 1) * W(src);
  }
  int64_t send_off(int src, int dst, int step, int B) const {
    int64_t o = 0;
    for (int q = 0; q < dst; ++q) o += block(src, q, step, B);
    return o;
  }
  int64_t recv_off(int dst, int src, int step, int B) const {
    int64_t o = 0;
    for (int p = 0; p < src; ++p) o += block(p, dst, step, B);
    return o;
  }
  void pack(SlabRank& r, int dst, int step, int B, size_t cs, cudaStream_t s) const {
    const int p = r.rank;
    char* out = (char*)r.send + send_off(p, dst, step, B) * (int64_t)cs;
    const int64_t Wd = W(dst), Wp = W(p);
    if (step == 0) {   // from the row buffer (x-transformed rows) -> [B][Nz][rows_p][W_dst]
      const int64_t rp = rows(p, 0);
      const int64_t d[4] = {B, Nz, rp, Wd}, so[3] = {r.hr.sA, rp * 8 * Nx, 8 * Nx}, to[3] = {Nz * rp * Wd, rp * Wd, Wd};
      copy4(out, to, (const char*)r.hr.bufA + 4 * (int64_t)c->plans[dst][3] * (int64_t)cs, so, d, cs, s);
    } else {           // from the column buffer rows [y0_dst, yh1_dst) -> [B][Nz][rows_dst][W_p]
      const int64_t rd = rows(dst, 1);
      const int64_t d[4] = {B, Nz, rd, Wp}, so[3] = {r.hc.sA, Ny * Wp, Wp}, to[3] = {Nz * rd * Wp, rd * Wp, Wp};
      copy4(out, to, (const char*)r.hc.bufC + (int64_t)c->plans[dst][0] * Wp * (int64_t)cs, so, d, cs, s);
    }
  }
  void unpack(SlabRank& r, int src, int step, int B, size_t cs, cudaStream_t s) const {
    const int q = r.rank;
    const char* in = (const char*)r.recv + recv_off(q, src, step, B) * (int64_t)cs;
    if (step == 0) {   // [B][Nz][rows_src][W_q] -> column buffer rows y0_src..
      const int64_t rs = rows(src, 0), Wq = W(q);
      const int64_t d[4] = {B, Nz, rs, Wq}, so[3] = {Nz * rs * Wq, rs * Wq, Wq}, to[3] = {r.hc.sA, Ny * Wq, Wq};
      copy4((char*)r.hc.bufA + (int64_t)c->plans[src][0] * Wq * (int64_t)cs, to, in, so, d, cs, s);
    } else {           // [B][Nz][rows_q][W_src] -> row buffer at kx0_src
      const int64_t rq = rows(q, 1), Ws = W(src);
      const int64_t d[4] = {B, Nz, rq, Ws}, so[3] = {Nz * rq * Ws, rq * Ws, Ws}, to[3] = {r.hx.sA, rq * 8 * Nx, 8 * Nx};
      copy4((char*)r.hx.bufC + 4 * (int64_t)c->plans[src][3] * (int64_t)cs, to, in, so, d, cs, s);
    }
  }
};

// all ranks in this process: pack, device copies between the virtual ranks, unpack
struct EmulatedExchange : SlabExchange {
  XchgGeom g;
  explicit EmulatedExchange(const XchgGeom& g_) : g(g_) {}
  void run(std::vector<SlabRank*>& ranks, int step, int B, size_t cs, cudaStream_t s) override {
    const int P = (int)ranks.size();
    for (SlabRank* r : ranks)
      for (int q = 0; q < P; ++q) g.pack(*r, q, step, B, cs, s);
    for (SlabRank* src : ranks)
      for (SlabRank* dst : ranks) {
        const int64_t n = g.block(src->rank, dst->rank, step, B);
        if (n > 0)
          AIMX_CUDA(cudaMemcpyAsync((char*)dst->recv + g.recv_off(dst->rank, src->rank, step, B) * (int64_t)cs,
                                    (const char*)src->send + g.send_off(src->rank, dst->rank, step, B) * (int64_t)cs,
                                    n * cs, cudaMemcpyDeviceToDevice, s));
      }
    for (SlabRank* r : ranks)
      for (int p = 0; p < P; ++p) g.unpack(*r, p, step, B, cs, s);
  }
};

// this process is one rank: pack, grouped ncclSend / ncclRecv, unpack
struct NcclExchange : SlabExchange {
  XchgGeom g;
  int world;
  ncclComm_t comm;
  NcclExchange(const XchgGeom& g_, int w, ncclComm_t cm) : g(g_), world(w), comm(cm) {}
  void run(std::vector<SlabRank*>& ranks, int step, int B, size_t cs, cudaStream_t s) override {
    SlabRank& r = *ranks[0];
    for (int q = 0; q < world; ++q) g.pack(r, q, step, B, cs, s);
    NcclApi& api = nccl();
    AIMX_NCCL(api.groupStart());
    for (int q = 0; q < world; ++q) {
      const int64_t ns = g.block(r.rank, q, step, B) * (int64_t)cs, nr = g.block(q, r.rank, step, B) * (int64_t)cs;
      if (ns > 0)
        AIMX_NCCL(api.send((const char*)r.send + g.send_off(r.rank, q, step, B) * (int64_t)cs, (size_t)ns,
                           ncclInt8, q, comm, s));
      if (nr > 0)
        AIMX_NCCL(api.recv((char*)r.recv + g.recv_off(r.rank, q, step, B) * (int64_t)cs, (size_t)nr, ncclInt8,
                           q, comm, s));
    }
    AIMX_NCCL(api.groupEnd());
    for (int p = 0; p < world; ++p) g.unpack(r, p, step, B, cs, s);
  }
};

void do_setup_slab(aimx_ctx* c, const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, int rank, int world,
                   const uint8_t* nccl_id) {
  setup_static(c, mesh, grid);
  const Topology& t = c->topo;
  const int Nx = t.n[0], Ny = t.n[1], Nz = t.n[2];
  c->slab = true;
  c->world = world;
  c->rank = nccl_id ? rank : 0;
  for (int r = 0; r < world; ++r) {
    int32_t o[6];
    aimx_status st = aimx_slab_plan(t.n, t.order, world, r, o);
    if (st != AIMX_OK) throw Error(st, "slab plan: 2 N_x / world must be a power of two and N_y >= world");
    c->plans.push_back({o[0], o[1], o[2], o[3], o[4]});
  }
  hot_common(c, c->hot);
  const int slots = c->slots = choose_slots(c);
  c->hot.batch = slots;
  setup_spectrum(c);
  const bool f32 = c->prec == AIMX_C64;
  const size_t cs = f32 ? sizeof(float2) : sizeof(double2);
  const int64_t noct = (int64_t)(Nx + 1) * (Ny + 1) * (Nz + 1);
  const NodeMap& full = c->nodes;
  std::vector<uint8_t> zo(Nz, 0);
  for (int z : full.zplanes) zo[z] = 1;
  XchgGeom geo{c, Nz, Ny, Nx};
  std::vector<int> mine;
  if (nccl_id) mine.push_back(rank);
  else for (int r = 0; r < world; ++r) mine.push_back(r);
  c->slabs.resize(mine.size());
  for (size_t i = 0; i < mine.size(); ++i) {
    SlabRank& R = c->slabs[i];
    const auto& pl = c->plans[mine[i]];
    R.rank = mine[i];
    R.y0 = pl[0]; R.y1 = pl[1]; R.yh1 = pl[2]; R.kx0 = pl[3]; R.kx1 = pl[4];
    const int ny = R.y1 - R.y0, nyh = R.yh1 - R.y0, W = 4 * (R.kx1 - R.kx0);
    // rows: gather + x fwd, S4+S5 of the RWGs anchored in the rows
    HotDev& hr = R.hr;
    hot_common(c, hr);
    NodeMap m;
    nodemap_rows(t, full, R.y0, R.y1, m);
    build_gather(c, hr, m);
    std::vector<int32_t>& owned = R.owned;
    for (int64_t e = 0; e < t.nb; ++e)
      if (t.anchor[3 * e + 1] >= R.y0 && t.anchor[3 * e + 1] < R.y1) owned.push_back((int32_t)e);
    if (!owned.empty()) build_near(c, hr, owned);
    hr.batch = slots;
    hr.sS = (int64_t)hr.nlines * Nx * 4;
    hr.sA = (int64_t)Nz * ny * 2 * Nx * 4;
    hr.sP = (int64_t)Nx * Ny * Nz * 4;
    hr.S = zalloc<char>(c, hr.sS * slots * (int64_t)cs + 64);
    hr.bufA = zalloc<char>(c, hr.sA * slots * (int64_t)cs);
    hr.phi = zalloc<char>(c, hr.sP * slots * (int64_t)cs + 64);
    hr.twx = make_twiddles(c, 2 * Nx);
    hr.xt = dalloc<char>(c, (int64_t)t.nb * kMaxBatch * (int64_t)cs + 64);
    // kx slab: y / z passes over all (y, z)
    HotDev& hc = R.hc;
    hot_common(c, hc);
    hc.W = W;
    hc.kx0 = R.kx0;
    hc.nzocc = (int)full.zplanes.size();
    hc.zplanes = dupload(c, full.zplanes);
    hc.zplane0 = full.zplanes.empty() ? 0 : full.zplanes[0];
    hc.zocc = dupload(c, zo);
    hc.line_occ = dupload(c, full.line_occ);
    hc.batch = slots;
    hc.sA = (int64_t)Nz * Ny * W;
    hc.sB = (int64_t)Nz * 2 * Ny * W;
    hc.sH = noct;
    hc.bufA = zalloc<char>(c, hc.sA * slots * (int64_t)cs);
    hc.bufB = zalloc<char>(c, hc.sB * slots * (int64_t)cs);
    hc.bufC = zalloc<char>(c, hc.sA * slots * (int64_t)cs);
    hc.Hoct = c->Hoct;
    hc.twy_tab = make_twiddles(c, 2 * Ny);
    hc.twz_tab = make_twiddles(c, 2 * Nz);
    attach_z_map(c, hc);
    // x inverse of rows [y0, yh1) into phi (global line numbering)
    HotDev& hx = R.hx;
    hot_common(c, hx);
    std::vector<int32_t> lid, plid;
    for (int32_t line : full.line_id) {
      const int y = line % Ny, z = line / Ny;
      if (y >= R.y0 && y < R.yh1) {
        lid.push_back((y - R.y0) + nyh * z);
        plid.push_back(line);
      }
    }
    hx.nlines = (int)lid.size();
    hx.line_id = dupload(c, lid);
    hx.phi_line = dupload(c, plid);
    hx.batch = slots;
    hx.sA = (int64_t)Nz * nyh * 2 * Nx * 4;
    hx.bufC = zalloc<char>(c, hx.sA * slots * (int64_t)cs);
    hx.phi = hr.phi;
    hx.twx = hr.twx;
    // exchange staging: the larger of the two steps, send and receive
    int64_t sn = 0, rn = 0;
    for (int step = 0; step < 2; ++step) {
      int64_t a = 0, b = 0;
      for (int q = 0; q < world; ++q) {
        a += geo.block(R.rank, q, step, slots);
        b += geo.block(q, R.rank, step, slots);
      }
      sn = std::max(sn, a);
      rn = std::max(rn, b);
    }
    R.send = dalloc<char>(c, sn * (int64_t)cs + 64);
    R.recv = dalloc<char>(c, rn * (int64_t)cs + 64);
  }
  if (nccl_id) {
    NcclApi& api = nccl();
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclComm_t comm = nullptr;
    AIMX_NCCL(api.commInitRank(&comm, world, id, rank));
    c->comm = comm;
    c->xchg.reset(new NcclExchange(geo, world, comm));
  } else {
    c->xchg.reset(new EmulatedExchange(geo));
  }
  finish_setup(c);
}

// Normalisation folded into the bound spectra: the inverse DFT's 1/M, M the
// padded grid size (planar: the padded plane, 4 N_x N_y).
double spectrum_scale(const aimx_ctx* c) {
  const HotDev& h = c->hot;
  return c->planar ? 1.0 / (4.0 * (double)h.Nx * h.Ny) : 1.0 / (8.0 * (double)h.Nx * h.Ny * h.Nz);
}

// S1 for B frequency points into spectrum slots 0..B-1.
void spectra(aimx_ctx* c, int B, const double* f, cudaStream_t s, void* out = nullptr) {
  if (!out) out = c->Hoct;
  double k0[kMaxBatch];
  for (int b = 0; b < B; ++b) {
    if (!(f[b] > 0.0) || !std::isfinite(f[b])) throw Error(AIMX_E_INVALID_ARG, "frequency must be finite and > 0");
    k0[b] = 2.0 * kPi * f[b] / kC0;
  }
  const double sc1 = spectrum_scale(c);
  StageScope sc(&c->prof, 0, s);
  if (c->prec == AIMX_C64)
    spectrum_dynamic_f32(c->sp, B, k0, (const float2*)c->Hs_T, (float)sc1, (float2*)out, s);
  else
    spectrum_dynamic_f64(c->sp, B, k0, c->Hs, sc1, (double2*)out, s);
}

// K's spectra at f into c->HF: the three gradient spectra d_a G_hat(k0)
// ([3][noct], kinds 2-4, odd along a), or the radial F_hat(k0) (kind 1)
void kop_spectrum(aimx_ctx* c, double f, cudaStream_t s, void* out = nullptr) {
  if (!out) out = c->HF;
  double k0[1] = {2.0 * kPi * f / kC0};
  const double sc1 = spectrum_scale(c);
  const int64_t noct = c->sp.noct;
  for (int a = 0; a < (c->kgrad ? 3 : 1); ++a) {
    const int kind = c->kgrad ? 2 + a : 1;
    if (c->prec == AIMX_C64)
      spectrum_dynamic_f32(c->sp, 1, k0, (const float2*)c->HsF_T + a * noct, (float)sc1,
                           (float2*)out + a * noct, s, kind);
    else
      spectrum_dynamic_f64(c->sp, 1, k0, c->HsF + a * noct, sc1, (double2*)out + a * noct, s, kind);
  }
}

void bind_frequency(aimx_ctx* c, double f, cudaStream_t s) {
  spectra(c, 1, &f, s);
  if (c->kop_on) kop_spectrum(c, f, s);
  c->f = f;
  c->k0 = 2.0 * kPi * f / kC0;
  c->omega = 2.0 * kPi * f;
  c->freq_set = true;
  if (c->aim_on)   // conventional AIM: the per-frequency near fill
    launch_aim_fill(c->topo, c->sd, c->k0, c->prec == AIMX_C64, c->aimDA, c->aimDR, s);
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

// slab contexts: every rank's part; NCCL: owned rows summed over ranks
void run_slab(aimx_ctx* c, const void* x, void* y0, void* y1, const Combine& cb, cudaStream_t s) {
  const size_t cs = c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2);
  const size_t ybytes = (size_t)cb.B * c->hot.nb * cs;
  if (c->comm) {   // rows owned elsewhere stay zero before the sum
    if (y0) AIMX_CUDA(cudaMemsetAsync(y0, 0, ybytes, s));
    if (y1) AIMX_CUDA(cudaMemsetAsync(y1, 0, ybytes, s));
  }
  std::vector<SlabRank*> rk;
  for (auto& r : c->slabs) rk.push_back(&r);
  slab_matvec(rk, c->topo.n[1], c->topo.n[2], c->topo.n[0], c->prec == AIMX_C64, *c->xchg, x, y0, y1, cb, s,
              &c->prof);
  if (c->comm) {
    NcclApi& api = nccl();
    const ncclDataType_t dt = c->prec == AIMX_C64 ? ncclFloat32 : ncclFloat64;
    const size_t n = (size_t)cb.B * c->hot.nb * 2;
    AIMX_NCCL(api.groupStart());
    if (y0) AIMX_NCCL(api.allReduce(y0, y0, n, dt, ncclSum, (ncclComm_t)c->comm, s));
    if (y1) AIMX_NCCL(api.allReduce(y1, y1, n, dt, ncclSum, (ncclComm_t)c->comm, s));
    AIMX_NCCL(api.groupEnd());
  }
}

// HotDev for a B-column launch: the potentials laid out for the power-of-two
// column bucket of B (the kernels' bucket; <= the slots), not for all slots,
// so small batches read dense node rows
HotDev batch_view(const aimx_ctx* c, int B) {
  HotDev h = c->hot;
  int b = 1;
  while (b < B) b <<= 1;
  h.batch = std::min(h.batch, b);
  return h;
}

void clear_graphs(aimx_ctx* c) {
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  c->last_mv = {nullptr, nullptr, nullptr, -1, 0.0, nullptr, 0};
}

void run_matvec(aimx_ctx* c, const void* x, void* y0, void* y1, int mode, cudaStream_t s) {
  Combine cb = make_combine(1, &c->f, mode, c->hot.nb);
  if (c->slab) return run_slab(c, x, y0, y1, cb, s);
  // one column: the potentials compact ([node][channel], batch 1), so the
  // interpolation's node rows are dense whatever the context's slot count
  HotDev h1 = c->hot;
  h1.batch = 1;
  auto eager = [&](cudaStream_t q) {
    if (c->prec == AIMX_C64) hot_matvec_f32(h1, x, y0, y1, cb, q, &c->prof);
    else hot_matvec_f64(h1, x, y0, y1, cb, q, &c->prof);
    if (c->aim_on)
      aim_spmv(c->prec == AIMX_C64, c->hot.nb, c->sd.rowptr, c->sd.col, c->aimDA, c->aimDR, x, y0, y1, cb, q);
    if (c->cfie_on && mode == 0) {   // eq:CFIEdis P:422: (-j w mu0 L - eta0 K) x
      kop_matvec(c->prec == AIMX_C64, c->hot, x, c->ktmp, c->HF, c->kphi1, c->kphi2, c->sd.lam, c->topo.h,
                 c->sd.rowptr, c->sd.col, c->ck_T, q, c->kgrad);
      gm_axpy(c->prec == AIMX_C64, c->hot.nb, -kMu0 * kC0, c->ktmp, y0, q);
    }
  };
  if (c->prof.on || std::getenv("AIMX_NO_GRAPH")) return eager(s);
  auto same = [&](const aimx_ctx::MvGraph& g) {
    return g.x == x && g.y0 == y0 && g.y1 == y1 && g.mode == mode && g.f == c->f;
  };
  for (auto& g : c->graphs)
    if (same(g)) {   // replay: the kernels' launch latencies go away
      AIMX_CUDA(cudaGraphLaunch(g.exec, s));
      launch_counter() += g.launches;
      return;
    }
  const bool repeat = same(c->last_mv);
  c->last_mv = {x, y0, y1, mode, c->f, nullptr, 0};
  if (!repeat) return eager(s);
  const int64_t n0 = launch_counter();
  AIMX_CUDA(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeRelaxed));
  cudaGraph_t graph = nullptr;
  try {
    eager(c->cap);
  } catch (...) {
    cudaStreamEndCapture(c->cap, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  AIMX_CUDA(cudaStreamEndCapture(c->cap, &graph));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  AIMX_CUDA(e);
  if (c->graphs.size() >= 8) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back({x, y0, y1, mode, c->f, exec, launch_counter() - n0});
  AIMX_CUDA(cudaGraphLaunch(exec, s));
}

// B frequency points: spectra into slots, then one batched matvec.
void run_batch(aimx_ctx* c, int B, const double* f, const void* X, void* Y, cudaStream_t s) {
  if (c->aim_on || c->cfie_on) {   // conventional AIM / CFIE: per frequency
    const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
    for (int b = 0; b < B; ++b) {
      bind_frequency(c, f[b], s);
      run_matvec(c, (const char*)X + b * vb, (char*)Y + b * vb, nullptr, 0, s);
    }
    return;
  }
  spectra(c, B, f, s);
  Combine cb = make_combine(B, f, 0, c->hot.nb);
  if (c->slab) return run_slab(c, X, Y, nullptr, cb, s);
  const HotDev hb = batch_view(c, B);
  if (c->prec == AIMX_C64) hot_matvec_f32(hb, X, Y, nullptr, cb, s, &c->prof);
  else hot_matvec_f64(hb, X, Y, nullptr, cb, s, &c->prof);
}

aimx_status fail(aimx_ctx* c, const Error& e) {
  if (c) c->last_error = e.what();
  return e.code;
}

// abort the context's NCCL communicator (a hung or failed peer must not
// deadlock this rank); later calls return AIMX_E_NCCL
void nccl_abort(aimx_ctx* c, const std::string& why) {
  if (c->comm && !c->nccl_dead) {
    NcclApi& api = nccl();
    if (api.commAbort) api.commAbort((ncclComm_t)c->comm);
    c->comm = nullptr;
  }
  c->nccl_dead = true;
  c->last_error = why;
}

// asynchronous NCCL error of the context's communicator, if any
void poll_nccl(aimx_ctx* c) {
  if (c->nccl_dead) throw Error(AIMX_E_NCCL, "the NCCL communicator was aborted");
  if (!c->comm) return;
  NcclApi& api = nccl();
  if (!api.getAsyncError) return;
  ncclResult_t r = ncclSuccess;
  if (api.getAsyncError((ncclComm_t)c->comm, &r) != ncclSuccess || (r != ncclSuccess && r != ncclInProgress)) {
    const std::string why = std::string("NCCL asynchronous error: ") + (api.errorString ? api.errorString(r) : "?");
    nccl_abort(c, why);
    throw Error(AIMX_E_NCCL, why);
  }
}

void check_sticky(aimx_ctx* c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(AIMX_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
  poll_nccl(c);
}

cudaStream_t pick(aimx_ctx* c, void* s) { return s ? (cudaStream_t)s : c->stream; }

// Stream ordering (include/aimx.h): every call that enqueues work waits, on
// its stream, for the spectra it reads (ev_spec) and for the last call that
// used the context's buffers on any stream (ev_use); when done it records
// ev_use (and ev_spec if it rewrote the bound spectra) and, on a user stream,
// makes the context stream wait for it.  So calls on different streams never
// overlap on the shared buffers (S, bufA-C, phi, xt, the spectra).  A wait on
// an event last recorded on the same stream costs nothing.
void enter_stream(aimx_ctx* c, cudaStream_t s) {
  AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_spec, 0));
  AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_use, 0));
}
void leave_stream(aimx_ctx* c, cudaStream_t s, bool spec_written = false) {
  if (spec_written) AIMX_CUDA(cudaEventRecord(c->ev_spec, s));
  AIMX_CUDA(cudaEventRecord(c->ev_use, s));
  if (s != c->stream) AIMX_CUDA(cudaStreamWaitEvent(c->stream, c->ev_use, 0));
}
// host-side state changes (set_kop / cfie / linear term / conventional):
// every call in flight on any stream has finished
void quiesce(aimx_ctx* c) {
  AIMX_CUDA(cudaEventSynchronize(c->ev_use));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
}

void destroy_impl(aimx_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm) {
    try {
      nccl().commDestroy((ncclComm_t)c->comm);
    } catch (...) {
    }
  }
  clear_graphs(c);
  if (c->cap) cudaStreamDestroy(c->cap);
  for (void* p : c->allocs) if (p) cudaFree(p);
  spectrum_plan_free(c->sp);
  if (c->stage) cudaFree(c->stage);
  if (c->gm_ws) cudaFree(c->gm_ws);
  if (c->gm_host) cudaFreeHost(c->gm_host);
  if (c->ev_gm) cudaEventDestroy(c->ev_gm);
  if (c->ev_spec) cudaEventDestroy(c->ev_spec);
  if (c->ev_use) cudaEventDestroy(c->ev_use);
  for (cudaStream_t q : {c->s2, c->s3})
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (int k = 0; k < 2; ++k)
    if (c->sc[k]) {
      cudaStreamSynchronize(c->sc[k]);
      cudaStreamDestroy(c->sc[k]);
    }
  for (cudaEvent_t e : c->ev_io) cudaEventDestroy(e);
  for (cudaEvent_t e : {c->ev_start, c->ev_sp[0], c->ev_sp[1], c->ev_mv[0], c->ev_mv[1], c->ev_grid[0], c->ev_grid[1],
                        c->ev_xt[0], c->ev_xt[1]})
    if (e) cudaEventDestroy(e);
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

aimx_status aimx_setup_slab(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, aimx_prec prec, int device,
                            int32_t rank, int32_t world, const uint8_t* nccl_id, void* stream, aimx_ctx** out) {
  g_setup_error.clear();
  if (!out) { g_setup_error = "out is NULL"; return AIMX_E_INVALID_ARG; }
  *out = nullptr;
  if (prec != AIMX_C64 && prec != AIMX_C128) { g_setup_error = "bad precision"; return AIMX_E_INVALID_ARG; }
  if (world < 1 || rank < 0 || rank >= world) { g_setup_error = "bad rank / world"; return AIMX_E_INVALID_ARG; }
  aimx_ctx* c = nullptr;
  try {
    auto t0 = std::chrono::steady_clock::now();
    AIMX_CUDA(cudaSetDevice(device));
    c = new aimx_ctx;
    c->device = device;
    c->prec = prec;
    c->stream = (cudaStream_t)stream;
    do_setup_slab(c, mesh, grid, rank, world, nccl_id);
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

aimx_status aimx_setup_cached(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, aimx_prec prec, int device,
                              const char* path, void* stream, aimx_ctx** out) {
  g_setup_error.clear();
  if (!out || !path) { g_setup_error = "out or path is NULL"; return AIMX_E_INVALID_ARG; }
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
    do_setup(c, mesh, grid, path);
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

aimx_status aimx_save_static(const aimx_ctx* cc, const char* path) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c || !path) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  const Topology& t = c->topo;
  const int64_t nb = t.nb, nnz = t.rowptr[nb], p3 = t.p3;
  std::FILE* fp = std::fopen(path, "wb");
  if (!fp) throw Error(AIMX_E_INVALID_ARG, std::string("cannot write ") + path);
  std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(fp, std::fclose);
  CacheHeader hd;
  std::memcpy(hd.magic, kCacheMagic, 8);
  hd.version = kCacheVersion;
  hd.key = (int64_t)static_key(t);
  hd.nb = nb;
  hd.nnz = nnz;
  hd.p3 = p3;
  bool ok = std::fwrite(&hd, sizeof(hd), 1, fp) == 1;
  std::vector<double> buf((size_t)std::max<int64_t>(nnz, nb * p3 * 4));
  auto put = [&](const double* src, int64_t n) {
    AIMX_CUDA(cudaMemcpy(buf.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost));
    ok = ok && std::fwrite(buf.data(), sizeof(double), (size_t)n, fp) == (size_t)n;
  };
  const SetupDev& d = c->sd;
  put(d.CA, nnz);
  put(d.CR, nnz);
  put(d.LA_NR, nnz);
  put(d.YR_NR, nnz);
  put(d.LA_P, nnz);
  put(d.YR_P, nnz);
  put(d.lam, nb * p3 * 4);
  ok = ok && std::fwrite(c->nz.data(), 1, c->nz.size(), fp) == c->nz.size();
  if (!ok) throw Error(AIMX_E_INVALID_ARG, std::string("write failed: ") + path);
  AIMX_API_END(c)
}

// ---- batched GMRES (right-preconditioned, restarted)
// One device batch of B frequencies iterates together; every column has its
// own Arnoldi basis, Hessenberg matrix and Givens rotations (host, fp64).
// Arnoldi: classical Gram-Schmidt applied twice (CGS2: two batched dot /
// update sweeps per step instead of j dependent ones).
static void solve_batch(aimx_ctx* c, int B, const double* f, const char* RHS, char* X, double tol, int m,
                        int maxit, int32_t* iters, double* relres, cudaStream_t s) {
  const bool f32 = c->prec == AIMX_C64;
  const int64_t N = c->hot.nb;
  const size_t cs = f32 ? sizeof(float2) : sizeof(double2);
  const int64_t blk = (int64_t)B * N;   // complex per [B][N] block
  // workspace: V[m+1] blocks, W, U, R blocks; device scalars
  const int64_t need = (int64_t)(m + 4) * blk * (int64_t)cs + (int64_t)(m + 2) * B * 16 * 4 + B * 8 * 2;
  if (c->gm_ws_bytes < need) {
    if (c->gm_ws) AIMX_CUDA(cudaFree(c->gm_ws));
    c->gm_ws = nullptr;
    AIMX_CUDA(cudaMalloc(&c->gm_ws, need));
    c->gm_ws_bytes = need;
  }
  char* V = (char*)c->gm_ws;
  char* W = V + (int64_t)(m + 1) * blk * cs;
  char* U = W + blk * cs;
  char* Rb = U + blk * cs;
  double2* ddots = (double2*)(Rb + blk * cs);
  double2* dcoef = ddots + (int64_t)(m + 2) * B;
  double2* dit = dcoef + (int64_t)(m + 2) * B;   // one Arnoldi step: [h pass 1 | h pass 2 | |w|^2]
  double* dsc = (double*)(dit + (int64_t)(2 * m + 4) * B);
  std::vector<double2> hd((size_t)(m + 2) * B);
  // pinned host copy of dit: one synchronisation per Arnoldi step
  const size_t hit_bytes = (size_t)(2 * m + 4) * B * sizeof(double2);
  if (c->gm_host_bytes < hit_bytes) {
    if (c->gm_host) AIMX_CUDA(cudaFreeHost(c->gm_host));
    c->gm_host = nullptr;
    AIMX_CUDA(cudaMallocHost(&c->gm_host, hit_bytes));
    c->gm_host_bytes = hit_bytes;
  }
  double2* hit = (double2*)c->gm_host;
  if (!c->ev_gm) AIMX_CUDA(cudaEventCreateWithFlags(&c->ev_gm, cudaEventDisableTiming));
  std::vector<double> hs(B);
  spectra(c, B, f, s);
  Combine cb = make_combine(B, f, 0, N);
  PcArgs pa;
  for (int b = 0; b < kMaxBatch; ++b) pa.alpha_im[b] = pa.beta[b] = 0.0;
  for (int b = 0; b < B; ++b) {
    pa.alpha_im[b] = cb.alpha_im[b];
    pa.beta[b] = cb.beta[b];
  }
  if (c->aim_on) {   // conventional AIM: this frequency's near fill (one column per batch)
    if (B != 1) throw Error(AIMX_E_INTERNAL, "conventional AIM solve runs one frequency per batch");
    launch_aim_fill(c->topo, c->sd, 2.0 * kPi * f[0] / kC0, f32, c->aimDA, c->aimDR, s);
  }
  if (c->cfie_on) {   // CFIE: this frequency's F spectrum
    if (B != 1) throw Error(AIMX_E_INTERNAL, "CFIE solve runs one frequency per batch");
    kop_spectrum(c, f[0], s);
  }
  const HotDev hsv = batch_view(c, B);
  auto matvec = [&](const void* in, void* out) {
    if (f32) hot_matvec_f32(hsv, in, out, nullptr, cb, s, &c->prof);
    else hot_matvec_f64(hsv, in, out, nullptr, cb, s, &c->prof);
    if (c->aim_on) aim_spmv(f32, N, c->sd.rowptr, c->sd.col, c->aimDA, c->aimDR, in, out, nullptr, cb, s);
    if (c->cfie_on) {
      kop_matvec(f32, c->hot, in, c->ktmp, c->HF, c->kphi1, c->kphi2, c->sd.lam, c->topo.h, c->sd.rowptr,
                 c->sd.col, c->ck_T, s, c->kgrad);
      gm_axpy(f32, N, -kMu0 * kC0, c->ktmp, out, s);
    }
  };
  auto norms = [&](const void* A, std::vector<double>& out) {   // ||A_b||
    gm_dots(f32, 1, B, N, A, 0, A, ddots, s);
    AIMX_CUDA(cudaMemcpyAsync(hd.data(), ddots, B * sizeof(double2), cudaMemcpyDeviceToHost, s));
    AIMX_CUDA(cudaStreamSynchronize(s));
    out.resize(B);
    for (int b = 0; b < B; ++b) out[b] = std::sqrt(std::max(0.0, hd[b].x));
  };
  auto colscale = [&](const void* A, const std::vector<double>& sc, void* out) {
    AIMX_CUDA(cudaMemcpyAsync(dsc, sc.data(), B * sizeof(double), cudaMemcpyHostToDevice, s));
    gm_colscale(f32, B, N, A, dsc, out, s);
  };
  using cd = std::complex<double>;
  std::vector<double> bnorm, beta;
  norms(RHS, bnorm);
  AIMX_CUDA(cudaMemsetAsync(X, 0, blk * cs, s));
  std::vector<int> it(B, 0), done(B, 0);
  for (int b = 0; b < B; ++b)
    if (bnorm[b] == 0.0) done[b] = 1;
  AIMX_CUDA(cudaMemcpyAsync(Rb, RHS, blk * cs, cudaMemcpyDeviceToDevice, s));
  int total = 0;
  while (total < maxit) {
    norms(Rb, beta);
    bool all = true;
    for (int b = 0; b < B; ++b) {
      if (!done[b] && beta[b] <= tol * bnorm[b]) done[b] = 1;
      all = all && done[b];
    }
    if (all) break;
    std::vector<double> inv(B);
    for (int b = 0; b < B; ++b) inv[b] = (done[b] || beta[b] == 0.0) ? 0.0 : 1.0 / beta[b];
    colscale(Rb, inv, V);   // v_0
    std::vector<std::vector<cd>> H(B, std::vector<cd>((size_t)(m + 1) * m, 0.0));
    std::vector<std::vector<cd>> csn(B, std::vector<cd>(2 * m, 0.0)), g(B, std::vector<cd>(m + 1, 0.0));
    std::vector<int> kb(B, 0), conv(B, 0);
    for (int b = 0; b < B; ++b) g[b][0] = done[b] ? 0.0 : beta[b];
    int j = 0;
    bool pre = false;   // the step's preconditioned matvec is already queued
    for (; j < m && total < maxit; ++j, ++total) {
      char* Vj = V + (int64_t)j * blk * cs;
      if (!pre) {
        gm_pc(f32, B, N, Vj, U, c->dA, c->dR, pa, false, s);
        matvec(U, W);
      }
      pre = false;
      // CGS2: h = V^H w ; w -= V h ; twice (coefficients stay on the device),
      // then |w|^2 and v_{j+1} = w / |w| on the device; ONE copy + sync
      const int64_t hs_ = (int64_t)(j + 1) * B;
      for (int pass = 0; pass < 2; ++pass) {
        gm_dots(f32, j + 1, B, N, V, blk, W, dit + pass * hs_, s);
        gm_lincomb(f32, j + 1, B, N, V, blk, dit + pass * hs_, W, false, s);
      }
      gm_dots(f32, 1, B, N, W, 0, W, dit + 2 * hs_, s);
      gm_colscale_rsqrt(f32, B, N, W, dit + 2 * hs_, V + (int64_t)(j + 1) * blk * cs, s);
      AIMX_CUDA(cudaMemcpyAsync(hit, dit, (size_t)(2 * hs_ + B) * sizeof(double2), cudaMemcpyDeviceToHost, s));
      AIMX_CUDA(cudaEventRecord(c->ev_gm, s));
      // look ahead: the next step's M^-1 v_{j+1} and its matvec need nothing
      // from the host, so they run while the host does this step's rotations
      if (j + 1 < m && total + 1 < maxit) {
        gm_pc(f32, B, N, V + (int64_t)(j + 1) * blk * cs, U, c->dA, c->dR, pa, false, s);
        matvec(U, W);
        pre = true;
      }
      AIMX_CUDA(cudaEventSynchronize(c->ev_gm));
      for (int pass = 0; pass < 2; ++pass)
        for (int b = 0; b < B; ++b)
          for (int i = 0; i <= j; ++i)
            H[b][(size_t)i * m + j] += cd(hit[pass * hs_ + (int64_t)i * B + b].x, hit[pass * hs_ + (int64_t)i * B + b].y);
      std::vector<double> hn(B);
      for (int b = 0; b < B; ++b) hn[b] = std::sqrt(std::max(0.0, hit[2 * hs_ + b].x));
      for (int b = 0; b < B; ++b) {
        if (done[b] || conv[b]) continue;
        cd* Hb = H[b].data();
        Hb[(size_t)(j + 1) * m + j] = hn[b];
        for (int i = 0; i < j; ++i) {   // previous rotations [[conj c, conj s], [-s, c]]
          const cd ci = csn[b][2 * i], si = csn[b][2 * i + 1];
          const cd t = std::conj(ci) * Hb[(size_t)i * m + j] + std::conj(si) * Hb[(size_t)(i + 1) * m + j];
          Hb[(size_t)(i + 1) * m + j] = -si * Hb[(size_t)i * m + j] + ci * Hb[(size_t)(i + 1) * m + j];
          Hb[(size_t)i * m + j] = t;
        }
        const cd a = Hb[(size_t)j * m + j], bb = Hb[(size_t)(j + 1) * m + j];
        const double den = std::sqrt(std::norm(a) + std::norm(bb));
        const cd cj = den != 0.0 ? a / den : cd(1.0), sj = den != 0.0 ? bb / den : cd(0.0);
        csn[b][2 * j] = cj;
        csn[b][2 * j + 1] = sj;
        Hb[(size_t)j * m + j] = den;
        Hb[(size_t)(j + 1) * m + j] = 0.0;
        g[b][j + 1] = -sj * g[b][j];
        g[b][j] = std::conj(cj) * g[b][j];
        kb[b] = j + 1;
        it[b] += 1;
        if (std::abs(g[b][j + 1]) <= tol * bnorm[b]) conv[b] = 1;
      }
      bool cyc_done = true;
      for (int b = 0; b < B; ++b) cyc_done = cyc_done && (done[b] || conv[b]);
      if (cyc_done) {
        ++total;
        break;
      }
    }
    // y = H^-1 g per column (back substitution), x += M^-1 V y
    int kmax = 0;
    for (int b = 0; b < B; ++b) kmax = std::max(kmax, done[b] ? 0 : kb[b]);
    if (kmax > 0) {
      std::vector<double2> coef((size_t)kmax * B, make_double2(0.0, 0.0));
      for (int b = 0; b < B; ++b) {
        if (done[b]) continue;
        const int k = kb[b];
        std::vector<cd> y(k);
        for (int i = k - 1; i >= 0; --i) {
          cd acc = g[b][i];
          for (int l = i + 1; l < k; ++l) acc -= H[b][(size_t)i * m + l] * y[l];
          y[i] = acc / H[b][(size_t)i * m + i];
        }
        for (int i = 0; i < k; ++i) coef[(size_t)i * B + b] = make_double2(y[i].real(), y[i].imag());
      }
      AIMX_CUDA(cudaMemcpyAsync(dcoef, coef.data(), coef.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
      gm_lincomb(f32, kmax, B, N, V, blk, dcoef, U, true, s);
      gm_pc(f32, B, N, U, X, c->dA, c->dR, pa, true, s);
    }
    // true residual for the restart / the convergence test
    matvec(X, W);
    gm_sub(f32, blk, RHS, W, Rb, s);
  }
  std::vector<double> rn;
  norms(Rb, rn);
  for (int b = 0; b < B; ++b) {
    if (iters) iters[b] = it[b];
    if (relres) relres[b] = bnorm[b] > 0.0 ? rn[b] / bnorm[b] : 0.0;
  }
}

static int sweep_batch(const aimx_ctx* c, int32_t batch, int64_t nf);

aimx_status aimx_solve(aimx_ctx* c, int64_t nf, const double* f_hz, const void* RHS, void* X, double tol,
                       int32_t restart, int32_t maxiter, int32_t* iters, double* relres, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (nf < 0 || (nf > 0 && (!f_hz || !RHS || !X)) || !(tol > 0.0) || restart < 1 || maxiter < 1)
    throw Error(AIMX_E_INVALID_ARG, "bad solve arguments");
  if (RHS == X) throw Error(AIMX_E_INVALID_ARG, "input and output alias");
  if (c->slab || !c->dA) throw Error(AIMX_E_UNSUPPORTED, "aimx_solve needs a one-GPU context");
  for (int64_t i = 0; i < nf; ++i)
    if (!(f_hz[i] > 0.0) || !std::isfinite(f_hz[i])) throw Error(AIMX_E_INVALID_ARG, "bad frequency");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  enter_stream(c, s);
  const bool had = c->freq_set;
  const double f0 = c->f;
  const int B = (c->aim_on || c->cfie_on) ? 1 : sweep_batch(c, 0, nf);   // AIM / CFIE: one frequency at a time
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  for (int64_t i = 0; i < nf; i += B) {
    const int nb_ = (int)std::min<int64_t>(B, nf - i);
    solve_batch(c, nb_, f_hz + i, (const char*)RHS + i * vb, (char*)X + i * vb, tol, restart, maxiter,
                iters ? iters + i : nullptr, relres ? relres + i : nullptr, s);
  }
  if (had) bind_frequency(c, f0, s);
  else c->freq_set = false;
  leave_stream(c, s, true);
  AIMX_API_END(c)
}

aimx_status aimx_sweep_status(aimx_ctx* c, int64_t nf, const void* Y, int32_t* status, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (nf < 0 || (nf > 0 && (!Y || !status))) throw Error(AIMX_E_INVALID_ARG, "bad status arguments");
  if (nf == 0) return AIMX_OK;
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  int32_t* flag = nullptr;
  AIMX_CUDA(cudaMallocAsync((void**)&flag, nf * sizeof(int32_t), s));
  AIMX_CUDA(cudaMemsetAsync(flag, 0, nf * sizeof(int32_t), s));
  const int64_t n2 = 2 * c->topo.nb;
  if (c->prec == AIMX_C64)
    k_nonfinite<float><<<nblk(n2 * nf), 256, 0, s>>>(n2, nf, (const float*)Y, flag);
  else
    k_nonfinite<double><<<nblk(n2 * nf), 256, 0, s>>>(n2, nf, (const double*)Y, flag);
  AIMX_CHECK_LAUNCH();
  AIMX_CUDA(cudaMemcpyAsync(status, flag, nf * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  AIMX_CUDA(cudaFreeAsync(flag, s));
  AIMX_CUDA(cudaStreamSynchronize(s));
  AIMX_API_END(c)
}

aimx_status aimx_sync(aimx_ctx* c, double timeout_s) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  AIMX_CUDA(cudaEventRecord(c->ev_use, c->stream));   // ev_use: the context stream waits for every user stream
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(c->ev_use);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) AIMX_CUDA(q);
    poll_nccl(c);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (timeout_s > 0 && el > timeout_s) {
      const std::string why = "aimx_sync: no completion within " + std::to_string(timeout_s) + " s";
      if (c->comm) nccl_abort(c, why + " (NCCL communicator aborted)");
      throw Error(AIMX_E_TIMEOUT, why);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  AIMX_API_END(c)
}

aimx_status aimx_nccl_unique_id(uint8_t id[128]) {
  if (!id) return AIMX_E_INVALID_ARG;
  try {
    ncclUniqueId u;
    AIMX_NCCL(nccl().getUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return AIMX_OK;
  } catch (const Error& e) {
    g_setup_error = e.what();
    return e.code;
  }
}

aimx_status aimx_set_frequency(aimx_ctx* c, double f_hz) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  enter_stream(c, c->stream);
  bind_frequency(c, f_hz, c->stream);
  leave_stream(c, c->stream, true);
  AIMX_API_END(c)
}

// C_lin on the overlapping pairs, once per context; the per-RWG
// geometry records are rebuilt first when the static matrices came from a cache.
static void ensure_side(aimx_ctx* c) {
  const Topology& t = c->topo;
  SetupDev& d = c->sd;
  if (!d.side) {
    d.V = dupload(c, t.V);
    d.T = dupload(c, t.T);
    d.ea = dupload(c, t.ea); d.eb = dupload(c, t.eb);
    d.tp = dupload(c, t.tp); d.tm = dupload(c, t.tm);
    d.pp = dupload(c, t.pp); d.pm = dupload(c, t.pm);
    d.side = dalloc<double>(c, 2 * t.nb * kSideStride);
    launch_rwg_sides(t, d, c->stream);
  }
}

static void build_linear(aimx_ctx* c) {
  const Topology& t = c->topo;
  SetupDev& d = c->sd;
  ensure_side(c);
  std::vector<int32_t> cols;
  build_overlap(t, cols);
  c->lin_col = dupload(c, cols);
  const bool f32 = c->prec == AIMX_C64;
  c->lin_c = dalloc<char>(c, t.nb * kLinW * (int64_t)(f32 ? sizeof(float2) : sizeof(double2)));
  launch_lin_entries(t, d, c->lin_col, f32, c->lin_c, c->stream);
  for (SlabRank& r : c->slabs) {   // each rank applies the rows it tests
    std::vector<int32_t> own((size_t)t.nb * kLinW, -1);
    for (int32_t e : r.owned) std::copy(cols.begin() + (int64_t)e * kLinW, cols.begin() + (int64_t)(e + 1) * kLinW,
                                        own.begin() + (int64_t)e * kLinW);
    r.lin_col = dupload(c, own);
  }
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
}

aimx_status aimx_set_linear_term(aimx_ctx* c, int enable) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  quiesce(c);
  if (enable && c->aim_on) throw Error(AIMX_E_INVALID_ARG, "the linear-term modification is an AIMx option (conventional AIM mode is on)");
  if (enable && !c->lin_col) build_linear(c);
  clear_graphs(c);
  c->lin_on = enable != 0;
  c->hot.lin_col = c->lin_on ? c->lin_col : nullptr;
  c->hot.lin_c = c->lin_c;
  for (SlabRank& r : c->slabs) {
    r.hr.lin_col = c->lin_on && !r.owned.empty() ? r.lin_col : nullptr;
    r.hr.lin_c = c->lin_c;
  }
  AIMX_API_END(c)
}

aimx_status aimx_set_conventional(aimx_ctx* c, int enable) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  if (enable && c->slab) throw Error(AIMX_E_UNSUPPORTED, "conventional AIM mode: one-GPU contexts only");
  if (enable && c->lin_on) throw Error(AIMX_E_INVALID_ARG, "turn the linear-term modification off first");
  if (enable && c->cfie_on) throw Error(AIMX_E_INVALID_ARG, "turn the CFIE off first");
  quiesce(c);
  if (enable && !c->aimDA) {
    ensure_side(c);
    const int64_t nnz = c->topo.rowptr[c->topo.nb];
    const size_t cs = c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2);
    c->aimDA = dalloc<char>(c, nnz * (int64_t)cs);
    c->aimDR = dalloc<char>(c, nnz * (int64_t)cs);
  }
  clear_graphs(c);
  c->aim_on = enable != 0;
  if (c->aim_on && c->freq_set) {   // the bound frequency's near fill
    enter_stream(c, c->stream);
    launch_aim_fill(c->topo, c->sd, c->k0, c->prec == AIMX_C64, c->aimDA, c->aimDR, c->stream);
    leave_stream(c, c->stream, true);
  }
  AIMX_API_END(c)
}

aimx_status aimx_get_aim_entries(const aimx_ctx* cc, double* DA, double* DR) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (!c->aim_on || !c->freq_set) throw Error(AIMX_E_STATE, "conventional AIM mode off or no frequency bound");
  AIMX_CUDA(cudaSetDevice(c->device));
  const int64_t nnz = c->topo.rowptr[c->topo.nb];
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  for (int part = 0; part < 2; ++part) {
    double* out = part ? DR : DA;
    const void* src = part ? c->aimDR : c->aimDA;
    if (!out) continue;
    if (c->prec == AIMX_C64) {
      std::vector<float> tmp((size_t)(2 * nnz));
      AIMX_CUDA(cudaMemcpy(tmp.data(), src, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
      std::copy(tmp.begin(), tmp.end(), out);
    } else {
      AIMX_CUDA(cudaMemcpy(out, src, (size_t)(2 * nnz) * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
  AIMX_API_END(c)
}

aimx_status aimx_get_linear_term(const aimx_ctx* c, int* enabled) {
  if (!c || !enabled) return AIMX_E_INVALID_ARG;
  *enabled = c->lin_on ? 1 : 0;
  return AIMX_OK;
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
  enter_stream(c, s);
  run_matvec(c, x, y0, y1, mode, s);
  leave_stream(c, s);
  AIMX_API_END(c)
}

aimx_status aimx_matvec(aimx_ctx* c, const void* x, void* y, void* stream) {
  return matvec_common(c, x, y, nullptr, 0, stream);
}

aimx_status aimx_matvec_parts(aimx_ctx* c, const void* x, void* yA, void* yPhi, void* stream) {
  return matvec_common(c, x, yA, yPhi, 1, stream);
}

// Several device batches: the spectra of batch i+1 are generated on a side
// stream (double-buffered) while batch i's matvec runs, so S1 overlaps S2-S5.
// before(i) / after(i): hooks on the compute stream around device batch i
// (the host sweep orders its copies with them).
static void sweep_impl(aimx_ctx* c, const std::vector<int64_t>& off, const double* f, const char* X, char* Y,
                       cudaStream_t s, const std::function<void(int64_t)>& before = nullptr,
                       const std::function<void(int64_t, cudaStream_t)>& after = nullptr,
                       const std::function<void(int64_t, cudaStream_t)>& before_side = nullptr) {
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  const int64_t nbat = (int64_t)off.size() - 1;
  auto count = [&](int64_t i) { return (int)(off[i + 1] - off[i]); };
  if (c->slab || nbat < 2 || !c->s2 || c->aim_on || c->cfie_on || (c->prof.on && c->prof.serial)) {
    for (int64_t i = 0; i < nbat; ++i) {
      if (before) before(i);
      run_batch(c, count(i), f + off[i], X + off[i] * vb, Y + off[i] * vb, s);
      if (after) after(i, s);
    }
    return;
  }
  AIMX_CUDA(cudaEventRecord(c->ev_start, s));
  AIMX_CUDA(cudaStreamWaitEvent(c->s2, c->ev_start, 0));
  // side stream, per batch: its interleaved columns (xt), then its spectra,
  // double-buffered; `before` (the host sweep's copy) gates the columns.  The
  // batch's gather and x transform wait only for its columns (ev_xt), its
  // spectrum multiply for its spectra (ev_sp; HotDev::spec_ready), so the
  // first batch's spectra overlap its projection
  auto spec = [&](int64_t i) {
    if (i >= 2) AIMX_CUDA(cudaStreamWaitEvent(c->s2, c->ev_mv[i % 2], 0));   // matvec i-2 read these buffers
    HotDev hh = c->hot;
    hh.xt = c->XT[i % 2];
    Combine cb = make_combine(count(i), f + off[i], 0, c->hot.nb);
    if (before_side) {   // host sweep: the spectra (independent of x) run during the batch's copy in
      spectra(c, count(i), f + off[i], c->s2, c->HB[i % 2]);
      AIMX_CUDA(cudaEventRecord(c->ev_sp[i % 2], c->s2));
      before_side(i, c->s2);
    }
    if (c->prec == AIMX_C64) interleave_f32(hh, X + off[i] * vb, cb, c->s2);
    else interleave_f64(hh, X + off[i] * vb, cb, c->s2);
    AIMX_CUDA(cudaEventRecord(c->ev_xt[i % 2], c->s2));
    if (!before_side) {
      spectra(c, count(i), f + off[i], c->s2, c->HB[i % 2]);
      AIMX_CUDA(cudaEventRecord(c->ev_sp[i % 2], c->s2));
    }
  };
  // overlap: the grid part of batch i+1 (stream s) runs while S4+S5 of batch
  // i (stream s3) does; phi is double-buffered (PHI), xt and the spectra are
  // (XT, HB), and spec(i+2) waits for S4+S5 of batch i (ev_mv)
  const bool ov = c->s3 && !std::getenv("AIMX_NO_OVERLAP");
  spec(0);
  for (int64_t i = 0; i < nbat; ++i) {
    if (i + 1 < nbat) spec(i + 1);
    AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_xt[i % 2], 0));
    if (before) before(i);
    HotDev hh = batch_view(c, count(i));
    hh.spec_ready = c->ev_sp[i % 2];
    hh.Hoct = c->HB[i % 2];
    hh.xt = c->XT[i % 2];
    Combine cb = make_combine(count(i), f + off[i], 0, c->hot.nb);
    cb.xt_ready = 1;
    const bool f32 = c->prec == AIMX_C64;
    if (!ov) {
      if (f32) hot_matvec_f32(hh, X + off[i] * vb, Y + off[i] * vb, nullptr, cb, s, &c->prof);
      else hot_matvec_f64(hh, X + off[i] * vb, Y + off[i] * vb, nullptr, cb, s, &c->prof);
      AIMX_CUDA(cudaEventRecord(c->ev_mv[i % 2], s));
      if (after) after(i, s);
      continue;
    }
    hh.phi = c->PHI[i % 2];
    if (f32) hot_grid_f32(hh, X + off[i] * vb, cb, s, &c->prof);
    else hot_grid_f64(hh, X + off[i] * vb, cb, s, &c->prof);
    AIMX_CUDA(cudaEventRecord(c->ev_grid[i % 2], s));
    AIMX_CUDA(cudaStreamWaitEvent(c->s3, c->ev_grid[i % 2], 0));
    if (f32) hot_near_f32(hh, X + off[i] * vb, Y + off[i] * vb, nullptr, cb, c->s3, &c->prof);
    else hot_near_f64(hh, X + off[i] * vb, Y + off[i] * vb, nullptr, cb, c->s3, &c->prof);
    AIMX_CUDA(cudaEventRecord(c->ev_mv[i % 2], c->s3));
    if (after) after(i, c->s3);
  }
  if (ov) AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_mv[(nbat - 1) % 2], 0));
}

// device batch of a sweep: the caller's, else the slots, balanced over the
// number of batches the sweep needs (e.g. 100 points in 32 slots: 4 x 25)
static int sweep_batch(const aimx_ctx* c, int32_t batch, int64_t nf) {
  if (batch > 0) return std::max(1, std::min<int>(batch, c->hot.batch));
  const int64_t S = c->hot.batch, nb = (nf + S - 1) / S;
  return (int)std::max<int64_t>(1, std::min<int64_t>(S, nb > 0 ? (nf + nb - 1) / nb : S));
}

// Batch offsets of a sweep (size nbat + 1): batches of the caller's size, else
// full slots with the remainder last (a short last batch also shortens the
// host sweep's final device->host copy); AIMX_SWEEP_PLAN="s0,s1,..." sets the
// leading batch sizes (experiments).
static std::vector<int64_t> sweep_plan(const aimx_ctx* c, int32_t batch, int64_t nf, bool host = false) {
  const int64_t S = c->hot.batch;
  const int64_t B = batch > 0 ? std::max<int64_t>(1, std::min<int64_t>(batch, S)) : S;
  std::vector<int64_t> off{0};
  const bool auto_host = host && batch <= 0 && !std::getenv("AIMX_SWEEP_PLAN");
  const double vbytes = (double)c->hot.nb * (c->prec == AIMX_C64 ? 8.0 : 16.0);
  if (auto_host && nf >= 32 && nf * vbytes >= 64e6) {
    // host buffers, copy-bound sweeps (>= 64 MB each way): at least four equal
    // batches, so the exposed first copy in and last copy out are a quarter of
    // the data (cfg5 64 points: 16 x 4 -- 6.33 against 7.90 ms for 24, 32, 8
    // end to end; the copies alone take 4.60 ms both ways at once)
    const int64_t B4 = std::min<int64_t>(S, std::max<int64_t>(8, ((nf + 3) / 4 + 7) / 8 * 8));
    while (off.back() < nf) off.push_back(std::min(nf, off.back() + B4));
    return off;
  }
  // host buffers: a 3/4 first batch starts the compute after a shorter first
  // copy (cfg2 100 points: 24, 32, 32, 12 -- 0.754 against 0.772 ms end to end)
  if (auto_host && nf > S && S >= 4) off.push_back(3 * S / 4);
  if (batch <= 0)
    if (const char* e = std::getenv("AIMX_SWEEP_PLAN")) {
      for (const char* p = e; *p && off.back() < nf;) {
        const int64_t v = std::max<int64_t>(1, std::min<int64_t>(S, std::atoll(p)));
        off.push_back(std::min(nf, off.back() + v));
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
      }
    }
  while (off.back() < nf) off.push_back(std::min(nf, off.back() + B));
  return off;
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
  enter_stream(c, s);
  sweep_impl(c, sweep_plan(c, batch, nf), f_hz, (const char*)X, (char*)Y, s);
  if (had) bind_frequency(c, f0, s);
  else c->freq_set = false;
  leave_stream(c, s, true);
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
  const std::vector<int64_t> plan = sweep_plan(c, batch, nf, true);
  const int64_t nbat_all = (int64_t)plan.size() - 1;
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  // staging: chunks of whole batches within 1 GB (all of them for cfg1/cfg2), so
  // the device batches pipeline; copies of the next chunk wait for this one
  const int64_t fit = std::max<int64_t>((int64_t)c->hot.batch, (int64_t)(1ll << 30) / (2 * (int64_t)vb));
  std::vector<int64_t> cuts{0};   // chunk boundaries, as batch indices
  for (int64_t i = 0; i < nbat_all; ++i)
    if (plan[i + 1] - plan[cuts.back()] > fit) cuts.push_back(i);
  cuts.push_back(nbat_all);
  int64_t CH = 0, nbat_max = 0;
  for (size_t k = 0; k + 1 < cuts.size(); ++k) {
    CH = std::max(CH, plan[cuts[k + 1]] - plan[cuts[k]]);
    nbat_max = std::max(nbat_max, cuts[k + 1] - cuts[k]);
  }
  const int64_t need = 2 * std::max<int64_t>(CH, 1) * (int64_t)vb;
  if (c->stage_bytes < need) {
    if (c->stage) AIMX_CUDA(cudaFree(c->stage));
    c->stage = nullptr;
    AIMX_CUDA(cudaMalloc(&c->stage, need));
    c->stage_bytes = need;
  }
  char* dX = (char*)c->stage;
  char* dY = dX + CH * vb;
  const bool had = c->freq_set;
  const double f0 = c->f;
  enter_stream(c, s);
  // per device batch: host->device copy on one copy stream, device->host on
  // another, ordered with the batch's compute by events, so both directions
  // overlap the other batches' compute
  if (!c->sc[0]) {
    for (int k = 0; k < 2; ++k) AIMX_CUDA(cudaStreamCreateWithFlags(&c->sc[k], cudaStreamNonBlocking));
  }
  while ((int64_t)c->ev_io.size() < 2 * nbat_max + 1) {
    cudaEvent_t e;
    AIMX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->ev_io.push_back(e);
  }
  for (size_t k = 0; k + 1 < cuts.size(); ++k) {
    const int64_t i0 = plan[cuts[k]];
    std::vector<int64_t> sub;   // the chunk's batch offsets, relative to i0
    for (int64_t i = cuts[k]; i <= cuts[k + 1]; ++i) sub.push_back(plan[i] - i0);
    const int64_t nbat = (int64_t)sub.size() - 1;
    cudaEvent_t go = c->ev_io[2 * nbat_max];
    AIMX_CUDA(cudaEventRecord(go, s));   // staging free: the previous chunk's work is done
    AIMX_CUDA(cudaStreamWaitEvent(c->sc[0], go, 0));
    AIMX_CUDA(cudaStreamWaitEvent(c->sc[1], go, 0));
    for (int64_t i = 0; i < nbat; ++i) {
      AIMX_CUDA(cudaMemcpyAsync(dX + sub[i] * vb, (const char*)X + (i0 + sub[i]) * vb, (sub[i + 1] - sub[i]) * vb,
                                cudaMemcpyHostToDevice, c->sc[0]));
      AIMX_CUDA(cudaEventRecord(c->ev_io[2 * i], c->sc[0]));
    }
    auto before = [&](int64_t i) { AIMX_CUDA(cudaStreamWaitEvent(s, c->ev_io[2 * i], 0)); };
    auto before_side = [&](int64_t i, cudaStream_t s2) { AIMX_CUDA(cudaStreamWaitEvent(s2, c->ev_io[2 * i], 0)); };
    auto after = [&](int64_t i, cudaStream_t sy) {
      AIMX_CUDA(cudaEventRecord(c->ev_io[2 * i + 1], sy));
      AIMX_CUDA(cudaStreamWaitEvent(c->sc[1], c->ev_io[2 * i + 1], 0));
      AIMX_CUDA(cudaMemcpyAsync((char*)Y + (i0 + sub[i]) * vb, dY + sub[i] * vb, (sub[i + 1] - sub[i]) * vb,
                                cudaMemcpyDeviceToHost, c->sc[1]));
    };
    sweep_impl(c, sub, f_hz + i0, dX, dY, s, before, after, before_side);
    AIMX_CUDA(cudaEventRecord(go, c->sc[1]));
    AIMX_CUDA(cudaStreamWaitEvent(s, go, 0));   // results are home before the next chunk / return
  }
  if (had) bind_frequency(c, f0, s);
  else c->freq_set = false;
  leave_stream(c, s, true);
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
  o->planar = c->planar ? 1 : 0;
  o->kop_grad = c->HsF && c->kgrad ? 1 : 0;
  o->grid_channels = c->hot.nc;
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

aimx_status aimx_get_linear_entries(const aimx_ctx* cc, int32_t* cols, double* CA_lin, double* Crho_lin) {
  aimx_ctx* c = const_cast<aimx_ctx*>(cc);
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (!c->lin_col) throw Error(AIMX_E_STATE, "aimx_set_linear_term has not been enabled");
  AIMX_CUDA(cudaSetDevice(c->device));
  const int64_t n = c->topo.nb * kLinW;
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  if (cols) AIMX_CUDA(cudaMemcpy(cols, c->lin_col, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
  const bool f32 = c->prec == AIMX_C64;
  std::vector<double> v((size_t)(2 * n));
  if (f32) {
    std::vector<float> tmp((size_t)(2 * n));
    AIMX_CUDA(cudaMemcpy(tmp.data(), c->lin_c, tmp.size() * sizeof(float), cudaMemcpyDeviceToHost));
    std::copy(tmp.begin(), tmp.end(), v.begin());
  } else {
    AIMX_CUDA(cudaMemcpy(v.data(), c->lin_c, v.size() * sizeof(double), cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i < n; ++i) {
    if (CA_lin) CA_lin[i] = v[2 * i];
    if (Crho_lin) Crho_lin[i] = v[2 * i + 1];
  }
  AIMX_API_END(c)
}

// double-layer operator K (NEXT #1): static near part, static F spectrum and
// buffers, built once on the first enable
static void build_kop(aimx_ctx* c) {
  const Topology& t = c->topo;
  ensure_side(c);
  if (!c->sd.T) c->sd.T = dupload(c, t.T);
  const int64_t nnz = t.rowptr[t.nb];
  const bool f32 = c->prec == AIMX_C64;
  const size_t cs = f32 ? sizeof(float2) : sizeof(double2);
  double* ck = dalloc<double>(c, nnz);
  double* ckpv = dalloc<double>(c, nnz);
  launch_K_static(t, c->sd, ck, c->stream, ckpv);
  if (f32) {
    float* ckf = dalloc<float>(c, nnz);
    float* ckpvf = dalloc<float>(c, nnz);
    k_d2f_real<<<nblk(nnz), 256, 0, c->stream>>>(nnz, ck, ckf);
    AIMX_CHECK_LAUNCH();
    k_d2f_real<<<nblk(nnz), 256, 0, c->stream>>>(nnz, ckpv, ckpvf);
    AIMX_CHECK_LAUNCH();
    AIMX_CUDA(cudaStreamSynchronize(c->stream));
    dfree(c, ck, nnz * (int64_t)sizeof(double));
    dfree(c, ckpv, nnz * (int64_t)sizeof(double));
    c->ck_T = ckf;
    c->ckpv_T = ckpvf;
  } else {
    c->ck_T = ck;
    c->ckpv_T = ckpv;
  }
  // the gradient-of-kernel form where the grid passes support its spectral
  // cross product (AIMX_K_RADIAL=1 or an unsupported grid: the radial form)
  c->kgrad = kop_grad_supported(f32, c->hot) && !std::getenv("AIMX_K_RADIAL");
  const int ns = c->kgrad ? 3 : 1;
  const int64_t noct = c->sp.noct;
  c->HsF = dalloc<double2>(c, ns * noct);
  for (int a = 0; a < ns; ++a) spectrum_static(c->sp, c->HsF + a * noct, c->stream, c->kgrad ? 2 + a : 1);
  if (f32) {
    c->HsF_T = dalloc<float2>(c, ns * noct);
    k_d2f<<<nblk(ns * noct), 256, 0, c->stream>>>(ns * noct, c->HsF, (float2*)c->HsF_T);
    AIMX_CHECK_LAUNCH();
  } else {
    c->HsF_T = c->HsF;
  }
  c->HF = dalloc<char>(c, ns * noct * (int64_t)cs);
  if (c->hot.nc != 4 && !c->hot.S4)   // K's passes keep 4 channels (s x J has a z part)
    c->hot.S4 = zalloc<char>(c, (int64_t)c->hot.nlines * c->hot.Nx * 4 * (int64_t)cs);
  const int64_t nP = c->hot.sP;   // one column, compact potentials (batch 1)
  c->kphi1 = zalloc<char>(c, nP * (int64_t)cs + 64);
  c->kphi2 = zalloc<char>(c, nP * (int64_t)cs + 64);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
}

aimx_status aimx_set_kop(aimx_ctx* c, int enable) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (enable && c->slab) throw Error(AIMX_E_UNSUPPORTED, "the double-layer operator: one-GPU contexts only");
  if (!enable && c->cfie_on) throw Error(AIMX_E_INVALID_ARG, "turn the CFIE off first");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  quiesce(c);
  if (enable && !c->HsF) build_kop(c);
  c->kop_on = enable != 0;
  if (c->kop_on && c->freq_set) {
    kop_spectrum(c, c->f, c->stream);
    leave_stream(c, c->stream, true);
  }
  AIMX_API_END(c)
}

// Several right-hand sides at the bound frequency, in device batches of the
// context's slots: the batched kernels with every column reading spectrum
// slot 0 (slot stride 0), so one spectrum serves the whole batch.
aimx_status aimx_matvec_multi(aimx_ctx* c, int64_t nrhs, const void* X, void* Y, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (nrhs < 0 || (nrhs > 0 && (!X || !Y))) throw Error(AIMX_E_INVALID_ARG, "bad arguments");
  if (nrhs > 0 && X == Y) throw Error(AIMX_E_INVALID_ARG, "input and output alias");
  if (!c->freq_set) throw Error(AIMX_E_STATE, "aimx_set_frequency has not been called");
  if (c->slab || c->aim_on || c->cfie_on)
    throw Error(AIMX_E_UNSUPPORTED, "aimx_matvec_multi: one-GPU AIMx contexts (no AIM / CFIE mode)");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  enter_stream(c, s);
  const size_t vb = (size_t)c->hot.nb * (c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2));
  for (int64_t i = 0; i < nrhs; i += c->hot.batch) {
    const int B = (int)std::min<int64_t>(c->hot.batch, nrhs - i);
    HotDev h = batch_view(c, B);
    h.sH = 0;   // every column reads the bound spectrum (slot 0)
    std::vector<double> f(B, c->f);
    Combine cb = make_combine(B, f.data(), 0, c->hot.nb);
    if (c->prec == AIMX_C64) hot_matvec_f32(h, (const char*)X + i * vb, (char*)Y + i * vb, nullptr, cb, s, &c->prof);
    else hot_matvec_f64(h, (const char*)X + i * vb, (char*)Y + i * vb, nullptr, cb, s, &c->prof);
  }
  leave_stream(c, s);
  AIMX_API_END(c)
}

aimx_status aimx_set_cfie(aimx_ctx* c, int enable) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (enable && c->slab) throw Error(AIMX_E_UNSUPPORTED, "CFIE: one-GPU contexts only");
  if (enable && c->aim_on) throw Error(AIMX_E_INVALID_ARG, "turn the conventional AIM mode off first");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  quiesce(c);
  if (enable) {
    if (!c->HsF) build_kop(c);
    if (!c->ktmp) c->ktmp = dalloc<char>(c, c->topo.nb * (int64_t)(c->prec == AIMX_C64 ? sizeof(float2) : sizeof(double2)));
    if (!c->kop_on) {
      c->kop_on = true;
      if (c->freq_set) kop_spectrum(c, c->f, c->stream);
    }
  }
  clear_graphs(c);
  c->cfie_on = enable != 0;
  leave_stream(c, c->stream, true);
  AIMX_API_END(c)
}

aimx_status aimx_matvec_kop(aimx_ctx* c, const void* x, void* y, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (!x || !y) throw Error(AIMX_E_INVALID_ARG, "null vector");
  if (x == y) throw Error(AIMX_E_INVALID_ARG, "input and output alias");
  if (!c->kop_on) throw Error(AIMX_E_STATE, "aimx_set_kop has not been enabled");
  if (!c->freq_set) throw Error(AIMX_E_STATE, "aimx_set_frequency has not been called");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  enter_stream(c, s);
  kop_matvec(c->prec == AIMX_C64, c->hot, x, y, c->HF, c->kphi1, c->kphi2, c->sd.lam, c->topo.h, c->sd.rowptr,
             c->sd.col, c->ck_T, s, c->kgrad);
  leave_stream(c, s);
  AIMX_API_END(c)
}

// PMCHWT (reading R27): x = [J; M], y = [y_E; y_H],
//   y_E = (Z0 + Z1) J - (K0 + K1) M,  y_H = (K0 + K1) J + (Z0/eta0^2 + Z1/eta1^2) M,
// medium 1 = the interior, k1 = k0 sqrt(eps_r), eta1 = eta0 / sqrt(eps_r); the
// interior operators are the free-space ones at the frequency f sqrt(eps_r)
// (same static matrices), the Z prefactor keeps the physical omega.
aimx_status aimx_matvec_pmchwt(aimx_ctx* c, double eps_r, const void* x, void* y, void* stream) {
  if (!c) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (!x || !y || x == y) throw Error(AIMX_E_INVALID_ARG, "null or aliased vectors");
  if (!(eps_r >= 1.0) || !std::isfinite(eps_r)) throw Error(AIMX_E_INVALID_ARG, "eps_r must be finite and >= 1");
  if (!c->HsF) throw Error(AIMX_E_STATE, "aimx_set_kop has not been enabled");
  if (!c->freq_set) throw Error(AIMX_E_STATE, "aimx_set_frequency has not been called");
  if (c->aim_on || c->cfie_on) throw Error(AIMX_E_INVALID_ARG, "PMCHWT runs the AIMx operators (AIM / CFIE off)");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  cudaStream_t s = pick(c, stream);
  enter_stream(c, s);
  const bool f32 = c->prec == AIMX_C64;
  const int64_t nb = c->hot.nb;
  const size_t cs = f32 ? sizeof(float2) : sizeof(double2);
  const int64_t noct = c->sp.noct;
  if (!c->pm_H1) {
    c->pm_H1 = dalloc<char>(c, noct * (int64_t)cs);
    c->pm_HF1 = dalloc<char>(c, (c->kgrad ? 3 : 1) * noct * (int64_t)cs);
    c->pm_t = dalloc<char>(c, 3 * nb * (int64_t)cs);
  }
  if (!c->kop_on) kop_spectrum(c, c->f, s);   // F_hat(k0) (aimx_set_kop(0) left it stale)
  const double f0 = c->f, f1 = c->f * std::sqrt(eps_r);
  spectra(c, 1, &f1, s, c->pm_H1);
  kop_spectrum(c, f1, s, c->pm_HF1);
  char* tA = (char*)c->pm_t;
  char* tP = tA + nb * cs;
  char* tK = tP + nb * cs;
  const char* J = (const char*)x;
  const char* Mc = J + nb * cs;
  char* yE = (char*)y;
  char* yH = yE + nb * cs;
  AIMX_CUDA(cudaMemsetAsync(y, 0, 2 * nb * cs, s));
  const double w = 2.0 * kPi * f0, eta0 = kMu0 * kC0, eta1 = eta0 / std::sqrt(eps_r);
  for (int i = 0; i < 2; ++i) {
    const double fi = i ? f1 : f0, k = 2.0 * kPi * fi / kC0;
    HotDev h = c->hot;
    if (i) h.Hoct = c->pm_H1;
    const void* HFi = i ? c->pm_HF1 : c->HF;
    Combine cb = make_combine(1, &fi, 1, nb);   // parts: tA = y^A, tP = -y^rho
    // Z = -j w mu0 (y^A - y^rho / k^2) = -j w mu0 (tA + tP / k^2)
    const double a = -w * kMu0, b = -w * kMu0 / (k * k);   // imaginary coefficients
    for (int src = 0; src < 2; ++src) {
      const void* xs = src ? (const void*)Mc : (const void*)J;
      if (f32) hot_matvec_f32(h, xs, tA, tP, cb, s, nullptr);
      else hot_matvec_f64(h, xs, tA, tP, cb, s, nullptr);
      const double sc = src ? 1.0 / ((i ? eta1 : eta0) * (i ? eta1 : eta0)) : 1.0;
      char* yz = src ? yH : yE;
      gm_caxpy(f32, nb, 0.0, a * sc, tA, yz, s);
      gm_caxpy(f32, nb, 0.0, b * sc, tP, yz, s);
      kop_matvec(f32, h, xs, tK, HFi, c->kphi1, c->kphi2, c->sd.lam, c->topo.h, c->sd.rowptr, c->sd.col,
                 c->ckpv_T, s, c->kgrad);
      gm_axpy(f32, nb, src ? -1.0 : 1.0, tK, src ? yE : yH, s);   // y_E -= K M, y_H += K J
    }
  }
  leave_stream(c, s);
  AIMX_API_END(c)
}

aimx_status aimx_get_kop_static(aimx_ctx* c, double* CK) {
  if (!c || !CK) return AIMX_E_INVALID_ARG;
  AIMX_API_BEGIN
  if (c->slab) throw Error(AIMX_E_UNSUPPORTED, "one-GPU contexts only");
  AIMX_CUDA(cudaSetDevice(c->device));
  check_sticky(c);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  ensure_side(c);
  if (!c->sd.T) {
    c->sd.T = dupload(c, c->topo.T);
  }
  const int64_t nnz = c->topo.rowptr[c->topo.nb];
  double* d = nullptr;
  AIMX_CUDA(cudaMalloc(&d, (size_t)std::max<int64_t>(nnz, 1) * sizeof(double)));
  std::unique_ptr<double, decltype(&cudaFree)> guard(d, &cudaFree);
  launch_K_static(c->topo, c->sd, d, c->stream);
  AIMX_CUDA(cudaStreamSynchronize(c->stream));
  AIMX_CUDA(cudaMemcpy(CK, d, (size_t)nnz * sizeof(double), cudaMemcpyDeviceToHost));
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
    const double M = 1.0 / spectrum_scale(c);
    if (c->prec == AIMX_C64) {
      std::vector<float2> tmp(n);
      AIMX_CUDA(cudaMemcpy(tmp.data(), c->Hoct, n * sizeof(float2), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < n; ++i) { out[2 * i] = tmp[i].x * M; out[2 * i + 1] = tmp[i].y * M; }
    } else {
      AIMX_CUDA(cudaMemcpy(out, c->Hoct, n * sizeof(double2), cudaMemcpyDeviceToHost));
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

aimx_status aimx_profile_stages(aimx_ctx* c, int32_t mask) {
  if (!c) return AIMX_E_INVALID_ARG;
  c->prof.mask = mask & 0x7f;
  c->prof.serial = (mask & AIMX_PROFILE_SERIAL) != 0;
  return AIMX_OK;
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
    case AIMX_E_NCCL: return "NCCL error (communicator aborted)";
    case AIMX_E_TIMEOUT: return "timed out";
    case AIMX_E_INTERNAL: return "internal error";
  }
  return "unknown status";
}

const char* aimx_last_error(const aimx_ctx* c) { return c ? c->last_error.c_str() : ""; }
const char* aimx_last_setup_error(void) { return g_setup_error.c_str(); }
const char* aimx_version(void) { return "aimx-b200 0.1 (sm_100a)"; }

}  // extern "C"
