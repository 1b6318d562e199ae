// Internal declarations of the AIMx B200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/aimx.h"
#include <nvtx3/nvToolsExt.h>

namespace aimx {

struct Error : std::runtime_error {
  aimx_status code;
  Error(aimx_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define AIMX_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      throw ::aimx::Error(e_ == cudaErrorMemoryAllocation ? AIMX_E_OOM : AIMX_E_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));       \
    }                                                                                \
  } while (0)

// Every kernel launch is followed by AIMX_CHECK_LAUNCH(), which also counts it
// (aimx_profile_read reports the count).
int64_t& launch_counter();
#define AIMX_STR2(x) #x
#define AIMX_STR(x) AIMX_STR2(x)
#define AIMX_CHECK_LAUNCH()                                                                       \
  do {                                                                                            \
    ++::aimx::launch_counter();                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                          \
    if (e_ != cudaSuccess)                                                                        \
      throw ::aimx::Error(AIMX_E_CUDA, std::string("kernel launch at " __FILE__ ":" AIMX_STR(__LINE__) ": ") + \
                                           cudaGetErrorString(e_));                              \
  } while (0)

// Launch with programmatic stream serialization (PDL, see fft.cuh pdl_wait).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AIMX_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

constexpr double kPi = 3.14159265358979323846;
constexpr double kC0 = 299792458.0;          // m/s (exact)
constexpr double kMu0 = 1.25663706212e-6;    // H/m (CODATA 2018), reading R1

// ---------------------------------------------------------------- host topology
struct Topology {
  int64_t nv = 0, nt = 0, nb = 0;
  std::vector<double> V;        // [nv][3]
  std::vector<int32_t> T;       // [nt][3]
  std::vector<int32_t> ea, eb, tp, tm, pp, pm;   // RWG table (external order)
  int32_t n[3] = {0, 0, 0};
  int32_t order = 2, p = 3, p3 = 27, near_cells = 2;
  double h = 0, origin[3] = {0, 0, 0};
  std::vector<int32_t> anchor;  // [nb][3]
  std::vector<int64_t> rowptr;  // [nb+1]
  std::vector<int32_t> col;     // [nnz]
};

void build_topology(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, Topology& t);

// Occupied-node (transposed stencil) structure, built after the weights are
// known so that exactly-zero weights (planar meshes) are pruned.
struct NodeMap {
  std::vector<int32_t> node_lin;   // [nocc] linear grid index, ascending
  std::vector<int32_t> node_ptr;   // [nocc+1]
  std::vector<int32_t> node_line;  // [nocc] index into line_id
  std::vector<int32_t> ent_rwg;    // [nent]
  std::vector<int32_t> ent_slot;   // [nent] stencil slot s
  std::vector<int32_t> line_id;    // [nlines] y + Ny z, ascending
  std::vector<int32_t> line_ptr;   // [nlines+1] into node arrays
  std::vector<int32_t> zplanes;    // occupied z planes, ascending
  std::vector<uint8_t> line_occ;   // [Ny*Nz]
};

void build_nodemap(const Topology& t, const std::vector<uint8_t>& nz_slot, NodeMap& m);

// Near matrix in row-group form (host_setup.cpp build_near_groups): groups of
// R spatially ordered rows sharing one sorted column union.
struct NearGroups {
  int R = 8;
  int order_kind = 0;              // 0: anchor linear index, 1: anchor Morton code
  int64_t ngrp = 0;
  std::vector<int32_t> rows;       // [ngrp][R] external row ids, -1 = padding
  std::vector<int64_t> ptr;        // [ngrp+1] into ucol
  std::vector<int32_t> ucol;       // [U] union columns (external ids), ascending per group
  std::vector<int64_t> slot;       // [nnz] CSR entry k -> value slot u*R + r
  std::vector<int64_t> wptr;       // [ngrp+1] into wnode
  std::vector<int32_t> wnode;      // [Uw] union of the rows' stencil nodes (linear grid index)
  std::vector<int64_t> wslot;      // [nb][p3] weight slot (w*R + r), -1 = exactly zero weight
};

// rows: the testing functions grouped (empty = all); entries of other rows keep slot -1
void build_near_groups(const Topology& t, const std::vector<uint8_t>& nz_slot, NearGroups& g,
                       const std::vector<int32_t>& rows = {});
void nodemap_rows(const Topology& t, const NodeMap& full, int y0, int y1, NodeMap& m);

// Work list of the S4+S5 kernel: chunks {group, flags, payload offset / 16,
// count} (flags: bit0 = near (C) chunk, else interpolation (W) chunk; bit1
// first, bit2 last chunk of its group).  Chunk c's payload, moved by ONE bulk
// copy: [count coefficient tuples (C: R (C_A, C_rho) pairs; W: R real4
// weights) | count row indices, 16-byte padded | descriptor of chunk c + kNearD].
constexpr int kNearD = 3;          // S4+S5 pipeline depth (chunks in flight)
struct NearChunks {
  std::vector<int32_t> chunks;     // [nchunk][4]
  std::vector<unsigned char> payload;
  std::vector<int64_t> uoff_c;     // [U] payload byte offset of union entry u's C pairs
  std::vector<int64_t> uoff_w;     // [Uw] ... of the W weights
  std::vector<int64_t> gfirst;     // [ngrp] first chunk of each group
  int64_t nchunk = 0;
  std::vector<double> cost;        // [ngrp] work estimate
};
// cs = bytes of one complex (= one real pair) in the compute precision; the
// chunks follow the groups in `order` (a permutation of 0..ngrp-1)
void build_near_chunks(const NearGroups& g, int chw, int chc, int cs, NearChunks& ck,
                       const std::vector<int64_t>& order);
// the S4+S5 kernel's group order for `ncta` CTAs: CTA k's groups are
// order[cta_begin[k] .. cta_begin[k+1]) (k, k + ncta, k + 2 ncta, ...)
std::vector<int64_t> near_round_order(int64_t ngrp, int ncta, std::vector<int64_t>& cta_begin);

// ---------------------------------------------------------------- device setup (fp64)
struct SetupDev {
  double* V = nullptr;        // [nv][3]
  int32_t* T = nullptr;       // [nt][3]
  int32_t* tp = nullptr;      // RWG tables
  int32_t* tm = nullptr;
  int32_t* pp = nullptr;
  int32_t* pm = nullptr;
  int32_t* ea = nullptr;
  int32_t* eb = nullptr;
  int32_t* anchor = nullptr;  // [nb][3]
  int64_t* rowptr = nullptr;  // [nb+1]
  int32_t* col = nullptr;     // [nnz]
  double* side = nullptr;     // per (rwg, side) geometry record, kSideStride doubles
  double* lam = nullptr;      // [nb][p3][4] fp64 weights
  double* LA_un = nullptr;    // unsymmetrised static entries [nnz]
  double* YR_un = nullptr;
  double* LA_NR = nullptr;    // symmetrised
  double* YR_NR = nullptr;
  double* LA_P = nullptr;     // precorrection
  double* YR_P = nullptr;
  double* CA = nullptr;       // C_A = LA_NR - LA_P
  double* CR = nullptr;
};
constexpr int kSideStride = 16;  // v0[3] v1[3] v2[3] free[3] coef div area pad

void launch_rwg_sides(const Topology& t, SetupDev& d, cudaStream_t s);
void launch_weights(const Topology& t, SetupDev& d, cudaStream_t s, uint8_t* nzflag);
void launch_static_near(const Topology& t, SetupDev& d, cudaStream_t s);
void launch_precorrect(const Topology& t, SetupDev& d, cudaStream_t s);

// ---------------------------------------------------------------- conventional AIM mode
// D(k0) = L_d,NR(k0) - W H_d,NR(k0) P on the near CSR pattern (external
// order), fp64 arithmetic, stored in the compute precision (float2 / double2).
void launch_aim_fill(const Topology& t, const SetupDev& d, double k0, bool f32, void* DA, void* DR, cudaStream_t s);

// ---------------------------------------------------------------- double-layer operator K (NEXT #1)
// C_K = sym(K_s,PV) + residue - K_s,P on the near CSR pattern (fp64; the oracle kop module,
// readings R23-R25).  Needs d.side, d.T, d.tp, d.tm.
void launch_K_static(const Topology& t, const SetupDev& d, double* CK, cudaStream_t s, double* CKpv = nullptr);
struct HotDev;
// y = Kmat x (one column, bound frequency): two passes of the grid transforms
// with the radial spectrum HF (slot 0), the curl combination, interpolation
// with the fp64 weights lam, + C_K x (ck: compute precision, CSR order)
// grad: the gradient-of-kernel form (HF = the three spectra d_a G_hat [3][noct],
// phi1 the potentials, phi2 unused), else the radial form (HF = F_hat)
void kop_matvec(bool f32, const HotDev& h, const void* x, void* y, const void* HF, void* phi1, void* phi2,
                const double* lam, double hg, const int64_t* rowptr, const int32_t* col, const void* ck,
                cudaStream_t s, bool grad = false);
// the gradient form runs on this context's grid (not planar; a fused short y/z
// pass or the TMA z pass)
bool kop_grad_supported(bool f32, const HotDev& h);

// ---------------------------------------------------------------- linear-term modification
// P:382-398 (sec:methods:aimx:acc): k0^2 G_lin, G_lin = -r/(8 pi) (eq:linterm
// P:365), by direct integration on overlapping pairs only (supports share a
// triangle, reading R21): at most kLinW columns per row.
constexpr int kLinW = 5;
// cols: [nb][kLinW] overlapping columns, ascending, -1 padded
void build_overlap(const Topology& t, std::vector<int32_t>& cols);
// C_lin = (L^A_lin - sum_c W^c H_lin P^c, y^rho_lin - W^rho H_lin P^rho) on the
// pairs of `cols` (device, [nb][kLinW]), symmetrised entries, written as
// real pairs in the compute precision (f32: float2, else double2) to out.
void launch_lin_entries(const Topology& t, const SetupDev& d, const int32_t* cols, bool f32, void* out,
                        cudaStream_t s);

// ---------------------------------------------------------------- batching
constexpr int kMaxBatch = 32;

// CTAs per SM of the S4+S5 kernel (its register budget, __launch_bounds__)
constexpr int near_ctas_per_sm(bool f32, bool single, int R = 8) { return R >= 16 ? 3 : (f32 ? 5 : 4); }
// CTAs per SM of the single-column c64 kernel (k_interp_near1; HALF: half-length chunks, 64 registers)
constexpr int near1_ctas_per_sm(bool half) { return half ? 8 : 5; }
// S4+S5 chunk lengths (entries) in the payload: C chunks 1024 / s, W chunks
// 256 / s, halved when the context holds 32 batch slots (the 32-column kernel
// keeps the same registers per lane)
constexpr int near_chc(bool f32, int slots) { return (f32 ? 128 : 64) / (slots >= 32 ? 2 : 1); }
constexpr int near_chw(bool f32, int slots) { return (f32 ? 32 : 16) / (slots >= 32 ? 2 : 1); }

// ---------------------------------------------------------------- spectrum
// Octant layout (all spectra): index ((ky (N_z+1) + kz) (N_x+1) + kx), x fastest.
struct SpectrumPlan {
  int Nx = 0, Ny = 0, Nz = 0;
  int nz1 = 0;                // z samples: Nz+1, or 1 (planar: the dz = 0 slice, 2-D transform); 0 -> Nz+1
  int64_t noct = 0;           // (Nx+1)(Ny+1) nz1
  double h = 0;
  int batch = 0;              // work buffers hold `batch` octants
  void* tw64[3] = {nullptr, nullptr, nullptr};   // fp64 twiddles, L = 2N per axis
  void* tw32[3] = {nullptr, nullptr, nullptr};   // fp32 twiddles
  void* work0 = nullptr;      // [batch][noct] complex (double2-sized)
  void* work1 = nullptr;
};

void spectrum_plan_init(SpectrumPlan& sp, int batch, cudaStream_t s);
void spectrum_plan_free(SpectrumPlan& sp);
// H_hat octant (unnormalised) of the static kernel, fp64.
// kind 0: the Green's function K = G (eq:hgf); 1: the radial factor F of
// grad G = -r F (double-layer operator, NEXT #1)
void spectrum_static(SpectrumPlan& sp, double2* out, cudaStream_t s, int kind = 0);
// Per-frequency, B frequencies: out[b] = scale * (Hs + DFT3(K_d(k0[b]))) in the
// compute precision (out stride noct).
void spectrum_dynamic_f32(SpectrumPlan& sp, int B, const double* k0, const float2* Hs, float scale,
                          float2* out, cudaStream_t s, int kind = 0);
void spectrum_dynamic_f64(SpectrumPlan& sp, int B, const double* k0, const double2* Hs,
                          double scale, double2* out, cudaStream_t s, int kind = 0);

// ---------------------------------------------------------------- profiler
// Per-stage CUDA-event timer (aimx_profile_*).
struct Profiler {
  bool on = false;
  int mask = 0x7f;             // stages bracketed while on (bit i = stage i)
  bool serial = false;         // sweeps on one stream while on (AIMX_PROFILE_SERIAL)
  std::vector<cudaEvent_t> pool;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  double ms[8] = {0};
  int64_t n[8] = {0};
  cudaEvent_t get();
  void begin(int stage, cudaStream_t s, cudaEvent_t& a);
  void end(int stage, cudaStream_t s, cudaEvent_t a);
  void collect();
  ~Profiler();
};

// A hot-path stage: an NVTX range on the host thread (named like bench.py's
// stages; visible to nsys / ncu --nvtx, a no-op without a tool attached)
// and, when the profiler is on for it, CUDA events around its launches.
constexpr const char* kStageNames[8] = {"aimx:spectrum", "aimx:proj_xfft", "aimx:yfwd", "aimx:zconv",
                                        "aimx:yinv", "aimx:xinv", "aimx:interp_near", "aimx:other"};
struct StageScope {
  Profiler* p;
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  StageScope(Profiler* p_, int st, cudaStream_t s_) : p(p_), stage(st), s(s_) {
    nvtxRangePushA(kStageNames[stage & 7]);
    if (p && p->on && ((p->mask >> stage) & 1)) p->begin(stage, s, a);
  }
  ~StageScope() {
    if (a) p->end(stage, s, a);
    nvtxRangePop();
  }
};

// ---------------------------------------------------------------- hot path
struct HotDev {
  // grid geometry
  int Nx = 0, Ny = 0, Nz = 0, p = 0, p3 = 0;
  int nb = 0, nocc = 0, nlines = 0, nzocc = 0;
  int W = 0;                     // row width (complex) of the y / z passes: 8 Nx, or 4 x (kx slab width)
  int kx0 = 0;                   // first kx of the column slab (slab-decomposed FFT), else 0
  int32_t* phi_line = nullptr;   // [nlines] phi line (y + Ny z) of each x-inverse line; null: line_id
  const void* tmB = nullptr;     // HOST pointer to the CUtensorMap of bufB (k_zconv_tma), or null
  int G = 8;                     // lanes per node in the projection gather
  int64_t nnz = 0;
  int batch = 0;                 // batch slots allocated
  // per-batch-slot strides (complex elements)
  int64_t sS = 0, sA = 0, sB = 0, sP = 0, sH = 0;
  // stencil / weights
  int32_t* rwg_base = nullptr;   // [nb] linear index of the stencil anchor node
  int32_t* node_lin = nullptr;   // [nocc]
  int32_t* node_line = nullptr;  // [nocc] index of the node's line in line_id
  int32_t* node_ptr = nullptr;   // [nocc+1]
  int32_t* ent_rwg = nullptr;    // [nent]
  void* ent_w = nullptr;         // [nent] real4
  int32_t* line_id = nullptr;    // [nlines] y + Ny z
  int32_t* zplanes = nullptr;    // [nzocc]
  int zplane0 = 0;               // the first occupied z plane (the z pass's one-plane form)
  // planar path (one occupied z plane, one-GPU contexts): bufA / bufC / phi hold
  // that plane only (line ids y, node indices lin - phi_off), bufB is absent and
  // S3 is x fwd -> y fwd * H_hat2 * y inv (k_yconv_plane) -> x inv with the
  // 2-D spectrum of the dz = 0 kernel slice [ky][kx]
  int planar = 0;
  int64_t phi_off = 0;           // linear grid index of phi's node 0 (planar: z0 Nx Ny)
  int nc = 4;                    // channels stored in S / bufA / bufC / phi: 4 (x, y, z, rho), or 3
                                 // (x, y, rho) on planar grids, where Lambda^z = 0 exactly (R12)
  void* S4 = nullptr;            // nc = 3: a 4-channel S for the double-layer operator's passes
  cudaEvent_t spec_ready = nullptr;   // HOST handle: the launch stream waits on it before the
                                      // spectrum multiply (sweep pipeline), or null
  uint8_t* line_occ = nullptr;   // [Ny*Nz]
  uint8_t* zocc = nullptr;       // [Nz] plane occupied
  // near matrix C = L_s,NR - L_s,P in row-group form (NearGroups)
  int R = 8;                     // rows per group
  int near_half = 0;            // 1: the payload's chunks are half length (32-slot contexts: near_chc / near_chw)
  int near1_old = 0;            // 1: single-column c64 launches keep the entry-per-lane kernel (AIMX_NEAR1_OLD=1 at setup; A/B)
  int near_mma = 0;              // 1: batched c64 launches take the tensor-core kernel (AIMX_NEAR_MMA=1 at setup)
  int ngrp = 0;
  int32_t* grp_rows = nullptr;   // [ngrp][R]
  unsigned char* payload = nullptr;   // NearChunks payloads: C pairs / W weights (zero where
                                      // not near / off-stencil), row indices, next descriptors
  int32_t* chunks = nullptr;     // [nchunk][4] NearChunks work list
  int32_t* cta_ptr = nullptr;    // [near_ctas+1] whole-group chunk ranges per CTA (batched launches)
  int near_ctas = 0;
  int32_t* warp_ptr1 = nullptr;  // [near_warps1+1] chunk ranges of whole groups per WARP (k_interp_near1w), or null
  int near_warps1 = 0;
  int32_t* cta_ptr1 = nullptr;   // [near_ctas1+1] the same for single-column launches
  int near_ctas1 = 0;
  // grid buffers (complex, 4 channels innermost), `batch` slots each
  void* S = nullptr;             // [nlines][Nx][4] gathered grid sources
  void* bufA = nullptr;          // [Nz][Ny][2Nx][4]
  void* bufB = nullptr;          // [Nz][2Ny][2Nx][4]
  void* bufC = nullptr;          // [Nz][Ny][2Nx][4]
  void* phi = nullptr;           // [Nz][Ny][Nx][4]
  void* twx = nullptr;           // exp(-2 pi i m / L), L = 2Nx, 2Ny, 2Nz (compute precision)
  void* twy_tab = nullptr;
  void* twz_tab = nullptr;
  void* Hoct = nullptr;          // [batch][noct] bound spectra / M (compute precision)
  void* xt = nullptr;            // [nb][16] batch-interleaved right-hand sides (near SpMM)
  // linear-term modification; null lin_col = off
  int32_t* lin_col = nullptr;    // [nb][kLinW] overlapping columns of the rows this HotDev tests, -1 padded
  void* lin_c = nullptr;         // [nb][kLinW] (C^A_lin, C^rho_lin) real pairs, compute precision
};

// ---------------------------------------------------------------- slab-decomposed FFT
// One rank of the y-slab / kx-slab decomposition (aimx_slab_plan): the
// projection, x transforms and S4+S5 run on the rank's rows, the y / z
// transforms on its kx slab; two all-to-all exchanges (NCCL, or device
// copies between the virtual ranks of one process) re-partition the grid.
struct SlabRank {
  int rank = 0;
  int y0 = 0, y1 = 0, yh1 = 0;   // owned rows [y0, y1); phi rows [y0, yh1)
  int kx0 = 0, kx1 = 0;          // kx slab of the y / z passes
  HotDev hr;                     // gather + x fwd on own rows (bufA: [Nz][y1-y0][2Nx][4]); S4+S5 of owned RWGs
  HotDev hc;                     // y fwd / z conv / y inv on the kx slab ([Nz][Ny or 2Ny][4 (kx1-kx0)])
  HotDev hx;                     // x inv of rows [y0, yh1) (bufC: [Nz][yh1-y0][2Nx][4]) -> phi
  std::vector<int32_t> owned;    // RWGs whose S4+S5 rows this rank computes
  int32_t* lin_col = nullptr;    // kLinW columns of the owned rows (others -1), when built
  void* send = nullptr;          // exchange staging (both exchanges share it)
  void* recv = nullptr;
};

// Per-launch batch arguments (by value).
struct Combine {
  int B = 1;                     // frequency points in this launch (<= batch slots)
  int mode = 0;                  // 0: y = alpha (yA - beta yR); 1: parts y0 = yA, y1 = -yR
  int64_t xstride = 0, ystride = 0;   // complex elements between batch vectors
  int xt_ready = 0;              // 1: h.xt already holds the interleaved columns (sweep pipeline)
  double alpha_im[kMaxBatch];    // alpha = j * alpha_im = -j w mu0
  double beta[kMaxBatch];        // k0^-2
};

// y += D(k0) x on the CSR pattern: combined (y += j alpha (D_A x - beta D_R x)) or parts
// (y0 += D_A x, y1 -= D_R x), one column
void aim_spmv(bool f32, int64_t nb, const int64_t* rowptr, const int32_t* col, const void* DA, const void* DR,
              const void* x, void* y0, void* y1, const Combine& cb, cudaStream_t s);

// ---- batched GMRES building blocks (solve.cu); B columns of N per block
struct PcArgs {
  double alpha_im[kMaxBatch];   // M_b = j alpha_im[b] (dA - beta[b] dR): the static diagonal preconditioner
  double beta[kMaxBatch];
};
void gm_pc(bool f32, int B, int64_t N, const void* in, void* out, const double* dA, const double* dR, const PcArgs& pa,
           bool accumulate, cudaStream_t s);
void gm_dots(bool f32, int nv, int B, int64_t N, const void* V, int64_t vstride, const void* W, double2* out,
             cudaStream_t s);
void gm_lincomb(bool f32, int nv, int B, int64_t N, const void* V, int64_t vstride, const double2* coef, void* W,
                bool assign, cudaStream_t s);
void gm_colscale(bool f32, int B, int64_t N, const void* W, const double* sc, void* out, cudaStream_t s);
void gm_colscale_rsqrt(bool f32, int B, int64_t N, const void* W, const double2* n2, void* out, cudaStream_t s);
void gm_sub(bool f32, int64_t n, const void* a, const void* b, void* out, cudaStream_t s);
void gm_axpy(bool f32, int64_t n, double a, const void* t, void* y, cudaStream_t s);   // y += a t
void gm_caxpy(bool f32, int64_t n, double ar, double ai, const void* t, void* y, cudaStream_t s);   // y += (ar + j ai) t
void gm_take(int64_t n, const int64_t* idx, const double* src, double* d, cudaStream_t s);

bool fft_length_supported(int L);
// bufB tensor map for the TMA z pass (out: 128-byte CUtensorMap); false if unavailable
bool make_z_tensor_map(const HotDev& h, bool f32, void* out);
void hot_matvec_f32(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c,
                    cudaStream_t s, Profiler* prof);
// xt <- the batch-interleaved columns of x (Combine: B, xstride)
void interleave_f32(const HotDev& h, const void* x, const Combine& c, cudaStream_t s);
// the two halves of hot_matvec: S2 + S3 up to phi, and S4 + S5 from phi and xt
void hot_grid_f32(const HotDev& h, const void* x, const Combine& c, cudaStream_t s, Profiler* prof);
void hot_grid_f64(const HotDev& h, const void* x, const Combine& c, cudaStream_t s, Profiler* prof);
void hot_near_f32(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                  Profiler* prof);
void hot_near_f64(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s,
                  Profiler* prof);
void interleave_f64(const HotDev& h, const void* x, const Combine& c, cudaStream_t s);
void hot_matvec_f64(const HotDev& h, const void* x, void* y0, void* y1, const Combine& c,
                    cudaStream_t s, Profiler* prof);
// Slab-decomposed hot path: every rank's S2-S5; the exchanges go through
// `xchg` (step 0: rows -> kx slabs, step 1: kx slabs -> rows incl. halo).
struct SlabExchange {
  virtual void run(std::vector<SlabRank*>& ranks, int step, int B, size_t csize, cudaStream_t s) = 0;
  virtual ~SlabExchange() {}
};
void slab_matvec(std::vector<SlabRank*>& ranks, int Ny, int Nz, int Nx, bool f32, SlabExchange& xchg,
                 const void* x, void* y0, void* y1, const Combine& c, cudaStream_t s, Profiler* prof);
// block copy [d0][d1][d2][d3 complex] between strided layouts (strides in complex)
void copy4(void* dst, const int64_t dstr[3], const void* src, const int64_t sstr[3], const int64_t dims[4],
           size_t csize, cudaStream_t s);

}  // namespace aimx
