// Internal declarations of the AIMx B200 library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/aimx.h"

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

#define AIMX_CHECK_LAUNCH() AIMX_CUDA(cudaGetLastError())

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
  std::vector<int32_t> ent_rwg;    // [nent]
  std::vector<int32_t> ent_slot;   // [nent] stencil slot s
  std::vector<int32_t> line_id;    // [nlines] y + Ny z, ascending
  std::vector<int32_t> line_ptr;   // [nlines+1] into node arrays
  std::vector<int32_t> zplanes;    // occupied z planes, ascending
  std::vector<uint8_t> line_occ;   // [Ny*Nz]
};

void build_nodemap(const Topology& t, const std::vector<uint8_t>& nz_slot, NodeMap& m);

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

// ---------------------------------------------------------------- spectrum
struct SpectrumPlan {
  int Nx, Ny, Nz;
  int64_t noct;               // (Nx+1)(Ny+1)(Nz+1)
  double h;
  double* cosx = nullptr;     // DCT-I matrices [(N+1)][(N+1)] per axis (fp64)
  double* cosy = nullptr;
  double* cosz = nullptr;
  float* cosx_f = nullptr;    // fp32 copies for the c64 per-frequency path
  float* cosy_f = nullptr;
  float* cosz_f = nullptr;
  void* work0 = nullptr;      // octant work buffers (complex, compute precision)
  void* work1 = nullptr;
};

void spectrum_plan_init(SpectrumPlan& sp, cudaStream_t s);
void spectrum_plan_free(SpectrumPlan& sp);
// H_hat octant (unnormalised) of the static kernel, fp64.
void spectrum_static(SpectrumPlan& sp, double2* out, cudaStream_t s);
// Per-frequency: out = scale * (Hs + DCT3(K_d(k0))) in precision T.
void spectrum_dynamic_f32(SpectrumPlan& sp, double k0, const float2* Hs, float scale, float2* out,
                          cudaStream_t s);
void spectrum_dynamic_f64(SpectrumPlan& sp, double k0, const double2* Hs, double scale,
                          double2* out, cudaStream_t s);

// ---------------------------------------------------------------- hot path
struct HotDev {
  // grid geometry
  int Nx, Ny, Nz, p, p3;
  int nb, nocc, nlines, nzocc;
  int64_t nnz;
  // stencil / weights
  int32_t* rwg_base = nullptr;   // [nb] linear index of the stencil anchor node
  void* lam = nullptr;           // [nb][p3] real4 (x,y,z,rho), compute precision
  int32_t* node_lin = nullptr;
  int32_t* node_ptr = nullptr;
  int32_t* ent_rwg = nullptr;
  void* ent_w = nullptr;         // [nent] real4
  int32_t* line_id = nullptr;
  int32_t* line_ptr = nullptr;
  int32_t* zplanes = nullptr;
  uint8_t* line_occ = nullptr;
  // near matrix (CSR, int32 offsets)
  int32_t* rowptr = nullptr;
  int32_t* col = nullptr;
  void* cval = nullptr;          // [nnz] real2 (C_A, C_rho)
  // grid buffers (complex, 4 channels innermost)
  void* bufA = nullptr;          // [Nz][Ny][2Nx][4]
  void* bufB = nullptr;          // [Nz][2Ny][2Nx][4]
  void* bufC = nullptr;          // [Nz][Ny][2Nx][4]
  void* phi = nullptr;           // [Nz][Ny][Nx][4]
  // twiddles exp(-2 pi i m / L) for L = 2Nx, 2Ny, 2Nz (compute precision)
  void* twx = nullptr;
  void* twy = nullptr;
  void* twz = nullptr;
  void* Hoct = nullptr;          // bound spectrum octant / M (compute precision)
};

// Per-stage CUDA-event timer (aimx_profile_*).
struct Profiler {
  bool on = false;
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

struct StageScope {
  Profiler* p;
  int stage;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  StageScope(Profiler* p_, int st, cudaStream_t s_) : p(p_), stage(st), s(s_) {
    if (p && p->on) p->begin(stage, s, a);
  }
  ~StageScope() {
    if (p && p->on) p->end(stage, s, a);
  }
};

struct Combine {
  // y = alpha (yA - beta yR), alpha = -j w mu0 (purely imaginary), beta = k0^-2;
  // mode 0: combined into y0; mode 1: parts y0 = yA, y1 = -yR.
  double alpha_im;
  double beta;
  int mode;
};

bool fft_length_supported(int L);
void hot_matvec_f32(const HotDev& h, const void* x, void* y0, void* y1, Combine c, cudaStream_t s,
                    Profiler* prof);
void hot_matvec_f64(const HotDev& h, const void* x, void* y0, void* y1, Combine c, cudaStream_t s,
                    Profiler* prof);

}  // namespace aimx
