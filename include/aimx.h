/*
 * aimx.h -- C ABI of the B200-native AIMx matrix-vector product.
 *
 * Method: Sharma & Triverio, "AIMx: An Extended Adaptive Integral Method for
 * the Fast Electromagnetic Modeling of Complex Structures" (arxiv 2009.02281).
 * Citations "P:<line>" refer to that paper's LaTeX source with the
 * equation label.  The library computes, for the EFIE of a PEC surface in free
 * space (eq:EFIEdis P:179-181),
 *
 *     y = Z(k0) x = -j w mu0 ( L_A + k0^-2 L_phi ) x,
 *     L   ~= L_s,NR - L_s,P + W H(k0) P                  (eq:LAIMx P:283)
 *
 * split as eq:EFIEAIMx: the sparse, frequency-independent near matrix
 * L_s,NR and precorrection L_s,P = W H_s,NR P (eq:aimLPs P:276) are built ONCE
 * with the static kernel G_s = 1/(4 pi r) (change (a)); the grid
 * convolution H(k0) (eq:Hmn P:305, three-level Toeplitz) carries all
 * frequency dependence, with the modified self term H^(m,m) = -j k0/(4 pi)
 * (eq:Hmm P:335).  Its spectrum is H_hat_s (static, built once) + DFT(K_d(k0))
 * (regenerated per frequency on the device).
 *
 * Conventions
 * -----------
 * - Every function returns an aimx_status; no C++ exception crosses the ABI.
 * - All host arrays passed in are BORROWED for the duration of the call and
 *   copied; the library never keeps a host pointer.
 * - Device vectors x / y / X / Y are owned by the caller (e.g. torch tensors
 *   via data_ptr()); they are contiguous complex numbers, interleaved
 *   (re, im), complex64 (float2) for AIMX_C64 and complex128 (double2) for
 *   AIMX_C128, in the EXTERNAL RWG order (ascending lexicographic vertex pair,
 *   see aimx_get_rwg).  Input and output must not alias.
 * - `stream` is a cudaStream_t passed as void*; NULL means the context's own
 *   stream (the one given to aimx_setup).  Work is enqueued asynchronously:
 *   no host synchronisation and no buffer allocation happens in aimx_matvec /
 *   aimx_matvec_parts / aimx_sweep, with one exception: the second call of
 *   aimx_matvec / aimx_matvec_parts with the same (x, y, mode, frequency)
 *   captures its launch sequence and instantiates a CUDA graph (driver
 *   memory for the graph; at most 8 are kept; AIMX_NO_GRAPH=1 disables it),
 *   which later identical calls replay.  aimx_matvec_pmchwt allocates its
 *   interior-medium spectra on its first call.  A context owns one set of
 *   work buffers: calls on different streams are ordered by the library with
 *   events (each waits for the previous call on any stream), never run
 *   concurrently on those buffers; a context is not thread-safe.
 * - Asynchronous CUDA faults surface as AIMX_E_CUDA on the next call.
 * - Independent contexts are independent (one per GPU / process in the
 *   multi-GPU frequency-sharded sweep).
 */
#ifndef AIMX_H
#define AIMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AIMX_OK = 0,
  AIMX_E_INVALID_ARG = 1,  /* NULL pointer, size/precision mismatch, f <= 0 or not finite */
  AIMX_E_MESH = 2,         /* index out of range, repeated vertex, zero-area triangle,
                              edge in > 2 triangles, inconsistent orientation, no RWG */
  AIMX_E_GRID = 3,         /* grid too small: a stencil does not fit, bad order/threshold */
  AIMX_E_STATE = 4,        /* matvec before aimx_set_frequency */
  AIMX_E_OOM = 5,          /* device or host allocation failed */
  AIMX_E_CUDA = 6,         /* CUDA runtime error (message in aimx_last_error) */
  AIMX_E_UNSUPPORTED = 7,  /* grid length with no compiled FFT kernel (see aimx.h notes) */
  AIMX_E_INTERNAL = 8,
  AIMX_E_NCCL = 9,         /* NCCL failure, or an asynchronous NCCL error found by polling: the
                              communicator has been aborted (sticky for the context) */
  AIMX_E_TIMEOUT = 10      /* aimx_sync: the work did not finish in time (NCCL contexts: the
                              communicator has been aborted, e.g. a peer rank hung or died) */
} aimx_status;

typedef enum {
  AIMX_C64 = 0,   /* complex64 storage and arithmetic on the hot path; setup in fp64 */
  AIMX_C128 = 1   /* complex128 throughout */
} aimx_prec;

/* Triangle mesh: vertices [nv][3] in metres (row-major float64),
 * triangles [nt][3] 0-based vertex indices (int32).  Triangles must be
 * consistently oriented (closed surfaces: outward).  Interior edges (shared by
 * exactly two triangles) carry the RWG unknowns; boundary edges none. */
typedef struct {
  int64_t nv;
  const double* vertices;
  int64_t nt;
  const int32_t* triangles;
} aimx_mesh_desc;

/* AIM grid: n[3] = (N_x, N_y, N_z) unpadded points; order = stencil
 * order n (n+1 points per axis), 1..3; near_cells = near-region
 * threshold T in grid cells (pairs whose stencils are within T cells,
 * Euclidean, are "near").  h <= 0 derives spacing and origin from the
 * mesh bounding box (margin ceil(n/2) nodes, isotropic h =
 * max_a ext_a / (N_a - 1 - 2 margin), origin = min - margin*h); otherwise h
 * and origin[3] are used as given.  Supported FFT lengths: 2*N_a must be a
 * power of two in [8, 1024]. */
typedef struct {
  int32_t n[3];
  int32_t order;
  int32_t near_cells;
  double h;
  double origin[3];
} aimx_grid_desc;

typedef struct aimx_ctx aimx_ctx;

typedef struct {
  int64_t num_unknowns;       /* N_b */
  int64_t nnz;                /* near pairs */
  int64_t occupied_nodes;     /* grid nodes carrying a non-zero projection weight */
  int64_t occupied_lines;     /* x-lines (y, z) with an occupied node */
  int64_t occupied_planes;    /* z planes with an occupied node */
  int64_t projection_entries; /* (RWG, node) pairs with a non-zero projection weight */
  int64_t device_bytes;       /* device memory owned by the context */
  int64_t batch_slots;        /* frequency points per device batch (aimx_sweep) */
  double setup_seconds;       /* wall time of aimx_setup */
  int32_t n[3];
  int32_t order;
  double h;
  double origin[3];
  int32_t near_group_rows;    /* R: rows per group of the near matrix's row-group layout */
  int32_t near_row_order;     /* 0: rows ordered by anchor linear index, 1: by anchor Morton code */
  int64_t near_union;         /* stored (column, group) entries; fill = nnz / (near_union * R) */
  int32_t planar;             /* 1: one occupied z plane, S3 runs in its exact 2-D form with the
                                 dz = 0 kernel slice (AIMX_NO_PLANAR=1 at setup keeps the 3-D path) */
  int32_t kop_grad;           /* 1: the double-layer operator K runs through the gradient-of-kernel
                                 spectra (set after aimx_set_kop; 0: the radial form or not built) */
  int32_t grid_channels;      /* channels of the grid passes: 4 (x, y, z, rho), or 3 on planar grids
                                 whose Lambda^z is exactly zero (AIMX_NO_ZSKIP=1 keeps 4) */
  int32_t reserved;
} aimx_stats;

/* S0 (the paper's "one-time static matrix-fill", tab:prof P:715): RWG basis,
 * grid, stencil anchors, near-region map, projection weights, static near
 * integrals L_s,NR (analytic inner, 7-point outer, symmetrised), precorrection
 * L_s,P, C = L_s,NR - L_s,P (fp64, stored in `prec`), static spectrum H_hat_s.
 * The only host->device copies of the context happen here.  `stream` becomes
 * the context stream (NULL = legacy default stream).  On failure *out is NULL
 * and aimx_last_setup_error() describes the cause. */
aimx_status aimx_setup(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid,
                       aimx_prec prec, int device, void* stream, aimx_ctx** out);

/* Static-setup cache (P:905-906 suggests storing the
 * frequency-independent near matrix to disk and reusing it across sweeps).
 * aimx_save_static writes the fp64 static matrices (C_A, C_rho and their four
 * constituents, CSR order), the projection weights and their exact-zero flags,
 * keyed by a hash of the mesh arrays and the grid descriptor.
 * aimx_setup_cached is aimx_setup that reads them instead of computing the
 * static fill: the integer topology is rebuilt from `mesh` and must match the
 * file (else AIMX_E_INVALID_ARG); results are bit-identical to aimx_setup. */
aimx_status aimx_save_static(const aimx_ctx* ctx, const char* path);
aimx_status aimx_setup_cached(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, aimx_prec prec,
                              int device, const char* path, void* stream, aimx_ctx** out);

/* S1: bind the frequency f (Hz): k0 = 2 pi f / c0; H_hat(k0) = H_hat_s +
 * DFT3(K_d(k0)) with K_d = (e^{-j k0 r} - 1)/(4 pi r) (eq:hgfd P:231) and
 * K_d(0) = -j k0/(4 pi) (eq:Hdmm P:331), generated on the device on the
 * context stream.  Does not touch C or the weights (byte-identical across
 * frequencies).  Idempotent.  f must be finite and > 0 (k0 = 0 rejected). */
aimx_status aimx_set_frequency(aimx_ctx* ctx, double f_hz);

/* Linear-term accuracy modification (sec:methods:aimx:acc P:361-398):
 * k0^2 G_lin, G_lin(r) = -r/(8 pi) (eq:linterm P:365), is integrated directly
 * on the pairs whose supports share a triangle (at most 5 per row, "O(N)"
 * P:396) and applied on the fly scaled by k0^2 (eq:Lmatdecomplin P:388):
 *   y^A   += k0^2 C^A_lin x,   C^A_lin   = L^A_lin   - sum_c W^c H_lin P^c,
 *   y^rho += k0^2 C^rho_lin x, C^rho_lin = y^rho_lin - W^rho H_lin P^rho,
 * with H_lin(delta) = G_lin(h |delta|) (the grid operator itself is unchanged:
 * its samples already contain k0^2 G_lin).  enable != 0 turns it on for every
 * later matvec, sweep and solve of the context (the first call builds C_lin on
 * the device, fp64, stored in `prec`; synchronises the context stream);
 * enable == 0 turns it off.  Off by default (the paper's results do not use it,
 * P:648).  aimx_get_linear_term reports the current state. */
aimx_status aimx_set_linear_term(aimx_ctx* ctx, int enable);
aimx_status aimx_get_linear_term(const aimx_ctx* ctx, int* enabled);

/* Conventional AIM mode (sec:methods:aim P:186-210), the method AIMx is
 * measured against: the near region is regenerated by direct integration at
 * every frequency ("Both L_NR(k0) and L_P(k0) must be generated for each
 * frequency").  With the same grid, weights and static matrices it is
 * AIMx plus, on the near pattern,
 *   D(k0) = L_d,NR(k0) - W H_d,NR(k0) P
 * (L_d,NR by the 7 x 7 product rule with G_d = G - G_s, H_d the grid samples
 * of G_d with H_d(0) = -j k0/(4 pi)), so near entries are direct integration
 * and far entries the grid.  enable != 0: every later aimx_set_frequency (and
 * each frequency of a sweep) runs that fill on the device (fp64, stored in
 * `prec`), matvec / parts / sweep add D(k0) x; sweeps run frequency by
 * frequency.  Exclusive with the linear-term modification (AIMX_E_INVALID_ARG);
 * one-GPU contexts only; aimx_solve then runs one frequency at a time, each
 * with its near fill (same static diagonal preconditioner).
 * aimx_get_aim_entries: D_A, D_rho of the bound frequency as complex128 in CSR
 * order ([nnz] interleaved re/im; AIMX_E_STATE when off or unbound). */
aimx_status aimx_set_conventional(aimx_ctx* ctx, int enable);
aimx_status aimx_get_aim_entries(const aimx_ctx* ctx, double* DA, double* Drho);

/* S2-S5: y = Z(k0) x = -j w mu0 (y^A - k0^-2 y^rho) (eq:EFIEAIMx P:288), where
 * y^A = W^(A) H P^(A) x + C_A x and y^rho = W^(phi) H P^(phi) x + C_rho x.
 * x, y: device vectors of N_b complex numbers (see conventions). */
aimx_status aimx_matvec(aimx_ctx* ctx, const void* x, void* y, void* stream);

/* Several right-hand sides at the bound frequency: Y[i,:] = Z(k0) X[i,:] for
 * i < nrhs (device [nrhs][N_b]), in device batches of the context's slots
 * (the batched kernels, one spectrum for all columns).  AIMX_E_UNSUPPORTED
 * for slab contexts and in conventional-AIM / CFIE mode. */
aimx_status aimx_matvec_multi(aimx_ctx* ctx, int64_t nrhs, const void* X, void* Y, void* stream);

/* Parts, unscaled: yA = L_A x = y^A, yPhi = L_phi x = -y^rho (the divergence is
 * moved to the testing function).  Either output may be NULL. */
aimx_status aimx_matvec_parts(aimx_ctx* ctx, const void* x, void* yA, void* yPhi,
                              void* stream);

/* Frequency sweep: for i < nf, Y[i,:] = Z(f_hz[i]) X[i,:] (per frequency: S1
 * then S2-S5).  f_hz is a HOST array; X, Y device arrays [nf][N_b] row-major.
 * Frequencies run in device batches of `batch` points, the remainder last
 * (<= 0 or more than the context's batch slots: all slots; slots are chosen at
 * setup from the grid size, at most 32, environment variable AIMX_BATCH
 * overrides): the spectra of
 * a batch are generated together and one batched matvec reads the near matrix
 * and the weights once for all of its right-hand sides.  Results are
 * deterministic (fixed-order reductions, no atomics); across batch sizes the
 * near-row sums are partitioned differently and agree to rounding.  The context's bound
 * frequency is restored afterwards if one was set. */
aimx_status aimx_sweep(aimx_ctx* ctx, int64_t nf, const double* f_hz, const void* X,
                       void* Y, int32_t batch, void* stream);

/* Iterative solve: for i < nf, Z(f_hz[i]) X[i,:] = RHS[i,:]
 * by restarted GMRES(restart) as the paper's sweep does (GMRES,
 * relative residual `tol`, the paper uses 1e-4), right-preconditioned with the
 * diagonal of the frequency-independent near matrix (M(k0) =
 * diag(-j w mu0 (L^A_s,NR[m,m] + k0^-2 L^phi_s,NR[m,m]))), x0 = 0.
 * Frequencies run in device batches (the slots, balanced over the batches
 * needed): each batch's spectra
 * are generated once and all its columns iterate together, each with its own
 * Krylov basis (Arnoldi by classical Gram-Schmidt applied twice, Givens on the
 * host).  RHS, X: device [nf][N_b]; f_hz, iters (iterations used, may be
 * NULL) and relres (final true residual ||RHS - Z X|| / ||RHS||, may be NULL)
 * are HOST arrays.  maxiter bounds the iterations per batch.  One-GPU contexts
 * only (AIMX_E_UNSUPPORTED for slab contexts).  Synchronises `stream` per
 * iteration (the Hessenberg work is on the host). */
aimx_status aimx_solve(aimx_ctx* ctx, int64_t nf, const double* f_hz, const void* RHS, void* X, double tol,
                       int32_t restart, int32_t maxiter, int32_t* iters, double* relres, void* stream);

/* The same sweep with X, Y in HOST memory (pinned or pageable): the library
 * stages each batch host->device and the results device->host on `stream`
 * and synchronises the stream before returning.  With batch <= 0 the first
 * device batch is 3/4 of the slots (its copy is shorter, the compute starts
 * sooner), so results equal aimx_sweep's to rounding; with an explicit batch
 * the batches, and the results bit for bit, are aimx_sweep's. */
aimx_status aimx_sweep_host(aimx_ctx* ctx, int64_t nf, const double* f_hz, const void* X,
                            void* Y, int32_t batch, void* stream);

/* Per-frequency status of a sweep's (or a solve's) result: status[i] (HOST,
 * int32[nf]) = 0 when every element of Y[i,:] is finite, 1 when Y[i,:] holds a
 * NaN or an infinity (e.g. a frequency whose inputs overflowed).  Y: device
 * [nf][N_b] as written by aimx_sweep / aimx_solve; one device pass over Y on
 * `stream`, then a host synchronisation of `stream`. */
aimx_status aimx_sweep_status(aimx_ctx* ctx, int64_t nf, const void* Y, int32_t* status, void* stream);

/* ---- introspection (parity tests; all host buffers, caller-allocated) ---- */
int64_t aimx_num_unknowns(const aimx_ctx* ctx);
aimx_status aimx_get_stats(const aimx_ctx* ctx, aimx_stats* out);
/* edge_ab[N_b][2] (a < b), tri_pm[N_b][2] (T+, T-), free_pm[N_b][2] (p+, p-);
 * any pointer may be NULL. */
aimx_status aimx_get_rwg(const aimx_ctx* ctx, int32_t* edge_ab, int32_t* tri_pm,
                         int32_t* free_pm);
/* anchors[N_b][3]: lowest stencil node index per axis. */
aimx_status aimx_get_anchors(const aimx_ctx* ctx, int32_t* anchors);
/* Two-call: with rowptr == NULL and col == NULL only *nnz is written.
 * rowptr[N_b+1] (int64), col[nnz] ascending per row. */
aimx_status aimx_get_near_csr(const aimx_ctx* ctx, int64_t* rowptr, int32_t* col,
                              int64_t* nnz);
/* C_A = L^A_s,NR - L^A_s,P and C_rho = y^rho_s,NR - y^rho_s,P (fp64, CSR order);
 * optional: the four constituent matrices (any pointer may be NULL). */
aimx_status aimx_get_static(const aimx_ctx* ctx, double* CA, double* Crho,
                            double* LA_NR, double* Yrho_NR, double* LA_P, double* Yrho_P);
/* Linear-term modification (aimx_set_linear_term; AIMX_E_STATE before its
 * first enable): cols[N_b][5] overlapping columns (ascending, -1 padded) and
 * C^A_lin, C^rho_lin [N_b][5] as stored (compute precision, widened to fp64).
 * Any pointer may be NULL. */
aimx_status aimx_get_linear_entries(const aimx_ctx* ctx, int32_t* cols, double* CA_lin, double* Crho_lin);
/* Double-layer operator K (sec:methods:K P:400-474):
 * aimx_set_kop(ctx, 1) builds its static near part C_K (below) and the static
 * spectrum of F_s = 1/(4 pi r^3); every later aimx_set_frequency also forms
 * F_hat(k0).  aimx_matvec_kop: y = Kmat x (reading R24: -int f_m . PV K[f_n]
 * + the exterior residue), eq:KAIMx with the grid part through the even radial
 * factor F of grad G = -r F: sum_ab eps_cab (d_a G (*) J_b) = -h [s x (F (*) J)
 * - F (*) (s x J)] (two passes of the hot-path transforms), W^(K) = -P^T of
 * the current channels, + C_K x.  One column, device vectors as aimx_matvec;
 * AIMX_E_STATE when not enabled or no frequency bound; one-GPU contexts. */
aimx_status aimx_set_kop(aimx_ctx* ctx, int enable);
/* CFIE (eq:CFIEdis P:422, closed PEC surfaces): enable != 0 makes every later
 * combined matvec, sweep point and solve apply (-j w mu0 L - eta0 Kmat)
 * (eta0 = mu0 c0; parts stay the L parts); sweeps and solves then run one
 * frequency at a time.  Enables K (aimx_set_kop) if needed; exclusive with
 * the conventional-AIM mode. */
aimx_status aimx_set_cfie(aimx_ctx* ctx, int enable);
/* PMCHWT for a homogeneous dielectric body (cfg4's formulation; reading R27,
 * AMB-17 -- the paper names PMCHWT but never states it): x = [J; M] and
 * y = [y_E; y_H], device vectors of 2 N_b complex,
 *   y_E = (Z0 + Z1) J - (K0 + K1) M,   y_H = (K0 + K1) J + (Z0/eta0^2 + Z1/eta1^2) M,
 * medium 0 outside (k0 of the bound frequency), medium 1 inside (k1 = k0
 * sqrt(eps_r), eta1 = eta0/sqrt(eps_r), mu_r = 1); Z_i = -j w mu0 (L_A(k_i) +
 * k_i^-2 L_phi(k_i)) with the physical w; K_i the tested principal-value K
 * (the exterior and interior residues cancel).  Both media share the static
 * matrices (G_s is medium-free).  Needs aimx_set_kop's static part
 * (AIMX_E_STATE otherwise); AIMX_E_INVALID_ARG in conventional-AIM or CFIE
 * mode. */
aimx_status aimx_matvec_pmchwt(aimx_ctx* ctx, double eps_r, const void* x, void* y, void* stream);
aimx_status aimx_matvec_kop(aimx_ctx* ctx, const void* x, void* y, void* stream);
/* Double-layer operator K, static near part (SURVEY 8(f) NEXT #1 groundwork;
 * sec:methods:K P:400-474, readings R23-R25): CK[nnz] (fp64, CSR order) =
 * sym(K_s,PV) + 1/2 int f_m . (n x f_n) - K_s,P, computed on the device on
 * demand (introspection for the parity tests).  One-GPU contexts only. */
aimx_status aimx_get_kop_static(aimx_ctx* ctx, double* CK);
/* Projection weights (fp64) lam[N_b][4][(n+1)^3], channels (x, y, z, rho),
 * node s = i + (n+1)(j + (n+1) k). */
aimx_status aimx_get_weights(const aimx_ctx* ctx, double* lam);
/* Spectrum octant, complex128 interleaved, index ((ky (N_z+1) + kz)(N_x+1) + kx):
 * which = 0 static H_hat_s, 1 the bound H_hat(k0) (unnormalised DFT).
 * Planar contexts (aimx_stats.planar = 1): the 2-D spectrum of the dz = 0
 * kernel slice, index (ky (N_x+1) + kx); it equals the 3-D octant summed over
 * all 2 N_z values of kz, divided by 2 N_z. */
aimx_status aimx_get_spectrum(const aimx_ctx* ctx, int which, double* out);

/* ---- stage profiling (CUDA events recorded on the launching stream) ----
 * Stages: 0 spectrum (S1: sample + 3 DCT passes), 1 proj_xfft (S2 + x fwd),
 * 2 yfwd, 3 zconv (z fwd * H_hat * z inv), 4 yinv, 5 xinv, 6 interp_near
 * (S4 + S5).  When enabled, every launch of a stage is bracketed by a pair of
 * events; aimx_profile_read synchronises the context, adds up the elapsed
 * device time per stage (ms) and the number of bracketed launches since the
 * previous read, and resets them.  Arrays have AIMX_NUM_STAGES entries.
 * *kernels (optional) receives the number of kernels this thread launched
 * through the library since the last aimx_profile_enable / aimx_profile_read. */
#define AIMX_NUM_STAGES 7
aimx_status aimx_profile_enable(aimx_ctx* ctx, int on);
aimx_status aimx_profile_read(aimx_ctx* ctx, double* ms, int64_t* launches, int64_t* kernels);
/* Which stages are bracketed while profiling is on (bit i = stage i; default
 * all).  Each bracket is a pair of events on the stream, which also ends the
 * overlap of consecutive kernels' launches (programmatic dependent launch)
 * at that point, so a timed run brackets only the stage it reports.
 * AIMX_PROFILE_SERIAL in the mask: while profiling is on, sweeps run their
 * device batches on one stream (no overlap of one batch's spectra or S4+S5
 * with the next batch's grid stages), so each stage's time is its own. */
#define AIMX_PROFILE_SERIAL 0x80
aimx_status aimx_profile_stages(aimx_ctx* ctx, int32_t mask);

/* ---- slab-decomposed FFT (multi-GPU for the largest grid) ----
 * Host-only plan (no GPU needed): for `world` ranks, rank `rank` owns the
 * unpadded grid rows y in [out[0], out[1]) (the RWGs whose stencil anchor row
 * lies there: projection, x transforms, interpolation and near rows), needs
 * potentials on rows [out[0], out[2]) (stencils reach `order` rows past the
 * block) and transforms the padded kx slab [out[3], out[4]) along y and z.
 * 2 N_x / world must be a power of two and N_y >= world (else UNSUPPORTED). */
aimx_status aimx_slab_plan(const int32_t n[3], int32_t order, int32_t world, int32_t rank,
                           int32_t out[6]);

/* Slab-decomposed context.  nccl_id == NULL: EMULATION -- the `world` ranks
 * all live in this context on one device and the two all-to-all exchanges of
 * every matvec are device copies between them (same kernels, same exchange
 * buffers as the NCCL path; for testing on one GPU).  nccl_id != NULL: this
 * process is rank `rank` of `world`, one GPU each; nccl_id is the 128-byte
 * ncclUniqueId from aimx_nccl_unique_id on rank 0, broadcast by the caller;
 * the exchanges are grouped ncclSend/ncclRecv and the owned rows of y are
 * summed over ranks with ncclAllReduce, so every rank returns the full y.
 * matvec / matvec_parts / sweep / set_frequency then behave as for
 * aimx_setup (x is replicated on every rank). */
aimx_status aimx_setup_slab(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, aimx_prec prec,
                            int device, int32_t rank, int32_t world, const uint8_t* nccl_id,
                            void* stream, aimx_ctx** out);
/* Wait on the host until every call enqueued on the context (any stream)
 * has finished, polling every 0.2 ms.  NCCL (slab) contexts also poll
 * ncclCommGetAsyncError: an asynchronous NCCL error, or no completion within
 * timeout_s seconds (<= 0: no limit), aborts the communicator
 * (ncclCommAbort) so the rank cannot deadlock on a dead or hung peer, and
 * returns AIMX_E_NCCL / AIMX_E_TIMEOUT; every later call on the context then
 * returns AIMX_E_NCCL.  Every API call also polls the asynchronous error
 * first. */
aimx_status aimx_sync(aimx_ctx* ctx, double timeout_s);

/* ncclGetUniqueId (NCCL loaded at run time; AIMX_E_UNSUPPORTED if absent). */
aimx_status aimx_nccl_unique_id(uint8_t id[128]);

void aimx_destroy(aimx_ctx* ctx);
const char* aimx_status_string(aimx_status s);
const char* aimx_last_error(const aimx_ctx* ctx);
const char* aimx_last_setup_error(void);
const char* aimx_version(void);

#ifdef __cplusplus
}
#endif
#endif /* AIMX_H */
