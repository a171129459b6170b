// fem_internal.cuh -- shared device/host declarations of the CUDA path (libfem.so).
// Not part of the ABI.  Independent of oracle/ (no shared code, tables or constants).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fem {

// Geometry of the rank-local problem, in GLOBAL node-plane indices.
struct Grid {
  int64_t nx, ny, nz;    // cells per direction (global)
  double h;              // cell side
  int64_t k0, k1;        // owned node planes [k0, k1)
  int64_t plane;         // nodes per plane = (nx+1)(ny+1)
};

// Source of a node-plane-indexed vector: node (i, j) comp c of owned plane k at
//   main[(k - k0) * ppitch + j * rpitch + i * C + c]
// (dense ABI layout: rpitch = (nx+1) C, ppitch = (nx+1)(ny+1) C; the library's padded layout has
// even pitches), optional ghost planes below/above (multi-GPU halo) with the same
// row pitch; other planes are outside the domain.
struct PlaneSrc {
  const double* main;
  const double* lo;  // plane k0-1 (may be null: outside domain or not exchanged)
  const double* hi;  // plane k1
  int64_t rpitch, ppitch;
};

// Output vector: node (i, j) comp c of owned plane k at y[(k - k0) * ppitch + j * rpitch + i*C + c].
struct OutVec {
  double* y;
  int64_t rpitch, ppitch;
};

// Peer halo (option "peer_halo"): tensor maps over the NEIGHBOUR ranks' padded
// vectors (CUDA IPC over NVLink / NVSwitch) for the ghost planes klo = k0-1 and khi = k1, so the
// apply's producer warp loads them straight from peer memory -- no separate halo exchange.
// on = 0: the ghost planes come from the local padded buffer (NCCL halo).
struct __align__(64) PeerMaps {
  CUtensorMap lo, hi;    // u ghost planes
  CUtensorMap lo2, hi2;  // u2 (mode 2: p_old) ghost planes
  int64_t klo, khi;      // global plane index served by lo / hi (-2^62: none)
  int on;
};

// Row-pair view of a dense caller vector with odd rows (PlaneRing PAIR, kernels_common.cuh)
struct PairGeom {
  int64_t lr, lp;  // row / plane length of the caller vector in elements
  int64_t nz;      // last node plane of the view (global index)
  int64_t k0 = 0;  // first node plane of the view (a slab's owned planes start at k0; plane pairs
                   // and parities count from there; other planes come from PeerMaps or read as 0)
};

// TMA tensor maps of one apply launch (u plane: padded layout; material: interleaved lambda/mu)
// mode 2 (fused CG): the operator input is p = r + beta p_old formed in the kernel; u is r,
// u2 is p_old, p is written to pnew (owned nodes, padded layout of x).
struct ApplyMaps {
  const CUtensorMap* u;    // nullptr: use the bulk-row path
  int64_t t_i0, t_j0, t_k0;  // global node of the u tensor origin
  const CUtensorMap* mat;  // elasticity only
  int64_t mat_layer0;
  const CUtensorMap* u2;   // mode 2: p_old
  const double* pold;      // mode 2: p_old owned plane k0 (same layout as x)
  double* pnew;            // mode 2: p output owned plane k0 (same layout as x)
  int interior;            // 1: u tensor spans only the Dirichlet interior (zero fill = mask)
  int quad;                // 0: 2x2x2 Gauss-Legendre (default), 1: 2x2x2 Gauss-Lobatto (BP5/BP6)
  const PeerMaps* peer;    // ghost planes from peer memory (nullptr / on = 0: local)
  const PairGeom* pair = nullptr;  // u is a row-pair view of a caller vector (kernels_common.cuh)
  // halo overlap (fem_api.cu, launch_split): a fixed z-chunking instead of the launcher's --
  // zc_force chunks starting kchunk_force planes apart, each kspan planes long (0: automatic)
  int64_t kchunk_force = 0, kspan = 0;
  int zc_force = 0;
  // elasticity fused apply: interior / edge CTAs as two grids (fem_api.cu passes a second stream
  // and two events to run them concurrently; nullptr: one after the other on the same stream)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

// Device scalars of one CG solve (rank-global after the allreduce steps).
struct CgScalars {
  double rr;        // r.r of the current iterate
  double pq;        // p.Ap (global after allreduce)
  double rr_new;    // r.r after the update (global after allreduce)
  double rr0;       // r0.r0
  double stop_rr;   // tol^2 * rr0
  double alpha;     // Chronopoulos-Gear CG: alpha of the last update
  double rr_acc;    // dot_mode 2: atomic accumulator of the update's r.r
  double alpha_h[7];  // deferred x update: alphas of the pending iterations of the group
  int32_t done;     // 0 running, 1 converged, 2 breakdown, 3 maxit reached
  int32_t it;       // iterations completed
  int32_t maxit;
  int32_t breakdown_iter;
  int32_t first;    // fused CG: 1 before the first apply (beta = 0, p = r)
  int32_t xp;       // deferred x update: number of pending x += alpha_h[j] P_j (P_j in p buffer j)
};

// Last-block reduction workspace: per-CTA partials + ticket counter.
struct Reduce {
  double* partials;       // >= max CTAs of any reducing launch
  unsigned int* ticket;   // zero-initialised, reset by the last block
  int64_t capacity;
  // how the fused Hestenes-Stiefel CG computes its two dots (option "dot_mode"; the paper's dot
  // ablation): 0 in the producing kernel's epilogue (block tree + last-block pass over
  // the CTA partials, deterministic); 1 none in the producing kernel -- separate dot kernels
  // re-read the vectors; 2 in the epilogue, CTA partials added with FP64 atomics (run-order
  // dependent).  Kernels other than the fused apply / update always use 0.
  int dot_mode = 0;
  // split applies (halo overlap): acc = 1 adds this launch's dots to the scalars instead of
  // writing them; roll = 0 leaves the fused-CG recurrence roll (rr = rr_new) to a later launch
  int acc = 0, roll = 1;
  // two grids sharing one reduction (the elasticity fused apply's interior / edge grids): this
  // grid's CTAs take partial slots boff .. boff + grid - 1 and the ticket counts btot CTAs in all
  // (0: this grid alone)
  int boff = 0, btot = 0;
};

constexpr int kMaxCtas = 1 << 16;

// Tile shapes of the apply kernels (kernel templates and host tensor-map boxes must agree).
#ifndef FEM_HEX_PREFETCH
#define FEM_HEX_PREFETCH 1  // general-hex apply: persistent grid + cp.async gather pipeline
#endif
constexpr bool kHexPrefetch = FEM_HEX_PREFETCH != 0;
#ifndef FEM_LAP_MINCHUNK
#define FEM_LAP_MINCHUNK 16  // Laplace z-chunks: minimum planes per chunk
#endif
#ifndef FEM_LAP_ROUNDS
#define FEM_LAP_ROUNDS 4  // Laplace z-chunks: minimum rounds of resident CTAs
#endif
#ifndef FEM_LAP_TY
#define FEM_LAP_TY 7
#endif
#ifndef FEM_LAP_R1
#define FEM_LAP_R1 3
#endif
#ifndef FEM_LAP_MINB
#define FEM_LAP_MINB 2  // resident CTAs per SM the Laplace apply is compiled for (register cap)
#endif
#ifndef FEM_LAP_S1
#define FEM_LAP_S1 4  // ring stages of the scalar fused CG apply
#endif
#ifndef FEM_LAP_R3
#define FEM_LAP_R3 2  // node rows per thread of the vector kernel (1: 2 CTAs / SM at 127 registers)
#endif
#ifndef FEM_LAP_MINB3
#define FEM_LAP_MINB3 (FEM_LAP_R3 > 1 ? 1 : FEM_LAP_MINB)  // resident CTAs per SM of the vector kernel
#endif
constexpr int kLapTX = 32, kLapTY = FEM_LAP_TY, kLapR1 = FEM_LAP_R1, kLapR3 = FEM_LAP_R3;  // Laplace: C=1 / C=3 rows per thread
#ifndef FEM_LAP_SELF1
#define FEM_LAP_SELF1 1  // scalar TMA path without producer warp (consumer warp 0 issues the loads)
#endif
#ifndef FEM_LAP_TY1
#define FEM_LAP_TY1 8  // consumer warps of the scalar TMA path
#endif
constexpr int kLapMinB = FEM_LAP_MINB, kLapMinB3 = FEM_LAP_MINB3, kLapS1 = FEM_LAP_S1, kLapTY1 = FEM_LAP_TY1;
constexpr bool kLapSelf1 = FEM_LAP_SELF1 != 0;
#ifndef FEM_LAP_SELF3
#define FEM_LAP_SELF3 0  // vector TMA path without producer warp
#endif
#ifndef FEM_LAP_TY3
#define FEM_LAP_TY3 7  // consumer warps of the vector TMA path
#endif
constexpr bool kLapSelf3 = FEM_LAP_SELF3 != 0;
constexpr int kLapTY3 = FEM_LAP_TY3;
#ifndef FEM_LAP_INTERIOR
#define FEM_LAP_INTERIOR 0  // 1: Laplace CG tensors span the Dirichlet interior only (round-1 layout)
#endif
#ifndef FEM_EL_TY
#define FEM_EL_TY 15
#endif
constexpr int kElTY = FEM_EL_TY;                                      // elasticity consumer warps
#ifndef FEM_EL_CY
#define FEM_EL_CY 2  // cell rows per thread of the elasticity apply (1: elastic_kernel, 2: elastic2_kernel)
#endif
#ifndef FEM_EL2_TY
#define FEM_EL2_TY 8  // consumer warps of elastic2_kernel (2 cell rows each)
#endif
#ifndef FEM_EL2_S
#define FEM_EL2_S 4  // ring stages of elastic2_kernel in fused CG (x2 for one input box)
#endif
#ifndef FEM_EL2_SELF
#define FEM_EL2_SELF 1  // elastic2_kernel without producer warp: consumer warp 0 issues the TMA loads
#endif
constexpr int kEl2HW = 3;  // doubles per thread per y hand-off of elastic2_kernel
constexpr int kElCY = FEM_EL_CY, kEl2TY = FEM_EL2_TY, kEl2S = FEM_EL2_S;
constexpr bool kEl2Self = FEM_EL2_SELF != 0;
constexpr int kElCellRows = kElCY == 2 ? 2 * kEl2TY : kElTY;  // cell rows per TMA tile (= u box rows - 1)
// material box rows: shared by elastic2_kernel (TMA path) and elastic_kernel (caller vectors)
constexpr int kElMatRows = kElCellRows > kElTY ? kElCellRows : kElTY;
// u-plane TMA box (doubles x rows) per kind: width = (((cols * C) + 1) & ~1) + 2
inline void u_box(int kind, unsigned* w, unsigned* h) {
  if (kind == 0) { *w = ((((kLapTX + 2) * 1) + 1) & ~1) + 2; *h = kLapTY1 * kLapR1 + 2; }
  else if (kind == 1) { *w = ((((kLapTX + 2) * 3) + 1) & ~1) + 2; *h = kLapTY3 * kLapR3 + 2; }
  else { *w = ((((32 + 1) * 3) + 1) & ~1) + 2; *h = kElCellRows + 1; }
}
inline void mat_box(unsigned* w, unsigned* h) { *w = 2 * 32; *h = kElMatRows; }

// ---- launchers (return cudaError_t of the launch) -----------------------------------------
// mode: 0 plain apply (y = A_c x), 1 CG apply (also pq partial -> sc->pq; skips if sc->done),
//       2 fused CG apply (p = r + beta p_old in the kernel, writes p and q, pq)
cudaError_t launch_laplace(int comps, int bc, const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps,
                           int mode, CgScalars* sc, Reduce red, cudaStream_t s, int sm_count);
cudaError_t launch_elastic(int bc, const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps, int mode,
                           CgScalars* sc, Reduce red, cudaStream_t s, int sm_count);
// dense ABI <-> padded layout (owned planes): n_planes planes of (nx+1)(ny+1) nodes x C
cudaError_t launch_pack(const double* dense, double* padded, int64_t rpitch, int64_t ppitch,
                        int64_t n_planes, int64_t nxn, int64_t nyn, int comps, int to_padded,
                        cudaStream_t s, int sm_count);
// CG vector kernels (n = owned DOFs)
cudaError_t launch_cg_init(const double* b, const double* ax, double* r, double* p, int64_t n,
                           CgScalars* sc, Reduce red, cudaStream_t s, int sm_count);
cudaError_t launch_cg_finish_init(CgScalars* sc, double tol, int maxit, cudaStream_t s);
cudaError_t launch_cg_update(double* x, double* r, const double* p, const double* q, int64_t n,
                             CgScalars* sc, Reduce red, cudaStream_t s, int sm_count, int nold = 0,
                             const double* const* pold = nullptr, int jpend = 0);
cudaError_t launch_cg_pupdate(const double* r, const double* pr, double* pw, int64_t n, CgScalars* sc, Reduce red,
                              cudaStream_t s, int sm_count);
// fused CG: x += alpha p; r -= alpha q; rr_new = r.r; iteration bookkeeping (p update is in the apply)
cudaError_t launch_cg_update_fused(double* x, double* r, const double* p, const double* q, int64_t n,
                                   CgScalars* sc, Reduce red, cudaStream_t s, int sm_count, int nold = 0,
                                   const double* const* pold = nullptr, int jpend = 0);
// deferred x update: x += alpha_h[j] P_j for the sc->xp pending iterations (end of a solve)
cudaError_t launch_cg_xdefer_flush(double* x, const double* const* pend, int64_t n, const CgScalars* sc,
                                   cudaStream_t s, int sm_count);
// general hexahedral meshes (kernels_hex.cu): cells = 2 int4 per cell (node ids in corner-bit
// order, bit 31 = Dirichlet node), xyz = node coordinates (w unused), lm = (lambda, mu) per cell.
// mode 0: y += A (P x) at unconstrained nodes (y zeroed by the caller); mode 1: + sc->pq = the
// sum of the element energies (P x)^T A (P x).
// E != nullptr: deterministic scatter -- element outputs E[cell][8][C] instead of FP64 atomics
// into y, then launch_hex_gather sums them per node (node -> entry CSR of launch_hex_node_csr)
cudaError_t launch_hex_apply(int kind, int bc, int quad, const int4* cells, const double4* xyz, const double2* lm,
                             const double* x, double* y, double* E, int64_t ncells, int mode, CgScalars* sc,
                             Reduce red, cudaStream_t s, int sm_count);
cudaError_t launch_hex_node_csr(const int4* cells, int64_t ncells, int64_t nnodes, int32_t* off, int32_t* list,
                                int sm_count);
cudaError_t launch_hex_gather(int comps, const int32_t* off, const int32_t* list, const double* E, double* y,
                              int64_t nnodes, cudaStream_t s, int sm_count);
// partial assembly on general hex meshes: per-Gauss-point geometry stored once (setup), then
// applied without recomputing J (Laplace kinds share the 6-value D'; elasticity 9-value B)
int64_t hex_pa_doubles(int kind, int64_t ncells);
cudaError_t launch_hex_pa_setup(int kind, int quad, const int4* cells, const double4* xyz, double* pa,
                                int64_t ncells, cudaStream_t s, int sm_count);
cudaError_t launch_hex_pa_apply(int kind, int bc, int quad, const int4* cells, const double* pa, const double2* lm,
                                const double* x, double* y, double* E, int64_t ncells, int mode, CgScalars* sc,
                                Reduce red, cudaStream_t s, int sm_count);
// partial assembly on the box (kernels_pa.cu): 21 values per Gauss point and cell,
// D_q = w_q det J_q C_e (Voigt, upper triangle), SoA [q][k][cell]
int64_t pa21_doubles(int64_t ncells);
cudaError_t launch_pa21_setup(const double2* lm, int64_t ncells, double h, double* D, cudaStream_t s, int sm_count);
cudaError_t launch_pa21_apply(int bc, int quad, const Grid& g, PlaneSrc x, OutVec y, const double* D, int mode,
                              CgScalars* sc, Reduce red, cudaStream_t s, int sm_count);
// y = x on the constrained nodes; mode 1: sc->pq += sum x_b^2
cudaError_t launch_hex_dirichlet(const int32_t* nodes, int64_t nb, int comps, const double* x, double* y,
                                 int mode, CgScalars* sc, Reduce red, cudaStream_t s, int sm_count);
// bad[0] += cells with an out-of-range node, bad[1] += cells with det J <= 0 at a point of the
// rule (0: the 2x2x2 Gauss points, 1: the Gauss-Lobatto points = the nodes)
cudaError_t launch_hex_check(const int4* cells, const double4* xyz, int64_t ncells, int64_t nnodes, int rule,
                             unsigned long long* bad, cudaStream_t s, int sm_count);
// VTK-ordered int32 node map (+ optional uint8 Dirichlet flags) -> internal cell records
cudaError_t launch_hex_pack_cells(const int32_t* vtk, const uint8_t* dir, int64_t ncells, int64_t nnodes,
                                  int* out, unsigned long long* bad, cudaStream_t s, int sm_count);
// Chronopoulos-Gear CG (single reduction, NEXT #1): with gamma = r.r and delta = w.r from the
// apply (mode 3): beta = gamma / gamma_prev, alpha = gamma / (delta - beta gamma / alpha_prev);
// p = r + beta p, s = w + beta s, x += alpha p, r -= alpha s (first step: p = r, s = w)
cudaError_t launch_cg_cgcg_update(double* x, double* r, const double* pr, double* pw, double* s, const double* w,
                                  int64_t n, CgScalars* sc, Reduce red, cudaStream_t st, int sm_count, int nold = 0,
                                  const double* const* pold = nullptr, int jpend = 0);
// loopback allreduce: out[i] = sum over ranks q = 0..P-1 (in order) of stage[q * stride + i]
cudaError_t launch_loop_sum(const double* stage, int P, int stride, int count, double* out, cudaStream_t s);
// dot_mode 1 of the fused CG: which = 0: sc->pq = a.b, then roll rr = rr_new, first = 0;
// which = 1: sc->rr_new = a.b, it++, maxit -> done = 3 (the update kernel's bookkeeping)
cudaError_t launch_cg_dot(const double* a, const double* b, int64_t n, int which, CgScalars* sc, Reduce red,
                          cudaStream_t s, int sm_count);
// deterministic dot -> *out (device)
cudaError_t launch_dot(const double* a, const double* b, int64_t n, double* out, Reduce red,
                       cudaStream_t s, int sm_count);
// residual helper: out = b - ax (for true residual)
cudaError_t launch_sub(const double* b, const double* ax, double* out, int64_t n, cudaStream_t s,
                       int sm_count);
// material validation: count of invalid cells -> *bad (device int64)
cudaError_t launch_check_material(const double2* lm, int64_t n, unsigned long long* bad,
                                  cudaStream_t s, int sm_count);

// CSR baseline
cudaError_t launch_csr_rowcount(int comps, int bc, const Grid& g, int64_t* rowptr, cudaStream_t s);
cudaError_t launch_csr_fill(int kind, int bc, const Grid& g, const double2* lm,
                            const int64_t* rowptr, int32_t* col, double* val, cudaStream_t s);
cudaError_t launch_csr_spmv(int comps, int64_t nrows, const int64_t* rowptr, const int32_t* col,
                            const double* val, const double* x, double* y, cudaStream_t s,
                            int sm_count);

void add_launches(int64_t n);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, smem) once per (kernel, current device): the
// attribute belongs to the device context, so a process driving several GPUs sets it on each.
cudaError_t ensure_smem_attr(const void* kernel, int smem);

}  // namespace fem

// ---- small device helpers -------------------------------------------------------------------
#ifdef __CUDACC__
namespace fem {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed tree); result valid in thread 0. `sh` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int wid = tid >> 5;
  const int nw = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
  // use linear lane from tid so 2-D blocks work
  v = warp_sum(v);
  __syncthreads();
  if ((tid & 31) == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (tid < nw) ? sh[tid] : 0.0;
    r = warp_sum(r);
  }
  (void)lane;
  return r;
}

// Last-block-done finalisation: every block writes its partial; the last block to arrive sums
// the partials in block order (deterministic) and returns true in thread 0 with *total set.
__device__ __forceinline__ bool last_block_reduce(double partial, Reduce red, double* sh,
                                                  double* total) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const unsigned int bid = red.boff + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned int nblk = red.btot ? (unsigned)red.btot : gridDim.x * gridDim.y * gridDim.z;
  __shared__ unsigned int s_is_last;
  if (tid == 0) {
    red.partials[bid] = partial;
    __threadfence();
    unsigned int t = atomicAdd(red.ticket, 1u);
    s_is_last = (t == nblk - 1);
  }
  __syncthreads();
  if (!s_is_last) return false;
  __threadfence();
  double v = 0.0;
  // fixed assignment of partials to threads, fixed tree -> bitwise deterministic
  for (unsigned int b = tid; b < nblk; b += nthr) v += ((volatile double*)red.partials)[b];
  double s = block_sum(v, sh);
  if (tid == 0) {
    *total = s;
    *red.ticket = 0u;
  }
  return tid == 0;
}

// Epilogue of a CG apply (mode 1 / 2): p.Ap of this CTA's nodes -> sc->pq, per red.dot_mode.
// roll (fused CG, mode 2): once every CTA has read rr / rr_new / first (i.e. in the last CTA),
// advance the recurrence rr = rr_new, first = 0 -- dot_mode 1 leaves that to the dot kernel.
__device__ __forceinline__ void cg_apply_epilogue(double pq, bool roll, CgScalars* sc, Reduce red, double* sh) {
  if (red.dot_mode == 1) return;  // separate dot kernel (launch_cg_dot) after this kernel
  const double bsum = block_sum(pq, sh);
  if (red.dot_mode == 2) {
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    if (tid == 0) atomicAdd(&sc->pq, bsum);  // zeroed by the previous update's last CTA
    if (!roll || !red.roll) return;
    double unused;
    if (last_block_reduce(0.0, red, sh, &unused)) {  // ticket only: the last CTA rolls
      sc->rr = sc->rr_new;
      sc->first = 0;
      sc->rr_acc = 0.0;  // the update's atomic target
    }
    return;
  }
  double total;
  if (last_block_reduce(bsum, red, sh, &total)) {
    sc->pq = red.acc ? sc->pq + total : total;
    if (roll && red.roll) {  // every block has read rr / rr_new / first: roll the recurrence
      sc->rr = sc->rr_new;
      sc->first = 0;
    }
  }
}

// the same for two sums at once (partials of b at red.partials + red.capacity)
__device__ __forceinline__ bool last_block_reduce2(double a, double b, Reduce red, double* sh,
                                                   double* ta, double* tb) {
  const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  const int nthr = blockDim.x * blockDim.y * blockDim.z;
  const unsigned int bid = red.boff + blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned int nblk = red.btot ? (unsigned)red.btot : gridDim.x * gridDim.y * gridDim.z;
  __shared__ unsigned int s_is_last2;
  if (tid == 0) {
    red.partials[bid] = a;
    red.partials[red.capacity + bid] = b;
    __threadfence();
    unsigned int t = atomicAdd(red.ticket, 1u);
    s_is_last2 = (t == nblk - 1);
  }
  __syncthreads();
  if (!s_is_last2) return false;
  __threadfence();
  double va = 0.0, vb = 0.0;
  for (unsigned int k = tid; k < nblk; k += nthr) {
    va += ((volatile double*)red.partials)[k];
    vb += ((volatile double*)red.partials)[red.capacity + k];
  }
  const double sa = block_sum(va, sh);
  const double sb = block_sum(vb, sh);
  if (tid == 0) {
    *ta = sa;
    *tb = sb;
    *red.ticket = 0u;
  }
  return tid == 0;
}

}  // namespace fem
#endif
