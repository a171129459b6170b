// fem_api.cu -- host side of libfem.so: the C ABI declared in include/fem.h.
// Handles, validation, workspace, slab partition + NCCL halo/allreduce, the CG driver
// (CUDA-graph captured iteration) and the CSR baseline.  Kernels live in kernels_*.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fem.h"
#include "fem_internal.cuh"

#ifndef FEM_X_DEFER
#define FEM_X_DEFER 8  // fused CG: x updated every FEM_X_DEFER-th iteration (1, 2, 4 or 8; option x_defer)
#endif

namespace fem {

// NVTX range over a host-side scope (SURVEY §5 "Tracing"): fem:apply, fem:halo, fem:allreduce,
// fem:interior / fem:boundary of the overlapped apply, fem:cg_iterate ...  Visible to nsys / ncu
// --nvtx when a tool is attached; a no-op otherwise.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
cudaError_t upload_unit_matrices(const double* K, const double* Kl, const double* Km);
static std::atomic<int64_t> g_launches{0};
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

struct SmemAttr {
  const void* fn;
  int dev, smem;
};
static std::vector<SmemAttr> g_smem_attr;
static std::mutex g_smem_mu;
cudaError_t ensure_smem_attr(const void* kernel, int smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_smem_mu);
  for (const SmemAttr& a : g_smem_attr)
    if (a.fn == kernel && a.dev == dev && a.smem >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  for (SmemAttr& a : g_smem_attr)
    if (a.fn == kernel && a.dev == dev) {
      a.smem = smem;
      return cudaSuccess;
    }
  g_smem_attr.push_back(SmemAttr{kernel, dev, smem});
  return cudaSuccess;
}
}  // namespace fem

using namespace fem;

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string t_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(FEM_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),     \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define NCCL_TRY(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess)                                                                \
      return fail(FEM_ENCCL, "%s failed: %s (%s:%d)", #expr, ncclGetErrorString(_r),      \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define FEM_TRY(expr)                \
  do {                               \
    int _s = (expr);                 \
    if (_s != FEM_OK) return _s;     \
  } while (0)

// ------------------------------------------------------------------------------------------
// handles
// ------------------------------------------------------------------------------------------
// In-process loopback group (fem_comm_create_loopback): the P slab ranks of one
// process on one device, each driven by its own host thread and stream.  Every NCCL call site
// (halo_pitch, allreduce1, the peer-halo handle exchange) has a loopback branch: stream-ordered
// device copies / a fixed-order sum kernel, ordered across the ranks' streams by CUDA events that
// the ranks exchange through a host rendezvous.  Like NCCL, every collective is entered by every
// rank in the same order.
struct LoopRec {
  const void* p = nullptr;  // halo: owned base of the published vector; peer exchange: fem_op_s*
  int64_t np = 0, pitch = 0;
};
struct LoopGroup {
  static constexpr int K = 64;  // event / record ring per rank (>= P: see loop_publish)
  static constexpr int KR = 4;  // allreduce staging ring
  static constexpr int MAXC = 8;  // values per allreduce
  int P = 0, device = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<int64_t> seq;       // [P] collectives published by each rank
  std::vector<LoopRec> rec;       // [P][K]
  std::vector<cudaEvent_t> ev;    // [P][K]
  double* red = nullptr;          // device [KR][P][MAXC] allreduce contributions
};

struct fem_comm_s {
  int nranks = 1, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  LoopGroup* loop = nullptr;  // loopback group (no NCCL)
  int64_t loop_seq = 0, loop_ar = 0;  // this rank's collective / allreduce counters
};

struct fem_mesh_s {
  Grid g{};  // global sizes, owned planes [k0, k1)
  fem_comm_s* comm = nullptr;
  int nranks = 1, rank = 0, device = 0, sm_count = 148;
  // general hexahedral mesh (fem_mesh_create_hex; Alg. 1 as written): explicit node map and
  // coordinates, single GPU.  hx_cells: 2 int4 per cell (corner-bit order, bit 31 = Dirichlet)
  bool hex = false;
  int64_t hx_nodes = 0, hx_ncells = 0, hx_nb = 0;
  double4* hx_xyz = nullptr;
  int4* hx_cells = nullptr;
  int32_t* hx_bnodes = nullptr;  // constrained nodes (identity rows)
  // deterministic scatter (option "deterministic"): node -> (cell, corner) entry CSR, ascending
  // entries per node, built on first use
  int32_t* hx_n2e_off = nullptr;  // [hx_nodes + 1]
  int32_t* hx_n2e = nullptr;      // [8 hx_ncells]: cell * 8 + corner
};

struct fem_op_s {
  fem_mesh_s* mesh = nullptr;
  int kind = 0, bc = 0, comps = 1;
  int64_t n_local = 0, n_global = 0, plane_dofs = 0, nloc_planes = 0;
  // material (local cell layers [mat_layer0, mat_layer0 + mat_layers)), (lambda, mu) interleaved
  double2* lm = nullptr;
  int64_t mat_layer0 = 0, mat_layers = 0;
  bool has_mat = false;
  // dense-layout workspace (fem_apply on caller vectors, host staging)
  double *ghost_lo = nullptr, *ghost_hi = nullptr;
  double *stage_a = nullptr, *stage_b = nullptr;
  // CG vectors in the library padded layout: node (i,j) comp c of local plane kk
  // (kk = 0 is the ghost plane k0-1) at v[pl_lead + kk*pl_pp + j*pl_rp + i*C + c]
  int64_t pl_lead = 0, pl_rp = 0, pl_pp = 0, pl_n = 0;
  int64_t pl_off = 0;  // offset of the owned range (pl_lead + pl_pp; 0 on general hex meshes)
  double *x_pl = nullptr, *r_pl = nullptr, *p_pl = nullptr, *q_pl = nullptr, *p2_pl = nullptr;
  // deferred x update over m = 4 / 8 iterations: m - 2 more p buffers (allocated on use)
  double* pex[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  CUtensorMap tm_x{}, tm_p{}, tm_mat{}, tm_r{}, tm_p2{}, tm_pex[7]{};
  int cg_parity = 0;  // fused CG: iteration phase mod 8 (selects the p buffers)
  bool tm_ok = false;
  bool tm_interior = false;  // u tensor spans the interior only (Laplace + Dirichlet)
  int64_t tm_i0 = 0, tm_j0 = 0, tm_k0 = 0;
  CgScalars* sc = nullptr;
  CgScalars* sc_host = nullptr;
  double* dot_dev = nullptr;
  double* dot_host = nullptr;
  unsigned long long* bad = nullptr;
  Reduce red{};
  // CG state
  const double* cg_b = nullptr;
  double* cg_x = nullptr;
  bool cg_active = false;
  cudaGraphExec_t graph1 = nullptr, graphN = nullptr, graph1b = nullptr;
  // options
  int use_graph = 1, check_every = 16, time_apply = 0;
  int direct_tm = 1;  // fem_apply on 16-B-strided caller vectors: tensor map straight over x
  int last_path = 0;  // staging of the last fem_apply: 0 bulk rows, 1 tensor map, 2 row-pair tensor map
  // general hex meshes: partial assembly (per-Gauss-point geometry stored once)
  int use_pa = 0;
  double* pa = nullptr;
  int pa_quad = -1;  // rule the stored geometry was computed for
  int quad = 0;      // 0: 2x2x2 Gauss-Legendre, 1: 2x2x2 Gauss-Lobatto (BP5/BP6; reading R1)
  int cg_variant = 0;  // 0: fused Hestenes-Stiefel (Table 4), 1: Chronopoulos-Gear single reduction
  int dot_mode = 0;    // fused Hestenes-Stiefel dots: 0 epilogue, 1 separate kernels, 2 atomics
  // general hexes: deterministic scatter (element outputs + per-node gather) instead of FP64 atomics
  int det = 0;
  double* hx_E = nullptr;  // [ncells][8][C]
  // fused CG: deferred x update (x advanced every x_defer-th iteration from the p buffers of the
  // group: 1, 2 or 4; option "x_defer")
  int x_defer = FEM_X_DEFER;
  int x_defer_cap = 8;  // lowered when the p ring does not fit in device memory
  // peer halo: the neighbour ranks' padded vectors x, p, r, p2 (CUDA IPC or, for single-process
  // tests, the other operator's buffers) and tensor maps over their ghost-plane sources
  bool peer_on = false, peer_ipc = false;
  double* nb_lo[4] = {nullptr, nullptr, nullptr, nullptr};
  double* nb_hi[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t nb_lo_nloc = 0;
  CUtensorMap pm_lo[4]{}, pm_hi[4]{};
  // fem_apply on caller vectors at P > 1: tensor maps over the ghost-plane buffers (direct view,
  // row-pair view), built on first use
  CUtensorMap gm_dir[2]{}, gm_pair[2]{};
  bool gm_dir_ok = false, gm_pair_ok = false;
  // P = 1 row-pair view without slack after the caller's vector: the last plane from a copy
  double* last_plane = nullptr;
  CUtensorMap gm_last{};
  int64_t pm_klo = -(int64_t(1) << 62), pm_khi = -(int64_t(1) << 62);
  std::vector<cudaEvent_t> ev;
  size_t ev_used = 0;
  bool ev_capture = false;   // events are being captured as graph nodes
  // halo overlap (apply_split): comm stream + fork / join events; option "halo_overlap"
  int overlap = 1;
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // option "trace": timing events of the last exchange apply (apply_split) -- [0] start on the
  // caller's stream, [1] halo done (comm stream), [2] interior planes done, [3] boundary planes
  // done; read back as trace_{halo,interior,boundary,total}_ns (the overlap timeline)
  int trace = 0;
  cudaEvent_t tr_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // elasticity fused apply: second stream for the edge grid beside the interior grid
  cudaStream_t astream = nullptr;
  cudaEvent_t ev_a0 = nullptr, ev_a1 = nullptr;
  bool tr_valid = false;
  struct MapEnt {
    const void* p = nullptr;
    unsigned long long id = 0;
    int path = 0;
    CUtensorMap map{};
  };
  std::vector<MapEnt> map_cache;  // fem_apply tensor maps over caller vectors
  size_t map_next = 0;
  // time_apply with graphs: one graph of exactly graphT_iters iterations (from parity
  // graphT_parity) with event-record nodes around every apply
  struct TimedGraph {
    cudaGraphExec_t exec = nullptr;
    int iters = 0, parity = 0;
    int64_t launches = 0;  // kernel launches the graph replays (counted during its capture)
  };
  std::vector<TimedGraph> graphT;  // up to 4 (iteration count, parity) shapes
  std::vector<TimedGraph> graphK;  // plain graphs of exactly k iterations (k <= 64), up to 6 shapes
};

struct fem_csr_s {
  int comps = 1, device = 0, sm_count = 148;
  int64_t nrows = 0, nnz = 0;
  int64_t* rowptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
};

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------
// One driver query per caller pointer: memory type, the allocation it lies in and that
// allocation's unique id (cuPointerGetAttributes, no error for plain host pointers).
struct PtrInfo {
  bool device = false;
  unsigned long long id = 0;  // CU_POINTER_ATTRIBUTE_BUFFER_ID (0: not a CUDA allocation)
  uintptr_t base = 0;         // allocation range
  size_t size = 0;
};
static PtrInfo ptr_info(const void* p) {
  using PFN = CUresult (*)(unsigned int, CUpointer_attribute*, void**, CUdeviceptr);
  static PFN fn = nullptr;
  PtrInfo r;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttributes", &f, cudaEnableDefault, &q) != cudaSuccess || !f) {
      cudaGetLastError();
      cudaPointerAttributes a;
      if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return r;
      }
      r.device = a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
      return r;
    }
    fn = reinterpret_cast<PFN>(f);
  }
  unsigned int mtype = 0, managed = 0;
  CUdeviceptr start = 0;
  size_t size = 0;
  unsigned long long id = 0;
  CUpointer_attribute at[5] = {CU_POINTER_ATTRIBUTE_MEMORY_TYPE, CU_POINTER_ATTRIBUTE_IS_MANAGED,
                               CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, CU_POINTER_ATTRIBUTE_RANGE_SIZE,
                               CU_POINTER_ATTRIBUTE_BUFFER_ID};
  void* data[5] = {&mtype, &managed, &start, &size, &id};
  if (fn(5, at, data, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS) return r;
  r.device = mtype == CU_MEMORYTYPE_DEVICE || managed;
  r.id = id;
  r.base = (uintptr_t)start;
  r.size = size;
  return r;
}
static bool is_device_ptr(const void* p) { return ptr_info(p).device; }

static int check_vec(const void* p, const char* name) {
  if (!p) return fail(FEM_EINVAL, "%s is NULL", name);
  if (((uintptr_t)p) & 7) return fail(FEM_EINVAL, "%s is not 8-byte aligned", name);
  return FEM_OK;
}

static int set_device(int dev) {
  int cur = -1;
  CUDA_TRY(cudaGetDevice(&cur));
  if (cur != dev) CUDA_TRY(cudaSetDevice(dev));
  return FEM_OK;
}

template <class T>
static int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FEM_ENOMEM, "cudaMalloc of %zu bytes failed: %s", count * sizeof(T),
                cudaGetErrorString(e));
  }
  return FEM_OK;
}

// unit-cube element matrices by the library's own 2x2x2 Gauss quadrature (h = 1), corner
// index a = dx + 2 dy + 4 dz.  Eq. 4 (scalar) and Eq. 6 split into its lambda and mu parts.
static void unit_element_matrices(double K[64], double Kl[576], double Km[576], int quad = 0) {
  // 2-point rule on [0, 1]: Gauss-Legendre (default) or Gauss-Lobatto (quad 1: the nodes)
  const double g = quad == 1 ? 1.0 : 1.0 / std::sqrt(3.0);
  const double gp[2] = {0.5 - 0.5 * g, 0.5 + 0.5 * g};
  std::memset(K, 0, 64 * sizeof(double));
  std::memset(Kl, 0, 576 * sizeof(double));
  std::memset(Km, 0, 576 * sizeof(double));
  for (int q = 0; q < 8; ++q) {
    const double X[3] = {gp[q & 1], gp[(q >> 1) & 1], gp[(q >> 2) & 1]};
    const double w = 1.0 / 8.0;
    double G[8][3];
    for (int a = 0; a < 8; ++a) {
      const int o[3] = {a & 1, (a >> 1) & 1, (a >> 2) & 1};
      for (int d = 0; d < 3; ++d) {
        double v = 1.0;
        for (int e = 0; e < 3; ++e) {
          const double f = o[e] ? X[e] : 1.0 - X[e];
          const double df = o[e] ? 1.0 : -1.0;
          v *= (e == d) ? df : f;
        }
        G[a][d] = v;
      }
    }
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        const double gg = G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2];
        K[a * 8 + b] += w * gg;
        for (int k = 0; k < 3; ++k)
          for (int l = 0; l < 3; ++l) {
            const int ix = (3 * a + k) * 24 + 3 * b + l;
            Kl[ix] += w * G[a][k] * G[b][l];
            Km[ix] += w * ((k == l ? gg : 0.0) + G[a][l] * G[b][k]);
          }
      }
  }
}

static std::vector<int> g_unit_devices;
static std::mutex g_unit_mu;

static int ensure_unit_matrices(int dev) {
  std::lock_guard<std::mutex> lk(g_unit_mu);
  if (std::find(g_unit_devices.begin(), g_unit_devices.end(), dev) != g_unit_devices.end())
    return FEM_OK;
  double K[64], Kl[576], Km[576];
  unit_element_matrices(K, Kl, Km);
  CUDA_TRY(upload_unit_matrices(K, Kl, Km));
  g_unit_devices.push_back(dev);
  return FEM_OK;
}

static int need_comm(fem_op_s* op) {
  fem_mesh_s* m = op->mesh;
  if (m->nranks > 1 && (!m->comm || (!m->comm->nccl && !m->comm->loop)))
    return fail(FEM_EUNSUPPORTED, "virtual communicator: use fem_apply_ghost (no exchange available)");
  return FEM_OK;
}

// ---- loopback collectives ------------------------------------------------------------------
// Publish this rank's record (+ an event recorded on its stream) for its next collective and wait
// until the ranks `who` have published theirs; their records / events are returned.
// Ring reuse: a rank re-records its slot of collective n at n + K only after the rendezvous of
// n + K - 1, by which every rank within distance K - 1 in the slab chain has published n + 1,
// i.e. finished consuming collective n (K = 64 >= P, fem_comm_create_loopback).
static int loop_publish(fem_comm_s* c, const LoopRec& mine, cudaStream_t s, const int* who, int nwho,
                        LoopRec* out, cudaEvent_t* out_ev) {
  LoopGroup* G = c->loop;
  const int64_t n = c->loop_seq++;
  const int slot = (int)(n % LoopGroup::K);
  const int me = c->rank;
  CUDA_TRY(cudaEventRecord(G->ev[me * LoopGroup::K + slot], s));
  std::unique_lock<std::mutex> lk(G->mu);
  G->rec[me * LoopGroup::K + slot] = mine;
  G->seq[me] = n + 1;
  G->cv.notify_all();
  const bool ok = G->cv.wait_for(lk, std::chrono::seconds(120), [&] {
    for (int t = 0; t < nwho; ++t)
      if (G->seq[who[t]] <= n) return false;
    return true;
  });
  if (!ok) return fail(FEM_ESTATE, "loopback collective %lld: a rank did not arrive within 120 s", (long long)n);
  for (int t = 0; t < nwho; ++t) {
    out[t] = G->rec[who[t] * LoopGroup::K + slot];
    out_ev[t] = G->ev[who[t] * LoopGroup::K + slot];
  }
  return FEM_OK;
}

// halo: (1) publish the owned vector, copy the neighbours' boundary planes after their producers;
// (2) publish "consumed", and the neighbours' streams wait for it before they can overwrite the
// planes this rank read (the synchronising semantics of ncclSend / ncclRecv)
static int loop_halo(fem_mesh_s* m, const double* owned, double* lo, double* hi, int64_t pitch,
                     cudaStream_t s) {
  fem_comm_s* c = m->comm;
  int who[2], nw = 0;
  if (m->rank > 0) who[nw++] = m->rank - 1;
  if (m->rank < m->nranks - 1) who[nw++] = m->rank + 1;
  LoopRec rec[2];
  cudaEvent_t ev[2];
  FEM_TRY(loop_publish(c, LoopRec{owned, m->g.k1 - m->g.k0, pitch}, s, who, nw, rec, ev));
  for (int t = 0; t < nw; ++t) {
    const double* src = static_cast<const double*>(rec[t].p);
    const bool below = who[t] < m->rank;
    const double* plane = below ? src + (rec[t].np - 1) * rec[t].pitch : src;
    CUDA_TRY(cudaStreamWaitEvent(s, ev[t], 0));
    CUDA_TRY(cudaMemcpyAsync(below ? lo : hi, plane, (size_t)pitch * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  FEM_TRY(loop_publish(c, LoopRec{}, s, who, nw, rec, ev));
  for (int t = 0; t < nw; ++t) CUDA_TRY(cudaStreamWaitEvent(s, ev[t], 0));
  return FEM_OK;
}

// allreduce(sum) of `count` device doubles: contributions staged in the group's ring, summed by
// every rank in rank order (bitwise the same result on every rank)
static int loop_allreduce(fem_mesh_s* m, double* dev, int count, cudaStream_t s) {
  fem_comm_s* c = m->comm;
  LoopGroup* G = c->loop;
  if (count > LoopGroup::MAXC) return fail(FEM_EINVAL, "loopback allreduce of more than %d values", LoopGroup::MAXC);
  double* stage = G->red + (c->loop_ar++ % LoopGroup::KR) * G->P * LoopGroup::MAXC;
  CUDA_TRY(cudaMemcpyAsync(stage + m->rank * LoopGroup::MAXC, dev, count * sizeof(double),
                           cudaMemcpyDeviceToDevice, s));
  std::vector<int> who(G->P);
  for (int q = 0; q < G->P; ++q) who[q] = q;
  std::vector<LoopRec> rec(G->P);
  std::vector<cudaEvent_t> ev(G->P);
  FEM_TRY(loop_publish(c, LoopRec{}, s, who.data(), G->P, rec.data(), ev.data()));
  for (int q = 0; q < G->P; ++q)
    if (q != m->rank) CUDA_TRY(cudaStreamWaitEvent(s, ev[q], 0));
  cudaError_t e = launch_loop_sum(stage, G->P, LoopGroup::MAXC, count, dev, s);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "loopback sum: %s", cudaGetErrorString(e));
  return FEM_OK;
}

// one node-plane halo per neighbour (ncclSend/Recv pairs in one group); planes `pitch` apart
static int halo_pitch(fem_op_s* op, const double* owned, double* lo, double* hi, int64_t pitch,
                      cudaStream_t s) {
  fem_mesh_s* m = op->mesh;
  if (m->nranks == 1) return FEM_OK;
  NvtxRange nv("fem:halo");
  if (m->comm->loop) return loop_halo(m, owned, lo, hi, pitch, s);
  const size_t cnt = (size_t)pitch;
  const int64_t np = m->g.k1 - m->g.k0;
  ncclComm_t c = m->comm->nccl;
  NCCL_TRY(ncclGroupStart());
  if (m->rank > 0) {
    NCCL_TRY(ncclSend(owned, cnt, ncclDouble, m->rank - 1, c, s));
    NCCL_TRY(ncclRecv(lo, cnt, ncclDouble, m->rank - 1, c, s));
  }
  if (m->rank < m->nranks - 1) {
    NCCL_TRY(ncclSend(owned + (np - 1) * pitch, cnt, ncclDouble, m->rank + 1, c, s));
    NCCL_TRY(ncclRecv(hi, cnt, ncclDouble, m->rank + 1, c, s));
  }
  NCCL_TRY(ncclGroupEnd());
  return FEM_OK;
}
static int halo(fem_op_s* op, const double* owned, double* lo, double* hi, cudaStream_t s) {
  return halo_pitch(op, owned, lo, hi, op->plane_dofs, s);
}

static int allreduce1(fem_op_s* op, double* dev_scalar, cudaStream_t s, int count = 1) {
  fem_mesh_s* m = op->mesh;
  if (m->nranks == 1) return FEM_OK;
  NvtxRange nv("fem:allreduce");
  if (m->comm->loop) return loop_allreduce(m, dev_scalar, count, s);
  NCCL_TRY(ncclAllReduce(dev_scalar, dev_scalar, count, ncclDouble, ncclSum, m->comm->nccl, s));
  return FEM_OK;
}

// ---- TMA tensor maps (driver entry point; no link against libcuda) --------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static int get_encode() {
  if (g_encode) return FEM_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(FEM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return FEM_OK;
}

// 3-D FP64 tiled map: dims (d0 contiguous, d1 rows of stride s1 bytes, d2 planes of stride s2),
// box (b0, b1, 1); out-of-range elements of a box are zero-filled by the copy engine.
static int make_map3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
                      uint64_t s1, uint64_t s2, uint32_t b0, uint32_t b1) {
  FEM_TRY(get_encode());
  if (((uintptr_t)base & 15) || (s1 & 15) || (s2 & 15) || ((b0 * 8) & 15))
    return fail(FEM_EINVAL, "tensor map alignment violated");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {b0, b1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FEM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return FEM_OK;
}

// u-plane maps of the padded CG vectors: only the nodes the operator may read (the interior
// with the Dirichlet box) lie inside the tensor, so the TMA zero fill is the mask P.
static int make_pl_maps(fem_op_s* op) {
  const Grid& g = op->mesh->g;
  const int C = op->comps;
  // Elasticity: the tensor spans the whole box (boundary nodes included: the Dirichlet mask P is
  // applied in registers and the unmasked boundary values feed the identity rows without a
  // global load).  Laplace with the Dirichlet box: the tensor spans only the interior, so the
  // copy engine's zero fill is the mask (boundary rows read x from global memory).
  const bool interior = op->tm_interior;
  const int64_t lo = interior ? 1 : 0;
  const int64_t i1 = interior ? g.nx - 1 : g.nx, j1 = interior ? g.ny - 1 : g.ny;
  const int64_t k0 = std::max<int64_t>(lo, g.k0 - 1), k1 = std::min<int64_t>(interior ? g.nz - 1 : g.nz, g.k1);
  op->tm_ok = false;
  if (i1 < lo || j1 < lo || k1 < k0) return FEM_OK;  // degenerate: bulk-row path, unfused CG
  unsigned bw, bh;
  u_box(op->kind, &bw, &bh);
  op->tm_i0 = lo;
  op->tm_j0 = lo;
  op->tm_k0 = k0;
  const int64_t off = op->pl_lead + (k0 - (g.k0 - 1)) * op->pl_pp + lo * op->pl_rp + lo * C;
  double* vecs[11] = {op->x_pl, op->p_pl, op->r_pl, op->p2_pl};
  CUtensorMap* maps[11] = {&op->tm_x, &op->tm_p, &op->tm_r, &op->tm_p2};
  for (int e = 0; e < 7; ++e) { vecs[4 + e] = op->pex[e]; maps[4 + e] = &op->tm_pex[e]; }
  for (int v = 0; v < 11; ++v) {
    if (!vecs[v]) continue;  // (pex: allocated for x_defer >= 4 only)
    FEM_TRY(make_map3d(maps[v], vecs[v] + off, (uint64_t)((i1 - lo + 1) * C), (uint64_t)(j1 - lo + 1),
                       (uint64_t)(k1 - k0 + 1), op->pl_rp * 8, op->pl_pp * 8, bw, bh));
  }
  op->tm_ok = true;
  return FEM_OK;
}

// Peer halo: tensor maps over the neighbours' ghost-plane sources (their last / first owned node
// plane), same origin, box and pitches as the local maps; ghost planes outside the operator's
// tensor range (the Dirichlet faces of the Laplace interior tensor) stay zero-filled locally.
extern "C" {
static void drop_graphs(fem_op_s* op);  // (defined inside the ABI block below)
}
static int build_peer_maps(fem_op_s* op) {
  const Grid& g = op->mesh->g;
  const int C = op->comps;
  const bool interior = op->tm_interior;
  const int64_t lo = interior ? 1 : 0;
  const int64_t i1 = interior ? g.nx - 1 : g.nx, j1 = interior ? g.ny - 1 : g.ny;
  const int64_t kmax = interior ? g.nz - 1 : g.nz;
  unsigned bw, bh;
  u_box(op->kind, &bw, &bh);
  constexpr int64_t kNone = -(int64_t(1) << 62);  // never a plane index (planes start at -1)
  op->pm_klo = (op->nb_lo[0] && g.k0 - 1 >= lo) ? g.k0 - 1 : kNone;
  op->pm_khi = (op->nb_hi[0] && g.k1 <= kmax) ? g.k1 : kNone;
  const int64_t off = op->pl_lead + lo * op->pl_rp + lo * C;
  for (int v = 0; v < 4; ++v) {
    if (op->pm_klo >= 0)
      FEM_TRY(make_map3d(&op->pm_lo[v], op->nb_lo[v] + off + op->nb_lo_nloc * op->pl_pp,
                         (uint64_t)((i1 - lo + 1) * C), (uint64_t)(j1 - lo + 1), 1, op->pl_rp * 8, op->pl_pp * 8,
                         bw, bh));
    if (op->pm_khi >= 0)
      FEM_TRY(make_map3d(&op->pm_hi[v], op->nb_hi[v] + off + op->pl_pp, (uint64_t)((i1 - lo + 1) * C),
                         (uint64_t)(j1 - lo + 1), 1, op->pl_rp * 8, op->pl_pp * 8, bw, bh));
  }
  op->peer_on = true;
  drop_graphs(op);  // captured iterations hold the halo path (and the x_defer group length) of their capture
  return FEM_OK;
}

static int make_mat_map(fem_op_s* op) {
  const Grid& g = op->mesh->g;
  unsigned bw, bh;
  mat_box(&bw, &bh);
  return make_map3d(&op->tm_mat, op->lm, (uint64_t)(2 * g.nx), (uint64_t)g.ny, (uint64_t)op->mat_layers,
                    (uint64_t)g.nx * 16, (uint64_t)g.nx * g.ny * 16, bw, bh);
}

// apply kernel dispatch
static int vec_index(const fem_op_s* op, const double* v) {  // x, p, r, p2 -> 0..3
  const double* b[4] = {op->x_pl, op->p_pl, op->r_pl, op->p2_pl};
  for (int i = 0; i < 4; ++i)
    if (b[i] == v) return i;
  return -1;
}

// peer-halo maps of one launch: u = padded vector v, u2 = v2 (mode 2), or none
static bool fill_peer(const fem_op_s* op, const double* v, const double* v2, PeerMaps* pm) {
  const int i = vec_index(op, v), i2 = v2 ? vec_index(op, v2) : i;
  if (!op->peer_on || i < 0 || i2 < 0) return false;
  pm->lo = op->pm_lo[i]; pm->hi = op->pm_hi[i];
  pm->lo2 = op->pm_lo[i2]; pm->hi2 = op->pm_hi[i2];
  pm->klo = op->pm_klo; pm->khi = op->pm_khi;
  pm->on = 1;
  return true;
}

static int ensure_aux_stream(fem_op_s* op) {
  if (op->astream) return FEM_OK;
  CUDA_TRY(cudaStreamCreateWithFlags(&op->astream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&op->ev_a0, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&op->ev_a1, cudaEventDisableTiming));
  return FEM_OK;
}

// elasticity applies run as an interior and an edge grid side by side (kernels_elastic.cu,
// TileMap): hand the launcher the operator's second stream and fork / join events
static int with_aux(fem_op_s* op, ApplyMaps* maps) {
  if (op->kind != FEM_ELASTICITY) return FEM_OK;
  FEM_TRY(ensure_aux_stream(op));
  maps->aux = op->astream;
  maps->ev_fork = op->ev_a0;
  maps->ev_join = op->ev_a1;
  return FEM_OK;
}

static int launch_apply(fem_op_s* op, PlaneSrc x, OutVec y, const CUtensorMap* umap, int mode,
                        cudaStream_t s, const double* vsrc = nullptr, const PairGeom* pair = nullptr) {
  fem_mesh_s* m = op->mesh;
  static thread_local PeerMaps pm;
  const bool peer = umap && vsrc && fill_peer(op, vsrc, nullptr, &pm);
  ApplyMaps maps{umap, op->tm_i0, op->tm_j0, op->tm_k0, &op->tm_mat, op->mat_layer0, nullptr, nullptr, nullptr,
                 op->tm_interior ? 1 : 0, op->quad, peer ? &pm : nullptr, pair};
  FEM_TRY(with_aux(op, &maps));
  cudaError_t e;
  if (op->use_pa)  // partial assembly on the box (21 stored values per Gauss point, bulk-row staging)
    e = launch_pa21_apply(op->bc, op->quad, m->g, x, y, op->pa, mode, op->sc, op->red, s, m->sm_count);
  else if (op->kind == FEM_ELASTICITY)
    e = launch_elastic(op->bc, m->g, x, y, maps, mode, op->sc, op->red, s, m->sm_count);
  else
    e = launch_laplace(op->comps, op->bc, m->g, x, y, maps, mode, op->sc, op->red, s, m->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "apply launch failed: %s", cudaGetErrorString(e));
  return FEM_OK;
}

static int launch_maps(fem_op_s* op, const Grid& g, PlaneSrc x, OutVec y, const ApplyMaps& maps, int mode,
                       Reduce red, cudaStream_t s) {
  fem_mesh_s* m = op->mesh;
  ApplyMaps mm = maps;
  FEM_TRY(with_aux(op, &mm));
  const cudaError_t e = op->kind == FEM_ELASTICITY
                            ? launch_elastic(op->bc, g, x, y, mm, mode, op->sc, red, s, m->sm_count)
                            : launch_laplace(op->comps, op->bc, g, x, y, maps, mode, op->sc, red, s, m->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "apply launch failed: %s", cudaGetErrorString(e));
  return FEM_OK;
}

static int ensure_comm_stream(fem_op_s* op) {
  if (op->cstream) return FEM_OK;
  CUDA_TRY(cudaStreamCreateWithFlags(&op->cstream, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming));
  CUDA_TRY(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming));
  return FEM_OK;
}

// Apply with an exchange step (NCCL or loopback halo, nranks > 1): the halo runs
// on the operator's comm stream while the interior output planes [k0+1, k1-1) -- which read
// owned planes only -- run on the caller's stream; after the join one launch covers the two
// boundary planes k0 and k1-1 (two one-plane z-chunks, kchunk_force).  The dots of the two
// launches add up (Reduce::acc); the fused-CG roll happens in the second.  Per node the sums
// are those of a single launch, so the result stays bitwise slab invariant.  `halo(stream)`
// posts the exchange; src / out / maps describe the whole owned range.
static int apply_split(fem_op_s* op, cudaStream_t s, PlaneSrc src, OutVec out, ApplyMaps maps, int mode,
                       Reduce red, const std::function<int(cudaStream_t)>& halo) {
  const Grid& g = op->mesh->g;
  const int64_t nl = g.k1 - g.k0;
  // trace events are plain records on the eager path (inside a graph capture they would be
  // nodes recorded at replay; the trace is a diagnostic of eager applies)
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(s, &cst));
  const bool tr = op->trace && cst == cudaStreamCaptureStatusNone;
  if (tr) {
    for (auto& e : op->tr_ev)
      if (!e) CUDA_TRY(cudaEventCreate(&e));
    CUDA_TRY(cudaEventRecord(op->tr_ev[0], s));
    op->tr_valid = true;
  }
  if (!op->overlap || nl < 3) {
    FEM_TRY(halo(s));
    if (tr) CUDA_TRY(cudaEventRecord(op->tr_ev[1], s));
    {
      NvtxRange nv("fem:apply_planes");
      FEM_TRY(launch_maps(op, g, src, out, maps, mode, red, s));
    }
    if (tr) {
      CUDA_TRY(cudaEventRecord(op->tr_ev[2], s));
      CUDA_TRY(cudaEventRecord(op->tr_ev[3], s));
    }
    return FEM_OK;
  }
  FEM_TRY(ensure_comm_stream(op));
  CUDA_TRY(cudaEventRecord(op->ev_fork, s));
  CUDA_TRY(cudaStreamWaitEvent(op->cstream, op->ev_fork, 0));
  FEM_TRY(halo(op->cstream));
  if (tr) CUDA_TRY(cudaEventRecord(op->tr_ev[1], op->cstream));
  CUDA_TRY(cudaEventRecord(op->ev_join, op->cstream));
  Grid gi = g;
  gi.k0 = g.k0 + 1;
  gi.k1 = g.k1 - 1;
  const PlaneSrc si{src.main + src.ppitch, src.main, src.main + (nl - 1) * src.ppitch, src.rpitch, src.ppitch};
  const OutVec oi{out.y + out.ppitch, out.rpitch, out.ppitch};
  ApplyMaps mi = maps;
  if (mi.pold) mi.pold += src.ppitch;  // (pold / pnew share the input's layout)
  if (mi.pnew) mi.pnew += src.ppitch;
  Reduce ri = red;
  ri.acc = 0;
  ri.roll = 0;
  {
    NvtxRange nv("fem:interior");
    FEM_TRY(launch_maps(op, gi, si, oi, mi, mode, ri, s));
  }
  if (tr) CUDA_TRY(cudaEventRecord(op->tr_ev[2], s));
  CUDA_TRY(cudaStreamWaitEvent(s, op->ev_join, 0));
  ApplyMaps mb = maps;
  mb.kchunk_force = nl - 1;
  mb.zc_force = 2;
  mb.kspan = 1;
  Reduce rb = red;
  rb.acc = 1;
  {
    NvtxRange nv("fem:boundary");
    FEM_TRY(launch_maps(op, g, src, out, mb, mode, rb, s));
  }
  if (tr) CUDA_TRY(cudaEventRecord(op->tr_ev[3], s));
  return FEM_OK;
}

static PlaneSrc dense_src(fem_op_s* op, const double* x, const double* lo, const double* hi) {
  const Grid& g = op->mesh->g;
  return PlaneSrc{x, lo, hi, (g.nx + 1) * op->comps, g.plane * op->comps};
}
static OutVec dense_out(fem_op_s* op, double* y) {
  const Grid& g = op->mesh->g;
  return OutVec{y, (g.nx + 1) * op->comps, g.plane * op->comps};
}
static double* pl_owned(fem_op_s* op, double* v) { return v + op->pl_off; }
static PlaneSrc pl_src(fem_op_s* op, double* v) {
  fem_mesh_s* m = op->mesh;
  return PlaneSrc{pl_owned(op, v), m->rank > 0 ? v + op->pl_lead : nullptr,
                  m->rank < m->nranks - 1 ? v + op->pl_lead + (op->nloc_planes + 1) * op->pl_pp : nullptr,
                  op->pl_rp, op->pl_pp};
}
static OutVec pl_out(fem_op_s* op, double* v) { return OutVec{pl_owned(op, v), op->pl_rp, op->pl_pp}; }
static int64_t pl_count(fem_op_s* op) { return op->nloc_planes * op->pl_pp; }  // owned range

// general hex mesh: y = A_c x (zero y, element kernel with red.add scatter, identity rows); with
// option "deterministic": element outputs to hx_E, then the per-node gather writes every y entry
static int apply_hex(fem_op_s* op, const double* x, double* y, int mode, cudaStream_t s) {
  fem_mesh_s* m = op->mesh;
  double* E = op->det ? op->hx_E : nullptr;
  if (!E) CUDA_TRY(cudaMemsetAsync(y, 0, op->n_local * sizeof(double), s));
  cudaError_t e = op->use_pa
                      ? launch_hex_pa_apply(op->kind, op->bc, op->quad, m->hx_cells, op->pa, op->lm, x, y, E,
                                            m->hx_ncells, mode, op->sc, op->red, s, m->sm_count)
                      : launch_hex_apply(op->kind, op->bc, op->quad, m->hx_cells, m->hx_xyz, op->lm, x, y, E,
                                         m->hx_ncells, mode, op->sc, op->red, s, m->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "hex apply launch: %s", cudaGetErrorString(e));
  if (E) {
    e = launch_hex_gather(op->comps, m->hx_n2e_off, m->hx_n2e, E, y, m->hx_nodes, s, m->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "hex gather launch: %s", cudaGetErrorString(e));
  }
  if (op->bc && m->hx_nb) {
    e = launch_hex_dirichlet(m->hx_bnodes, m->hx_nb, op->comps, x, y, mode, op->sc, op->red, s, m->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "hex identity-row launch: %s", cudaGetErrorString(e));
  }
  return FEM_OK;
}

// Tensor maps over caller vectors, cached per (pointer, allocation id, staging path): fem_apply
// on the same buffers (the usual case: a solver's work vectors) re-encodes nothing.
static const CUtensorMap* cached_map(fem_op_s* op, const void* p, unsigned long long id, int path) {
  for (const auto& e : op->map_cache)
    if (e.p == p && e.id == id && e.path == path && id != 0) return &e.map;
  return nullptr;
}
static CUtensorMap* new_map_slot(fem_op_s* op, const void* p, unsigned long long id, int path) {
  constexpr size_t kSlots = 8;
  if (op->map_cache.size() < kSlots) op->map_cache.emplace_back();
  auto& e = op->map_cache[op->map_next++ % op->map_cache.size()];
  e.p = p;
  e.id = id;
  e.path = path;
  return &e.map;
}

// y = A_c x for a DEVICE dense owned vector x (halo via op ghost buffers); xi describes x's
// allocation (ptr_info)
static int apply_device(fem_op_s* op, const double* x, double* y, cudaStream_t s, const PtrInfo& xi) {
  if (op->mesh->hex) return apply_hex(op, x, y, 0, s);
  fem_mesh_s* m = op->mesh;
  const Grid& g = m->g;
  const int64_t rp = (g.nx + 1) * op->comps;
  // A caller vector whose rows are 16-B multiples ((nx+1) c even) and whose base is 16-B aligned
  // is described by a tensor map directly (full box, like the CG vectors), so the apply stages ONE
  // TMA box per plane instead of one bulk copy per row.  Single rank: the ghost planes of a slab
  // are not adjacent to the caller's memory.
  if (op->direct_tm && !op->use_pa && m->nranks == 1 && op->tm_ok && !op->tm_interior && (rp & 1) == 0 &&
      ((uintptr_t)x & 15) == 0) {
    const CUtensorMap* map = cached_map(op, x, xi.id, 1);
    if (!map) {
      unsigned bw, bh;
      u_box(op->kind, &bw, &bh);
      CUtensorMap* slot = new_map_slot(op, x, xi.id, 1);
      FEM_TRY(make_map3d(slot, x, (uint64_t)rp, (uint64_t)(g.ny + 1), (uint64_t)(g.nz + 1), (uint64_t)rp * 8,
                         (uint64_t)(g.plane * op->comps) * 8, bw, bh));
      map = slot;
    }
    op->last_path = 1;
    return launch_apply(op, dense_src(op, x, nullptr, nullptr), dense_out(op, y), map, 0, s);
  }
  // Odd rows (Dirichlet box): the row-pair view (kernels_common.cuh, PairGeom) --
  // dim 0 spans two rows plus the plane parity, dims 1 / 2 step by row pairs / plane pairs (16-B
  // strides) -- so the apply still stages two TMA boxes per plane.  Boxes read up to one row and
  // two box widths past the vector's end (last plane): taken only when the caller's allocation
  // extends that far (cuMemGetAddressRange), else the bulk-row path.
  if (op->direct_tm && !op->use_pa && m->nranks == 1 && op->tm_ok && !op->tm_interior && op->bc && (rp & 1) &&
      (op->kind != FEM_ELASTICITY || kElCY == 2) && ((uintptr_t)x & 15) == 0) {
    unsigned bw, bh;
    u_box(op->kind, &bw, &bh);
    const int64_t lp = g.plane * op->comps;
    const size_t need = (size_t)(op->n_local + rp + 2 * (int64_t)bw) * sizeof(double);
    if (xi.id && (uintptr_t)x + need <= xi.base + xi.size) {
      const PairGeom pg{rp, lp, g.nz};
      const CUtensorMap* map = cached_map(op, x, xi.id, 2);
      if (!map) {
        CUtensorMap* slot = new_map_slot(op, x, xi.id, 2);
        FEM_TRY(make_map3d(slot, x, (uint64_t)(lp + 2 * rp), (uint64_t)((g.ny + 2) / 2), (uint64_t)((g.nz + 2) / 2),
                           (uint64_t)(2 * rp) * 8, (uint64_t)(2 * lp) * 8, bw, (bh + 1) / 2));
        map = slot;
      }
      op->last_path = 2;
      return launch_apply(op, dense_src(op, x, nullptr, nullptr), dense_out(op, y), map, 0, s, nullptr, &pg);
    }
    if (g.nz >= 1 && xi.id) {
      // No slack after the vector (e.g. an exact-size cudaMalloc): the view covers planes
      // [0, nz - 1] only -- its boxes then stay inside the vector -- and the last plane is served
      // from a one-plane copy with slack (3.6 MB at C4) through the PeerMaps plane substitution
      if (!op->last_plane) {
        FEM_TRY(dalloc(&op->last_plane, lp + rp + 2 * 128));
        CUDA_TRY(cudaMemset(op->last_plane, 0, (lp + rp + 2 * 128) * sizeof(double)));
        FEM_TRY(make_map3d(&op->gm_last, op->last_plane, (uint64_t)(lp + 2 * rp), (uint64_t)((g.ny + 2) / 2), 1,
                           (uint64_t)(2 * rp) * 8, (uint64_t)(2 * lp) * 8, bw, (bh + 1) / 2));
      }
      CUDA_TRY(cudaMemcpyAsync(op->last_plane, x + g.nz * lp, lp * sizeof(double), cudaMemcpyDeviceToDevice, s));
      const CUtensorMap* map = cached_map(op, x, xi.id, 5);
      if (!map) {
        CUtensorMap* slot = new_map_slot(op, x, xi.id, 5);
        FEM_TRY(make_map3d(slot, x, (uint64_t)(lp + 2 * rp), (uint64_t)((g.ny + 2) / 2), (uint64_t)((g.nz + 1) / 2),
                           (uint64_t)(2 * rp) * 8, (uint64_t)(2 * lp) * 8, bw, (bh + 1) / 2));
        map = slot;
      }
      static thread_local PeerMaps pm;
      pm.lo = pm.hi = pm.lo2 = pm.hi2 = op->gm_last;
      pm.klo = -(int64_t(1) << 62);
      pm.khi = g.nz;
      pm.on = 1;
      const PairGeom pg{rp, lp, g.nz - 1, 0};
      ApplyMaps maps{map, 0, 0, 0, &op->tm_mat, op->mat_layer0, nullptr, nullptr, nullptr, 0, op->quad, &pm, &pg};
      op->last_path = 2;
      return launch_maps(op, g, dense_src(op, x, nullptr, nullptr), dense_out(op, y), maps, 0, op->red, s);
    }
  }
  // P > 1: the same two TMA views over the rank's owned planes [k0, k1) (tensor origin k0), the
  // ghost planes k0 - 1 / k1 from the library's ghost buffers -- filled by the halo, overlapped
  // with the interior planes (apply_split) -- through the PeerMaps plane substitution
  if (op->direct_tm && !op->use_pa && m->nranks > 1 && op->tm_ok && !op->tm_interior && ((uintptr_t)x & 15) == 0 &&
      ((rp & 1) == 0 || (op->bc && (op->kind != FEM_ELASTICITY || kElCY == 2)))) {
    unsigned bw, bh;
    u_box(op->kind, &bw, &bh);
    const int64_t lp = g.plane * op->comps;
    const int64_t nloc = g.k1 - g.k0;
    const bool pair = (rp & 1) != 0;
    const size_t need = (size_t)(op->n_local + rp + 2 * (int64_t)bw) * sizeof(double);
    if (!pair || (xi.id && (uintptr_t)x + need <= xi.base + xi.size)) {
      const int path = pair ? 4 : 3;
      const CUtensorMap* map = cached_map(op, x, xi.id, path);
      if (!map) {
        CUtensorMap* slot = new_map_slot(op, x, xi.id, path);
        if (pair)
          FEM_TRY(make_map3d(slot, x, (uint64_t)(lp + 2 * rp), (uint64_t)((g.ny + 2) / 2), (uint64_t)((nloc + 1) / 2),
                             (uint64_t)(2 * rp) * 8, (uint64_t)(2 * lp) * 8, bw, (bh + 1) / 2));
        else
          FEM_TRY(make_map3d(slot, x, (uint64_t)rp, (uint64_t)(g.ny + 1), (uint64_t)nloc, (uint64_t)rp * 8,
                             (uint64_t)lp * 8, bw, bh));
        map = slot;
      }
      CUtensorMap* gm = pair ? op->gm_pair : op->gm_dir;
      bool& gm_ok = pair ? op->gm_pair_ok : op->gm_dir_ok;
      if (!gm_ok) {
        double* gb[2] = {op->ghost_lo, op->ghost_hi};
        for (int k = 0; k < 2; ++k) {
          if (pair)
            FEM_TRY(make_map3d(&gm[k], gb[k], (uint64_t)(lp + 2 * rp), (uint64_t)((g.ny + 2) / 2), 1,
                               (uint64_t)(2 * rp) * 8, (uint64_t)(2 * lp) * 8, bw, (bh + 1) / 2));
          else
            FEM_TRY(make_map3d(&gm[k], gb[k], (uint64_t)rp, (uint64_t)(g.ny + 1), 1, (uint64_t)rp * 8,
                               (uint64_t)lp * 8, bw, bh));
        }
        gm_ok = true;
      }
      static thread_local PeerMaps pm;
      constexpr int64_t kNone = -(int64_t(1) << 62);
      pm.lo = gm[0];
      pm.hi = gm[1];
      pm.lo2 = gm[0];
      pm.hi2 = gm[1];
      pm.klo = m->rank > 0 ? g.k0 - 1 : kNone;
      pm.khi = m->rank < m->nranks - 1 ? g.k1 : kNone;
      pm.on = 1;
      const PairGeom pg{rp, lp, g.k1 - 1, g.k0};
      ApplyMaps maps{map, 0, 0, g.k0, &op->tm_mat, op->mat_layer0, nullptr, nullptr, nullptr, 0, op->quad, &pm,
                     pair ? &pg : nullptr};
      op->last_path = pair ? 2 : 1;
      return apply_split(op, s, dense_src(op, x, op->ghost_lo, op->ghost_hi), dense_out(op, y), maps, 0, op->red,
                         [&](cudaStream_t hs) { return halo(op, x, op->ghost_lo, op->ghost_hi, hs); });
    }
  }
  op->last_path = 0;
  PlaneSrc src = dense_src(op, x, op->mesh->rank > 0 ? op->ghost_lo : nullptr,
                           op->mesh->rank < op->mesh->nranks - 1 ? op->ghost_hi : nullptr);
  if (m->nranks == 1) return launch_apply(op, src, dense_out(op, y), nullptr, 0, s);
  ApplyMaps maps{nullptr, op->tm_i0, op->tm_j0, op->tm_k0, &op->tm_mat, op->mat_layer0, nullptr, nullptr, nullptr,
                 op->tm_interior ? 1 : 0, op->quad, nullptr, nullptr};
  return apply_split(op, s, src, dense_out(op, y), maps, 0, op->red,
                     [&](cudaStream_t hs) { return halo(op, x, op->ghost_lo, op->ghost_hi, hs); });
}

// q_pl = A_c v for a padded CG vector v (x_pl or p_pl): halo into its ghost planes, TMA path
static int apply_pl(fem_op_s* op, double* v, const CUtensorMap* map, int mode, cudaStream_t s) {
  fem_mesh_s* m = op->mesh;
  if (m->hex) return apply_hex(op, pl_owned(op, v), pl_owned(op, op->q_pl), mode, s);
  if (m->nranks > 1 && !(op->peer_on && op->tm_ok)) {
    ApplyMaps maps{op->tm_ok ? map : nullptr, op->tm_i0, op->tm_j0, op->tm_k0, &op->tm_mat, op->mat_layer0,
                   nullptr, nullptr, nullptr, op->tm_interior ? 1 : 0, op->quad, nullptr, nullptr};
    return apply_split(op, s, pl_src(op, v), pl_out(op, op->q_pl), maps, mode, op->red, [&](cudaStream_t hs) {
      return halo_pitch(op, pl_owned(op, v), v + op->pl_lead, v + op->pl_lead + (op->nloc_planes + 1) * op->pl_pp,
                        op->pl_pp, hs);
    });
  }
  return launch_apply(op, pl_src(op, v), pl_out(op, op->q_pl), op->tm_ok ? map : nullptr, mode, s, v);
}

// (re)compute the stored Gauss-point geometry when partial assembly is on and the rule changed
static int pa_setup(fem_op_s* op, bool force = false) {
  if (!op->use_pa) return FEM_OK;
  if (!op->mesh->hex) {  // box: D_q = w_q det J_q C_e from the material (quadrature independent)
    if (!op->has_mat) return FEM_OK;  // computed by fem_set_material
    if (op->pa_quad >= 0 && !force) return FEM_OK;
    const int64_t ncells = op->mesh->g.nx * op->mesh->g.ny * op->mesh->g.nz;
    if (!op->pa) FEM_TRY(dalloc(&op->pa, pa21_doubles(ncells)));
    cudaError_t e = launch_pa21_setup(op->lm, ncells, op->mesh->g.h, op->pa, 0, op->mesh->sm_count);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(FEM_ECUDA, "partial-assembly setup: %s", cudaGetErrorString(e));
    op->pa_quad = 0;
    return FEM_OK;
  }
  if (op->pa_quad == op->quad) return FEM_OK;
  if (!op->pa) FEM_TRY(dalloc(&op->pa, hex_pa_doubles(op->kind, op->mesh->hx_ncells)));
  cudaError_t e = launch_hex_pa_setup(op->kind, op->quad, op->mesh->hx_cells, op->mesh->hx_xyz, op->pa,
                                      op->mesh->hx_ncells, 0, op->mesh->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "partial-assembly setup: %s", cudaGetErrorString(e));
  CUDA_TRY(cudaDeviceSynchronize());
  op->pa_quad = op->quad;
  return FEM_OK;
}


static int pack(fem_op_s* op, const double* dense, double* v, int to_padded, cudaStream_t s) {
  if (op->mesh->hex) {  // CG vectors are dense on general meshes
    if (to_padded)
      CUDA_TRY(cudaMemcpyAsync(pl_owned(op, v), dense, op->n_local * sizeof(double), cudaMemcpyDeviceToDevice, s));
    else
      CUDA_TRY(cudaMemcpyAsync(const_cast<double*>(dense), pl_owned(op, v), op->n_local * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    return FEM_OK;
  }
  const Grid& g = op->mesh->g;
  cudaError_t e = launch_pack(dense, pl_owned(op, v), op->pl_rp, op->pl_pp, op->nloc_planes, g.nx + 1,
                              g.ny + 1, op->comps, to_padded, s, op->mesh->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "pack launch: %s", cudaGetErrorString(e));
  return FEM_OK;
}

static int ensure_stage(fem_op_s* op) {
  if (!op->stage_a) FEM_TRY(dalloc(&op->stage_a, op->n_local));
  if (!op->stage_b) FEM_TRY(dalloc(&op->stage_b, op->n_local));
  return FEM_OK;
}

static int dot_device(fem_op_s* op, const double* a, const double* b, cudaStream_t s,
                      double* result, int64_t n = -1) {
  cudaError_t e = launch_dot(a, b, n < 0 ? op->n_local : n, op->dot_dev, op->red, s, op->mesh->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "dot launch failed: %s", cudaGetErrorString(e));
  FEM_TRY(allreduce1(op, op->dot_dev, s));
  CUDA_TRY(cudaMemcpyAsync(op->dot_host, op->dot_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *result = *op->dot_host;
  return FEM_OK;
}

// ------------------------------------------------------------------------------------------
// ABI
// ------------------------------------------------------------------------------------------
extern "C" {

const char* fem_last_error(void) { return t_err.c_str(); }
const char* fem_version(void) { return "paper_2308_09839_b200 libfem 0.1 (sm_100a, fp64)"; }
int64_t fem_launch_count(void) { return g_launches.load(); }

int fem_get_unique_id(void* id_out, int64_t id_bytes) {
  if (!id_out || id_bytes < (int64_t)sizeof(ncclUniqueId))
    return fail(FEM_EINVAL, "id buffer must hold %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return FEM_OK;
}

int fem_comm_create(int32_t nranks, int32_t rank, const void* id, fem_comm_t* out) {
  if (!out) return fail(FEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FEM_EINVAL, "bad nranks/rank %d/%d", nranks, rank);
  auto* c = new (std::nothrow) fem_comm_s();
  if (!c) return fail(FEM_ENOMEM, "host allocation failed");
  c->nranks = nranks;
  c->rank = rank;
  cudaError_t e = cudaGetDevice(&c->device);
  if (e != cudaSuccess) {
    delete c;
    return fail(FEM_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  }
  if (nranks > 1 && id) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(FEM_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
  }
  *out = c;
  return FEM_OK;
}

int fem_comm_create_loopback(int32_t nranks, fem_comm_t* out) {
  if (!out) return fail(FEM_EINVAL, "out is NULL");
  if (nranks < 1 || nranks > LoopGroup::K) return fail(FEM_EINVAL, "loopback nranks must be in [1, %d]", LoopGroup::K);
  for (int r = 0; r < nranks; ++r) out[r] = nullptr;
  auto* G = new (std::nothrow) LoopGroup();
  if (!G) return fail(FEM_ENOMEM, "host allocation failed");
  G->P = nranks;
  cudaGetDevice(&G->device);
  G->seq.assign(nranks, 0);
  G->rec.resize((size_t)nranks * LoopGroup::K);
  G->ev.assign((size_t)nranks * LoopGroup::K, nullptr);
  auto bail = [&](int st) {
    for (cudaEvent_t e : G->ev)
      if (e) cudaEventDestroy(e);
    cudaFree(G->red);
    for (int r = 0; r < nranks; ++r) { delete out[r]; out[r] = nullptr; }
    delete G;
    return st;
  };
  for (auto& e : G->ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(FEM_ECUDA, "cudaEventCreate failed"));
  if (dalloc(&G->red, (size_t)LoopGroup::KR * nranks * LoopGroup::MAXC) != FEM_OK) return bail(FEM_ENOMEM);
  for (int r = 0; r < nranks; ++r) {
    out[r] = new (std::nothrow) fem_comm_s();
    if (!out[r]) return bail(fail(FEM_ENOMEM, "host allocation failed"));
    out[r]->nranks = nranks;
    out[r]->rank = r;
    out[r]->device = G->device;
    out[r]->loop = G;
  }
  G->refs = nranks;
  return FEM_OK;
}

void fem_comm_destroy(fem_comm_t c) {
  if (!c) return;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (LoopGroup* G = c->loop) {
    bool last;
    {
      std::lock_guard<std::mutex> lk(G->mu);
      last = --G->refs == 0;
    }
    if (last) {
      set_device(G->device);
      for (cudaEvent_t e : G->ev)
        if (e) cudaEventDestroy(e);
      cudaFree(G->red);
      delete G;
    }
  }
  delete c;
}

int fem_partition(int64_t nz, int32_t nranks, int32_t rank, int64_t* pb, int64_t* pe) {
  if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !pb || !pe)
    return fail(FEM_EINVAL, "bad partition arguments");
  if (nz + 1 < nranks) return fail(FEM_EINVAL, "fewer node planes (%lld) than ranks (%d)", (long long)(nz + 1), nranks);
  const int64_t N = nz + 1, base = N / nranks, rem = N % nranks;
  *pb = rank * base + std::min<int64_t>(rank, rem);
  *pe = *pb + base + (rank < rem ? 1 : 0);
  return FEM_OK;
}

int fem_mesh_create(int64_t nx, int64_t ny, int64_t nz, double h, fem_comm_t comm, fem_mesh_t* out) {
  if (!out) return fail(FEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (nx < 1 || ny < 1 || nz < 1) return fail(FEM_EINVAL, "dims must be >= 1 (got %lld %lld %lld)", (long long)nx, (long long)ny, (long long)nz);
  if (!(h > 0.0) || !std::isfinite(h)) return fail(FEM_EINVAL, "h must be finite and > 0");
  // 32-bit global node index limit and int32 CSR column headroom
  const double nn = (double)(nx + 1) * (double)(ny + 1) * (double)(nz + 1);
  if (nn >= 4294967296.0) return fail(FEM_EOVERFLOW, "global node count %.0f >= 2^32", nn);
  const int P = comm ? comm->nranks : 1;
  const int R = comm ? comm->rank : 0;
  if (nz + 1 < P) return fail(FEM_EINVAL, "fewer node planes (%lld) than ranks (%d)", (long long)(nz + 1), P);
  auto* m = new (std::nothrow) fem_mesh_s();
  if (!m) return fail(FEM_ENOMEM, "host allocation failed");
  m->comm = comm;
  m->nranks = P;
  m->rank = R;
  cudaGetDevice(&m->device);
  cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, m->device);
  int64_t k0 = 0, k1 = 0;
  fem_partition(nz, P, R, &k0, &k1);
  m->g = Grid{nx, ny, nz, h, k0, k1, (nx + 1) * (ny + 1)};
  *out = m;
  return FEM_OK;
}

int fem_mesh_local(fem_mesh_t m, int64_t* pb, int64_t* pe, int64_t* nloc) {
  if (!m) return fail(FEM_EINVAL, "mesh is NULL");
  if (m->hex) {  // one "plane": all nodes
    if (pb) *pb = 0;
    if (pe) *pe = 1;
    if (nloc) *nloc = m->hx_nodes;
    return FEM_OK;
  }
  if (pb) *pb = m->g.k0;
  if (pe) *pe = m->g.k1;
  if (nloc) *nloc = (m->g.k1 - m->g.k0) * m->g.plane;
  return FEM_OK;
}

int fem_mesh_create_hex(int64_t n_nodes, int64_t n_cells, const double* coords, const int32_t* cells,
                        const uint8_t* dirichlet, fem_mesh_t* out) {
  if (!out) return fail(FEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_nodes < 1 || n_cells < 1) return fail(FEM_EINVAL, "n_nodes and n_cells must be >= 1");
  if (n_nodes > 2147483647LL) return fail(FEM_EOVERFLOW, "node count %lld exceeds 2^31 - 1", (long long)n_nodes);
  if (!coords || !cells) return fail(FEM_EINVAL, "coords / cells is NULL");
  if ((reinterpret_cast<uintptr_t>(coords) & 7) || (reinterpret_cast<uintptr_t>(cells) & 3))
    return fail(FEM_EINVAL, "coords must be 8-byte and cells 4-byte aligned");
  auto* m = new (std::nothrow) fem_mesh_s();
  if (!m) return fail(FEM_ENOMEM, "host allocation failed");
  cudaGetDevice(&m->device);
  cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, m->device);
  m->hex = true;
  m->hx_nodes = n_nodes;
  m->hx_ncells = n_cells;
  m->g = Grid{0, 0, 0, 0.0, 0, 1, n_nodes};
  int32_t* d_vtk = nullptr;
  uint8_t* d_dir = nullptr;
  unsigned long long* d_bad = nullptr;
  auto cleanup = [&]() { cudaFree(d_vtk); cudaFree(d_dir); cudaFree(d_bad); };
  auto bail = [&](int st) { cleanup(); fem_mesh_destroy(m); return st; };
  // coordinates -> double4 records (cudaMemcpy2D: 24-B source rows, 32-B destination rows)
  if (dalloc(&m->hx_xyz, n_nodes) != FEM_OK) return bail(FEM_ENOMEM);
  const cudaMemcpyKind kc = is_device_ptr(coords) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (cudaMemset(m->hx_xyz, 0, n_nodes * sizeof(double4)) != cudaSuccess ||
      cudaMemcpy2D(m->hx_xyz, sizeof(double4), coords, 3 * sizeof(double), 3 * sizeof(double), n_nodes, kc) !=
          cudaSuccess)
    return bail(fail(FEM_ECUDA, "coordinate copy failed"));
  // node map (+ Dirichlet flags) -> internal cell records, validated on the device
  if (dalloc(&d_vtk, n_cells * 8) != FEM_OK || dalloc(&d_bad, 2) != FEM_OK ||
      dalloc(&m->hx_cells, n_cells * 2) != FEM_OK)
    return bail(FEM_ENOMEM);
  if (cudaMemcpy(d_vtk, cells, n_cells * 8 * sizeof(int32_t),
                 is_device_ptr(cells) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(d_bad, 0, 2 * sizeof(unsigned long long)) != cudaSuccess)
    return bail(fail(FEM_ECUDA, "node map copy failed"));
  std::vector<uint8_t> hdir;
  if (dirichlet) {
    if (dalloc(&d_dir, n_nodes) != FEM_OK) return bail(FEM_ENOMEM);
    hdir.resize(n_nodes);
    const cudaMemcpyKind kd = is_device_ptr(dirichlet) ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost;
    if (cudaMemcpy(hdir.data(), dirichlet, n_nodes, kd) != cudaSuccess ||
        cudaMemcpy(d_dir, hdir.data(), n_nodes, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(FEM_ECUDA, "Dirichlet flag copy failed"));
  }
  if (launch_hex_pack_cells(d_vtk, d_dir, n_cells, n_nodes, reinterpret_cast<int*>(m->hx_cells), d_bad, 0,
                            m->sm_count) != cudaSuccess ||
      launch_hex_check(m->hx_cells, m->hx_xyz, n_cells, n_nodes, 0, d_bad, 0, m->sm_count) != cudaSuccess)
    return bail(fail(FEM_ECUDA, "mesh validation launch failed"));
  unsigned long long bad[2] = {0, 0};
  if (cudaMemcpy(bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost) != cudaSuccess)
    return bail(fail(FEM_ECUDA, "mesh validation failed: %s", cudaGetErrorString(cudaGetLastError())));
  if (bad[0]) return bail(fail(FEM_EINVAL, "%llu node-map entries outside [0, n_nodes)", bad[0]));
  if (bad[1]) return bail(fail(FEM_EINVAL, "%llu cells have det J <= 0 at a Gauss point (S:265, S:333)", bad[1]));
  // constrained node list (identity rows)
  std::vector<int32_t> bn;
  for (int64_t n = 0; n < (int64_t)hdir.size(); ++n)
    if (hdir[n]) bn.push_back((int32_t)n);
  m->hx_nb = (int64_t)bn.size();
  if (m->hx_nb) {
    if (dalloc(&m->hx_bnodes, m->hx_nb) != FEM_OK) return bail(FEM_ENOMEM);
    if (cudaMemcpy(m->hx_bnodes, bn.data(), bn.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(fail(FEM_ECUDA, "constrained-node copy failed"));
  }
  cleanup();
  *out = m;
  return FEM_OK;
}

int fem_mesh_info_hex(fem_mesh_t m, int64_t* n_nodes, int64_t* n_cells, int64_t* n_constrained) {
  if (!m) return fail(FEM_EINVAL, "mesh is NULL");
  if (!m->hex) return fail(FEM_EINVAL, "not a general hexahedral mesh");
  if (n_nodes) *n_nodes = m->hx_nodes;
  if (n_cells) *n_cells = m->hx_ncells;
  if (n_constrained) *n_constrained = m->hx_nb;
  return FEM_OK;
}

void fem_mesh_destroy(fem_mesh_t m) {
  if (!m) return;
  if (m->hex) {
    set_device(m->device);
    cudaFree(m->hx_xyz);
    cudaFree(m->hx_cells);
    cudaFree(m->hx_bnodes);
    cudaFree(m->hx_n2e_off);
    cudaFree(m->hx_n2e);
  }
  delete m;
}

static void op_free(fem_op_s* op) {
  if (!op) return;
  set_device(op->mesh->device);
  if (op->graph1) cudaGraphExecDestroy(op->graph1);
  if (op->graphN) cudaGraphExecDestroy(op->graphN);
  for (auto e : op->ev) cudaEventDestroy(e);
  if (op->cstream) cudaStreamDestroy(op->cstream);
  if (op->ev_fork) cudaEventDestroy(op->ev_fork);
  if (op->ev_join) cudaEventDestroy(op->ev_join);
  for (auto e : op->tr_ev)
    if (e) cudaEventDestroy(e);
  if (op->astream) cudaStreamDestroy(op->astream);
  if (op->ev_a0) cudaEventDestroy(op->ev_a0);
  if (op->ev_a1) cudaEventDestroy(op->ev_a1);
  if (op->peer_ipc)
    for (int v = 0; v < 4; ++v) {
      if (op->nb_lo[v]) cudaIpcCloseMemHandle(op->nb_lo[v]);
      if (op->nb_hi[v]) cudaIpcCloseMemHandle(op->nb_hi[v]);
    }
  cudaFree(op->lm);
  cudaFree(op->pa);
  cudaFree(op->hx_E);
  cudaFree(op->last_plane);
  cudaFree(op->x_pl); cudaFree(op->r_pl); cudaFree(op->p_pl); cudaFree(op->q_pl); cudaFree(op->p2_pl);
  for (double* e : op->pex) cudaFree(e);
  if (op->graph1b) cudaGraphExecDestroy(op->graph1b);
  for (const auto& t : op->graphT) cudaGraphExecDestroy(t.exec);
  for (const auto& t : op->graphK) cudaGraphExecDestroy(t.exec);
  cudaFree(op->ghost_lo); cudaFree(op->ghost_hi);
  cudaFree(op->stage_a); cudaFree(op->stage_b);
  cudaFree(op->sc); cudaFree(op->dot_dev); cudaFree(op->bad);
  cudaFree(op->red.partials); cudaFree(op->red.ticket);
  cudaFreeHost(op->sc_host); cudaFreeHost(op->dot_host);
  delete op;
}

static int op_common_alloc(fem_op_s* op) {
  FEM_TRY(dalloc(&op->sc, 1));
  FEM_TRY(dalloc(&op->dot_dev, 1));
  FEM_TRY(dalloc(&op->bad, 1));
  FEM_TRY(dalloc(&op->red.partials, 2 * kMaxCtas));  // (two sums: last_block_reduce2)
  FEM_TRY(dalloc(&op->red.ticket, 1));
  op->red.capacity = kMaxCtas;
  if (cudaMallocHost(&op->sc_host, sizeof(CgScalars)) != cudaSuccess ||
      cudaMallocHost(&op->dot_host, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    return fail(FEM_ENOMEM, "pinned host allocation failed");
  }
  if (cudaMemset(op->red.ticket, 0, sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(op->sc, 0, sizeof(CgScalars)) != cudaSuccess ||
      cudaMemset(op->dot_dev, 0, sizeof(double)) != cudaSuccess)  // (also the peer-halo sync allreduce)
    return fail(FEM_ECUDA, "cudaMemset failed");
  return FEM_OK;
}

// operator on a general hexahedral mesh: dense CG vectors (no padded layout, no tensor maps);
// CG runs the unfused iteration (apply + update + p-update)
static int op_create_hex(fem_op_s* op, fem_op_t* out) {
  const fem_mesh_s* m = op->mesh;
  op->plane_dofs = m->hx_nodes * op->comps;
  op->nloc_planes = 1;
  op->n_local = op->n_global = op->plane_dofs;
  op->pl_lead = 0;
  op->pl_rp = op->pl_pp = op->n_local;
  op->pl_off = 0;
  op->pl_n = op->n_local;
  op->tm_ok = false;
  int st = FEM_OK;
  for (double** v : {&op->x_pl, &op->r_pl, &op->p_pl, &op->q_pl})
    if (st == FEM_OK) st = dalloc(v, op->pl_n);
  if (st == FEM_OK) st = op_common_alloc(op);
  if (st != FEM_OK) {
    op_free(op);
    return st;
  }
  *out = op;
  return FEM_OK;
}

int fem_op_create(fem_mesh_t mesh, int32_t kind, int32_t bc, fem_op_t* out) {
  if (!out) return fail(FEM_EINVAL, "out is NULL");
  *out = nullptr;
  if (!mesh) return fail(FEM_EINVAL, "mesh is NULL");
  if (kind < 0 || kind > 2) return fail(FEM_EINVAL, "unknown kind %d", kind);
  if (bc < 0 || bc > 1) return fail(FEM_EINVAL, "unknown bc %d", bc);
  FEM_TRY(set_device(mesh->device));
  auto* op = new (std::nothrow) fem_op_s();
  if (!op) return fail(FEM_ENOMEM, "host allocation failed");
  op->mesh = mesh;
  op->kind = kind;
  op->bc = bc;
  op->comps = kind == FEM_SCALAR_LAPLACE ? 1 : 3;
  if (mesh->hex) return op_create_hex(op, out);
  const Grid& g = mesh->g;
  op->plane_dofs = g.plane * op->comps;
  op->nloc_planes = g.k1 - g.k0;
  op->n_local = op->nloc_planes * op->plane_dofs;
  op->n_global = (g.nz + 1) * op->plane_dofs;
  // padded layout: even row pitch, lead so that the tensor origin node is 16-B aligned
  op->pl_rp = ((g.nx + 1) * op->comps + 1) & ~1LL;
  op->pl_pp = op->pl_rp * (g.ny + 1);
  // Laplace tensors span the whole box like elasticity's (mask in registers, identity rows from
  // the staged planes); FEM_LAP_INTERIOR=1 restores interior-only tensors (zero fill = mask)
  op->tm_interior = FEM_LAP_INTERIOR && bc && kind != FEM_ELASTICITY;
  op->pl_lead = op->tm_interior ? (op->comps & 1) : 0;  // tensor-origin node 16-B aligned
  op->pl_n = (op->pl_lead + (op->nloc_planes + 2) * op->pl_pp + 1) & ~1LL;
  op->pl_off = op->pl_lead + op->pl_pp;
  int st = FEM_OK;
#define OP_TRY(x)                 \
  do {                            \
    st = (x);                     \
    if (st != FEM_OK) {           \
      op_free(op);                \
      return st;                  \
    }                             \
  } while (0)
  OP_TRY(dalloc(&op->x_pl, op->pl_n));
  OP_TRY(dalloc(&op->r_pl, op->pl_n));
  OP_TRY(dalloc(&op->p_pl, op->pl_n));
  OP_TRY(dalloc(&op->q_pl, op->pl_n));
  OP_TRY(dalloc(&op->p2_pl, op->pl_n));
  // (+ one row and two box widths: the row-pair tensor view of a ghost plane reads that far)
  OP_TRY(dalloc(&op->ghost_lo, op->plane_dofs + (g.nx + 1) * op->comps + 2 * 128));
  OP_TRY(dalloc(&op->ghost_hi, op->plane_dofs + (g.nx + 1) * op->comps + 2 * 128));
  OP_TRY(dalloc(&op->sc, 1));
  OP_TRY(dalloc(&op->dot_dev, 1));
  OP_TRY(dalloc(&op->bad, 1));
  OP_TRY(dalloc(&op->red.partials, 2 * kMaxCtas));
  OP_TRY(dalloc(&op->red.ticket, 1));
  op->red.capacity = kMaxCtas;
  if (cudaMallocHost(&op->sc_host, sizeof(CgScalars)) != cudaSuccess ||
      cudaMallocHost(&op->dot_host, sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    op_free(op);
    return fail(FEM_ENOMEM, "pinned host allocation failed");
  }
  if (cudaMemset(op->red.ticket, 0, sizeof(unsigned int)) != cudaSuccess ||
      cudaMemset(op->sc, 0, sizeof(CgScalars)) != cudaSuccess ||
      cudaMemset(op->dot_dev, 0, sizeof(double)) != cudaSuccess ||  // (also the peer-halo sync allreduce)
      cudaMemset(op->x_pl, 0, sizeof(double) * op->pl_n) != cudaSuccess ||
      cudaMemset(op->r_pl, 0, sizeof(double) * op->pl_n) != cudaSuccess ||
      cudaMemset(op->p_pl, 0, sizeof(double) * op->pl_n) != cudaSuccess ||
      cudaMemset(op->q_pl, 0, sizeof(double) * op->pl_n) != cudaSuccess ||
      cudaMemset(op->p2_pl, 0, sizeof(double) * op->pl_n) != cudaSuccess) {
    op_free(op);
    return fail(FEM_ECUDA, "cudaMemset failed");
  }
  OP_TRY(ensure_unit_matrices(mesh->device));
  OP_TRY(make_pl_maps(op));
#undef OP_TRY
  *out = op;
  return FEM_OK;
}

int fem_op_ndof(fem_op_t op, int64_t* nl, int64_t* ng) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (nl) *nl = op->n_local;
  if (ng) *ng = op->n_global;
  return FEM_OK;
}

static int set_material_hex(fem_op_s* op, const double* lam, const double* mu, int64_t layer_begin,
                            int64_t n_layers) {
  if (layer_begin != 0 || n_layers != 1)
    return fail(FEM_EINVAL, "general hex mesh: pass layer_begin 0, n_layers 1 (arrays of n_cells values)");
  const int64_t cnt = op->mesh->hx_ncells;
  if (!op->lm) FEM_TRY(dalloc(&op->lm, cnt));
  const cudaMemcpyKind kl = is_device_ptr(lam) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind km = is_device_ptr(mu) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUDA_TRY(cudaMemcpy2D(op->lm, 16, lam, 8, 8, cnt, kl));
  CUDA_TRY(cudaMemcpy2D(reinterpret_cast<double*>(op->lm) + 1, 16, mu, 8, 8, cnt, km));
  CUDA_TRY(cudaMemset(op->bad, 0, sizeof(unsigned long long)));
  CUDA_TRY(launch_check_material(op->lm, cnt, op->bad, 0, op->mesh->sm_count));
  unsigned long long bad = 0;
  CUDA_TRY(cudaMemcpy(&bad, op->bad, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad) {
    op->has_mat = false;
    return fail(FEM_EMATERIAL, "%llu cells violate mu > 0, lambda + 2 mu / 3 >= 0 (S:249)", bad);
  }
  op->has_mat = true;
  op->cg_active = false;
  return FEM_OK;
}

int fem_set_material(fem_op_t op, const double* lam, const double* mu, int64_t layer_begin,
                     int64_t n_layers) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (op->kind != FEM_ELASTICITY) return fail(FEM_EINVAL, "material given to a non-elastic operator");
  FEM_TRY(check_vec(lam, "lambda"));
  FEM_TRY(check_vec(mu, "mu"));
  FEM_TRY(set_device(op->mesh->device));
  if (op->mesh->hex) return set_material_hex(op, lam, mu, layer_begin, n_layers);
  const Grid& g = op->mesh->g;
  const int64_t need0 = std::max<int64_t>(g.k0 - 1, 0);
  const int64_t need1 = std::min<int64_t>(g.k1 - 1, g.nz - 1);  // inclusive
  if (layer_begin < 0 || n_layers < 1 || layer_begin > need0 || layer_begin + n_layers - 1 < need1)
    return fail(FEM_EINVAL, "material layers [%lld, %lld) do not cover the needed [%lld, %lld]",
                (long long)layer_begin, (long long)(layer_begin + n_layers), (long long)need0, (long long)need1);
  const int64_t nl = need1 - need0 + 1, nxy = g.nx * g.ny, cnt = nl * nxy;
  if (op->mat_layers != nl || !op->lm) {
    cudaFree(op->lm);
    op->lm = nullptr;
    op->mat_layers = 0;
    FEM_TRY(dalloc(&op->lm, cnt));
  }
  const size_t off = (size_t)(need0 - layer_begin) * nxy;
  const cudaMemcpyKind kl = is_device_ptr(lam) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const cudaMemcpyKind km = is_device_ptr(mu) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  // interleave (lambda, mu) per cell: one 16-B record ("cell constant C", 2 x 8 B)
  CUDA_TRY(cudaMemcpy2D(op->lm, 16, lam + off, 8, 8, cnt, kl));
  CUDA_TRY(cudaMemcpy2D(reinterpret_cast<double*>(op->lm) + 1, 16, mu + off, 8, 8, cnt, km));
  op->mat_layer0 = need0;
  op->mat_layers = nl;
  CUDA_TRY(cudaMemset(op->bad, 0, sizeof(unsigned long long)));
  CUDA_TRY(launch_check_material(op->lm, cnt, op->bad, 0, op->mesh->sm_count));
  unsigned long long bad = 0;
  CUDA_TRY(cudaMemcpy(&bad, op->bad, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad) {
    op->has_mat = false;
    return fail(FEM_EMATERIAL, "%llu cells violate mu > 0, lambda + 2 mu / 3 >= 0 (S:249)", bad);
  }
  FEM_TRY(make_mat_map(op));
  op->has_mat = true;
  op->cg_active = false;
  if (op->use_pa) FEM_TRY(pa_setup(op, true));  // D_q folds the material in
  return FEM_OK;
}

int fem_apply_ghost(fem_op_t op, const double* x, const double* glo, const double* ghi, double* y,
                    void* stream) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(check_vec(x, "x"));
  FEM_TRY(check_vec(y, "y"));
  if ((const void*)x == (const void*)y) return fail(FEM_EINVAL, "x and y alias");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  if (op->mesh->hex) return fail(FEM_EUNSUPPORTED, "fem_apply_ghost: general hex meshes are single-GPU");
  const Grid& g = op->mesh->g;
  if ((g.k0 > 0 && !glo) || (g.k1 <= g.nz && !ghi))
    return fail(FEM_EINVAL, "a ghost plane inside the box is NULL");
  if (!is_device_ptr(x) || !is_device_ptr(y) || (glo && !is_device_ptr(glo)) || (ghi && !is_device_ptr(ghi)))
    return fail(FEM_EINVAL, "fem_apply_ghost needs device pointers");
  FEM_TRY(set_device(op->mesh->device));
  PlaneSrc src = dense_src(op, x, g.k0 > 0 ? glo : nullptr, g.k1 <= g.nz ? ghi : nullptr);
  return launch_apply(op, src, dense_out(op, y), nullptr, 0, (cudaStream_t)stream);
}

int fem_apply_ghost_padded(fem_op_t op, const double* x, const double* glo, const double* ghi, double* y,
                           void* stream) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(check_vec(x, "x"));
  FEM_TRY(check_vec(y, "y"));
  if ((const void*)x == (const void*)y) return fail(FEM_EINVAL, "x and y alias");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  if (op->mesh->hex) return fail(FEM_EUNSUPPORTED, "fem_apply_ghost_padded: general hex meshes are single-GPU");
  const Grid& g = op->mesh->g;
  if (!op->peer_on && ((g.k0 > 0 && !glo) || (g.k1 <= g.nz && !ghi)))
    return fail(FEM_EINVAL, "a ghost plane inside the box is NULL");
  if (!is_device_ptr(x) || !is_device_ptr(y) || (glo && !is_device_ptr(glo)) || (ghi && !is_device_ptr(ghi)))
    return fail(FEM_EINVAL, "fem_apply_ghost_padded needs device pointers");
  FEM_TRY(set_device(op->mesh->device));
  cudaStream_t s = (cudaStream_t)stream;
  op->cg_active = false;  // x_pl / q_pl are the CG workspace
  FEM_TRY(pack(op, x, op->x_pl, 1, s));
  const fem_mesh_s* m = op->mesh;
  auto ghost = [&](const double* src, double* dst) -> int {
    cudaError_t e = launch_pack(src, dst, op->pl_rp, op->pl_pp, 1, g.nx + 1, g.ny + 1, op->comps, 1, s, m->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "ghost pack: %s", cudaGetErrorString(e));
    return FEM_OK;
  };
  if (!op->peer_on) {
    if (m->rank > 0 && glo) FEM_TRY(ghost(glo, op->x_pl + op->pl_lead));
    if (m->rank < m->nranks - 1 && ghi) FEM_TRY(ghost(ghi, op->x_pl + op->pl_lead + (op->nloc_planes + 1) * op->pl_pp));
  }
  FEM_TRY(launch_apply(op, pl_src(op, op->x_pl), pl_out(op, op->q_pl), op->tm_ok ? &op->tm_x : nullptr, 0, s,
                       op->x_pl));
  return pack(op, y, op->q_pl, 0, s);
}

int fem_op_link_peers(fem_op_t op, fem_op_t lo, fem_op_t hi) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (!op->tm_ok) return fail(FEM_EUNSUPPORTED, "peer halo needs the TMA (padded) path");
  const Grid& g = op->mesh->g;
  for (fem_op_s* nb : {lo, hi}) {
    if (!nb) continue;
    const Grid& h = nb->mesh->g;
    if (nb->kind != op->kind || nb->bc != op->bc || h.nx != g.nx || h.ny != g.ny || h.nz != g.nz ||
        nb->mesh->device != op->mesh->device || !nb->tm_ok)
      return fail(FEM_EINVAL, "peer operator does not match (kind, bc, mesh, device)");
  }
  if ((lo && lo->mesh->g.k1 != g.k0) || (hi && hi->mesh->g.k0 != g.k1))
    return fail(FEM_EINVAL, "peer slabs are not the neighbours of this slab");
  if ((g.k0 > 0) != (lo != nullptr) || (g.k1 <= g.nz) != (hi != nullptr))
    return fail(FEM_EINVAL, "a neighbour slab is missing (or given where there is none)");
  FEM_TRY(set_device(op->mesh->device));
  auto bufs = [](fem_op_s* o, double** b) { b[0] = o->x_pl; b[1] = o->p_pl; b[2] = o->r_pl; b[3] = o->p2_pl; };
  if (lo) { bufs(lo, op->nb_lo); op->nb_lo_nloc = lo->nloc_planes; }
  if (hi) bufs(hi, op->nb_hi);
  op->cg_active = false;
  return build_peer_maps(op);
}

// peer halo across processes: CUDA IPC handles of the padded vectors x, p, r, p2 + the slab's
// owned plane count (fem_op_peer_info), opened by the neighbours (fem_op_open_peers)
struct PeerInfo {
  cudaIpcMemHandle_t h[4];
  int64_t nloc;
};
static_assert(sizeof(PeerInfo) <= 320, "peer info exceeds the documented 320 bytes");

int fem_op_peer_info(fem_op_t op, void* info, int64_t bytes) {
  if (!op || !info) return fail(FEM_EINVAL, "op / info is NULL");
  if (bytes < (int64_t)sizeof(PeerInfo)) return fail(FEM_EINVAL, "info buffer must hold %zu bytes", sizeof(PeerInfo));
  if (!op->tm_ok) return fail(FEM_EUNSUPPORTED, "peer halo needs the TMA (padded) path");
  FEM_TRY(set_device(op->mesh->device));
  PeerInfo mine{};
  double* b[4] = {op->x_pl, op->p_pl, op->r_pl, op->p2_pl};
  for (int v = 0; v < 4; ++v) CUDA_TRY(cudaIpcGetMemHandle(&mine.h[v], b[v]));
  mine.nloc = op->nloc_planes;
  std::memcpy(info, &mine, sizeof(mine));
  return FEM_OK;
}

int fem_op_open_peers(fem_op_t op, const void* lo_info, const void* hi_info) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (!op->tm_ok) return fail(FEM_EUNSUPPORTED, "peer halo needs the TMA (padded) path");
  if (op->peer_on) return fail(FEM_ESTATE, "peers already linked");
  const Grid& g = op->mesh->g;
  if ((g.k0 > 0) != (lo_info != nullptr) || (g.k1 <= g.nz) != (hi_info != nullptr))
    return fail(FEM_EINVAL, "a neighbour's info is missing (or given where there is none)");
  FEM_TRY(set_device(op->mesh->device));
  PeerInfo nb[2]{};
  if (lo_info) std::memcpy(&nb[0], lo_info, sizeof(PeerInfo));
  if (hi_info) std::memcpy(&nb[1], hi_info, sizeof(PeerInfo));
  for (int v = 0; v < 4; ++v) {
    void* p = nullptr;
    if (lo_info) {
      CUDA_TRY(cudaIpcOpenMemHandle(&p, nb[0].h[v], cudaIpcMemLazyEnablePeerAccess));
      op->nb_lo[v] = static_cast<double*>(p);
    }
    if (hi_info) {
      CUDA_TRY(cudaIpcOpenMemHandle(&p, nb[1].h[v], cudaIpcMemLazyEnablePeerAccess));
      op->nb_hi[v] = static_cast<double*>(p);
    }
  }
  op->nb_lo_nloc = nb[0].nloc;
  op->peer_ipc = true;
  op->cg_active = false;
  return build_peer_maps(op);
}

// the same exchange over the operator's NCCL communicator (option "peer_halo")
static int peer_halo_ipc(fem_op_s* op) {
  fem_mesh_s* m = op->mesh;
  if (m->nranks == 1) return FEM_OK;
  if (m->comm && m->comm->loop) {  // same process and device: link the neighbours' operators
    int who[2], nw = 0;
    if (m->rank > 0) who[nw++] = m->rank - 1;
    if (m->rank < m->nranks - 1) who[nw++] = m->rank + 1;
    LoopRec rec[2];
    cudaEvent_t ev[2];
    FEM_TRY(loop_publish(m->comm, LoopRec{op, 0, 0}, 0, who, nw, rec, ev));
    fem_op_s* lo = nullptr;
    fem_op_s* hi = nullptr;
    for (int t = 0; t < nw; ++t)
      (who[t] < m->rank ? lo : hi) = static_cast<fem_op_s*>(const_cast<void*>(rec[t].p));
    const int st = fem_op_link_peers(op, lo, hi);
    // the neighbours hold this operator's pointer: nobody returns before everyone has linked
    FEM_TRY(loop_publish(m->comm, LoopRec{}, 0, who, nw, rec, ev));
    return st;
  }
  if (!m->comm || !m->comm->nccl) return fail(FEM_EUNSUPPORTED, "peer halo across processes needs an NCCL communicator");
  PeerInfo mine{};
  FEM_TRY(fem_op_peer_info(op, &mine, sizeof(mine)));
  char* d = nullptr;
  CUDA_TRY(cudaMalloc(&d, 3 * sizeof(PeerInfo)));
  CUDA_TRY(cudaMemcpy(d, &mine, sizeof(PeerInfo), cudaMemcpyHostToDevice));
  cudaStream_t s = 0;
  ncclComm_t c = m->comm->nccl;
  ncclResult_t r = ncclGroupStart();
  if (m->rank > 0) {
    if (r == ncclSuccess) r = ncclSend(d, sizeof(PeerInfo), ncclChar, m->rank - 1, c, s);
    if (r == ncclSuccess) r = ncclRecv(d + sizeof(PeerInfo), sizeof(PeerInfo), ncclChar, m->rank - 1, c, s);
  }
  if (m->rank < m->nranks - 1) {
    if (r == ncclSuccess) r = ncclSend(d, sizeof(PeerInfo), ncclChar, m->rank + 1, c, s);
    if (r == ncclSuccess) r = ncclRecv(d + 2 * sizeof(PeerInfo), sizeof(PeerInfo), ncclChar, m->rank + 1, c, s);
  }
  if (r == ncclSuccess) r = ncclGroupEnd();
  PeerInfo nb[2];
  cudaError_t e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemcpy(nb, d + sizeof(PeerInfo), 2 * sizeof(PeerInfo), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (r != ncclSuccess) return fail(FEM_ENCCL, "peer handle exchange: %s", ncclGetErrorString(r));
  if (e != cudaSuccess) return fail(FEM_ECUDA, "peer handle exchange: %s", cudaGetErrorString(e));
  return fem_op_open_peers(op, m->rank > 0 ? &nb[0] : nullptr, m->rank < m->nranks - 1 ? &nb[1] : nullptr);
}

int fem_apply(fem_op_t op, const double* x, double* y, void* stream) {
  NvtxRange nv("fem:apply");
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(need_comm(op));
  FEM_TRY(check_vec(x, "x"));
  FEM_TRY(check_vec(y, "y"));
  if ((const void*)x == (const void*)y) return fail(FEM_EINVAL, "x and y alias");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  FEM_TRY(set_device(op->mesh->device));
  cudaStream_t s = (cudaStream_t)stream;
  const PtrInfo xi = ptr_info(x);
  const bool xd = xi.device, yd = is_device_ptr(y);
  if (xd && yd) return apply_device(op, x, y, s, xi);
  FEM_TRY(ensure_stage(op));
  const size_t bytes = op->n_local * sizeof(double);
  const double* xs = x;
  if (!xd) {
    CUDA_TRY(cudaMemcpyAsync(op->stage_a, x, bytes, cudaMemcpyHostToDevice, s));
    xs = op->stage_a;
  }
  double* ys = yd ? y : op->stage_b;
  FEM_TRY(apply_device(op, xs, ys, s, xd ? xi : ptr_info(xs)));
  if (!yd) {
    CUDA_TRY(cudaMemcpyAsync(y, ys, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return FEM_OK;
}

int fem_dot(fem_op_t op, const double* a, const double* b, double* result, void* stream) {
  NvtxRange nv("fem:dot");
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(need_comm(op));
  FEM_TRY(check_vec(a, "a"));
  FEM_TRY(check_vec(b, "b"));
  if (!result) return fail(FEM_EINVAL, "result is NULL");
  FEM_TRY(set_device(op->mesh->device));
  cudaStream_t s = (cudaStream_t)stream;
  const bool ad = is_device_ptr(a), bd = is_device_ptr(b);
  const double *as = a, *bs = b;
  if (!ad || !bd) {
    FEM_TRY(ensure_stage(op));
    const size_t bytes = op->n_local * sizeof(double);
    if (!ad) { CUDA_TRY(cudaMemcpyAsync(op->stage_a, a, bytes, cudaMemcpyHostToDevice, s)); as = op->stage_a; }
    if (!bd) { CUDA_TRY(cudaMemcpyAsync(op->stage_b, b, bytes, cudaMemcpyHostToDevice, s)); bs = op->stage_b; }
  }
  return dot_device(op, as, bs, s, result);
}

// ---- CG -----------------------------------------------------------------------------------
// option time_apply: CUDA events around every apply launch of the CG iterations (read back by
// fem_apply_time).  Inside a stream capture they become event-record nodes of the graph
// (cudaEventRecordExternal), so the graph-replayed iteration is timed as it runs.
static int ensure_events(fem_op_s* op, size_t n) {
  while (op->ev.size() < n) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    op->ev.push_back(e);
  }
  return FEM_OK;
}
static int apply_event(fem_op_s* op, int end, cudaStream_t s) {
  if (!end) FEM_TRY(ensure_events(op, op->ev_used + 2));
  cudaEvent_t e = op->ev[op->ev_used + end];
  CUDA_TRY(cudaEventRecordWithFlags(e, s, op->ev_capture ? cudaEventRecordExternal : cudaEventRecordDefault));
  if (end) op->ev_used += 2;
  return FEM_OK;
}

static void drop_graphs(fem_op_s* op);
// deferred x update (option "x_defer"): fused Hestenes-Stiefel CG on the box.  Returns the group
// length m (1: x += alpha p every iteration).  The peer halo maps the neighbours' p and p2 only,
// so with it m is at most 2.
// which CG iteration runs (iteration()): the fused Hestenes-Stiefel one, the single-reduction
// one, or the unfused one (partial assembly, general hexes, degenerate boxes)
static int iter_kind(const fem_op_s* op) {
  if (op->use_pa || !op->tm_ok) return 2;
  return op->cg_variant == 1 ? 1 : 0;
}
static int x_defer_m(const fem_op_s* op) {
  if (op->x_defer <= 1) return 1;
  // (the fused Hestenes-Stiefel apply reads p_old through the peer halo, which maps the
  // neighbours' p and p2 only; the other iterations' applies do not read old p vectors)
  return std::min((op->peer_on && iter_kind(op) == 0) ? 2 : op->x_defer, op->x_defer_cap);
}
// the p buffers of the deferral group: iteration phase j writes p into buf[j % m] and reads p_old
// from buf[(j - 1) % m]; buf[m - 1] is p_pl, the buffer cg_begin initialises (so the first
// iteration's p_old, multiplied by beta = 0, is finite)
// Single-reduction CG: p2_pl holds s, so its ring is pex[0 .. m-2] + p_pl (m = 1: p_pl alone).
// Unfused iteration: p_pl (cg_begin's p0), p2_pl, pex[0 .. m-3] (m = 1: p_pl alone, in place).
static void p_ring(fem_op_s* op, int m, double** buf, const CUtensorMap** maps) {
  if (iter_kind(op) == 2) {
    buf[0] = op->p_pl; maps[0] = &op->tm_p;
    if (m >= 2) { buf[1] = op->p2_pl; maps[1] = &op->tm_p2; }
    for (int i = 2; i < m; ++i) { buf[i] = op->pex[i - 2]; maps[i] = &op->tm_pex[i - 2]; }
    return;
  }
  if (iter_kind(op) == 1) {
    for (int i = 0; i < m - 1; ++i) { buf[i] = op->pex[i]; maps[i] = &op->tm_pex[i]; }
    buf[m - 1] = op->p_pl; maps[m - 1] = &op->tm_p;
    return;
  }
  const int g = m < 2 ? 2 : m;  // (m = 1 keeps the ping-pong pair)
  buf[0] = op->p2_pl; maps[0] = &op->tm_p2;
  for (int i = 1; i < g - 1; ++i) { buf[i] = op->pex[i - 1]; maps[i] = &op->tm_pex[i - 1]; }
  buf[g - 1] = op->p_pl; maps[g - 1] = &op->tm_p;
}
// (out of device memory for m - 2 more p vectors: the group length drops to what fits -- 4, then
// 2, which needs none -- and stays capped for the operator's lifetime)
static int ensure_p_ring(fem_op_s* op) {
  bool grew = false;
  if (iter_kind(op) == 2 && x_defer_m(op) >= 2 && !op->p2_pl) {  // (general hexes do not allocate it)
    if (cudaMalloc(&op->p2_pl, sizeof(double) * op->pl_n) != cudaSuccess) {
      cudaGetLastError();
      op->p2_pl = nullptr;
      op->x_defer_cap = 1;
      return FEM_OK;
    }
    CUDA_TRY(cudaMemset(op->p2_pl, 0, sizeof(double) * op->pl_n));
    grew = true;
  }
  for (int e = 0; e < x_defer_m(op) - (iter_kind(op) == 1 ? 1 : 2); ++e) {
    if (op->pex[e]) continue;
    if (cudaMalloc(&op->pex[e], sizeof(double) * op->pl_n) != cudaSuccess) {
      cudaGetLastError();
      op->pex[e] = nullptr;
      // extra buffers 0 .. e-1 exist: a ring of e + 2 (single-reduction CG: e + 1) >= m fits
      const int fit = e + (iter_kind(op) == 1 ? 1 : 2);
      op->x_defer_cap = fit >= 4 ? 4 : (fit >= 2 ? 2 : 1);
      e = -1;  // re-check with the cap
      continue;
    }
    CUDA_TRY(cudaMemset(op->pex[e], 0, sizeof(double) * op->pl_n));
    grew = true;
  }
  if (!grew) return FEM_OK;
  drop_graphs(op);
  return op->mesh->hex ? FEM_OK : make_pl_maps(op);
}

static int cg_iteration_body(fem_op_s* op, int phase, cudaStream_t s, bool timed) {
  fem_mesh_s* m = op->mesh;
  const int64_t n = pl_count(op);
  // deferred x update (§5.3): p_k in ring buffer k mod m, p_{k+1} written to the next one
  const int xm = x_defer_m(op);
  double* pb[8];
  const CUtensorMap* pmap[8];
  p_ring(op, xm, pb, pmap);
  const int j = phase % xm;
  double* pc = pb[j];
  double* pn = pb[(j + 1) % xm];
  if (timed) FEM_TRY(apply_event(op, 0, s));
  FEM_TRY(apply_pl(op, pc, pmap[j], 1, s));  // q = A p, pq (halo inside when P > 1)
  if (timed) FEM_TRY(apply_event(op, 1, s));
  FEM_TRY(allreduce1(op, &op->sc->pq, s));
  const double* po[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int nold = 0;
  if (xm > 1) {
    if (j < xm - 1) {
      nold = -1;
    } else {
      nold = xm - 1;
      for (int k = 0; k < nold; ++k) po[k] = pl_owned(op, pb[k]);
    }
  }
  cudaError_t e = launch_cg_update(pl_owned(op, op->x_pl), pl_owned(op, op->r_pl), pl_owned(op, pc),
                                   pl_owned(op, op->q_pl), n, op->sc, op->red, s, m->sm_count, nold, po, j);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "update launch: %s", cudaGetErrorString(e));
  FEM_TRY(allreduce1(op, &op->sc->rr_new, s));
  e = launch_cg_pupdate(pl_owned(op, op->r_pl), pl_owned(op, pc), pl_owned(op, pn), n, op->sc, op->red, s,
                        m->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "pupdate launch: %s", cudaGetErrorString(e));
  return FEM_OK;
}

// fused CG iteration (TMA path): p = r + beta p_old formed inside the apply (NEXT #1 of the
// survey, 88 -> 80 B/DOF for Laplace); parity selects the p ping-pong buffers.

static int cg_fused_body(fem_op_s* op, int phase, cudaStream_t s, bool timed) {
  fem_mesh_s* m = op->mesh;
  const int xm = x_defer_m(op);
  double* pb[8];
  const CUtensorMap* pmap[8];
  p_ring(op, xm, pb, pmap);
  const int gm = xm < 2 ? 2 : xm;  // ring length (m = 1 keeps the ping-pong pair)
  const int jn = phase % gm, jo = (phase + gm - 1) % gm;
  double* pold = pb[jo];
  double* pnew = pb[jn];
  static thread_local PeerMaps pm;
  const bool peer = fill_peer(op, op->r_pl, pold, &pm);
  if (timed) FEM_TRY(apply_event(op, 0, s));
  ApplyMaps maps{&op->tm_r, op->tm_i0, op->tm_j0, op->tm_k0, &op->tm_mat, op->mat_layer0,
                 pmap[jo], pl_owned(op, pold), pl_owned(op, pnew),
                 op->tm_interior ? 1 : 0, op->quad, peer ? &pm : nullptr};
  // the two dots per option "dot_mode" (Reduce::dot_mode; the paper's dot ablation)
  Reduce rd = op->red;
  rd.dot_mode = op->dot_mode;
  if (m->nranks > 1 && !peer) {  // halo of r and p_old overlapped with the interior planes
    auto halos = [&](cudaStream_t hs) -> int {
      double* const vs[2] = {op->r_pl, pold};
      for (double* v : vs)
        FEM_TRY(halo_pitch(op, pl_owned(op, v), v + op->pl_lead, v + op->pl_lead + (op->nloc_planes + 1) * op->pl_pp,
                           op->pl_pp, hs));
      return FEM_OK;
    };
    FEM_TRY(apply_split(op, s, pl_src(op, op->r_pl), pl_out(op, op->q_pl), maps, 2, rd, halos));
  } else {
    FEM_TRY(launch_maps(op, m->g, pl_src(op, op->r_pl), pl_out(op, op->q_pl), maps, 2, rd, s));
  }
  if (timed) FEM_TRY(apply_event(op, 1, s));
  cudaError_t e;
  const int64_t n = pl_count(op);
  if (op->dot_mode == 1) {  // p.q by a separate kernel re-reading p and q
    e = launch_cg_dot(pl_owned(op, pnew), pl_owned(op, op->q_pl), n, 0, op->sc, op->red, s, m->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "dot launch: %s", cudaGetErrorString(e));
  }
  FEM_TRY(allreduce1(op, &op->sc->pq, s));
  // deferred x update: phases 0 .. m-2 of a group leave alpha p pending (p stays in its ring
  // buffer until the group's last phase), phase m-1 adds the group's m updates in order
  const double* po[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int nold = 0;
  if (xm > 1) {
    const int j = phase % xm;
    if (j < xm - 1) {
      nold = -1;
    } else {
      nold = xm - 1;
      for (int k = 0; k < nold; ++k) po[k] = pl_owned(op, pb[k]);
    }
  }
  e = launch_cg_update_fused(pl_owned(op, op->x_pl), pl_owned(op, op->r_pl), pl_owned(op, pnew),
                             pl_owned(op, op->q_pl), n, op->sc, rd, s, m->sm_count, nold, po, phase % xm);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "update launch: %s", cudaGetErrorString(e));
  if (op->dot_mode == 1) {  // r.r by a separate kernel re-reading r
    e = launch_cg_dot(pl_owned(op, op->r_pl), pl_owned(op, op->r_pl), n, 1, op->sc, op->red, s, m->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "dot launch: %s", cudaGetErrorString(e));
  }
  FEM_TRY(allreduce1(op, &op->sc->rr_new, s));
  return FEM_OK;
}

// Chronopoulos-Gear iteration (option "cg_variant" = 1; TMA path): w = A r with delta = w.r and
// gamma = r.r reduced together (one allreduce of 2 values), then one update kernel
static int cg_cgcg_body(fem_op_s* op, int phase, cudaStream_t s, bool timed) {
  fem_mesh_s* m = op->mesh;
  if (timed) FEM_TRY(apply_event(op, 0, s));
  FEM_TRY(apply_pl(op, op->r_pl, &op->tm_r, 3, s));  // w (q_pl) = A r; pq = w.r, rr_new = r.r
  if (timed) FEM_TRY(apply_event(op, 1, s));
  FEM_TRY(allreduce1(op, &op->sc->pq, s, 2));  // pq and rr_new are adjacent in CgScalars
  // deferred x update (§5.3a): p_k into ring buffer k mod m, x once per group of m iterations
  const int xm = x_defer_m(op);
  double* pb[8];
  const CUtensorMap* pmap[8];
  p_ring(op, xm, pb, pmap);
  const int j = phase % xm;
  const double* po[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int nold = 0;
  if (xm > 1) {
    if (j < xm - 1) {
      nold = -1;
    } else {
      nold = xm - 1;
      for (int k = 0; k < nold; ++k) po[k] = pl_owned(op, pb[k]);
    }
  }
  cudaError_t e = launch_cg_cgcg_update(pl_owned(op, op->x_pl), pl_owned(op, op->r_pl),
                                        pl_owned(op, pb[(j + xm - 1) % xm]), pl_owned(op, pb[j]),
                                        pl_owned(op, op->p2_pl), pl_owned(op, op->q_pl), pl_count(op), op->sc,
                                        op->red, s, m->sm_count, nold, po, j);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "cgcg update launch: %s", cudaGetErrorString(e));
  // peer halo: the next apply reads the neighbours' r -- wait for their updates
  if (op->peer_on && m->nranks > 1) FEM_TRY(allreduce1(op, op->dot_dev, s));
  return FEM_OK;
}

static int iteration(fem_op_s* op, int parity, cudaStream_t s, bool timed) {
  switch (iter_kind(op)) {
    case 0: return cg_fused_body(op, parity, s, timed);
    case 1: return cg_cgcg_body(op, parity, s, timed);
    default: return cg_iteration_body(op, parity, s, timed);  // partial assembly, hexes, degenerate
  }
}

static int capture(fem_op_s* op, int iters, int parity, cudaStream_t s, cudaGraphExec_t* out,
                   bool timed = false, int64_t* launches = nullptr) {
  // capture on a private stream (legacy stream 0 cannot be captured)
  if (timed) {
    op->ev_used = 0;
    FEM_TRY(ensure_events(op, 2 * (size_t)iters));
  }
  cudaStream_t cs;
  CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const int64_t before = g_launches.load();
  int st = FEM_OK;
  op->ev_capture = timed;
  for (int t = 0; t < iters && st == FEM_OK; ++t) st = iteration(op, (parity + t) & 7, cs, timed);
  op->ev_capture = false;
  if (timed) op->ev_used = 0;  // set at each replay
  if (launches) *launches = g_launches.load() - before;
  g_launches.store(before);  // captured launches are counted at replay
  cudaGraph_t graph;
  cudaError_t e = cudaStreamEndCapture(cs, &graph);
  if (st != FEM_OK) {
    if (e == cudaSuccess) cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    return st;
  }
  if (e != cudaSuccess) {
    cudaStreamDestroy(cs);
    return fail(FEM_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(e));
  }
  e = cudaGraphInstantiate(out, graph, 0);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e));
  (void)s;
  return FEM_OK;
}

// CG on the padded copies: x_pl = x0; r = b - A x0; p = r (the caller's x is written at the end)
static int cg_begin_dev(fem_op_s* op, const double* b, double* x, double tol, int maxit, cudaStream_t s) {
  fem_mesh_s* m = op->mesh;
  FEM_TRY(ensure_p_ring(op));  // (x_defer = m >= 4: m - 2 more p buffers on first use)
  FEM_TRY(pack(op, x, op->x_pl, 1, s));
  // peer halo: the neighbours must have packed their x0 before this rank's apply reads it
  if (op->peer_on && m->nranks > 1) FEM_TRY(allreduce1(op, op->dot_dev, s));
  FEM_TRY(apply_pl(op, op->x_pl, &op->tm_x, 0, s));  // q = A x0
  FEM_TRY(pack(op, b, op->r_pl, 1, s));              // r = b
  cudaError_t e = launch_cg_init(pl_owned(op, op->r_pl), pl_owned(op, op->q_pl), pl_owned(op, op->r_pl),
                                 pl_owned(op, op->p_pl), pl_count(op), op->sc, op->red, s, m->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "init launch: %s", cudaGetErrorString(e));
  FEM_TRY(allreduce1(op, &op->sc->rr_new, s));
  e = launch_cg_finish_init(op->sc, tol, maxit, s);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "init launch: %s", cudaGetErrorString(e));
  op->cg_parity = 0;
  op->cg_b = b;
  op->cg_x = x;
  op->cg_active = true;
  return FEM_OK;
}

static int cg_iterate_dev(fem_op_s* op, int iters, cudaStream_t s) {
  // loopback ranks rendezvous on the host inside every collective: not capturable, run eagerly
  const bool loop = op->mesh->comm && op->mesh->comm->loop && op->mesh->nranks > 1;
  if (op->time_apply && op->use_graph && !loop && iters > 0) {
    // timed AND graph-replayed: one graph of exactly `iters` iterations whose event-record nodes
    // bracket every apply (the events of the last replay are read by fem_apply_time)
    cudaGraphExec_t ge = nullptr;
    for (const auto& t : op->graphT)
      if (t.iters == iters && t.parity == op->cg_parity) ge = t.exec;
    if (!ge) {
      if (op->graphT.size() >= 4) {
        cudaGraphExecDestroy(op->graphT.front().exec);
        op->graphT.erase(op->graphT.begin());
      }
      int64_t nl = 0;
      FEM_TRY(capture(op, iters, op->cg_parity, s, &ge, true, &nl));
      op->graphT.push_back({ge, iters, op->cg_parity, nl});
    }
    for (const auto& t : op->graphT)
      if (t.exec == ge) add_launches(t.launches);
    CUDA_TRY(cudaGraphLaunch(ge, s));
    op->ev_used = 2 * (size_t)iters;
    op->cg_parity = (op->cg_parity + iters) & 7;
    return FEM_OK;
  }
  if (op->time_apply || !op->use_graph || loop) {
    for (int t = 0; t < iters; ++t) {
      FEM_TRY(iteration(op, op->cg_parity, s, op->time_apply != 0));
      op->cg_parity = (op->cg_parity + 1) & 7;
    }
    return FEM_OK;
  }
  // plain graphs of exactly k iterations (k <= 64; longer runs replay the 64-iteration graph),
  // cached per (k, parity): a K-step call is one or a few graph launches, so small problems pay
  // one launch latency per call instead of one per 8 iterations
  constexpr int KMAX = 64;
  auto launch_k = [&](int k) -> int {
    cudaGraphExec_t ge = nullptr;
    for (const auto& t : op->graphK)
      if (t.iters == k && t.parity == op->cg_parity) ge = t.exec;
    if (!ge) {
      if (op->graphK.size() >= 6) {
        cudaGraphExecDestroy(op->graphK.front().exec);
        op->graphK.erase(op->graphK.begin());
      }
      int64_t nl = 0;
      FEM_TRY(capture(op, k, op->cg_parity, s, &ge, false, &nl));
      op->graphK.push_back({ge, k, op->cg_parity, nl});
    }
    for (const auto& t : op->graphK)
      if (t.exec == ge) add_launches(t.launches);
    CUDA_TRY(cudaGraphLaunch(ge, s));
    op->cg_parity = (op->cg_parity + k) & 7;
    return FEM_OK;
  };
  int left = iters;
  while (left > 0) {
    const int k = std::min(left, KMAX);
    FEM_TRY(launch_k(k));
    left -= k;
  }
  return FEM_OK;
}

static int cg_end_dev(fem_op_s* op, fem_cg_info* info, cudaStream_t s) {
  const int xm = x_defer_m(op);
  if (xm > 1) {  // the pending updates of an unfinished group, if the solve ended inside one
    double* pb[8];
    const CUtensorMap* pmap[8];
    p_ring(op, xm, pb, pmap);
    const double* pend[7];
    for (int k = 0; k < 7; ++k) pend[k] = pl_owned(op, pb[k < xm - 1 ? k : 0]);
    const cudaError_t e = launch_cg_xdefer_flush(pl_owned(op, op->x_pl), pend, pl_count(op), op->sc, s,
                                                 op->mesh->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "x update launch: %s", cudaGetErrorString(e));
  }
  // peer halo: the true-residual apply below reads the neighbours' x -- wait for their last x update
  if (op->peer_on && op->mesh->nranks > 1 && xm > 1)
    FEM_TRY(allreduce1(op, op->dot_dev, s));
  FEM_TRY(pack(op, op->cg_x, op->x_pl, 0, s));  // x = x_pl (caller layout)
  CUDA_TRY(cudaMemcpyAsync(op->sc_host, op->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  const CgScalars h = *op->sc_host;
  int status = (h.done == 2) ? FEM_EBREAKDOWN : FEM_OK;
  if (info) {
    info->iterations = h.it;
    info->converged = (h.done == 1) || (h.rr_new == 0.0) || (h.rr_new <= h.stop_rr);
    info->breakdown_iter = h.breakdown_iter;
    info->status = status;
    info->r0_norm = std::sqrt(h.rr0);
    // rr_new is the last residual the recurrence computed (fused CG: the update's r.r; unfused:
    // equal to rr; single-reduction CG: gamma = r.r of the iterate the last update started from)
    info->r_norm = std::sqrt(h.rr_new);
    // true residual ||b - A x||
    FEM_TRY(apply_pl(op, op->x_pl, &op->tm_x, 0, s));
    FEM_TRY(pack(op, op->cg_b, op->r_pl, 1, s));
    double* r = pl_owned(op, op->r_pl);
    cudaError_t e = launch_sub(r, pl_owned(op, op->q_pl), r, pl_count(op), s, op->mesh->sm_count);
    if (e != cudaSuccess) return fail(FEM_ECUDA, "sub launch: %s", cudaGetErrorString(e));
    double tr = 0.0;
    FEM_TRY(dot_device(op, r, r, s, &tr, pl_count(op)));
    info->true_r_norm = std::sqrt(tr);
    op->cg_active = false;  // r was overwritten
  }
  if (status == FEM_EBREAKDOWN) return fail(FEM_EBREAKDOWN, "CG breakdown at iteration %d (p.Ap <= 0 or non-finite)", h.breakdown_iter);
  return FEM_OK;
}

int fem_cg_begin(fem_op_t op, const double* b, double* x, double tol, int32_t maxit, void* stream) {
  NvtxRange nv("fem:cg_begin");
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(need_comm(op));
  FEM_TRY(check_vec(b, "b"));
  FEM_TRY(check_vec(x, "x"));
  if ((const void*)b == (const void*)x) return fail(FEM_EINVAL, "b and x alias");
  if (!(tol >= 0.0) || !std::isfinite(tol)) return fail(FEM_EINVAL, "tol must be finite and >= 0");
  if (maxit < 0) return fail(FEM_EINVAL, "maxit must be >= 0");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  if (!is_device_ptr(b) || !is_device_ptr(x)) return fail(FEM_EINVAL, "fem_cg_begin needs device pointers");
  FEM_TRY(set_device(op->mesh->device));
  return cg_begin_dev(op, b, x, tol, maxit, (cudaStream_t)stream);
}

int fem_cg_iterate(fem_op_t op, int32_t iters, void* stream) {
  NvtxRange nv("fem:cg_iterate");
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (!op->cg_active) return fail(FEM_ESTATE, "fem_cg_begin not called");
  if (iters < 0) return fail(FEM_EINVAL, "iters < 0");
  FEM_TRY(set_device(op->mesh->device));
  return cg_iterate_dev(op, iters, (cudaStream_t)stream);
}

int fem_cg_end(fem_op_t op, fem_cg_info* info, void* stream) {
  NvtxRange nv("fem:cg_end");
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  if (!op->cg_active) return fail(FEM_ESTATE, "fem_cg_begin not called");
  FEM_TRY(set_device(op->mesh->device));
  fem_cg_info tmp;
  return cg_end_dev(op, info ? info : &tmp, (cudaStream_t)stream);
}

int fem_cg_solve(fem_op_t op, const double* b, double* x, double tol, int32_t maxit,
                 fem_cg_info* info, void* stream) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(need_comm(op));
  FEM_TRY(check_vec(b, "b"));
  FEM_TRY(check_vec(x, "x"));
  if ((const void*)b == (const void*)x) return fail(FEM_EINVAL, "b and x alias");
  if (!(tol >= 0.0) || !std::isfinite(tol)) return fail(FEM_EINVAL, "tol must be finite and >= 0");
  if (maxit < 0) return fail(FEM_EINVAL, "maxit must be >= 0");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  FEM_TRY(set_device(op->mesh->device));
  cudaStream_t s = (cudaStream_t)stream;
  const bool bd = is_device_ptr(b), xd = is_device_ptr(x);
  const size_t bytes = op->n_local * sizeof(double);
  const double* bs = b;
  double* xs = x;
  if (!bd || !xd) FEM_TRY(ensure_stage(op));
  if (!bd) { CUDA_TRY(cudaMemcpyAsync(op->stage_b, b, bytes, cudaMemcpyHostToDevice, s)); bs = op->stage_b; }
  if (!xd) { CUDA_TRY(cudaMemcpyAsync(op->stage_a, x, bytes, cudaMemcpyHostToDevice, s)); xs = op->stage_a; }
  FEM_TRY(cg_begin_dev(op, bs, xs, tol, maxit, s));
  int done_it = 0;
  // tol == 0 runs exactly maxit iterations unless r.r == 0 / breakdown, which the kernels stop on
  // by themselves (done flag): no intermediate host polls needed
  const int chunk = tol == 0.0 ? std::max(1, maxit) : std::max(1, op->check_every);
  while (done_it < maxit) {
    const int n = std::min(chunk, maxit - done_it);
    FEM_TRY(cg_iterate_dev(op, n, s));
    done_it += n;
    CUDA_TRY(cudaMemcpyAsync(op->sc_host, op->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const CgScalars& h = *op->sc_host;  // rr_new is rank-global here (after its allreduce)
    if (h.done || h.rr_new == 0.0 || h.rr_new <= h.stop_rr) break;
  }
  fem_cg_info tmp;
  int st = cg_end_dev(op, info ? info : &tmp, s);
  if (!xd) {
    CUDA_TRY(cudaMemcpyAsync(x, xs, bytes, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
  }
  return st;
}

// captured CG graphs hold the kernels / options of their capture
static void drop_graphs(fem_op_s* op) {
  for (cudaGraphExec_t* g : {&op->graph1, &op->graphN, &op->graph1b})
    if (*g) {
      cudaGraphExecDestroy(*g);
      *g = nullptr;
    }
  for (const auto& t : op->graphT) cudaGraphExecDestroy(t.exec);
  op->graphT.clear();
  for (const auto& t : op->graphK) cudaGraphExecDestroy(t.exec);
  op->graphK.clear();
}


int fem_set_option(fem_op_t op, const char* key, int64_t value) {
  if (!op || !key) return fail(FEM_EINVAL, "op/key is NULL");
  if (!std::strcmp(key, "use_graph")) op->use_graph = value != 0;
  else if (!std::strcmp(key, "check_every")) {
    if (value < 1) return fail(FEM_EINVAL, "check_every must be >= 1");
    op->check_every = (int)value;
  } else if (!std::strcmp(key, "time_apply")) op->time_apply = value != 0;
  else if (!std::strcmp(key, "direct_tma")) op->direct_tm = value != 0;
  else if (!std::strcmp(key, "partial_assembly")) {
    if (!op->mesh->hex && (op->kind != FEM_ELASTICITY || op->mesh->nranks != 1))
      return fail(FEM_EUNSUPPORTED, "partial_assembly: general hex meshes, or the single-rank elasticity box operator");
    if (op->cg_active) return fail(FEM_ESTATE, "partial_assembly cannot change during a CG solve");
    FEM_TRY(set_device(op->mesh->device));
    op->use_pa = value != 0;
    if (!op->use_pa && !op->mesh->hex && op->pa) {  // release the 1,344 B/cell
      cudaFree(op->pa);
      op->pa = nullptr;
      op->pa_quad = -1;
    }
    FEM_TRY(pa_setup(op));
    // captured CG graphs hold the other kernel
    drop_graphs(op);
  } else if (!std::strcmp(key, "peer_halo")) {
    // collective over the slab ranks (every rank must set it): ghost planes read in the apply
    // kernels straight from the neighbours' memory (CUDA IPC over NVLink), no NCCL halo
    if (!value) return fail(FEM_EINVAL, "peer_halo cannot be switched off once on");
    if (!op->tm_ok) return fail(FEM_EUNSUPPORTED, "peer halo needs the TMA (padded) path");
    if (op->cg_active) return fail(FEM_ESTATE, "peer_halo cannot change during a CG solve");
    FEM_TRY(set_device(op->mesh->device));
    if (!op->peer_on) FEM_TRY(peer_halo_ipc(op));
    drop_graphs(op);
  } else if (!std::strcmp(key, "cg_variant")) {
    if (value != 0 && value != 1) return fail(FEM_EINVAL, "cg_variant must be 0 (fused CG) or 1 (Chronopoulos-Gear)");
    if (op->cg_active) return fail(FEM_ESTATE, "cg_variant cannot change during a CG solve");
    op->cg_variant = (int)value;
    drop_graphs(op);
  } else if (!std::strcmp(key, "trace")) {
    op->trace = value != 0;
  } else if (!std::strcmp(key, "x_defer")) {
    if (value != 1 && value != 2 && value != 4 && value != 8) return fail(FEM_EINVAL, "x_defer must be 1, 2, 4 or 8");
    if (op->cg_active) return fail(FEM_ESTATE, "x_defer cannot change during a CG solve");
    op->x_defer = (int)value;
    drop_graphs(op);
  } else if (!std::strcmp(key, "deterministic")) {
    if (!op->mesh->hex) return fail(FEM_EUNSUPPORTED, "deterministic: general hex meshes (the box kernels are atomic-free)");
    if (op->cg_active) return fail(FEM_ESTATE, "deterministic cannot change during a CG solve");
    FEM_TRY(set_device(op->mesh->device));
    fem_mesh_s* m = op->mesh;
    if (value && !m->hx_n2e) {
      FEM_TRY(dalloc(&m->hx_n2e_off, m->hx_nodes + 1));
      FEM_TRY(dalloc(&m->hx_n2e, 8 * m->hx_ncells));
      const cudaError_t e = launch_hex_node_csr(m->hx_cells, m->hx_ncells, m->hx_nodes, m->hx_n2e_off, m->hx_n2e,
                                                m->sm_count);
      if (e != cudaSuccess) {
        cudaFree(m->hx_n2e_off); cudaFree(m->hx_n2e);
        m->hx_n2e_off = nullptr; m->hx_n2e = nullptr;
        return fail(FEM_ECUDA, "node-to-cell map: %s", cudaGetErrorString(e));
      }
    }
    if (value && !op->hx_E) FEM_TRY(dalloc(&op->hx_E, 8 * op->comps * m->hx_ncells));
    if (!value && op->hx_E) {
      cudaFree(op->hx_E);
  cudaFree(op->last_plane);
      op->hx_E = nullptr;
    }
    op->det = value != 0;
    drop_graphs(op);
  } else if (!std::strcmp(key, "halo_overlap")) {
    op->overlap = value != 0;
    drop_graphs(op);
  } else if (!std::strcmp(key, "dot_mode")) {
    if (value < 0 || value > 2) return fail(FEM_EINVAL, "dot_mode must be 0 (fused epilogue), 1 (separate dot kernels) or 2 (atomic partials)");
    if (op->cg_active) return fail(FEM_ESTATE, "dot_mode cannot change during a CG solve");
    op->dot_mode = (int)value;
    drop_graphs(op);
  } else if (!std::strcmp(key, "quadrature")) {
    if (value != 0 && value != 1) return fail(FEM_EINVAL, "quadrature must be 0 (Gauss) or 1 (Gauss-Lobatto)");
    if (value == 1 && op->mesh->hex) {  // the Lobatto points are the nodes: det J > 0 there too
      FEM_TRY(set_device(op->mesh->device));
      unsigned long long* d_bad = nullptr;
      FEM_TRY(dalloc(&d_bad, 2));
      unsigned long long bad[2] = {0, 0};
      cudaError_t e = cudaMemset(d_bad, 0, sizeof(bad));
      if (e == cudaSuccess)
        e = launch_hex_check(op->mesh->hx_cells, op->mesh->hx_xyz, op->mesh->hx_ncells, op->mesh->hx_nodes, 1, d_bad,
                             0, op->mesh->sm_count);
      if (e == cudaSuccess) e = cudaMemcpy(bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost);
      cudaFree(d_bad);
      if (e != cudaSuccess) return fail(FEM_ECUDA, "mesh check: %s", cudaGetErrorString(e));
      if (bad[1]) return fail(FEM_EINVAL, "%llu cells have det J <= 0 at a node (Gauss-Lobatto point)", bad[1]);
    }
    op->quad = (int)value;
    FEM_TRY(set_device(op->mesh->device));
    FEM_TRY(pa_setup(op));
    drop_graphs(op);
  } else return fail(FEM_EINVAL, "unknown option '%s'", key);
  return FEM_OK;
}

int fem_get_option(fem_op_t op, const char* key, int64_t* value) {
  if (!op || !key || !value) return fail(FEM_EINVAL, "op/key/value is NULL");
  if (!std::strcmp(key, "fused_cg")) *value = (op->tm_ok && !op->use_pa) ? 1 : 0;
  else if (!std::strcmp(key, "tma")) *value = op->tm_ok ? 1 : 0;
  else if (!std::strcmp(key, "use_graph")) *value = op->use_graph;
  else if (!std::strcmp(key, "check_every")) *value = op->check_every;
  else if (!std::strcmp(key, "time_apply")) *value = op->time_apply;
  else if (!std::strcmp(key, "direct_tma")) *value = op->direct_tm;
  else if (!std::strcmp(key, "last_apply_path")) *value = op->last_path;
  else if (!std::strcmp(key, "partial_assembly")) *value = op->use_pa;
  else if (!std::strcmp(key, "quadrature")) *value = op->quad;
  else if (!std::strcmp(key, "cg_variant")) *value = (op->tm_ok && !op->use_pa && op->cg_variant == 1) ? 1 : 0;
  else if (!std::strcmp(key, "peer_halo")) *value = op->peer_on ? 1 : 0;
  else if (!std::strcmp(key, "dot_mode")) *value = op->dot_mode;
  else if (!std::strcmp(key, "halo_overlap")) *value = op->overlap;
  else if (!std::strcmp(key, "trace")) *value = op->trace;
  else if (!std::strcmp(key, "deterministic")) *value = op->mesh->hex ? op->det : 1;
  else if (!std::strcmp(key, "x_defer")) *value = x_defer_m(op);
  else if (!std::strncmp(key, "trace_", 6)) {
    // trace_{halo,interior,boundary,total}_ns of the last traced exchange apply (blocks on it)
    static const char* names[4] = {"trace_halo_ns", "trace_interior_ns", "trace_boundary_ns", "trace_total_ns"};
    static const int from[4] = {0, 0, 0, 0}, to[4] = {1, 2, 3, 3};
    int k = -1;
    for (int t = 0; t < 4; ++t)
      if (!std::strcmp(key, names[t])) k = t;
    if (k < 0) return fail(FEM_EINVAL, "unknown option '%s'", key);
    if (!op->tr_valid) return fail(FEM_ESTATE, "%s: no traced exchange apply yet (option trace, nranks > 1)", key);
    FEM_TRY(set_device(op->mesh->device));
    CUDA_TRY(cudaEventSynchronize(op->tr_ev[3]));
    CUDA_TRY(cudaEventSynchronize(op->tr_ev[1]));
    float ms = 0.f;
    if (k == 2) CUDA_TRY(cudaEventElapsedTime(&ms, op->tr_ev[2], op->tr_ev[3]));  // boundary: after interior
    else CUDA_TRY(cudaEventElapsedTime(&ms, op->tr_ev[from[k]], op->tr_ev[to[k]]));
    *value = (int64_t)(ms * 1e6);
  }
  else return fail(FEM_EINVAL, "unknown option '%s'", key);
  return FEM_OK;
}

int fem_apply_time(fem_op_t op, double* total_ms, int64_t* count) {
  if (!op) return fail(FEM_EINVAL, "op is NULL");
  FEM_TRY(set_device(op->mesh->device));
  double tot = 0.0;
  int64_t n = 0;
  if (op->ev_used) CUDA_TRY(cudaEventSynchronize(op->ev[op->ev_used - 1]));
  for (size_t t = 0; t + 1 < op->ev_used; t += 2) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, op->ev[t], op->ev[t + 1]));
    tot += ms;
    ++n;
  }
  op->ev_used = 0;
  if (total_ms) *total_ms = tot;
  if (count) *count = n;
  return FEM_OK;
}

void fem_op_destroy(fem_op_t op) { op_free(op); }

// ---- CSR ----------------------------------------------------------------------------------
int fem_csr_create(fem_op_t op, fem_csr_t* out) {
  if (!op || !out) return fail(FEM_EINVAL, "op/out is NULL");
  *out = nullptr;
  if (op->mesh->nranks != 1) return fail(FEM_EUNSUPPORTED, "CSR baseline is single-rank only");
  if (op->mesh->hex) return fail(FEM_EUNSUPPORTED, "CSR baseline is built for the box mesh only");
  if (op->kind == FEM_ELASTICITY && !op->has_mat) return fail(FEM_ESTATE, "material not set");
  FEM_TRY(set_device(op->mesh->device));
  const Grid& g = op->mesh->g;
  const int64_t nrows = op->n_global;
  if (nrows >= 2147483647LL) return fail(FEM_EOVERFLOW, "CSR column index exceeds int32");
  auto* c = new (std::nothrow) fem_csr_s();
  if (!c) return fail(FEM_ENOMEM, "host allocation failed");
  c->comps = op->comps;
  c->device = op->mesh->device;
  c->sm_count = op->mesh->sm_count;
  c->nrows = nrows;
  int st = dalloc(&c->rowptr, nrows + 1);
  if (st) { delete c; return st; }
  cudaError_t e = launch_csr_rowcount(op->comps, op->bc, g, c->rowptr, 0);
  if (e != cudaSuccess) { fem_csr_destroy(c); return fail(FEM_ECUDA, "csr rowcount: %s", cudaGetErrorString(e)); }
  int64_t nnz = 0;
  e = cudaMemcpy(&nnz, c->rowptr + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { fem_csr_destroy(c); return fail(FEM_ECUDA, "csr nnz: %s", cudaGetErrorString(e)); }
  c->nnz = nnz;
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double need = (double)nnz * 12.0;
  if (need > (double)fr * 0.95) {
    fem_csr_destroy(c);
    return fail(FEM_ENOMEM, "CSR needs %.1f GB, %.1f GB free", need / 1e9, fr / 1e9);
  }
  if ((st = dalloc(&c->col, nnz)) || (st = dalloc(&c->val, nnz))) { fem_csr_destroy(c); return st; }
  {  // unit element matrices of the operator's quadrature rule (constant memory, this device)
    std::lock_guard<std::mutex> lk(g_unit_mu);
    double K[64], Kl[576], Km[576];
    unit_element_matrices(K, Kl, Km, op->quad);
    e = upload_unit_matrices(K, Kl, Km);
    if (e == cudaSuccess) e = launch_csr_fill(op->kind, op->bc, g, op->lm, c->rowptr, c->col, c->val, 0);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { fem_csr_destroy(c); return fail(FEM_ECUDA, "csr fill: %s", cudaGetErrorString(e)); }
  *out = c;
  return FEM_OK;
}

int fem_csr_info(fem_csr_t c, int64_t* nrows, int64_t* nnz, int64_t* bytes) {
  if (!c) return fail(FEM_EINVAL, "csr is NULL");
  if (nrows) *nrows = c->nrows;
  if (nnz) *nnz = c->nnz;
  if (bytes) *bytes = c->nnz * 12 + (c->nrows + 1) * 8;
  return FEM_OK;
}

int fem_csr_apply(fem_csr_t c, const double* x, double* y, void* stream) {
  if (!c) return fail(FEM_EINVAL, "csr is NULL");
  FEM_TRY(check_vec(x, "x"));
  FEM_TRY(check_vec(y, "y"));
  if ((const void*)x == (const void*)y) return fail(FEM_EINVAL, "x and y alias");
  if (!is_device_ptr(x) || !is_device_ptr(y)) return fail(FEM_EINVAL, "fem_csr_apply needs device pointers");
  FEM_TRY(set_device(c->device));
  cudaError_t e = launch_csr_spmv(c->comps, c->nrows, c->rowptr, c->col, c->val, x, y,
                                  (cudaStream_t)stream, c->sm_count);
  if (e != cudaSuccess) return fail(FEM_ECUDA, "spmv launch: %s", cudaGetErrorString(e));
  return FEM_OK;
}

int fem_csr_export(fem_csr_t c, int64_t* rowptr, int32_t* col, double* val, void* stream) {
  if (!c) return fail(FEM_EINVAL, "csr is NULL");
  FEM_TRY(set_device(c->device));
  cudaStream_t s = (cudaStream_t)stream;
  auto cp = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst) return FEM_OK;
    const cudaMemcpyKind k = is_device_ptr(dst) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, k, s));
    return FEM_OK;
  };
  FEM_TRY(cp(rowptr, c->rowptr, (c->nrows + 1) * sizeof(int64_t)));
  FEM_TRY(cp(col, c->col, c->nnz * sizeof(int32_t)));
  FEM_TRY(cp(val, c->val, c->nnz * sizeof(double)));
  CUDA_TRY(cudaStreamSynchronize(s));
  return FEM_OK;
}

void fem_csr_destroy(fem_csr_t c) {
  if (!c) return;
  set_device(c->device);
  cudaFree(c->rowptr);
  cudaFree(c->col);
  cudaFree(c->val);
  delete c;
}

}  // extern "C"
