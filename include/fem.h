/*
 * fem.h -- C ABI of the B200-native hot path of arXiv 2308.09839
 * ("low-order matrix-free finite element operators in CG").
 *
 * Library: paper_2308_09839_b200/libfem.so (CUDA sm_100a, FP64).  No torch types cross this
 * boundary: every argument is a plain integer, double, host pointer, device pointer or an
 * opaque handle.  Citations "P:n" are lines of the paper text, "S:n" of SPEC.md.
 *
 * Problem (Eq. 1-3): Q1 trilinear hexahedra on the box [0,nx h]x[0,ny h]x[0,nz h];
 *   kind FEM_SCALAR_LAPLACE  : A_ij = int grad phi_i . grad phi_j                 (Eq. 1 / 4)
 *   kind FEM_VECTOR_LAPLACE  : 3 components, (e_k (x) grad phi_i):(e_l (x) grad phi_j) (Eq. 2 / 5)
 *   kind FEM_ELASTICITY      : (e_k (x) grad phi_i) : sigma(e_l (x) grad phi_j),
 *                              sigma = lambda_e tr(eps) I + 2 mu_e eps, cell-wise lambda_e, mu_e
 *                                                                               (Eq. 3 / 6)
 * integrated with 2x2x2 Gauss-Legendre quadrature (reading R1), applied
 * matrix-free (three steps of P:188-196, Eq. 7-9, Alg. 1).
 *
 * Layouts (ABI level):
 *   node n = i + (nx+1)(j + (ny+1) k), x fastest;  DOF = c n + comp, c = 1 or 3
 *   ("3(i-1)+k").  Vectors are dense FP64, 8-byte aligned, length c * n_local_nodes,
 *   covering the rank's OWNED node planes [plane_begin, plane_end) only.
 *   Cells e = i + nx (j + ny k); lambda/mu are FP64 per cell.
 * Boundary conditions (reading R6): FEM_BC_DIRICHLET_BOX applies
 *   y = P A P x + (I - P) x, P zeroing every DOF of every node on the 6 box faces.
 *
 * Pointers: "device or host" arguments are classified with cudaPointerGetAttributes; host
 * arguments are staged through library-owned device buffers inside the call (the e2e path).
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  Every
 * call is stream-ordered on it; calls returning host values (fem_dot, fem_cg_solve with
 * info, fem_csr_create) synchronise that stream.
 * Errors: every int-returning function returns a fem_status; it never throws, never aborts;
 * on error a thread-local message is available from fem_last_error().
 * Ownership: handles are created and destroyed by the caller through this API; the library
 * owns everything behind a handle (workspace, ghost planes, material copies, CSR arrays).
 */
#ifndef PAPER_2308_09839_FEM_H
#define PAPER_2308_09839_FEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FEM_OK = 0,
  FEM_EINVAL = 1,       /* bad argument: dims < 1, h <= 0 or non-finite, NULL/misaligned pointer,
                           aliasing x == y, material on a non-elastic op, unknown kind/bc      */
  FEM_ENOMEM = 2,       /* device or host allocation failed                                    */
  FEM_ECUDA = 3,        /* a CUDA runtime call failed (message has the CUDA error string)      */
  FEM_ENCCL = 4,        /* an NCCL call failed                                                  */
  FEM_EOVERFLOW = 5,    /* global node count >= 2^32 or DOF index overflow              */
  FEM_EMATERIAL = 6,    /* some mu <= 0 or lambda + 2 mu / 3 < 0, or non-finite         */
  FEM_EBREAKDOWN = 7,   /* CG: p^T A p <= 0 or non-finite while r^T r > 0               */
  FEM_ESTATE = 8,       /* call out of order (e.g. elastic apply before fem_set_material)       */
  FEM_EUNSUPPORTED = 9  /* valid request this build does not implement (message says what)      */
} fem_status;

typedef enum { FEM_SCALAR_LAPLACE = 0, FEM_VECTOR_LAPLACE = 1, FEM_ELASTICITY = 2 } fem_kind;
typedef enum { FEM_BC_NONE = 0, FEM_BC_DIRICHLET_BOX = 1 } fem_bc;

typedef struct fem_comm_s* fem_comm_t;
typedef struct fem_mesh_s* fem_mesh_t;
typedef struct fem_op_s* fem_op_t;
typedef struct fem_csr_s* fem_csr_t;

/* CG report (reduced).  status is a fem_status of the solve itself. */
typedef struct {
  int32_t iterations;      /* iterations performed                                             */
  int32_t converged;       /* 1 if sqrt(r.r) <= tol * ||r0|| or r.r == 0 was reached            */
  int32_t breakdown_iter;  /* iteration at which p.Ap <= 0 / non-finite was seen, else -1       */
  int32_t status;          /* FEM_OK or FEM_EBREAKDOWN                                          */
  double r0_norm;          /* ||b - A x0||_2 (global)                                           */
  double r_norm;           /* recurrence residual norm sqrt(r.r) of the last residual the
                              recurrence computed: the exit iterate's (Hestenes-Stiefel); with
                              cg_variant 1 the iterate the last update started from, unless
                              converged (then the exit iterate's)                              */
  double true_r_norm;      /* ||b - A x||_2 recomputed at exit (one extra apply)                */
} fem_cg_info;

/* ---- diagnostics --------------------------------------------------------------------- */
const char* fem_last_error(void);           /* thread-local; "" if none                     */
const char* fem_version(void);
/* Number of CUDA kernels this process has launched through the library (graph replays count
 * every kernel node).  Used by bench.py's "gpu_launches". */
int64_t fem_launch_count(void);

/* ---- communicator (slab decomposition over NCCL) ------------------------ */
/* Rank 0 creates a 128-byte NCCL unique id; the caller broadcasts it (torch.distributed). */
int fem_get_unique_id(void* id_out, int64_t id_bytes /* >= 128 */);
/* nranks == 1: no NCCL is touched and id may be NULL.  The calling thread's current CUDA
 * device is the rank's device.  nranks > 1 with id == NULL creates a VIRTUAL communicator:
 * it only defines the slab partition (for single-process tests with fem_apply_ghost); calls that
 * need an exchange (fem_apply, fem_dot, fem_cg_*) then return FEM_EUNSUPPORTED. */
int fem_comm_create(int32_t nranks, int32_t rank, const void* id, fem_comm_t* out);
/* In-process loopback communicator: creates `nranks` (1..64) communicators out[0..nranks-1] of
 * one group on the calling thread's current device, with no NCCL.  Each is used by ONE host
 * thread (the rank), every rank with its own stream, all on that device.  The library's
 * collectives (node-plane halo, allreduce of the CG scalars, the peer-halo exchange) become
 * device copies and a rank-ordered sum kernel, ordered across the ranks' streams by CUDA events
 * the ranks exchange through a host rendezvous; so fem_apply, fem_dot, fem_cg_* and the
 * "peer_halo" option run the multi-rank code paths of the slab decomposition on one GPU (tests;
 * DESIGN.md §7).  Every rank must enter the same collectives in the same order (as with NCCL); a
 * rank missing for 120 s makes the others fail with FEM_ESTATE.  CG iterations are launched
 * eagerly (no CUDA graph: the rendezvous is on the host).  Destroy every returned communicator. */
int fem_comm_create_loopback(int32_t nranks, fem_comm_t* out);
/* Slab partition (pure host function, no CUDA): the nz+1 node planes split as evenly as
 * possible, rank r owns [plane_begin, plane_end); the first (nz+1) % nranks ranks get one more. */
int fem_partition(int64_t nz, int32_t nranks, int32_t rank, int64_t* plane_begin,
                  int64_t* plane_end);
void fem_comm_destroy(fem_comm_t comm);

/* ---- mesh ----------------------------------------------------------------- */
/* nx, ny, nz >= 1 cells; h > 0 cell side.  comm NULL means one GPU.  Node planes (z) are split
 * as evenly as possible over the ranks; rank r owns [plane_begin, plane_end). */
int fem_mesh_create(int64_t nx, int64_t ny, int64_t nz, double h, fem_comm_t comm,
                    fem_mesh_t* out);
int fem_mesh_local(fem_mesh_t mesh, int64_t* plane_begin, int64_t* plane_end,
                   int64_t* n_local_nodes);
void fem_mesh_destroy(fem_mesh_t mesh);

/* ---- general (deformed) hexahedral mesh: Algorithm 1 as written ------------- */
/* An explicit mesh of trilinear hexahedra, the input of Alg. 1 ("global support point
 * coordinates", node map; Table 2):
 *   coords[3 n + d]  FP64 coordinate d of node n (device or host, 8-byte aligned);
 *   cells[8 e + a]   int32 global node of local node a of cell e, VTK corner order:
 *                    (0,0,0) (1,0,0) (1,1,0) (0,1,0) (0,0,1) (1,0,1) (1,1,1) (0,1,1);
 *   dirichlet[n]     uint8, != 0 marks a constrained node (all components; device or host), or
 *                    NULL.  Operators created with FEM_BC_DIRICHLET_BOX on this mesh apply
 *                    y = P A P x + (I - P) x for these nodes.
 * The arrays are copied (the caller may free them).  The Jacobian, its determinant and inverse
 * are recomputed at each 2x2x2 Gauss point of every apply (Alg. 1 lines 4-5).  Errors:
 * FEM_EINVAL for n_nodes / n_cells < 1, a node index outside [0, n_nodes), or det J <= 0 at any
 * Gauss point; FEM_EOVERFLOW for n_nodes >= 2^31.  Single GPU.  Vectors on this
 * mesh are dense, DOF = c n + comp over all n_nodes nodes; fem_set_material takes n_cells values
 * with layer_begin = 0, n_layers = 1; fem_apply, fem_dot and fem_cg_* work as on the box (CG
 * unfused: apply + update + p-update); fem_apply_ghost and fem_csr_create return
 * FEM_EUNSUPPORTED.  The scatter adds element contributions with FP64 atomics, so results are
 * exact up to the (run-dependent) summation order of the <= 8 contributions per node. */
int fem_mesh_create_hex(int64_t n_nodes, int64_t n_cells, const double* coords, const int32_t* cells,
                        const uint8_t* dirichlet, fem_mesh_t* out);
int fem_mesh_info_hex(fem_mesh_t mesh, int64_t* n_nodes, int64_t* n_cells, int64_t* n_constrained);

/* ---- operator -------------------------------------------------------------------------- */
int fem_op_create(fem_mesh_t mesh, int32_t kind, int32_t bc, fem_op_t* out);
int fem_op_ndof(fem_op_t op, int64_t* n_local_dof, int64_t* n_global_dof);
/* Cell-wise Lame parameters (P:9, "cell constant C").  lambda/mu (device or host) hold
 * the cell layers [layer_begin, layer_begin + n_layers) of the global cell-lexicographic
 * arrays; they must cover every layer the rank touches (its owned planes' adjacent cells).
 * Values are validated (FEM_EMATERIAL) and copied; the caller may free them afterwards. */
int fem_set_material(fem_op_t op, const double* lambda, const double* mu, int64_t layer_begin,
                     int64_t n_layers);
/* y = A_c x on the rank's owned DOFs.  x, y: device or host, length n_local_dof,
 * x != y.  Collective when nranks > 1 (one node-plane halo per neighbour). */
int fem_apply(fem_op_t op, const double* x, double* y, void* stream);
/* y = A_c x with caller-supplied ghost node planes and no communication: ghost_lo is node
 * plane plane_begin-1, ghost_hi is plane plane_end (device pointers, plane_dofs = c (nx+1)(ny+1)
 * values each; NULL where the plane is outside the box).  x, y device, owned planes. */
int fem_apply_ghost(fem_op_t op, const double* x, const double* ghost_lo, const double* ghost_hi,
                    double* y, void* stream);
/* As fem_apply_ghost, but through the CG-internal padded layout and its TMA tensor maps (the
 * path every fused CG iteration runs, including the material tensor at the slab offset), for
 * single-process slab tests of that path: x and the ghost planes are packed into the library's
 * padded x, the apply writes the padded q, which is unpacked into y.  Interrupts an active
 * fem_cg_begin/iterate sequence (FEM_ESTATE on the next fem_cg_iterate). */
int fem_apply_ghost_padded(fem_op_t op, const double* x, const double* ghost_lo, const double* ghost_hi,
                           double* y, void* stream);
/* Single-process loopback of the peer halo ("peer_halo" option): this slab operator reads its
 * ghost planes directly from the padded vectors of the operators of the slabs below (lo) and
 * above (hi) -- NULL where the box ends -- which live in the same process on the same device.
 * For tests of the peer-halo kernel path with virtual communicators (fem_apply_ghost_padded then
 * takes NULL ghost planes); the cross-process version is fem_set_option(op, "peer_halo", 1). */
int fem_op_link_peers(fem_op_t op, fem_op_t lo, fem_op_t hi);
/* Peer halo across processes without NCCL for the handle exchange: fem_op_peer_info writes this
 * slab operator's CUDA IPC handles of its CG vectors and its plane count (<= 320 bytes) into
 * `info`; the caller sends it to both slab neighbours (any channel, e.g. torch.distributed) and
 * each rank calls fem_op_open_peers with the infos of the slabs below / above (NULL at the box
 * ends).  Equivalent to the "peer_halo" option, which does the same exchange over NCCL. */
int fem_op_peer_info(fem_op_t op, void* info, int64_t bytes);
int fem_op_open_peers(fem_op_t op, const void* lo_info, const void* hi_info);
/* Global sum_i a_i b_i over owned DOFs (Table 4 "ddot").  Deterministic for a
 * fixed rank count.  Result written to *result (host).  Collective. */
int fem_dot(fem_op_t op, const double* a, const double* b, double* result, void* stream);
/* Conjugate gradient (recurrences of Table 4) on A_c x = b.
 * x holds x0 on entry and the iterate on exit (device or host).  tol > 0: stop when
 * sqrt(r.r) <= tol * ||r0||; tol == 0: exactly maxit iterations unless r.r == 0.
 * info may be NULL.  Returns FEM_EBREAKDOWN on breakdown (info filled).  Collective. */
int fem_cg_solve(fem_op_t op, const double* b, double* x, double tol, int32_t maxit,
                 fem_cg_info* info, void* stream);
/* Split CG for benchmarking a fixed number of steps with inputs resident on the device:
 * fem_cg_begin initialises r = b - A x, p = r (b, x device pointers that must stay valid),
 * fem_cg_iterate runs `iters` iterations (CUDA-graph replay; stream-ordered, no host sync),
 * fem_cg_end synchronises and fills info. */
int fem_cg_begin(fem_op_t op, const double* b, double* x, double tol, int32_t maxit, void* stream);
int fem_cg_iterate(fem_op_t op, int32_t iters, void* stream);
int fem_cg_end(fem_op_t op, fem_cg_info* info, void* stream);
/* Options: "use_graph" (default 1), "check_every" (default 16 iterations between host
 * convergence polls in fem_cg_solve), "time_apply" (1: record CUDA events around every apply
 * launched by fem_cg_iterate; read back with fem_apply_time), "partial_assembly" (general hex
 * meshes, and the single-rank elasticity box operator; else FEM_EUNSUPPORTED; 1: store per Gauss
 * point what the matrix-free kernel recomputes and apply from it, the paper's comparison method
 * P:308-309 / Table 3 -- general hexes: the geometry, 6 values per point for the Laplace kinds,
 * 9 for elasticity; elasticity box: Table 3's 21 values per point, D_q = w_q det J_q C_e (the
 * symmetric 6x6 Voigt stiffness with the cell's lambda, mu folded in), 1,344 B per cell;
 * 0: matrix-free recomputation, the default), "quadrature" (0: the
 * 2x2x2 Gauss-Legendre rule, default; 1: the 2x2x2 Gauss-Lobatto rule collocated with the nodes,
 * the quadrature of the CEED benchmark problems BP5 / BP6 the paper names, P:581, P:638,
 * a different operator (the 7-point stencil for Laplace on the box); applies to
 * every kernel of the operator incl. fem_csr_create; on a general hex mesh, switching to 1
 * checks det J > 0 at the nodes, FEM_EINVAL otherwise), "cg_variant" (0: the fused
 * Hestenes-Stiefel CG of Table 4, default; 1: Chronopoulos-Gear single-reduction CG -- r.r and
 * w.r come out of the apply together, one allreduce of two values per iteration instead of two;
 * TMA path only, reads back 0 elsewhere), "dot_mode" (how the fused Hestenes-Stiefel CG
 * forms its two dots -- the dot-implementation ablation of P:714-728: 0, default, in the
 * epilogue of the producing kernel (p.Ap in the apply, r.r in the update) by a block tree plus a
 * last-block pass over the CTA partials in block order (deterministic); 1 by separate dot
 * kernels after the apply and the update, re-reading p, q and r (+24 B/DOF, +2 launches per
 * iteration); 2 in the epilogue with the CTA partials added by FP64 atomics (summation order
 * varies from run to run); TMA path, cg_variant 0 only), "halo_overlap" (1, default: with an
 * exchange step -- nranks > 1 without peer_halo -- the halo runs on a library stream while the
 * interior node planes are applied, then the two boundary planes; 0: halo, then one apply),
 * "x_defer" (every CG iteration -- fused, single-reduction and unfused; 1, 2, 4 or 8, default
 * 8: x is updated once per group of m iterations, x = ((x + alpha_0 p_0) + ...) + alpha_{m-1}
 * p_{m-1}, from the m p buffers the iteration writes in turn -- the same FMAs in the same order as
 * the per-iteration update, so x is bitwise the same; the other updates of the group leave x
 * alone: 32 + 16 / m instead of 48 B/DOF of update traffic per iteration in the fused CG (Table
 * 4's axpy rows); m >= 4 allocates up to m - 1 more p vectors on the first solve
 * (when they do not fit in device memory, m drops to 4 or 2 for the operator's lifetime and
 * reads back accordingly); cg_end adds the pending updates of an unfinished group; with
 * peer_halo the fused Hestenes-Stiefel iteration uses m <= 2; reads back the m in use;
 * FEM_EINVAL for other values), "deterministic" (general hex meshes: 1 replaces
 * the FP64 atomic scatter by element outputs E[cell][8][C] and a per-node gather over the node's
 * (cell, corner) entries in ascending order -- bitwise reproducible results run after run, at
 * 24 C extra bytes of traffic per cell each way; the node map is built on the first switch-on;
 * box operators read back 1, their kernels are atomic-free, and reject the setting with
 * FEM_EUNSUPPORTED), "trace" (1: CUDA timing events around the halo, the interior and the boundary launches of
 * every eager exchange apply; read back, blocking on the last traced apply, as the read-only
 * "trace_halo_ns", "trace_interior_ns", "trace_boundary_ns", "trace_total_ns" -- the
 * halo / interior overlap timeline; FEM_ESTATE before the first traced apply; host-side NVTX
 * ranges fem:apply, fem:halo, fem:allreduce, fem:interior, fem:boundary, fem:cg_* are always
 * emitted and cost nothing without a tool attached),
 * "peer_halo" (1: collective over the slab ranks --
 * every rank sets it -- exchanging CUDA IPC handles of the CG vectors with the neighbours over
 * NCCL; the apply kernels then load the ghost node planes straight from the neighbours' memory
 * over NVLink inside their TMA pipeline and the NCCL halo step disappears; the two CG allreduces
 * order the cross-rank reads and writes; TMA path only, cannot be switched off), "direct_tma"
 * (1, default: fem_apply on a single-rank box operator stages caller vectors whose rows are
 * 16-B multiples -- (nx+1)*comps even -- and whose base is 16-B aligned through a tensor map
 * straight over the caller's memory, one TMA box per node plane; 0 or any other vector: one
 * bulk copy per row; results are identical; with the Dirichlet box, Laplace kinds and odd rows
 * a "row-pair" tensor view -- two TMA boxes per plane -- is used when the caller's allocation
 * extends one row past the vector).  Read-only "last_apply_path": staging of the last fem_apply
 * (0 bulk rows, 1 tensor map, 2 row-pair tensor map). */
int fem_set_option(fem_op_t op, const char* key, int64_t value);
/* Read-only properties: "fused_cg" (1: CG iterations use the fused apply -- p = r + beta p_old
 * formed inside the TMA apply kernel -- and 2 kernels per iteration; 0: apply + update +
 * p-update), "tma" (1: CG applies stage planes with TMA tensor maps), plus the options above. */
int fem_get_option(fem_op_t op, const char* key, int64_t* value);
/* Total device time (ms) and count of the applies timed since the last call (time_apply). */
int fem_apply_time(fem_op_t op, double* total_ms, int64_t* count);
void fem_op_destroy(fem_op_t op);

/* ---- assembled CSR baseline (Table 1) ------------------------------ */
/* Builds A_c as CSR on the device from the same element matrices (int64 row offsets, int32
 * columns, FP64 values: 12 B per non-zero).  Single rank only (FEM_EUNSUPPORTED else).
 * Elasticity requires fem_set_material first. */
int fem_csr_create(fem_op_t op, fem_csr_t* out);
int fem_csr_info(fem_csr_t csr, int64_t* nrows, int64_t* nnz, int64_t* bytes);
int fem_csr_apply(fem_csr_t csr, const double* x, double* y, void* stream);
/* Copy the CSR arrays out (device or host destinations, any may be NULL): rowptr nrows + 1
 * int64, col nnz int32, val nnz FP64.  Synchronises the stream.  Used to hand the identical
 * matrix to a library SpMV (cuSPARSE) for the baseline comparison of bench.py. */
int fem_csr_export(fem_csr_t csr, int64_t* rowptr, int32_t* col, double* val, void* stream);
void fem_csr_destroy(fem_csr_t csr);

#ifdef __cplusplus
}
#endif
#endif /* PAPER_2308_09839_FEM_H */
