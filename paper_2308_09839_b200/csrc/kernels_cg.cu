// kernels_cg.cu -- CG vector kernels (Table 4 rows) and the deterministic dot
// ("the dot product ... implementation has dramatic impact").
//
// Per iteration, with p.Ap fused into the apply kernel's epilogue:
//   apply   : q = A_c p,  pq = p.q            (kernels_laplace / kernels_elastic, mode 1)
//   update  : alpha = rr/pq; x += alpha p; r -= alpha q; rr' = r.r     (48 B/DOF)
//   pupdate : beta = rr'/rr; p = r + beta p; rr = rr'; convergence     (24 B/DOF)
// Scalars live in device memory (CgScalars); kernels read them at start, so the iteration is
// host-sync free and CUDA-graph capturable.  Every dot is a warp-shuffle + block tree + a
// last-block-done pass summing the per-CTA partials in block order: bitwise reproducible for
// a fixed launch configuration, no floating-point atomics.
#include <algorithm>

#include "fem_internal.cuh"

namespace fem {

constexpr int kVecThreads = 256;
#ifndef FEM_UPD_MINB
#define FEM_UPD_MINB 3  // resident blocks per SM the fused update kernel is compiled for (80 registers)
#endif
#ifndef FEM_UPD_MINB_PEND
#define FEM_UPD_MINB_PEND 4  // ... its variants without the x group (64 registers: the 8-per-SM grid in two full waves)
#endif

// grid of a grid-stride vector kernel: at most one wave of resident blocks (per_sm per SM), so
// every block streams an equal share and no partial last wave idles part of the GPU
static inline unsigned vec_blocks(int64_t n, int sm_count, int per_sm = 8) {
  int64_t want = (n + kVecThreads * 4 - 1) / (kVecThreads * 4);
  int64_t cap = (int64_t)sm_count * per_sm;
  return (unsigned)std::max<int64_t>(1, std::min(want, cap));
}

__global__ void __launch_bounds__(kVecThreads) cg_init_kernel(const double* __restrict__ b,
                                                              const double* __restrict__ ax,
                                                              double* __restrict__ r,
                                                              double* __restrict__ p, int64_t n,
                                                              CgScalars* sc, Reduce red) {
  __shared__ double sh[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double ri = b[i] - ax[i];
    r[i] = ri;
    p[i] = ri;
    acc = fma(ri, ri, acc);
  }
  double bs = block_sum(acc, sh);
  double tot;
  if (last_block_reduce(bs, red, sh, &tot)) sc->rr_new = tot;
}

__global__ void cg_finish_init_kernel(CgScalars* sc, double tol, int maxit) {
  const double rr = sc->rr_new;
  sc->rr = rr;
  sc->rr0 = rr;
  sc->stop_rr = tol * tol * rr;
  sc->pq = 0.0;
  sc->rr_acc = 0.0;
  for (int k = 0; k < 7; ++k) sc->alpha_h[k] = 0.0;
  sc->xp = 0;
  sc->it = 0;
  sc->maxit = maxit;
  sc->breakdown_iter = -1;
  sc->first = 1;
  sc->done = (rr == 0.0 || rr <= sc->stop_rr) ? 1 : (maxit <= 0 ? 3 : 0);
}

struct OldP {
  const double* p[7];  // the pending p vectors P_0 .. P_{NOLD-1} (deferred x update)
};

// unfused iteration (general hexes, partial assembly, degenerate boxes): x += alpha p; r -= alpha
// q; rr_new = r.r.  NOLD: the deferred x update as in cg_update_fused_kernel below (-1: alpha
// pending in sc->alpha_h[jpend]; k: the k pending updates, then this one).
template <int NOLD>
__global__ void __launch_bounds__(kVecThreads) cg_update_kernel(double* __restrict__ x,
                                                                double* __restrict__ r,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ q,
                                                                int64_t n, CgScalars* sc,
                                                                Reduce red, OldP po, int jpend) {
  __shared__ double sh[32];
  if (sc->done) return;
  const double pq = sc->pq;
  if (!(pq > 0.0) || !isfinite(pq)) {  // breakdown: same decision in every block
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->breakdown_iter = sc->it;
      sc->done = 2;
    }
    return;
  }
  const double alpha = sc->rr / pq;
  if (NOLD < 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    sc->alpha_h[jpend] = alpha;
    sc->xp = jpend + 1;
  }
  double ah[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) ah[k] = sc->alpha_h[k];
  if (NOLD > 0 && blockIdx.x == 0 && threadIdx.x == 0) sc->xp = 0;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    if (NOLD >= 0) {
      double xv = x[i];
#pragma unroll
      for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) xv = fma(ah[k], po.p[k][i], xv);
      x[i] = fma(alpha, p[i], xv);
    }
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    acc = fma(ri, ri, acc);
  }
  double bs = block_sum(acc, sh);
  double tot;
  if (last_block_reduce(bs, red, sh, &tot)) sc->rr_new = tot;
}

// fused CG (mode-2 apply has formed p = r + beta p_old and q = A p):
//   alpha = rr / pq; x += alpha p; r -= alpha q; rr_new = r.r; it++; convergence -> done.
// The next mode-2 apply reads beta = rr_new / rr and rolls rr = rr_new in its last block.
// Deferred x update (option x_defer = m): the fused CG keeps the p of m
// consecutive iterations in m buffers (the apply writes p_k into buffer k mod m and reads p_{k-1}
// as p_old), so x needs updating only every m-th iteration.  NOLD selects the update's x work:
//   -1  x untouched: alpha is left pending (sc->alpha_h[j], sc->xp = j + 1)        (24 B/DOF)
//   k   x = (((x + alpha_0 P_0) + ...) + alpha_{k-1} P_{k-1}) + alpha p: the k pending updates,
//       then this one, in their sequential order -- bitwise the x of k + 1 per-iteration updates
//       (k = 0: the plain x += alpha p, 48 B/DOF; k = 1: 56; k = 3: 72; k = 7: 104)
// so a group of m iterations moves 32 m + 16 instead of 48 m B/DOF of update traffic.
template <int NOLD>
__global__ void __launch_bounds__(kVecThreads, NOLD <= 0 ? FEM_UPD_MINB_PEND : FEM_UPD_MINB) cg_update_fused_kernel(double* __restrict__ x,
                                                                      double* __restrict__ r,
                                                                      const double* __restrict__ p,
                                                                      const double* __restrict__ q,
                                                                      int64_t n, CgScalars* sc,
                                                                      Reduce red, OldP po, int jpend) {
  __shared__ double sh[32];
  if (sc->done) return;
  // convergence of the current iterate: rr_new is the allreduced (rank-global) r.r of the
  // previous update, so every rank decides alike (the apply before this kernel was wasted work)
  const double rrc = sc->rr_new;
  if (rrc == 0.0 || rrc <= sc->stop_rr) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->done = 1;
    return;
  }
  const double pq = sc->pq;
  if (!(pq > 0.0) || !isfinite(pq)) {  // breakdown: same decision in every block
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->breakdown_iter = sc->it;
      sc->done = 2;
    }
    return;
  }
  const double alpha = sc->rr / pq;
  // (alpha_h / xp are read by later kernels only: block 0 may write them)
  if (NOLD < 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    sc->alpha_h[jpend] = alpha;
    sc->xp = jpend + 1;
  }
  double ah[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) ah[k] = sc->alpha_h[k];
  if (NOLD > 0 && blockIdx.x == 0 && threadIdx.x == 0) sc->xp = 0;
  double acc = 0.0;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // 16-B vector accesses (the vectors share one layout, hence one alignment); a leading
  // unaligned element and a trailing odd element are handled by thread 0 / the last thread
  const int64_t head = (reinterpret_cast<uintptr_t>(r) & 15) ? 1 : 0;
  auto one = [&](int64_t i) {
    if (NOLD >= 0) {
      double xv = x[i];
#pragma unroll
      for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) xv = fma(ah[k], po.p[k][i], xv);
      x[i] = fma(alpha, p[i], xv);
    }
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    acc = fma(ri, ri, acc);
  };
  if (head && gtid == 0 && n > 0) one(0);
  const int64_t n2 = (n - head) / 2;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x + head);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r + head);
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p + head);
  const double2* __restrict__ q2 = reinterpret_cast<const double2*>(q + head);
  auto xupd = [&](int64_t j) {
    if (NOLD < 0) return;
    double2 xa = x2[j];
    double2 o[7];
#pragma unroll
    for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) o[k] = reinterpret_cast<const double2*>(po.p[k] + head)[j];
    const double2 pa = p2[j];
#pragma unroll
    for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) {
      xa.x = fma(ah[k], o[k].x, xa.x);
      xa.y = fma(ah[k], o[k].y, xa.y);
    }
    x2[j] = make_double2(fma(alpha, pa.x, xa.x), fma(alpha, pa.y, xa.y));
  };
  int64_t i = gtid;
  if (NOLD <= 1) {
    for (; i + stride < n2; i += 2 * stride) {  // two independent 16-B groups in flight per thread
      const double2 qa = q2[i], qb = q2[i + stride], ra = r2[i], rb = r2[i + stride];
      xupd(i);
      xupd(i + stride);
      const double2 na = make_double2(fma(-alpha, qa.x, ra.x), fma(-alpha, qa.y, ra.y));
      const double2 nb = make_double2(fma(-alpha, qb.x, rb.x), fma(-alpha, qb.y, rb.y));
      r2[i] = na;
      r2[i + stride] = nb;
      acc = fma(na.x, na.x, acc); acc = fma(na.y, na.y, acc);
      acc = fma(nb.x, nb.x, acc); acc = fma(nb.y, nb.y, acc);
    }
  }
  for (; i < n2; i += stride) {
    const double2 qa = q2[i], ra = r2[i];
    xupd(i);
    const double2 na = make_double2(fma(-alpha, qa.x, ra.x), fma(-alpha, qa.y, ra.y));
    r2[i] = na;
    acc = fma(na.x, na.x, acc); acc = fma(na.y, na.y, acc);
  }
  if (((n - head) & 1) && gtid == stride - 1) one(n - 1);
  if (red.dot_mode == 1) return;  // r.r and the bookkeeping: launch_cg_dot(which = 1)
  double bs = block_sum(acc, sh);
  if (red.dot_mode == 2) {
    if (threadIdx.x == 0) atomicAdd(&sc->rr_acc, bs);  // zeroed by the apply's last CTA
    double unused;
    if (last_block_reduce(0.0, red, sh, &unused)) {  // ticket only: the last CTA publishes
      sc->rr_new = sc->rr_acc;
      sc->pq = 0.0;  // the next apply's atomic target
      const int it = sc->it + 1;
      sc->it = it;
      if (it >= sc->maxit) sc->done = 3;
    }
    return;
  }
  double tot;
  if (last_block_reduce(bs, red, sh, &tot)) {
    // tot is this rank's partial of r.r: the allreduce that follows makes rr_new global, so the
    // convergence test runs at the start of the next fused apply (every rank, the same value)
    sc->rr_new = tot;
    const int it = sc->it + 1;
    sc->it = it;
    if (it >= sc->maxit) sc->done = 3;
  }
}

// Chronopoulos-Gear CG update (NEXT #1; single global reduction per iteration -- the apply
// (mode 3) delivered delta = w.r in pq and gamma = r.r in rr_new, reduced together).  Recurrences:
//   beta = gamma / gamma_prev, alpha = gamma / (delta - beta gamma / alpha_prev)  (first: beta = 0,
//   alpha = gamma / delta); p = r + beta p; s = w + beta s; x += alpha p; r -= alpha s.
// gamma is the residual of the iterate before this update, so convergence is decided here.
// Deferred x update in the single-reduction CG (option x_defer): p_k is written
// into ring buffer k mod m (pw) from p_{k-1} (pr), s stays in place; NOLD as in
// cg_update_fused_kernel (-1: alpha pending, k: the k pending updates, then this one).
template <int NOLD>
__global__ void __launch_bounds__(kVecThreads, FEM_UPD_MINB) cg_cgcg_update_kernel(double* __restrict__ x, double* __restrict__ r,
                                                                     const double* pr, double* pw,  // (alias when m = 1)
                                                                     double* __restrict__ s,
                                                                     const double* __restrict__ w, int64_t n,
                                                                     CgScalars* sc, Reduce red, OldP po, int jpend) {
  __shared__ double sh[32];
  if (sc->done) return;
  const double gam = sc->rr_new, delta = sc->pq;
  const bool first = sc->first != 0;
  // Early exits write only `done` / `breakdown_iter`: other blocks may still be reading rr, alpha
  // and first to take the same decision (the reported residual is rr_new, fem_cg_end).
  if (gam == 0.0 || gam <= sc->stop_rr) {  // converged at the current iterate (same test in every block)
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->done = 1;
    return;
  }
  const double beta = first ? 0.0 : gam / sc->rr;
  const double denom = first ? delta : delta - beta * gam / sc->alpha;
  const double alpha = gam / denom;
  if (!(denom > 0.0) || !isfinite(alpha)) {  // breakdown
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sc->breakdown_iter = sc->it;
      sc->done = 2;
    }
    return;
  }
  // (alpha_h / xp are read by later kernels only: block 0 may write them)
  if (NOLD < 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    sc->alpha_h[jpend] = alpha;
    sc->xp = jpend + 1;
  }
  double ah[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) ah[k] = sc->alpha_h[k];
  if (NOLD > 0 && blockIdx.x == 0 && threadIdx.x == 0) sc->xp = 0;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](int64_t i) {
    const double ri = r[i], wi = w[i];
    const double pi = first ? ri : fma(beta, pr[i], ri);
    const double si = first ? wi : fma(beta, s[i], wi);
    pw[i] = pi;
    s[i] = si;
    if (NOLD >= 0) {
      double xv = x[i];
#pragma unroll
      for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) xv = fma(ah[k], po.p[k][i], xv);
      x[i] = fma(alpha, pi, xv);
    }
    r[i] = fma(-alpha, si, ri);
  };
  // 16-B accesses (the vectors share one layout), head / tail elements scalar
  const int64_t head = (reinterpret_cast<uintptr_t>(r) & 15) ? 1 : 0;
  if (head && gtid == 0 && n > 0) one(0);
  const int64_t n2 = (n - head) / 2;
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x + head);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r + head);
  const double2* pr2 = reinterpret_cast<const double2*>(pr + head);
  double2* pw2 = reinterpret_cast<double2*>(pw + head);
  double2* __restrict__ s2 = reinterpret_cast<double2*>(s + head);
  const double2* __restrict__ w2 = reinterpret_cast<const double2*>(w + head);
  for (int64_t i = gtid; i < n2; i += stride) {
    const double2 rv = r2[i], wv = w2[i];
    double2 pv = rv, sv = wv;
    if (!first) {
      const double2 pov = pr2[i], sov = s2[i];
      pv = make_double2(fma(beta, pov.x, rv.x), fma(beta, pov.y, rv.y));
      sv = make_double2(fma(beta, sov.x, wv.x), fma(beta, sov.y, wv.y));
    }
    pw2[i] = pv;
    s2[i] = sv;
    if (NOLD >= 0) {
      double2 xv = x2[i];
#pragma unroll
      for (int k = 0; k < (NOLD > 0 ? NOLD : 0); ++k) {
        const double2 o = reinterpret_cast<const double2*>(po.p[k] + head)[i];
        xv.x = fma(ah[k], o.x, xv.x);
        xv.y = fma(ah[k], o.y, xv.y);
      }
      x2[i] = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
    }
    r2[i] = make_double2(fma(-alpha, sv.x, rv.x), fma(-alpha, sv.y, rv.y));
  }
  if (((n - head) & 1) && gtid == stride - 1) one(n - 1);
  double tot;
  if (last_block_reduce(0.0, red, sh, &tot)) {  // every block has read the scalars
    sc->rr = gam;
    sc->alpha = alpha;
    sc->first = 0;
    const int it = sc->it + 1;
    sc->it = it;
    if (it >= sc->maxit) sc->done = 3;
  }
}

// p_next = r + beta p (pw = pr: in place; a ring buffer of the deferred x update otherwise)
__global__ void __launch_bounds__(kVecThreads) cg_pupdate_kernel(const double* __restrict__ r,
                                                                 const double* pr, double* pw, int64_t n,
                                                                 CgScalars* sc, Reduce red) {
  __shared__ double sh[32];
  if (sc->done) return;
  const double rr_new = sc->rr_new;
  const double beta = rr_new / sc->rr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    pw[i] = fma(beta, pr[i], r[i]);
  double tot;
  if (last_block_reduce(0.0, red, sh, &tot)) {
    // all blocks have read rr / rr_new: advance the recurrence
    sc->rr = rr_new;
    const int it = sc->it + 1;
    sc->it = it;
    if (rr_new == 0.0 || rr_new <= sc->stop_rr)
      sc->done = 1;
    else if (it >= sc->maxit)
      sc->done = 3;
  }
}

__global__ void __launch_bounds__(kVecThreads) dot_kernel(const double* __restrict__ a,
                                                          const double* __restrict__ b, int64_t n,
                                                          double* out, Reduce red) {
  __shared__ double sh[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    acc = fma(a[i], b[i], acc);
  double bs = block_sum(acc, sh);
  double tot;
  if (last_block_reduce(bs, red, sh, &tot)) *out = tot;
}

// dot_mode 1 (separate dot kernels): 16-B loads like the update kernel, deterministic reduction
__global__ void __launch_bounds__(kVecThreads) cg_dot_kernel(const double* __restrict__ a,
                                                             const double* __restrict__ b, int64_t n,
                                                             int which, CgScalars* sc, Reduce red) {
  __shared__ double sh[32];
  if (sc->done) return;
  double acc = 0.0;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t head = (reinterpret_cast<uintptr_t>(a) & 15) ? 1 : 0;
  if (head && gtid == 0 && n > 0) acc = a[0] * b[0];
  const int64_t n2 = (n - head) / 2;
  const double2* __restrict__ a2 = reinterpret_cast<const double2*>(a + head);
  const double2* __restrict__ b2 = reinterpret_cast<const double2*>(b + head);
  for (int64_t i = gtid; i < n2; i += stride) {
    const double2 u = a2[i], v = b2[i];
    acc = fma(u.x, v.x, acc);
    acc = fma(u.y, v.y, acc);
  }
  if (((n - head) & 1) && gtid == stride - 1) acc = fma(a[n - 1], b[n - 1], acc);
  const double bs = block_sum(acc, sh);
  double tot;
  if (last_block_reduce(bs, red, sh, &tot)) {
    if (which == 0) {  // p.q; the apply has finished reading rr / rr_new / first
      sc->pq = tot;
      sc->rr = sc->rr_new;
      sc->first = 0;
    } else {  // r.r of the update (local partial: the allreduce follows)
      sc->rr_new = tot;
      const int it = sc->it + 1;
      sc->it = it;
      if (it >= sc->maxit) sc->done = 3;
    }
  }
}

__global__ void loop_sum_kernel(const double* __restrict__ stage, int P, int stride, int count,
                                double* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= count) return;
  double v = 0.0;
  for (int q = 0; q < P; ++q) v += stage[q * stride + i];
  out[i] = v;
}

__global__ void sub_kernel(const double* __restrict__ b, const double* __restrict__ ax,
                           double* __restrict__ out, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = b[i] - ax[i];
}

__global__ void check_material_kernel(const double2* __restrict__ lm, int64_t n,
                                      unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const double l = lm[i].x, m = lm[i].y;
    // mu > 0 and lambda + 2 mu / 3 >= 0, finite
    const bool ok = isfinite(l) && isfinite(m) && m > 0.0 && (l + 2.0 * m / 3.0) >= 0.0;
    cnt += ok ? 0 : 1;
  }
  if (cnt) atomicAdd(bad, cnt);  // validation counter only (not on the apply path)
}

cudaError_t launch_cg_init(const double* b, const double* ax, double* r, double* p, int64_t n,
                           CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  cg_init_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(b, ax, r, p, n, sc, red);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cg_finish_init(CgScalars* sc, double tol, int maxit, cudaStream_t s) {
  cg_finish_init_kernel<<<1, 1, 0, s>>>(sc, tol, maxit);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cg_update(double* x, double* r, const double* p, const double* q, int64_t n,
                             CgScalars* sc, Reduce red, cudaStream_t s, int sm_count, int nold,
                             const double* const* pold, int jpend) {
  const unsigned nb = vec_blocks(n, sm_count);  // (the same grid for every nold: the r.r grouping, hence x, is independent of x_defer)
  OldP po{{p, p, p, p, p, p, p}};
  for (int k = 0; k < nold && k < 7; ++k) po.p[k] = pold[k];
  switch (nold) {
    case -1: cg_update_kernel<-1><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, jpend); break;
    case 0: cg_update_kernel<0><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 1: cg_update_kernel<1><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 3: cg_update_kernel<3><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 7: cg_update_kernel<7><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    default: return cudaErrorInvalidValue;
  }
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cg_update_fused(double* x, double* r, const double* p, const double* q, int64_t n,
                                   CgScalars* sc, Reduce red, cudaStream_t s, int sm_count, int nold,
                                   const double* const* pold, int jpend) {
  const unsigned nb = vec_blocks(n, sm_count);  // (the same grid for every nold: the r.r grouping, hence x, is independent of x_defer)
  OldP po{{p, p, p, p, p, p, p}};
  for (int k = 0; k < nold && k < 7; ++k) po.p[k] = pold[k];
  switch (nold) {
    case -1: cg_update_fused_kernel<-1><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, jpend); break;
    case 0: cg_update_fused_kernel<0><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 1: cg_update_fused_kernel<1><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 3: cg_update_fused_kernel<3><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    case 7: cg_update_fused_kernel<7><<<nb, kVecThreads, 0, s>>>(x, r, p, q, n, sc, red, po, 0); break;
    default: return cudaErrorInvalidValue;
  }
  add_launches(1);
  return cudaGetLastError();
}

// deferred x update, end of a solve: the xp pending updates x += alpha_j P_j, in order
__global__ void __launch_bounds__(kVecThreads) cg_xdefer_flush_kernel(double* __restrict__ x, OldP po, int64_t n,
                                                                      const CgScalars* sc) {
  const int np = sc->xp;
  if (np <= 0) return;
  double ah[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) ah[k] = k < np ? sc->alpha_h[k] : 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double xv = x[i];
    for (int k = 0; k < np && k < 7; ++k) xv = fma(ah[k], po.p[k][i], xv);
    x[i] = xv;
  }
}
cudaError_t launch_cg_xdefer_flush(double* x, const double* const* pend, int64_t n, const CgScalars* sc,
                                   cudaStream_t s, int sm_count) {
  OldP po{{pend[0], pend[1], pend[2], pend[3], pend[4], pend[5], pend[6]}};
  cg_xdefer_flush_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(x, po, n, sc);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cg_cgcg_update(double* x, double* r, const double* pr, double* pw, double* s, const double* w,
                                  int64_t n, CgScalars* sc, Reduce red, cudaStream_t st, int sm_count, int nold,
                                  const double* const* pold, int jpend) {
  const unsigned nb = vec_blocks(n, sm_count);  // (the same grid for every nold: the r.r grouping, hence x, is independent of x_defer)
  OldP po{{pr, pr, pr, pr, pr, pr, pr}};
  for (int k = 0; k < nold && k < 7; ++k) po.p[k] = pold[k];
  switch (nold) {
    case -1: cg_cgcg_update_kernel<-1><<<nb, kVecThreads, 0, st>>>(x, r, pr, pw, s, w, n, sc, red, po, jpend); break;
    case 0: cg_cgcg_update_kernel<0><<<nb, kVecThreads, 0, st>>>(x, r, pr, pw, s, w, n, sc, red, po, 0); break;
    case 1: cg_cgcg_update_kernel<1><<<nb, kVecThreads, 0, st>>>(x, r, pr, pw, s, w, n, sc, red, po, 0); break;
    case 3: cg_cgcg_update_kernel<3><<<nb, kVecThreads, 0, st>>>(x, r, pr, pw, s, w, n, sc, red, po, 0); break;
    case 7: cg_cgcg_update_kernel<7><<<nb, kVecThreads, 0, st>>>(x, r, pr, pw, s, w, n, sc, red, po, 0); break;
    default: return cudaErrorInvalidValue;
  }
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cg_pupdate(const double* r, const double* pr, double* pw, int64_t n, CgScalars* sc, Reduce red,
                              cudaStream_t s, int sm_count) {
  cg_pupdate_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(r, pr, pw, n, sc, red);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_dot(const double* a, const double* b, int64_t n, double* out, Reduce red,
                       cudaStream_t s, int sm_count) {
  dot_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(a, b, n, out, red);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_cg_dot(const double* a, const double* b, int64_t n, int which, CgScalars* sc, Reduce red,
                          cudaStream_t s, int sm_count) {
  Reduce r = red;
  r.dot_mode = 0;
  cg_dot_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(a, b, n, which, sc, r);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_loop_sum(const double* stage, int P, int stride, int count, double* out, cudaStream_t s) {
  loop_sum_kernel<<<1, 32, 0, s>>>(stage, P, stride, count, out);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_sub(const double* b, const double* ax, double* out, int64_t n, cudaStream_t s,
                       int sm_count) {
  sub_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(b, ax, out, n);
  add_launches(1);
  return cudaGetLastError();
}
cudaError_t launch_check_material(const double2* lm, int64_t n, unsigned long long* bad,
                                  cudaStream_t s, int sm_count) {
  check_material_kernel<<<vec_blocks(n, sm_count), kVecThreads, 0, s>>>(lm, n, bad);
  add_launches(1);
  return cudaGetLastError();
}

}  // namespace fem

namespace fem {
// dense ABI layout <-> library padded layout for n_planes planes:
// dense (i,j,k,c) at ((k*nyn + j)*nxn + i)*C + c; padded at k*ppitch + j*rpitch + i*C + c.
__global__ void pack_kernel(const double* __restrict__ dense, double* __restrict__ padded,
                            int64_t rpitch, int64_t ppitch, int64_t n_planes, int64_t nxn,
                            int64_t nyn, int comps, int to_padded) {
  const int64_t rowlen = nxn * comps;
  const int64_t nrows = n_planes * nyn;
  // one warp-strided pass per row
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nrows; r += warps) {
    const int64_t k = r / nyn, j = r - k * nyn;
    const double* d = dense + r * rowlen;
    double* pd = padded + k * ppitch + j * rpitch;
    if (to_padded)
      for (int64_t e = lane; e < rowlen; e += 32) pd[e] = d[e];
    else
      for (int64_t e = lane; e < rowlen; e += 32) const_cast<double*>(d)[e] = pd[e];
  }
}

cudaError_t launch_pack(const double* dense, double* padded, int64_t rpitch, int64_t ppitch,
                        int64_t n_planes, int64_t nxn, int64_t nyn, int comps, int to_padded,
                        cudaStream_t s, int sm_count) {
  pack_kernel<<<(unsigned)sm_count * 8, 256, 0, s>>>(dense, padded, rpitch, ppitch, n_planes, nxn,
                                                      nyn, comps, to_padded);
  add_launches(1);
  return cudaGetLastError();
}
}  // namespace fem
