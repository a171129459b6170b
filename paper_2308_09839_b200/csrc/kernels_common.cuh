// kernels_common.cuh -- node-plane staging shared by the apply kernels (sm_100a).
//
// A CTA marches along z over node planes.  A dedicated producer warp streams plane k's halo tile
// (ROWS rows x COLS node columns x C components) into a ring slot of shared memory: lane r issues
// ONE bulk copy (cp.async.bulk, the TMA copy engine; SASS UBLKCP) for the 16-B aligned middle of
// row r and at most two 8-B cp.async for its ragged ends, all completing on the slot's `full`
// mbarrier; consumer warps release a slot through its `empty` mbarrier (no CTA-wide barrier).
// The caller's vectors keep the dense ABI layout whose rows are only 8-B aligned (257 or 385
// nodes per row), which is why tiled TMA tensor maps (16-B strides) are not used.  Per-row copy
// descriptors are computed once per CTA; per plane the producer only adds the plane base.
//
// Masking: only DOFs that the operator may read are copied -- domain nodes, and with the
// Dirichlet box only interior nodes.  Every other position of the ring is zero: zeroed
// once at kernel start, and the two positions adjacent to a row's valid range are re-zeroed per
// copy (the 8-B alignment shift `lead` of a row can differ between planes).  Planes with no
// operator data (outside the box, or a Dirichlet face plane) are served from a permanent zero
// slot.  The consumer therefore reads without any per-element mask.
//
// Optional second stream (elasticity): the cell-material layer k (lambda, mu interleaved as
// double2, always 16-B aligned) is copied with the same slot, one bulk copy per cell row.
#pragma once
#include "fem_internal.cuh"

namespace fem {

// Pointer to node plane k of a plane-indexed vector (nullptr: outside the domain / not held).
__device__ __forceinline__ const double* plane_ptr(const PlaneSrc& x, const Grid& g, int64_t k,
                                                   int comps) {
  if (k < 0 || k > g.nz) return nullptr;
  if (k >= g.k0 && k < g.k1) return x.main + (k - g.k0) * g.plane * comps;
  if (k == g.k0 - 1) return x.lo;
  if (k == g.k1) return x.hi;
  return nullptr;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Optional material stream (elasticity): interleaved (lambda, mu) per cell, cell layers.
struct MatSrc {
  const double2* lm;  // cell (i,j,k) at lm[(k - layer0) * nx * ny + j * nx + i]; nullptr: none
  int64_t layer0;
};

// Ring of S plane slots + one zero slot.  Slot layout: ROWS rows of PITCH doubles (PITCH even,
// >= COLS*C + 4); a row's data starts at element lead[slot][row] in {2, 3} (+ col*C + comp).
// With MROWS > 0 each slot also holds MROWS x MCOLS double2 of material.
// full[s]: completes when plane data landed (ROWS+1 arrivals + tx bytes);
// empty[s]: completes when the consumer warps released the slot.
template <int ROWS, int COLS, int C, int S, int MROWS = 0, int MCOLS = 0>
struct PlaneRing {
  static constexpr int PITCH = ((COLS * C + 4) + 1) & ~1;
  static constexpr int SLOT = ROWS * PITCH + 2 * MROWS * MCOLS;  // doubles
  static constexpr size_t BYTES = (size_t)(S + 1) * SLOT * sizeof(double);  // + zero slot
  static constexpr size_t META = 2 * S * sizeof(uint64_t) + ((S + 1) * ROWS + 2 * S) * sizeof(int);
  static_assert(ROWS <= 32 && MROWS <= 32, "one producer lane per row");
  static_assert((S & (S - 1)) == 0, "S must be a power of two");

  double* buf;      // (S+1) * SLOT doubles, 16-B aligned; slot S is the zero slot
  uint64_t* full;   // S mbarriers
  uint64_t* empty;  // S mbarriers
  int* lead;        // (S+1) * ROWS
  int* valid;       // S: plane holds operator data
  int* mvalid;      // S: material layer present

  __device__ __forceinline__ void carve(unsigned char* ring_base, unsigned char* meta_base) {
    buf = reinterpret_cast<double*>(ring_base);
    full = reinterpret_cast<uint64_t*>(meta_base);
    empty = full + S;
    lead = reinterpret_cast<int*>(empty + S);
    valid = lead + (S + 1) * ROWS;
    mvalid = valid + S;
  }

  // all threads: zero the ring, init barriers; ends with __syncthreads
  __device__ __forceinline__ void init(int tid, int nthreads, int n_consumer_warps) {
    double2* b2 = reinterpret_cast<double2*>(buf);
    for (int t = tid; t < (S + 1) * SLOT / 2; t += nthreads) b2[t] = make_double2(0.0, 0.0);
    for (int t = tid; t < (S + 1) * ROWS; t += nthreads) lead[t] = 2;
    if (tid == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], ROWS + 1);
        mbar_init(&empty[s], n_consumer_warps);
      }
      fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();
  }

  // producer warp: stream planes pfirst .. plast (and material layers) through the ring.
  //   ilo, jlo: global node index of tile column 0 / row 0 (may be -1); material tile cells
  //   start at (ilo, jlo) too.
  __device__ __forceinline__ void produce(const PlaneSrc& x, const Grid& g, int64_t pfirst, int64_t plast,
                                          int64_t ilo, int64_t jlo, int bc, int lane, MatSrc mat) {
    // ---- per-lane row descriptors (plane independent) ----
    const int64_t imin = bc ? 1 : 0, imax = bc ? g.nx - 1 : g.nx;
    const int64_t jmin = bc ? 1 : 0, jmax = bc ? g.ny - 1 : g.ny;
    const int64_t j = jlo + lane;
    const int64_t ca = max(ilo, imin), cb = min(ilo + COLS - 1, imax);
    const bool rvalid = lane < ROWS && j >= jmin && j <= jmax && cb >= ca;
    const int64_t offV = (j * (g.nx + 1) + ilo) * C;  // element offset of virtual column 0
    const int64_t offA0 = (j * (g.nx + 1) + ca) * C;
    const int64_t offA1 = (j * (g.nx + 1) + cb + 1) * C;
    // bytes of this row's bulk copy for an even / odd plane base element index
    uint32_t rb[2];
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const uint64_t a0 = (uint64_t)(offA0 + par) * 8, a1 = (uint64_t)(offA1 + par) * 8;
      const uint64_t b0 = (a0 + 15) & ~15ull, b1 = a1 & ~15ull;
      rb[par] = (rvalid && b1 > b0) ? (uint32_t)(b1 - b0) : 0u;
    }
    uint32_t tot0 = rb[0], tot1 = rb[1];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tot0 += __shfl_xor_sync(0xffffffffu, tot0, o);
      tot1 += __shfl_xor_sync(0xffffffffu, tot1, o);
    }
    // material rows (cells): lane r = cell row jlo + r, cells [max(ilo,0), min(ilo+MCOLS-1, nx-1)]
    const int64_t mi0 = max(ilo, (int64_t)0), mi1 = min(ilo + MCOLS - 1, g.nx - 1);
    const bool mrow = MROWS > 0 && mat.lm != nullptr && lane < MROWS && j >= 0 && j < g.ny && mi1 >= mi0;
    const uint32_t mbytes = mrow ? (uint32_t)((mi1 - mi0 + 1) * 16) : 0u;
    uint32_t mtot = mbytes;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mtot += __shfl_xor_sync(0xffffffffu, mtot, o);
    const int64_t moff = j * g.nx + mi0;
    const int mdst = (int)(mi0 - ilo);

#pragma unroll 1
    for (int64_t p = pfirst; p <= plast; ++p) {
      const int t = (int)(p - pfirst);
      const int s = t & (S - 1);
      if (t >= S) mbar_wait(&empty[s], (uint32_t)(((t / S) - 1) & 1));
      fence_proxy_async();
      const double* base = plane_ptr(x, g, p, C);
      const bool pvalid = base != nullptr && !(bc && (p == 0 || p == g.nz));
      const bool mlayer = MROWS > 0 && mat.lm != nullptr && p >= 0 && p < g.nz;
      const int par = (int)(((uintptr_t)base >> 3) & 1);
      double* row = buf + (size_t)s * SLOT + lane * PITCH;
      const bool go = pvalid && rvalid;
      uintptr_t A0 = 0, A1 = 0, B0 = 0, B1 = 0, V0 = 0;
      int ld = 2;
      if (go) {
        V0 = (uintptr_t)(base + offV);
        A0 = (uintptr_t)(base + offA0);
        A1 = (uintptr_t)(base + offA1);
        B0 = (A0 + 15) & ~(uintptr_t)15;
        B1 = A1 & ~(uintptr_t)15;
        ld = 2 + (int)((V0 >> 3) & 1);
        lead[s * ROWS + lane] = ld;
        const int v0 = ld + (int)((A0 - V0) >> 3), v1 = ld + (int)((A1 - V0) >> 3);
        if (v0 >= 1) row[v0 - 1] = 0.0;
        if (v1 < PITCH) row[v1] = 0.0;
      }
      if (lane == 0) {
        valid[s] = pvalid ? 1 : 0;
        mvalid[s] = mlayer ? 1 : 0;
        mbar_arrive_expect_tx(&full[s], (pvalid ? (par ? tot1 : tot0) : 0u) + (mlayer ? mtot : 0u));
      }
      __syncwarp();
      if (go) {
        auto dst = [&](uintptr_t a) { return row + ld + (int)((a - V0) >> 3); };
        if (B1 > B0) bulk_g2s(dst(B0), (const void*)B0, (uint32_t)(B1 - B0), &full[s]);
        if ((A0 & 15) && A0 < A1) cp_async8(dst(A0), (const void*)A0);
        if ((A1 & 15) && B1 >= A0) cp_async8(dst(B1), (const void*)B1);
      }
      if (MROWS > 0 && mlayer && mrow) {
        double2* md = reinterpret_cast<double2*>(buf + (size_t)s * SLOT + ROWS * PITCH) + lane * MCOLS + mdst;
        bulk_g2s(md, mat.lm + (p - mat.layer0) * g.nx * g.ny + moff, mbytes, &full[s]);
      }
      if (lane < ROWS) cp_async_arrive_noinc(&full[s]);
    }
  }

  // consumers: wait until slot s holds its plane (phase parity ph)
  __device__ __forceinline__ void wait(int s, uint32_t ph) { mbar_wait(&full[s], ph); }

  // consumer warp: release slot s after its last read
  __device__ __forceinline__ void release(int s, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // base of row r of slot s for reading (zero slot if the plane has no operator data)
  __device__ __forceinline__ const double* row_ptr(int s, int r) const {
    const int ss = valid[s] ? s : S;
    return buf + (size_t)ss * SLOT + r * PITCH + lead[ss * ROWS + r];
  }
  // material (lambda, mu) of tile cell (col, row) in slot s; zeros outside the box
  __device__ __forceinline__ double2 mat(int s, int row, int col) const {
    const int ss = mvalid[s] ? s : S;
    return reinterpret_cast<const double2*>(buf + (size_t)ss * SLOT + ROWS * PITCH)[row * MCOLS + col];
  }
};

}  // namespace fem
