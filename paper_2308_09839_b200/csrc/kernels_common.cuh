// kernels_common.cuh -- node-plane staging shared by the apply kernels (sm_100a).
//
// A CTA marches along z over node planes.  Plane k's halo tile (ROWS rows x COLS node columns x
// C components) is copied into a ring slot of shared memory by one warp: lane r issues ONE bulk
// copy (cp.async.bulk, the TMA copy engine; SASS UBLKCP) for the 16-B aligned middle of row r
// and at most two 8-B cp.async for its ragged ends, all completing on the slot's mbarrier.  The
// caller's vectors keep the dense ABI layout whose rows are only 8-B aligned (e.g. 257 or 385
// nodes per row), which is why tiled TMA tensor maps (16-B strides) are not used.
//
// Masking: only DOFs that the operator may read are copied -- domain nodes, and with the
// Dirichlet box only interior nodes.  Every other position of the ring is zero: zeroed
// once at kernel start, and the two positions adjacent to a row's valid range are re-zeroed per
// copy (the per-row 8-B alignment shift `lead` can differ between planes).  Planes with no
// operator data (outside the box, or a Dirichlet face plane) are served from a permanent zero
// slot.  The consumer therefore reads without any per-element mask.
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

// Ring of S plane slots + one zero slot.  Slot layout: ROWS rows of PITCH doubles (PITCH even,
// >= COLS*C + 4); a row's data starts at element lead[slot][row] in {2, 3} (+ col*C + comp).
// full[s]: completes when plane data landed (ROWS+1 arrivals + tx bytes);
// empty[s]: completes when the NCW consumer warps released the slot.
template <int ROWS, int COLS, int C, int S>
struct PlaneRing {
  static constexpr int PITCH = ((COLS * C + 4) + 1) & ~1;
  static constexpr int SLOT = ROWS * PITCH;
  static constexpr size_t BYTES = (size_t)(S + 1) * SLOT * sizeof(double);  // + zero slot
  static constexpr size_t META = 2 * S * sizeof(uint64_t) + ((S + 1) * ROWS + S) * sizeof(int);
  static_assert(ROWS <= 32, "one producer lane per row");
  static_assert((S & (S - 1)) == 0, "S must be a power of two");

  double* buf;      // (S+1) * SLOT doubles, 16-B aligned; slot S is the zero slot
  uint64_t* full;   // S mbarriers
  uint64_t* empty;  // S mbarriers
  int* lead;        // (S+1) * ROWS
  int* valid;       // S: plane holds operator data

  __device__ __forceinline__ void carve(unsigned char* ring_base, unsigned char* meta_base) {
    buf = reinterpret_cast<double*>(ring_base);
    full = reinterpret_cast<uint64_t*>(meta_base);
    empty = full + S;
    lead = reinterpret_cast<int*>(empty + S);
    valid = lead + (S + 1) * ROWS;
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

  // producer warp: stream planes pfirst .. plast through the ring
  __device__ __forceinline__ void produce(const PlaneSrc& x, const Grid& g, int64_t pfirst, int64_t plast,
                                          int64_t ilo, int64_t jlo, int bc, int lane) {
#pragma unroll 1
    for (int64_t p = pfirst; p <= plast; ++p) {
      const int t = (int)(p - pfirst);
      const int s = t & (S - 1);
      if (t >= S) mbar_wait(&empty[s], (uint32_t)(((t / S) - 1) & 1));
      issue(s, x, g, p, ilo, jlo, bc, lane);
    }
  }

  // consumer warp: release slot s after its last read
  __device__ __forceinline__ void release(int s, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  // warp 0 only (all 32 lanes): copy node plane k into slot s.
  //   ilo, jlo: global node index of tile column 0 / row 0 (may be -1)
  __device__ __forceinline__ void issue(int s, const PlaneSrc& x, const Grid& g, int64_t k,
                                        int64_t ilo, int64_t jlo, int bc, int lane) {
    fence_proxy_async();  // order earlier generic reads of this slot before the async writes
    const double* base = plane_ptr(x, g, k, C);
    const bool pvalid = base != nullptr && !(bc && (k == 0 || k == g.nz));
    const int64_t imin = bc ? 1 : 0, imax = bc ? g.nx - 1 : g.nx;
    const int64_t jmin = bc ? 1 : 0, jmax = bc ? g.ny - 1 : g.ny;
    const int64_t j = jlo + lane;
    const int64_t ca = max(ilo, imin), cb = min(ilo + COLS - 1, imax);
    uint32_t bytes = 0;
    uintptr_t A0 = 0, A1 = 0, B0 = 0, B1 = 0;
    int ld = 2;
    const bool rvalid = pvalid && lane < ROWS && j >= jmin && j <= jmax && cb >= ca;
    double* row = buf + (size_t)s * SLOT + lane * PITCH;
    if (rvalid) {
      const int64_t rowoff = j * (g.nx + 1);
      const uintptr_t V0 = (uintptr_t)(base + (rowoff + ilo) * C);  // virtual column 0
      A0 = (uintptr_t)(base + (rowoff + ca) * C);
      A1 = (uintptr_t)(base + (rowoff + cb + 1) * C);
      B0 = (A0 + 15) & ~(uintptr_t)15;
      B1 = A1 & ~(uintptr_t)15;
      ld = 2 + (int)((V0 >> 3) & 1);
      if (B1 > B0) bytes = (uint32_t)(B1 - B0);
      lead[s * ROWS + lane] = ld;
      // re-zero the neighbours of the valid range (shift may differ from the last use)
      const int v0 = ld + (int)((A0 - V0) >> 3), v1 = ld + (int)((A1 - V0) >> 3);
      if (v0 - 1 >= 0) row[v0 - 1] = 0.0;
      if (v1 < PITCH) row[v1] = 0.0;
    }
    if (lane == 0) valid[s] = pvalid ? 1 : 0;
    // total bytes of the bulk copies -> expect_tx before any copy is issued
    uint32_t tot = bytes;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane == 0) mbar_arrive_expect_tx(&full[s], tot);
    __syncwarp();
    if (rvalid) {
      const uintptr_t V0 = (uintptr_t)(base + (j * (g.nx + 1) + ilo) * C);
      auto dst = [&](uintptr_t a) { return row + ld + (int)((a - V0) >> 3); };
      if (bytes) bulk_g2s(dst(B0), (const void*)B0, bytes, &full[s]);
      if ((A0 & 15) && A0 < A1) cp_async8(dst(A0), (const void*)A0);
      if ((A1 & 15) && B1 >= A0) cp_async8(dst(B1), (const void*)B1);
    }
    if (lane < ROWS) cp_async_arrive_noinc(&full[s]);
  }

  // consumers: wait until slot s holds its plane (phase parity ph)
  __device__ __forceinline__ void wait(int s, uint32_t ph) { mbar_wait(&full[s], ph); }

  // base of row r of slot s for reading (zero slot if the plane has no operator data)
  __device__ __forceinline__ const double* row_ptr(int s, int r) const {
    const int ss = valid[s] ? s : S;
    return buf + (size_t)ss * SLOT + r * PITCH + lead[ss * ROWS + r];
  }
};

}  // namespace fem
