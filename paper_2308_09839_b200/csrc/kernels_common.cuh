// kernels_common.cuh -- node-plane staging shared by the apply kernels (sm_100a).
//
// A CTA marches along z over node planes.  A dedicated producer warp streams each plane's halo
// tile (ROWS rows x COLS node columns x C components) into a ring slot of shared memory; consumer
// warps wait on the slot's `full` mbarrier and release it through its `empty` mbarrier (no
// CTA-wide barrier on the data path).  Two staging policies for the u plane:
//
//  * TM = true  (library-internal "padded layout", used inside CG): ONE TMA tensor copy per plane
//    (cp.async.bulk.tensor.3d, SASS UTMALDG) of a ROWS x BOXW box.  The tensor map describes only
//    the nodes the operator may read (the interior with the Dirichlet box), so TMA's
//    out-of-bounds zero fill IS the mask P of y = P A P x + (I-P) x and the domain-edge padding.
//  * TM = false (caller vectors in the dense ABI layout, rows only 8-B aligned e.g. 257/385
//    nodes, which tensor maps cannot describe): lane r issues one bulk copy (cp.async.bulk, SASS
//    UBLKCP) for the 16-B aligned middle of row r and <= 2 8-B cp.async for its ragged ends.  Only
//    readable nodes are copied; every other ring position is zero (zeroed at start, the two
//    positions next to a row's valid range re-zeroed per copy because the 8-B shift `lead` can
//    change between planes; planes without operator data are served from a zero slot).
//
// Measured on this pool (tools/microbench/bulk_copy.cu, profiles/r01_microbench_bulk_copy.txt):
// the copy engine accepts ~65 bulk copies / us / SM, so copies must be >= 1 KB to reach HBM
// bandwidth -- the reason for the tensor path (one copy per plane) inside CG.
//
// Optional material stream (elasticity): the cell layer k of interleaved (lambda, mu) is fetched
// with the same slot by one TMA tensor copy (cells outside the box read as zero -> no
// contribution).
#pragma once
#include <cuda.h>

#include <algorithm>

#include "fem_internal.cuh"

namespace fem {

// Pointer to node plane k of a plane-indexed vector (nullptr: outside the domain / not held).
__device__ __forceinline__ const double* plane_ptr(const PlaneSrc& x, const Grid& g, int64_t k) {
  if (k < 0 || k > g.nz) return nullptr;
  if (k >= g.k0 && k < g.k1) return x.main + (k - g.k0) * x.ppitch;
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
// Wait for phase `parity` of an mbarrier.  The suspend-time hint lets the hardware park the warp
// until the phase completes instead of spinning on issue slots (warps that run ahead of the
// slowest consumer otherwise burn the issue bandwidth the slow warps need).
#ifndef FEM_WAIT_HINT
#define FEM_WAIT_HINT 1
#endif
__device__ __forceinline__ void mbar_wait_a(uint32_t addr, uint32_t parity) {
#if !FEM_WAIT_HINT
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(1000000)
      : "memory");
}
#ifndef FEM_REFILL_FENCE
#define FEM_REFILL_FENCE 1  // fence.proxy.async before every TMA refill of a released ring slot
#endif
#ifndef FEM_RING_FENCE
#define FEM_RING_FENCE 0
#endif
__device__ __forceinline__ void mbar_arrive_a(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(addr) : "memory");
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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Launch geometry of an apply: xt x yt tiles, zc z-chunks of kchunk node planes each.
struct WorkGrid {
  int xt, yt, zc;      // tiles in x, y; z-chunks
  int64_t kchunk;      // node planes per z-chunk
  __device__ __forceinline__ int items() const { return xt * yt * zc; }
};

// Host: choose the z-chunking so that the items (xt*yt*zc) spread evenly over `slots` resident
// CTAs (minimise the idle fraction of the last round), with chunks of >= min_chunk planes and at
// least min_rounds rounds of CTAs when the mesh allows it.
inline WorkGrid make_workgrid(int xt, int yt, int64_t nplanes, int64_t slots, int64_t min_chunk,
                              int64_t min_rounds = 1) {
  WorkGrid best{xt, yt, 1, nplanes};
  double best_eff = -1.0;
  const int64_t tiles = (int64_t)xt * yt;
  const int64_t zmax = std::max<int64_t>(1, nplanes / min_chunk);
  for (int64_t zc = 1; zc <= zmax; ++zc) {
    const int64_t kchunk = (nplanes + zc - 1) / zc;
    const int64_t z = (nplanes + kchunk - 1) / kchunk;
    const int64_t items = tiles * z;
    const int64_t rounds = (items + slots - 1) / slots;
    if (rounds < min_rounds && zc < zmax) continue;  // keep enough CTAs to balance the SMs
    // useful work / (rounds * slots * chunk length incl. the 2-plane halo)
    const double eff = (double)nplanes * tiles / ((double)rounds * slots * (kchunk + 2));
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = WorkGrid{xt, yt, (int)z, kchunk};
    }
  }
  return best;
}

// Host: cover n nodes with tiles of at most tmax, all tiles (but possibly the last) equally wide:
// returns the tile count, *per = nodes per tile.  (257 nodes at tmax 32 -> 9 tiles of 29 instead
// of 8 x 32 + a 1-node sliver that streams every plane for one column.)
inline int64_t balanced_tiles(int64_t n, int tmax, int* per) {
  const int64_t tiles = (n + tmax - 1) / tmax;
  *per = (int)((n + tiles - 1) / tiles);
  return (n + *per - 1) / *per;
}

// Tensor-map coordinates of a tile: box origin = node (ilo, jlo) of plane k, relative to the
// tensor origin (node (t_i0, t_j0) of plane t_k0).  Out-of-range coordinates zero-fill.
struct TmaOrigin {
  int64_t t_i0, t_j0, t_k0;
};

// Ring of S plane slots.  Slot: u region ROWS x PITCH doubles (+ material MROWS x MPITCH).
//   TM:  PITCH = BOXW (box width, doubles); data at row r, element col*C + comp.
//   !TM: PITCH even >= COLS*C + 4, row data start at lead[slot][row] in {2,3}; slot S = zeros.
// PAIR (TM only): the u tensor is a "row-pair" view of a dense caller vector whose rows are NOT
// 16-B multiples (odd (nx+1) C): dim 0 = elements of two consecutive rows plus the plane parity
// (extent Lp + 2 Lr), dim 1 = row pairs (stride 2 Lr), dim 2 = plane pairs (stride 2 Lp), so all
// strides are 16-B multiples.  A plane tile is TWO boxes: the rows of the parity of row jlo and
// the rows of the other parity, each HR = ceil(ROWS / 2) rows; ring row r lives in box r & 1 at
// box row r >> 1, shifted by the box's 8-B misalignment (set_pair_plane).  Columns / rows past the
// box edge read the neighbouring row: only the Dirichlet identity rows see them (bc = 1 only).
// (PairGeom: fem_internal.cuh)

template <bool TM, int ROWS, int COLS, int C, int S, int MROWS = 0, int MCOLS = 0, int NU = 1,
          bool PAIR = false>
struct PlaneRing {
  // box width: COLS*C rounded to even, +2 so the box can start one element early (the box x
  // origin must be 16-B aligned: odd element offsets are shifted, see tshift)
  static constexpr int BOXW = (((COLS * C) + 1) & ~1) + 2;
  static constexpr int PITCH = TM ? BOXW : (((COLS * C + 4) + 1) & ~1);
  static constexpr int HR = (ROWS + 1) / 2;                          // PAIR: rows per half box
  static constexpr int HALF = ((HR * BOXW) + 15) & ~15;             // PAIR: half-box stride (128 B)
  static constexpr int UDBL = (((PAIR ? 2 * HALF : ROWS * PITCH)) + 15) & ~15;  // 128-B multiple
  static constexpr int MPITCH = 2 * MCOLS;                           // doubles per material row
  static constexpr int MDBL = ((MROWS * MPITCH) + 15) & ~15;
  static constexpr int SLOT = NU * UDBL + MDBL;                      // doubles, 128-B multiple
  static_assert(NU == 1 || TM, "two u boxes only on the tensor path");
  static constexpr int NSLOT = TM ? S : S + 1;
  static constexpr size_t BYTES = (size_t)NSLOT * SLOT * sizeof(double);
  static constexpr size_t META = 2 * S * sizeof(uint64_t) + ((S + 1) * ROWS + 2 * S) * sizeof(int);
  static constexpr uint32_t UBOX_BYTES = (PAIR ? 2 * HR : ROWS) * BOXW * 8;
  static_assert(!PAIR || (TM && NU == 1), "row-pair staging: tensor path, one input box");
  static constexpr uint32_t MBOX_BYTES = MROWS * MPITCH * 8;
  static_assert(TM || ROWS <= 32, "one producer lane per row (row path)");
  static_assert(S >= 2, "at least two ring stages");
  static_assert(ROWS <= 256 && BOXW <= 256 && MPITCH <= 256, "TMA box dims <= 256");

  double* buf;      // NSLOT * SLOT doubles, 128-B aligned
  uint64_t* full;   // S mbarriers
  uint64_t* empty;  // S mbarriers
  int* lead;        // (S+1) * ROWS     (!TM)
  int* valid;       // S               (!TM)
  unsigned* cnt;    // S release counters (refill by the last consumer warp, no producer warp)
  int tshift = 0;   // TM: 1 if the tile's first element sits at an odd offset of the tensor
  int psh0 = 0, psh1 = 0;  // PAIR: 8-B shift of the two half boxes of the current plane
  int64_t pilo = 0, pjlo = 0;  // PAIR: tile origin (node column / row of ring column / row 0)
  PairGeom pg{};
  uint32_t full_a = 0, empty_a = 0;  // shared-window addresses of full[0], empty[0]

  // TM: the box must start at an even element (16 B); returns the (even) x coordinate
  __device__ __forceinline__ int set_tshift(int64_t ilo, const TmaOrigin& uorg) {
    const int64_t ux = (ilo - uorg.t_i0) * C;
    tshift = (int)(ux & 1);
    return (int)(ux - tshift);
  }

  __device__ __forceinline__ void carve(unsigned char* ring_base, unsigned char* meta_base) {
    buf = reinterpret_cast<double*>(ring_base);
    full = reinterpret_cast<uint64_t*>(meta_base);
    empty = full + S;
    full_a = smem_u32(full);
    empty_a = smem_u32(empty);
    lead = reinterpret_cast<int*>(empty + S);
    valid = lead + (S + 1) * ROWS;
    cnt = reinterpret_cast<unsigned*>(valid + S);
  }

  // all threads: zero the ring (row path), init barriers; ends with __syncthreads
  __device__ __forceinline__ void init(int tid, int nthreads, int n_consumer_warps) {
    if (!TM) {
      double2* b2 = reinterpret_cast<double2*>(buf);
      for (int t = tid; t < NSLOT * SLOT / 2; t += nthreads) b2[t] = make_double2(0.0, 0.0);
      for (int t = tid; t < (S + 1) * ROWS; t += nthreads) lead[t] = 2;
    }
    if (tid < S) cnt[tid] = 0u;
    if (tid == 0) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&full[s], TM ? 1 : ROWS + 1);
        mbar_init(&empty[s], n_consumer_warps);
      }
      fence_mbar_init();
    }
    fence_proxy_async();
    __syncthreads();
  }

  // TM, one thread: load plane p (u box(es) + material layer) into ring position t.  (ux, uy):
  // u box origin (set_tshift), (mx, my): material box origin.
  __device__ __forceinline__ void issue_tm(int t, int64_t p, int ux, int uy, int mx, int my, TmaOrigin uorg,
                                           const CUtensorMap* umap, const CUtensorMap* umap2,
                                           const CUtensorMap* mmap, int64_t mlayer0, const PeerMaps* peer) {
    const int s = t % S;
    double* slot = buf + (size_t)s * SLOT;
    mbar_arrive_expect_tx(&full[s], NU * UBOX_BYTES + (MROWS > 0 ? MBOX_BYTES : 0u));
    if (PAIR) {  // two half boxes (row parities); planes outside [k0, nz] read as zeros, except
                 // the ghost planes of a slab (PeerMaps: a row-pair view of a one-plane buffer)
      const CUtensorMap* m = umap;
      int64_t rel = p - pg.k0;
      bool in = p >= pg.k0 && p <= pg.nz;
      if (peer && peer->on && (p == peer->klo || p == peer->khi)) {
        m = (p == peer->klo) ? &peer->lo : &peer->hi;
        rel = 0;
        in = true;
      }
      const int z = in ? (int)(rel >> 1) : -1;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int64_t j = pjlo + b;
        const int64_t d0 = pilo * C + (j & 1) * pg.lr + (rel & 1) * pg.lp;
        tma_load_3d(slot + b * HALF, m, (int)(d0 & ~(int64_t)1), (int)(j >> 1), z, &full[s]);
      }
      if (MROWS > 0) tma_load_3d(slot + UDBL, mmap, mx, my, (int)(p - mlayer0), &full[s]);
      return;
    }
    const CUtensorMap *m1 = umap, *m2 = umap2;
    int z = (int)(p - uorg.t_k0);
    if (peer && peer->on) {  // ghost planes straight from the neighbour's memory
      if (p == peer->klo) { m1 = &peer->lo; m2 = &peer->lo2; z = 0; }
      else if (p == peer->khi) { m1 = &peer->hi; m2 = &peer->hi2; z = 0; }
    }
    tma_load_3d(slot, m1, ux, uy, z, &full[s]);
    if (NU == 2) tma_load_3d(slot + UDBL, m2, ux, uy, z, &full[s]);
    if (MROWS > 0) tma_load_3d(slot + NU * UDBL, mmap, mx, my, (int)(p - mlayer0), &full[s]);
  }
  // TM: wait until every consumer warp released ring position t (slot t % S)
  __device__ __forceinline__ void wait_released(int t) {
    mbar_wait_a(empty_a + 8u * (t % S), (uint32_t)((t / S) & 1));
  }

  // producer warp: stream planes pfirst .. plast (and material layers) through the ring.
  //   ilo, jlo: global node index of tile column 0 / row 0 (may be -1); material tile cells
  //   start at cell (ilo, jlo).  umap / uorg used when TM; mmap: material tensor (or nullptr).
  //   tbase: ring position of plane pfirst (persistent CTAs continue the ring across work items)
  __device__ __forceinline__ void produce(const PlaneSrc& x, const Grid& g, int64_t pfirst, int64_t plast,
                                          int64_t ilo, int64_t jlo, int bc, int lane,
                                          const CUtensorMap* umap, TmaOrigin uorg,
                                          const CUtensorMap* mmap, int64_t mlayer0,
                                          const CUtensorMap* umap2 = nullptr, int tbase = 0,
                                          const PeerMaps* peer = nullptr) {
    if (lane == 0) {
      if (TM) tma_prefetch_desc(umap);
      if (NU == 2) tma_prefetch_desc(umap2);
      if (MROWS > 0) tma_prefetch_desc(mmap);
    }
    // ---- row-path per-lane descriptors (plane independent) ----
    const int64_t imin = bc ? 1 : 0, imax = bc ? g.nx - 1 : g.nx;
    const int64_t jmin = bc ? 1 : 0, jmax = bc ? g.ny - 1 : g.ny;
    const int64_t j = jlo + lane;
    const int64_t ca = max(ilo, imin), cb = min(ilo + COLS - 1, imax);
    const bool rvalid = !TM && lane < ROWS && j >= jmin && j <= jmax && cb >= ca;
    const int64_t offV = j * x.rpitch + ilo * C;  // element offset of virtual column 0
    const int64_t offA0 = j * x.rpitch + ca * C;
    const int64_t offA1 = j * x.rpitch + (cb + 1) * C;
    uint32_t tot0 = 0, tot1 = 0;
    if (!TM) {
      uint32_t rb[2];
#pragma unroll
      for (int par = 0; par < 2; ++par) {
        const uint64_t a0 = (uint64_t)(offA0 + par) * 8, a1 = (uint64_t)(offA1 + par) * 8;
        const uint64_t b0 = (a0 + 15) & ~15ull, b1 = a1 & ~15ull;
        rb[par] = (rvalid && b1 > b0) ? (uint32_t)(b1 - b0) : 0u;
      }
      tot0 = rb[0];
      tot1 = rb[1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tot0 += __shfl_xor_sync(0xffffffffu, tot0, o);
        tot1 += __shfl_xor_sync(0xffffffffu, tot1, o);
      }
    }
    const int ux = TM ? set_tshift(ilo, uorg) : 0, uy = (int)(jlo - uorg.t_j0);
    const int mx = (int)(2 * ilo), my = (int)jlo;

#pragma unroll 1
    for (int64_t p = pfirst; p <= plast; ++p) {
      const int t = tbase + (int)(p - pfirst);
      const int s = t % S;
      if (t >= S) mbar_wait_a(empty_a + 8u * s, (uint32_t)(((t / S) - 1) & 1));
      double* slot = buf + (size_t)s * SLOT;
      if (TM) {
        if (lane == 0) {
          if (FEM_REFILL_FENCE) fence_proxy_async();  // the consumers' generic reads of the slot before the TMA write
          issue_tm(t, p, ux, uy, mx, my, uorg, umap, umap2, mmap, mlayer0, peer);
        }
        continue;
      }
      fence_proxy_async();
      const double* base = plane_ptr(x, g, p);
      const bool pvalid = base != nullptr && !(bc && (p == 0 || p == g.nz));
      const int par = (int)(((uintptr_t)base >> 3) & 1);
      double* row = slot + lane * PITCH;
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
        mbar_arrive_expect_tx(&full[s], (pvalid ? (par ? tot1 : tot0) : 0u) + (MROWS > 0 ? MBOX_BYTES : 0u));
        if (MROWS > 0) tma_load_3d(slot + UDBL, mmap, mx, my, (int)(p - mlayer0), &full[s]);
      }
      __syncwarp();
      if (go) {
        auto dst = [&](uintptr_t a) { return row + ld + (int)((a - V0) >> 3); };
        if (B1 > B0) bulk_g2s(dst(B0), (const void*)B0, (uint32_t)(B1 - B0), &full[s]);
        if ((A0 & 15) && A0 < A1) cp_async8(dst(A0), (const void*)A0);
        if ((A1 & 15) && B1 >= A0) cp_async8(dst(B1), (const void*)B1);
      }
      if (lane < ROWS) cp_async_arrive_noinc(&full[s]);
    }
  }

  // consumers: wait until slot s holds its plane (phase parity ph)
  __device__ __forceinline__ void wait(int s, uint32_t ph) { mbar_wait_a(full_a + 8u * s, ph); }

  // consumer warp, no-producer rings: count this warp's release of slot s; true in the warp whose
  // release was the last of the nwarps consumers (it refills the slot: fence_proxy_async, then
  // issue_tm).  The acq_rel atomic orders every warp's reads of the slot before the refill.
  __device__ __forceinline__ bool release_last(int s, int lane, int nwarps) {
    __syncwarp();
    unsigned last = 0;
    if (lane == 0) {
      unsigned old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n"
                   : "=r"(old) : "r"(smem_u32(cnt + s)) : "memory");
      last = ((old + 1) % (unsigned)nwarps) == 0u;
    }
    return __shfl_sync(0xffffffffu, last, 0) != 0u;
  }

  // release_last split in two (FEM_LAP_LATE_REFILL): the warp's arrive on the slot counter is
  // issued right after its last read of the slot, the "was it the last" test -- which waits for
  // the atomic's return -- only after the plane's arithmetic, so the atomic latency overlaps it
  __device__ __forceinline__ unsigned release_begin(int s, int lane) {
    __syncwarp();
    unsigned old = 0;
    if (lane == 0)
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;\n"
                   : "=r"(old) : "r"(smem_u32(cnt + s)) : "memory");
    return old;
  }
  __device__ __forceinline__ bool release_end(unsigned old, int lane, int nwarps) const {
    const unsigned last = (lane == 0) ? (unsigned)(((old + 1) % (unsigned)nwarps) == 0u) : 0u;
    return __shfl_sync(0xffffffffu, last, 0) != 0u;
  }

  // consumer warp: release slot s after its last read.  (The thread that refills the slot issues
  // fence.proxy.async between observing the release and the TMA: the generic-proxy reads of the
  // slot must be ordered before the async-proxy write.  Without that fence the vector Laplace
  // fused CG at 256^3 sporadically corrupted part of one warp row of one plane -- the TMA refill
  // landed before queued LDS of the releasing warp.  FEM_RING_FENCE=1 adds a consumer-side fence
  // as well: not needed, and 3-5 % slower.)
  __device__ __forceinline__ void release(int s, int lane) {
#if FEM_RING_FENCE
    fence_proxy_async();
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive_a(empty_a + 8u * s);
  }

  // base of row r of slot s for reading the u plane
  // PAIR: tile origin and geometry (all threads), then the shifts of each plane before reading it
  __device__ __forceinline__ void set_pair_tile(int64_t ilo, int64_t jlo, const PairGeom& g) {
    pilo = ilo; pjlo = jlo; pg = g;
  }
  // (ghost planes of a slab, p = k0 - 1 or nz + 1, are served at parity 0 -- PeerMaps)
  __device__ __forceinline__ void set_pair_plane(int64_t p) {
    const int64_t rel = (p >= pg.k0 && p <= pg.nz) ? p - pg.k0 : 0;
    psh0 = (int)((pilo * C + (pjlo & 1) * pg.lr + (rel & 1) * pg.lp) & 1);
    psh1 = (int)((pilo * C + ((pjlo + 1) & 1) * pg.lr + (rel & 1) * pg.lp) & 1);
  }
  __device__ __forceinline__ const double* row_ptr(int s, int r) const {
    if (PAIR) return buf + (size_t)s * SLOT + (r & 1) * HALF + (r >> 1) * BOXW + ((r & 1) ? psh1 : psh0);
    if (TM) return buf + (size_t)s * SLOT + r * PITCH + tshift;  // (second box: + UDBL)
    const int ss = valid[s] ? s : S;
    return buf + (size_t)ss * SLOT + r * PITCH + lead[ss * ROWS + r];
  }
  // material (lambda, mu) of tile cell (col, row) in slot s (zeros outside the box)
  __device__ __forceinline__ double2 mat(int s, int row, int col) const {
    return reinterpret_cast<const double2*>(buf + (size_t)s * SLOT + NU * UDBL)[row * MCOLS + col];
  }
};

}  // namespace fem
