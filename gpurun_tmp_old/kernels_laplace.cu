// kernels_laplace.cu -- scalar / vector Laplace apply y = A_c x (Eq. 7 / Eq. 8).
//
// B200 form: on the uniform box the 2x2x2-Gauss element operator of Eq. 4 is
// exact (the integrand is of degree <= 2 per direction), so the assembled operator is the
// tensor-product sum  A = (h/36) [Kz (x) My (x) Mx + Mz (x) Ky (x) Mx + Mz (x) My (x) Kx]  with
// the unit 1-D stencils  M~ = [1, 2m, 1],  K~ = [-1, m, -1]  (m = number of 1-D elements at the
// node: 2 inside, 1 on a face).  Evaluated node-centrically, no scatter and no atomics:
//   a = Mx x, b = Kx x           (per node row, from smem)
//   c1 = My a, c2 = My b + Ky a  (per node, from the thread's rows)
//   y(k) = (h/36) [Mz c2 + Kz c1] over the register window c(k-1), c(k), c(k+1).
// The CTA marches along z over node planes staged by the producer warp (PlaneRing: one TMA
// tensor copy per plane inside CG, bulk row copies for caller vectors); x is read from HBM once,
// the one-node xy halo from L2.  Vector Laplace (Eq. 8) is the same per component.
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "kernels_common.cuh"

#ifndef FEM_LAP_S3
#define FEM_LAP_S3 4  // ring stages of the vector fused CG apply
#endif
#ifndef FEM_LAP_LATE_REFILL
#define FEM_LAP_LATE_REFILL 1  // self-refilling scalar ring: the last-release test after the plane's arithmetic
#endif
#ifndef FEM_LAP_FORCE_EDGE
#define FEM_LAP_FORCE_EDGE 0  // 1: every CTA takes the Dirichlet-aware march (experiments)
#endif

namespace fem {

// GLL: 2-point Gauss-Lobatto quadrature (BP5/BP6, reading R1): the 1-D mass is
// lumped, M~ = [0, 3m, 0] instead of [1, 2m, 1]; K~ is exact under both rules.
template <bool TM, int MODE, int C, int TX, int TY, int R, int S, bool GLL, bool PAIR = false>
__global__ void __launch_bounds__(TX*(TY + ((TM && (C == 1 ? kLapSelf1 : kLapSelf3)) ? 0 : 1)), (C == 1 ? kLapMinB : kLapMinB3))
    laplace_kernel(Grid g, PlaneSrc x, OutVec yo, const __grid_constant__ CUtensorMap umap,
                   TmaOrigin uorg, const __grid_constant__ CUtensorMap umap2, const double* pold,
                   double* pnew, int bc, int tmint, int64_t kchunk, int64_t kspan, CgScalars* sc, Reduce red,
                   const __grid_constant__ PeerMaps peer, int txa, int rya, PairGeom pg) {
  // tmint = 1: the u tensor spans only the Dirichlet interior (TMA zero fill = the mask P, the
  // identity rows read x from global memory); 0: the tensor spans the whole box, the mask is
  // applied in registers and the identity rows use the staged values (no global loads).
  constexpr int mode = MODE;
  constexpr int NU = (MODE == 2) ? 2 : 1;
  // TY consumer warps (one node column per lane, R node rows each) + 1 producer warp
  // SELF: no producer warp -- the consumer warp that releases the slot of plane t last refills
  // it with plane t+S (Ring::release_last)
  constexpr bool SELF = TM && (C == 1 ? kLapSelf1 : kLapSelf3);
  constexpr int NT = TX * (TY + (SELF ? 0 : 1));
  constexpr int ROWS = TY * R + 2;
  constexpr int COLS = TX + 2;
  using Ring = PlaneRing<TM, ROWS, COLS, C, S, 0, 0, NU, PAIR>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red_sh[32];
  Ring ring;
  ring.carve(smem_raw, smem_raw + Ring::BYTES);

  if (mode >= 1 && sc->done) return;
  // fused CG (mode 2): operator input p = r + beta p_old, beta = rr_new / rr (0 on the first step)
  const double beta = (mode == 2) ? (sc->first ? 0.0 : sc->rr_new / sc->rr) : 0.0;

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + TX * ty;
  // tile = txa <= TX node columns x rya <= TY*R node rows: the launcher balances the tiles over
  // the mesh (e.g. 257 columns = 9 x 29, not 8 x 32 + 1) so no CTA streams planes for a sliver
  const int64_t i0 = (int64_t)blockIdx.x * txa;
  const int64_t j0 = (int64_t)blockIdx.y * rya;
  const int64_t kb = g.k0 + (int64_t)blockIdx.z * kchunk;
  const int64_t ke = min(g.k1, kb + kspan);
  const int64_t pfirst = kb - 1;
  ring.init(tid, NT, TY);
  if (PAIR) ring.set_pair_tile(i0 - 1, j0 - 1, pg);
  const int tux = TM ? ring.set_tshift(i0 - 1, uorg) : 0, tuy = (int)(j0 - 1 - uorg.t_j0);
  const int nplane = (int)(ke - pfirst + 1);
  if (SELF && tid == 0) {  // prologue: the first S planes
    tma_prefetch_desc(&umap);
    if (MODE == 2) tma_prefetch_desc(&umap2);
    for (int t = 0; t < S && t < nplane; ++t)
      ring.issue_tm(t, pfirst + t, tux, tuy, 0, 0, uorg, &umap, &umap2, nullptr, 0, &peer);
  }

  double pq = 0.0, rr2 = 0.0;  // (rr2: mode 3, sum of the input's squares)
  if (!SELF && ty == TY) {
    ring.produce(x, g, pfirst, ke, i0 - 1, j0 - 1, bc, tx, &umap, uorg, nullptr, 0, &umap2, 0, &peer);
  } else {
    const int64_t i = i0 + tx;
    const double h36 = g.h * (1.0 / 36.0);
    // CTAs whose tile (with its one-node halo) and z-chunk stay away from the box faces run the
    // march with constant 1-D multiplicities (m = 2) and without Dirichlet / identity-row logic
#if FEM_LAP_FORCE_EDGE
    const bool edge = true;
#else
    const bool edge = i0 <= 1 || i0 + TX >= g.nx || j0 <= 1 || j0 + TY * R >= g.ny || pfirst <= 0 || ke >= g.nz;
#endif
    auto march = [&](auto mkc) {
      constexpr bool MK = decltype(mkc)::value;
      // per-node 1-D multiplicities m = (#1-D elements touching the node) in x, y
      const double mx = MK ? (double)((i > 0) + (i < g.nx)) : 2.0;
      double my[R];
      bool active[R], bnode_xy[R];
      int64_t off_y[R], off_x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int64_t j = j0 + ty * R + r;
        my[r] = MK ? (double)((j > 0) + (j < g.ny)) : 2.0;
        active[r] = (i <= g.nx) && (j <= g.ny) && tx < txa && ty * R + r < rya;
        bnode_xy[r] = MK && bc && (i == 0 || i == g.nx || j == 0 || j == g.ny);
        off_y[r] = j * yo.rpitch + i * C;
        off_x[r] = j * x.rpitch + i * C;
      }
      // Dirichlet mask of the full-box tensor (TM && !tmint): node columns i-1, i, i+1 and the
      // R+2 node rows this thread reads; warp-uniform `wedge` selects the masked x-filter
      const bool rmask = MK && TM && bc && !tmint;
      const bool cmm = rmask && (i - 1 == 0 || i - 1 == g.nx), cm0 = rmask && (i == 0 || i == g.nx);
      const bool cmp = rmask && (i + 1 == 0 || i + 1 == g.nx);
      bool rmk[R + 2];
      bool anym = cmm || cm0 || cmp;
#pragma unroll
      for (int rr = 0; rr < R + 2; ++rr) {
        const int64_t jr = j0 + ty * R + rr - 1;
        rmk[rr] = rmask && (jr == 0 || jr == g.ny);
        anym = anym || rmk[rr];
      }
      const bool wedge = MK && __any_sync(0xffffffffu, anym);
      // 3-plane register windows (c1, c2 and the centre value), rotated instead of shifted: the
      // z-march is unrolled by three and at phase K the planes p-2, p-1, p sit in slots
      // K, K+1, K+2 (mod 3), so no registers are moved between planes
      double c1w[3][R][C], c2w[3][R][C], xcw[3][R][C];
#pragma unroll
      for (int w = 0; w < 3; ++w)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c) { c1w[w][r][c] = 0.0; c2w[w][r][c] = 0.0; xcw[w][r][c] = 0.0; }
      // output / identity-row pointers of the next output plane (advanced one plane per output)
      double* yq = yo.y + (kb - g.k0) * yo.ppitch;
      const double* xq = x.main + (kb - g.k0) * x.ppitch;
      const double* pq_old = (mode == 2) ? pold + (kb - g.k0) * x.ppitch : nullptr;
      double* pq_new = (mode == 2) ? pnew + (kb - g.k0) * x.ppitch : nullptr;

      auto plane = [&](int64_t p, auto kc) {
        constexpr int W0 = decltype(kc)::value % 3, W1 = (W0 + 1) % 3, W2 = (W0 + 2) % 3;
        const int t = (int)(p - pfirst);
        const int slot = t % S;
        ring.wait(slot, (uint32_t)((t / S) & 1));
        if (PAIR) ring.set_pair_plane(p);
        // x-direction filters for the R+2 rows this thread needs
        double a[R + 2][C], b[R + 2][C];
        auto xfilter = [&](auto masked) {
          constexpr bool XM = decltype(masked)::value;
          const bool pm = XM && (p == 0 || p == g.nz);  // Dirichlet face plane
#pragma unroll
          for (int rr = 0; rr < R + 2; ++rr) {
            const double* row = ring.row_ptr(slot, ty * R + rr) + tx * C;
            const double* row2 = row + Ring::UDBL;  // mode 2: p_old box
            const bool rz = XM && (pm || rmk[rr]);
#pragma unroll
            for (int c = 0; c < C; ++c) {
              double xm = row[c], x0 = row[C + c], xp = row[2 * C + c];
              if (mode == 2) {
                xm = fma(beta, row2[c], xm);
                x0 = fma(beta, row2[C + c], x0);
                xp = fma(beta, row2[2 * C + c], xp);
              }
              if (rr >= 1 && rr <= R) xcw[W2][rr - 1][c] = x0;  // unmasked (identity rows)
              if (XM) {
                xm = (rz || cmm) ? 0.0 : xm;
                x0 = (rz || cm0) ? 0.0 : x0;
                xp = (rz || cmp) ? 0.0 : xp;
              }
              const double sn = xm + xp;
              a[rr][c] = GLL ? (3.0 * mx) * x0 : fma(2.0 * mx, x0, sn);
              b[rr][c] = fma(mx, x0, -sn);
            }
          }
        };
        if (MK && rmask && (wedge || p == 0 || p == g.nz)) xfilter(std::true_type{});
        else xfilter(std::false_type{});
        unsigned rel = 0;
        if (SELF) {
          if (FEM_LAP_LATE_REFILL) {
            rel = ring.release_begin(slot, tx);  // the refill test follows the plane's arithmetic
          } else if (ring.release_last(slot, tx, TY) && t + S < nplane && tx == 0) {  // refill: plane t+S
            if (FEM_REFILL_FENCE) fence_proxy_async();
            ring.issue_tm(t + S, p + S, tux, tuy, 0, 0, uorg, &umap, &umap2, nullptr, 0, &peer);
          }
        } else {
          ring.release(slot, tx);
        }
        // y-direction
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const double an = a[r][c] + a[r + 2][c];
            const double bn = b[r][c] + b[r + 2][c];
            if (GLL) {
              c1w[W2][r][c] = (3.0 * my[r]) * a[r + 1][c];
              c2w[W2][r][c] = fma(3.0 * my[r], b[r + 1][c], fma(my[r], a[r + 1][c], -an));
            } else {
              c1w[W2][r][c] = fma(2.0 * my[r], a[r + 1][c], an);
              c2w[W2][r][c] = fma(2.0 * my[r], b[r + 1][c], bn) + fma(my[r], a[r + 1][c], -an);
            }
          }
        // z-direction: output plane q = p-1
        const int64_t q = p - 1;
        if (q >= kb) {
          const double mz = MK ? (double)((q > 0) + (q < g.nz)) : 2.0;
          const bool qface = MK && bc && (q == 0 || q == g.nz);
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (!active[r]) continue;
#pragma unroll
            for (int c = 0; c < C; ++c) {
              double v, xv = xcw[W1][r][c];
              if (MK && (qface || bnode_xy[r])) {
                if (!rmask) {  // interior tensor / row path: boundary values are not staged
                  xv = xq[off_x[r] + c];
                  if (mode == 2) xv = fma(beta, pq_old[off_x[r] + c], xv);
                }
                v = xv;
              } else {
                const double nb = (c2w[W0][r][c] - c1w[W0][r][c]) + (c2w[W2][r][c] - c1w[W2][r][c]);
                if (GLL)
                  v = h36 * fma(3.0 * mz, c2w[W1][r][c], fma(mz, c1w[W1][r][c], -(c1w[W0][r][c] + c1w[W2][r][c])));
                else
                  v = h36 * fma(2.0 * mz, c2w[W1][r][c], fma(mz, c1w[W1][r][c], nb));
              }
              yq[off_y[r] + c] = v;
              if (mode == 2) pq_new[off_x[r] + c] = xv;
              if (mode >= 1) pq = fma(v, xv, pq);
              if (mode == 3) rr2 = fma(xv, xv, rr2);
            }
          }
          yq += yo.ppitch;
          if (MK && !rmask) xq += x.ppitch;
          if (mode == 2) {
            if (MK && !rmask) pq_old += x.ppitch;
            pq_new += x.ppitch;
          }
        }
        if (SELF && FEM_LAP_LATE_REFILL && ring.release_end(rel, tx, TY) && t + S < nplane && tx == 0) {
          if (FEM_REFILL_FENCE) fence_proxy_async();  // refill: plane t+S
          ring.issue_tm(t + S, p + S, tux, tuy, 0, 0, uorg, &umap, &umap2, nullptr, 0, &peer);
        }
      };
      using K0 = std::integral_constant<int, 0>;
      using K1 = std::integral_constant<int, 1>;
      using K2 = std::integral_constant<int, 2>;
      if constexpr (C == 1) {
#pragma unroll 1
        for (int64_t p = pfirst; p <= ke; p += 3) {
          plane(p, K0{});
          if (p + 1 > ke) break;
          plane(p + 1, K1{});
          if (p + 2 > ke) break;
          plane(p + 2, K2{});
        }
      } else {  // vector: the three-fold body costs the 2nd CTA's registers (measured 0.371 -> 0.424 ms)
#pragma unroll 1
        for (int64_t p = pfirst; p <= ke; ++p) {
          plane(p, K0{});
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < C; ++c) {
              c1w[0][r][c] = c1w[1][r][c]; c2w[0][r][c] = c2w[1][r][c];
              c1w[1][r][c] = c1w[2][r][c]; c2w[1][r][c] = c2w[2][r][c];
              xcw[1][r][c] = xcw[2][r][c];
            }
        }
      }
    };
    if (edge) march(std::true_type{});
    else march(std::false_type{});
  }
  if (mode == 3) {  // single-reduction CG: delta = w.r and gamma = r.r in one pass
    const double bd = block_sum(pq, red_sh);
    const double bg = block_sum(rr2, red_sh);
    double td, tg;
    if (last_block_reduce2(bd, bg, red, red_sh, &td, &tg)) {
      sc->pq = red.acc ? sc->pq + td : td;
      sc->rr_new = red.acc ? sc->rr_new + tg : tg;
    }
  } else if (mode >= 1) {
    cg_apply_epilogue(pq, mode == 2, sc, red, red_sh);
  }
}

template <bool TM, int C, int TX, int TY, int R, int S, bool PAIR = false>
static cudaError_t launch_cfg(const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps, int bc, int mode,
                              CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  using Ring1 = PlaneRing<TM, TY * R + 2, TX + 2, C, S, 0, 0, 1, PAIR>;
  using Ring2 = PlaneRing<TM, TY * R + 2, TX + 2, C, S, 0, 0, (TM ? 2 : 1)>;
  const size_t smem = (mode == 2 ? Ring2::BYTES + Ring2::META : Ring1::BYTES + Ring1::META);
  if (mode == 3 && !TM) return cudaErrorInvalidValue;  // single-reduction CG: tensor path only
  const bool gll = maps.quad == 1;
  auto pick = [&](auto gl) {
    constexpr bool G = decltype(gl)::value;
    if constexpr (PAIR) return laplace_kernel<TM, 0, C, TX, TY, R, S, G, true>;  // fem_apply only
    else
      return mode == 3 ? laplace_kernel<TM, (TM ? 3 : 1), C, TX, TY, R, S, G>
           : mode == 2 ? laplace_kernel<TM, (TM ? 2 : 1), C, TX, TY, R, S, G>
           : mode == 1 ? laplace_kernel<TM, 1, C, TX, TY, R, S, G>
                       : laplace_kernel<TM, 0, C, TX, TY, R, S, G>;
  };
  auto kern = gll ? pick(std::true_type{}) : pick(std::false_type{});
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
  }
  int txa, rya;
  const int64_t xt = balanced_tiles(g.nx + 1, TX, &txa);
  const int64_t yt = balanced_tiles(g.ny + 1, TY * R, &rya);
  const int64_t nplanes = g.k1 - g.k0;
  // z-chunks: about 4 resident waves of CTAs (2 per SM), chunks of >= 16 planes
  constexpr int kRes = (C == 1) ? kLapMinB : kLapMinB3;  // resident CTAs per SM
  int64_t zc = (4LL * kRes * sm_count + xt * yt - 1) / (xt * yt);
  // chunks of >= 16 planes amortise the pipeline fill; a mesh too small to fill the GPU that
  // way takes chunks down to 2 planes (latency: the z-march is the serial part of a CTA)
  const int64_t minchunk = (xt * yt * (nplanes / 16) < sm_count) ? 2 : FEM_LAP_MINCHUNK;
  zc = std::max<int64_t>(1, std::min<int64_t>(zc, nplanes / minchunk));
  int64_t kchunk = (nplanes + zc - 1) / zc;
  zc = (nplanes + kchunk - 1) / kchunk;
  if (minchunk > 2) {  // wave-quantisation aware chunking (2 resident CTAs per SM)
    const WorkGrid w = make_workgrid((int)xt, (int)yt, nplanes, (int64_t)kRes * sm_count, minchunk, FEM_LAP_ROUNDS);
    zc = w.zc;
    kchunk = w.kchunk;
  }
  if (maps.kchunk_force > 0) {  // halo overlap: the caller's plane selection
    kchunk = maps.kchunk_force;
    zc = maps.zc_force;
  }
  const int64_t kspan = maps.kspan > 0 ? maps.kspan : kchunk;
  if (xt * yt * zc > kMaxCtas) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)xt, (unsigned)yt, (unsigned)zc), block(TX, TY + ((TM && (C == 1 ? kLapSelf1 : kLapSelf3)) ? 0 : 1));
  CUtensorMap um, um2;
  if (TM) um = *maps.u; else std::memset(&um, 0, sizeof(um));
  if (TM && mode == 2) um2 = *maps.u2; else std::memset(&um2, 0, sizeof(um2));
  TmaOrigin org{maps.t_i0, maps.t_j0, maps.t_k0};
  PeerMaps pm;
  if (maps.peer && maps.peer->on) pm = *maps.peer; else { std::memset(&pm, 0, sizeof(pm)); pm.klo = pm.khi = -(int64_t(1) << 62); }
  const PairGeom pg = maps.pair ? *maps.pair : PairGeom{0, 0, 0};
  kern<<<grid, block, smem, s>>>(g, x, y, um, org, um2, maps.pold, maps.pnew, bc, maps.interior, kchunk, kspan, sc, red, pm,
                                 txa, rya, pg);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_laplace(int comps, int bc, const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps,
                           int mode, CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  if (mode == 2 && (!maps.u || !maps.u2)) return cudaErrorInvalidValue;  // fused CG needs TMA maps
  if (mode == 3 && !maps.u) return cudaErrorInvalidValue;
  if (maps.pair) {  // caller vector with odd rows through a row-pair tensor (fem_apply)
    if (mode != 0 || !bc) return cudaErrorInvalidValue;
    if (comps == 1) return launch_cfg<true, 1, kLapTX, kLapTY1, kLapR1, 8, true>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    return launch_cfg<true, 3, kLapTX, kLapTY3, kLapR3, 8, true>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  }
  if (maps.u) {
    if (comps == 1 && mode == 2) return launch_cfg<true, 1, kLapTX, kLapTY1, kLapR1, kLapS1>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    if (comps == 1) return launch_cfg<true, 1, kLapTX, kLapTY1, kLapR1, 8>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    if (mode == 2) return launch_cfg<true, 3, kLapTX, kLapTY3, kLapR3, FEM_LAP_S3>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    return launch_cfg<true, 3, kLapTX, kLapTY3, kLapR3, 8>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  }
  if (comps == 1) return launch_cfg<false, 1, kLapTX, kLapTY, kLapR1, 8>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  return launch_cfg<false, 3, kLapTX, kLapTY, kLapR3, 8>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
}

}  // namespace fem
