// kernels_elastic.cu -- isotropic linear elasticity apply y = A_c u with cell-wise lambda_e, mu_e
// (Eq. 9 / Alg. 1), FP64.
//
// B200 form.  On the uniform box J = (h/2) I, so the 2x2x2-Gauss element
// operator of Eq. 6 equals the exact integral and is diagonalised, up to a 3x3 / 2x2 coupling,
// by the Hadamard ("modal") basis of the trilinear space: u(xi) = sum_m c_m xi^m over the eight
// monomials m in {1, x, y, xy, z, xz, yz, xyz}.  Per cell:
//   1. forward transform c' = H^T u^e: butterflies in x, y on each node face (the face of plane
//      k+1 is computed once and carried to the next cell layer), then z;
//   2. modal stress g = G(c'): the strain modes of grad u (Alg. 1 "gradient of input variable"),
//      sigma = lambda tr eps I + 2 mu eps and the w_q detJ scaling fold into 9 scalar
//      products per cell (lambda_e, mu_e premultiplied by h/16);
//   3. inverse transform v^e = H g (Alg. 1 "P grad phi_i" steps) into the two faces of the cell.
// Scatter without atomics: the bottom face of cell layer k is added to the top face of
// layer k-1 (register carry), the four cells sharing a node in xy exchange corner values through
// shared memory, and each node is written exactly once.  Summation order per node is fixed
// (independent of the tiling and of the z-chunk / slab boundaries).
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "kernels_common.cuh"

#ifndef FEM_EL2_REFILL2
#define FEM_EL2_REFILL2 1  // elastic2_kernel: warp 0 refills two ring slots every other plane
#endif
#ifndef FEM_EL2_HD
#define FEM_EL2_HD 8  // y hand-off ring depth of elastic2_kernel when shared memory allows (4 or 8)
#endif
#ifndef FEM_EL2_S0
#define FEM_EL2_S0 FEM_EL2_S  // ring stages outside fused CG (one input box); 4 + an 8-deep hand-off beat 8 + 4 (C5b fem_apply 0.73 -> 0.69 ms)
#endif
#ifndef FEM_EL2_NOEMPTY
#define FEM_EL2_NOEMPTY 0  // 1: drop the hand-off "consumed" barriers (redundant when HD >= S + 2; measured: no gain)
#endif
#ifndef FEM_EL2_ZFACE
#define FEM_EL2_ZFACE 1  // interior grid: z-face chunks with interior x/y tiles, mask-free except the face plane
#endif
#ifndef FEM_EL2_TWOGRID
#define FEM_EL2_TWOGRID 1  // fused CG apply: interior (mask-free) and edge CTAs as two kernels
#endif

namespace fem {

namespace {
// per-component face transform of 4 node values (x fastest, then y):
// returns (sum, y-diff, x-diff, xy) in the unnormalised Hadamard basis
struct Face {
  double s, y, x, xy;
};
__device__ __forceinline__ Face face_fwd(double u00, double u10, double u01, double u11) {
  const double s0 = u00 + u10, d0 = u10 - u00, s1 = u01 + u11, d1 = u11 - u01;
  return Face{s0 + s1, s1 - s0, d0 + d1, d1 - d0};
}
}  // namespace

// GLL: 2-point Gauss-Lobatto quadrature (BP6-style, reading R1): the quadrature
// moment w = <xi^2> is 1/3 under Gauss and 1 under Gauss-Lobatto.  Modal weights in terms of w:
// linear modes 1; bilinear modes mu 3w, lambda w (the "Seta" groups) and mu w (the T group);
// trilinear modes (4 mu + lambda) w^2.
template <bool TM, int MODE, int TY, int S, bool GLL>
__global__ void __launch_bounds__(32 * (TY + 1), (TY <= 7) ? 2 : 1)
    elastic_kernel(Grid g, PlaneSrc x, OutVec yo, const __grid_constant__ CUtensorMap umap,
                   TmaOrigin uorg, const __grid_constant__ CUtensorMap mmap, int64_t mat_layer0,
                   const __grid_constant__ CUtensorMap umap2, const double* pold, double* pnew,
                   int bc, int64_t kchunk, int64_t kspan, CgScalars* sc, Reduce red, const __grid_constant__ PeerMaps peer,
                   int txa, int tya) {
  constexpr int mode = MODE;
  constexpr int NU = (MODE == 2) ? 2 : 1;
  // TY consumer warps (lane = cell column, warp = cell row) + 1 producer warp
  constexpr int TX = 32;
  constexpr int NT = TX * (TY + 1);
  constexpr int ROWS = TY + 1;  // node rows j0-1 .. j0+TY-1
  constexpr int COLS = TX + 1;  // node cols i0-1 .. i0+TX-1
  constexpr int TPART = 4 * TY * TX * 3;  // y hand-off buffers (ring of 4)
  using Ring = PlaneRing<TM, ROWS, COLS, 3, S, kElMatRows, TX, NU>;
  static_assert(kElMatRows >= TY, "material box covers the tile's cell rows");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red_sh[32];
  Ring ring;
  double* tpart = reinterpret_cast<double*>(smem_raw + Ring::BYTES);  // [4][TY][TX][3]
  uint64_t* tfull = reinterpret_cast<uint64_t*>(tpart + TPART);        // [4][TY]
  uint64_t* tempty = tfull + 4 * TY;                                    // [4][TY]
  ring.carve(smem_raw, reinterpret_cast<unsigned char*>(tempty + 4 * TY));
  const uint32_t tfull_a = smem_u32(tfull), tempty_a = smem_u32(tempty);

  if (mode >= 1 && sc->done) return;
  // fused CG (mode 2): operator input p = r + beta p_old, beta = rr_new / rr (0 on the first step)
  const double beta = (mode == 2) ? (sc->first ? 0.0 : sc->rr_new / sc->rr) : 0.0;

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + TX * ty;
  // output tile: nodes i0 .. i0+txa-1, j0 .. j0+tya-1 (txa <= TX-1, tya <= TY-1, balanced over
  // the mesh by the launcher); thread (tx,ty) owns cell (i0-1+tx, j0-1+ty) and outputs node
  // (i0-1+tx, j0+ty) (when 1 <= tx <= txa, ty < tya) from its top corners + the bottom corners
  // handed down by the warp above
  const int64_t i0 = (int64_t)blockIdx.x * txa;
  const int64_t j0 = (int64_t)blockIdx.y * tya;
  const int64_t kb = g.k0 + (int64_t)blockIdx.z * kchunk;
  const int64_t ke = min(g.k1, kb + kspan);
  const int64_t pfirst = kb - 1;  // planes kb-1 .. ke (cell layers kb-1 .. ke-1)
  if (tid < 4 * TY) {
    mbar_init(&tfull[tid], 1);
    mbar_init(&tempty[tid], 1);
  }
  ring.init(tid, NT, TY);  // (fences + __syncthreads cover the hand-off barriers too)
  if (TM) ring.set_tshift(i0 - 1, uorg);

  double pq = 0.0, rr2 = 0.0;  // (rr2: mode 3, sum of the input's squares)
  if (ty == TY) {
    ring.produce(x, g, pfirst, ke, i0 - 1, j0 - 1, bc, tx, &umap, uorg, &mmap, mat_layer0, &umap2, 0, &peer);
  } else {
    const int64_t ci = i0 - 1 + tx, cj = j0 - 1 + ty;
    const double hs = g.h * (1.0 / 16.0);
    const int64_t nj = cj + 1;  // node row this thread outputs (top corners of its cell)
    // Dirichlet mask flags of the cell's node columns ci, ci+1 and rows cj, cj+1 (TMA path)
    const bool mc0 = bc && (ci == 0 || ci == g.nx), mc1 = bc && (ci + 1 == 0 || ci + 1 == g.nx);
    const bool mr0 = bc && (cj == 0 || cj == g.ny), mr1 = bc && (cj + 1 == 0 || cj + 1 == g.ny);
    const bool owner = tx >= 1 && tx <= txa && ty < tya && ci <= g.nx && nj <= g.ny;
    const bool bnode_xy = bc && (ci == 0 || ci == g.nx || nj == 0 || nj == g.ny);
    // output / boundary-read pointers, advanced by one plane per output plane
    double* yp = yo.y + (kb - g.k0) * yo.ppitch + (owner ? nj * yo.rpitch + ci * 3 : 0);
    const int64_t xoff0 = (kb - g.k0) * x.ppitch + (owner ? nj * x.rpitch + ci * 3 : 0);
    const double* xpb = x.main + xoff0;
    const double* ppb = (mode == 2) ? pold + xoff0 : nullptr;  // p_old (mode 2, boundary nodes)
    double* pnb = (mode == 2) ? pnew + xoff0 : nullptr;        // p written here (mode 2)
    const int nplane = (int)(ke - pfirst + 1);  // planes kb-1 .. ke
    const int qface0 = bc ? (int)(0 - kb) : -1000000;     // output index of node plane 0
    const int qface1 = bc ? (int)(g.nz - kb) : -1000000;  // ... of node plane nz
    // hand-off buffers / barriers (b = output parity)
    double* const tw0 = tpart + (ty * TX + tx) * 3;                 // + b * TY*TX*3
    const double* const tr0 = tpart + ((ty + 1) * TX + tx) * 3;
    const uint32_t tfw0 = tfull_a + 8u * ty, tew0 = tempty_a + 8u * ty;  // + b * 8*TY
    const uint32_t tfr0 = tfull_a + 8u * (ty + 1), ter0 = tempty_a + 8u * (ty + 1);

    Face fb[3];     // face transform of the bottom plane of the current cell layer
    double cb[12];  // carried top-face contribution of the previous cell layer (4 modes x 3 comps)
    double xc[3];   // this thread's node value at the bottom plane (for p.Ap)
#pragma unroll
    for (int t = 0; t < 12; ++t) cb[t] = 0.0;
    double Ln, Mn;  // material of the cell layer above the bottom plane (x h/16)

    auto load_plane = [&](int t, Face* ft, double* xn, double& L, double& M) {
      const int slot = t % S;
      ring.wait(slot, (uint32_t)((t / S) & 1));
      const double2 lmn = ring.mat(slot, ty, tx);  // material layer of this plane
      const double* r0 = ring.row_ptr(slot, ty) + tx * 3;
      const double* r1 = ring.row_ptr(slot, ty + 1) + tx * 3;
      // TMA path: the box holds every node of the box domain; the Dirichlet mask P is
      // applied here (boundary nodes read as 0 for the operator, unmasked for the identity rows)
      const int64_t pl = pfirst + t;
      const bool pface = TM && bc && (pl == 0 || pl == g.nz);
      const bool m00 = pface || mc0 || mr0, m10 = pface || mc1 || mr0;
      const bool m01 = pface || mc0 || mr1, m11 = pface || mc1 || mr1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a00 = r0[c], a10 = r0[3 + c], a01 = r1[c], a11 = r1[3 + c];
        if (mode == 2) {  // p = r + beta p_old (second box)
          const double* q0 = r0 + Ring::UDBL;
          const double* q1 = r1 + Ring::UDBL;
          a00 = fma(beta, q0[c], a00);
          a10 = fma(beta, q0[3 + c], a10);
          a01 = fma(beta, q1[c], a01);
          a11 = fma(beta, q1[3 + c], a11);
        }
        xn[c] = a01;  // node (ci, cj+1): the node this thread outputs (unmasked)
        if (TM && bc && (m00 || m10 || m01 || m11)) {
          a00 = m00 ? 0.0 : a00;
          a10 = m10 ? 0.0 : a10;
          a01 = m01 ? 0.0 : a01;
          a11 = m11 ? 0.0 : a11;
        }
        ft[c] = face_fwd(a00, a10, a01, a11);
      }
      ring.release(slot, tx);
      L = lmn.x * hs;
      M = lmn.y * hs;
    };
    load_plane(0, fb, xc, Ln, Mn);

#pragma unroll 1
    for (int t = 1; t < nplane; ++t) {
      // plane kb-1+t is available; cell layer kb-2+t lies below it
      Face ft[3];
      double xn[3];
      const double L0 = Ln, M0 = Mn;
      load_plane(t, ft, xn, Ln, Mn);
      // modal coefficients (unnormalised): component u=0, v=1, w=2
      // x = ds, y = sd, xy = dd summed over z; z, xz, yz, xyz = differences in z
      const double ux = fb[0].x + ft[0].x, uy = fb[0].y + ft[0].y, uxy = fb[0].xy + ft[0].xy;
      const double uz = ft[0].s - fb[0].s, uxz = ft[0].x - fb[0].x, uyz = ft[0].y - fb[0].y, uxyz = ft[0].xy - fb[0].xy;
      const double vx = fb[1].x + ft[1].x, vy = fb[1].y + ft[1].y, vxy = fb[1].xy + ft[1].xy;
      const double vz = ft[1].s - fb[1].s, vxz = ft[1].x - fb[1].x, vyz = ft[1].y - fb[1].y, vxyz = ft[1].xy - fb[1].xy;
      const double wx = fb[2].x + ft[2].x, wy = fb[2].y + ft[2].y, wxy = fb[2].xy + ft[2].xy;
      const double wz = ft[2].s - fb[2].s, wxz = ft[2].x - fb[2].x, wyz = ft[2].y - fb[2].y, wxyz = ft[2].xy - fb[2].xy;
      double xsave[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { fb[c] = ft[c]; xsave[c] = xc[c]; xc[c] = xn[c]; }

      // modal stress: weights 1 (linear modes), 1/3 (bilinear), 1/9 (trilinear)
      const double M2 = M0 + M0;
      const double S0 = ux + vy + wz;
      const double LS0 = L0 * S0;
      const double gux = fma(M2, ux, LS0), gvy = fma(M2, vy, LS0), gwz = fma(M2, wz, LS0);
      const double tuv = M0 * (uy + vx), tuw = M0 * (uz + wx), tvw = M0 * (vz + wy);
      const double guy = tuv, gvx = tuv, guz = tuw, gwx = tuw, gvz = tvw, gwy = tvw;
      const double L1 = GLL ? L0 : L0 * (1.0 / 3.0), M1 = GLL ? M0 : M0 * (1.0 / 3.0);
      const double Sxi = vxy + wxz, Seta = uxy + wyz, Szeta = uxz + vyz;
      const double LSxi = L1 * Sxi, LSeta = L1 * Seta, LSzeta = L1 * Szeta;
      // mu weight of these bilinear modes: 3 <xi^2> (1 under Gauss, 3 under Gauss-Lobatto)
      const double MB = GLL ? 3.0 * M0 : M0;
      const double guxy = fma(MB, uxy, LSeta), gwyz = fma(MB, wyz, LSeta);
      const double gvxy = fma(MB, vxy, LSxi), gwxz = fma(MB, wxz, LSxi);
      const double guxz = fma(MB, uxz, LSzeta), gvyz = fma(MB, vyz, LSzeta);
      const double T = uyz + vxz + wxy;
      const double guyz = M1 * (T + uyz), gvxz = M1 * (T + vxz), gwxy = M1 * (T + wxy);
      const double K3 = GLL ? fma(4.0, M0, L0) : fma(4.0, M0, L0) * (1.0 / 9.0);
      const double guxyz = K3 * uxyz, gvxyz = K3 * vxyz, gwxyz = K3 * wxyz;

      // inverse z: face mode f at bottom = g_f - g_fz, top = g_f + g_fz (g_1 = 0);
      // bottom face of this cell + carried top face of layer k-1 -> complete face at plane p-1
      double F[12];
      {
        const double gx[3] = {gux, gvx, gwx}, gy[3] = {guy, gvy, gwy}, gxy[3] = {guxy, gvxy, gwxy};
        const double gz[3] = {guz, gvz, gwz}, gxz[3] = {guxz, gvxz, gwxz}, gyz[3] = {guyz, gvyz, gwyz};
        const double gxyz[3] = {guxyz, gvxyz, gwxyz};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          F[4 * c + 0] = cb[4 * c + 0] - gz[c];
          F[4 * c + 1] = cb[4 * c + 1] + (gx[c] - gxz[c]);
          F[4 * c + 2] = cb[4 * c + 2] + (gy[c] - gyz[c]);
          F[4 * c + 3] = cb[4 * c + 3] + (gxy[c] - gxyz[c]);
          cb[4 * c + 0] = gz[c];
          cb[4 * c + 1] = gx[c] + gxz[c];
          cb[4 * c + 2] = gy[c] + gyz[c];
          cb[4 * c + 3] = gxy[c] + gxyz[c];
        }
      }
      if (t >= 2) {  // node plane q = kb + t - 2 is complete in xy-corner form
        const int qo = t - 2;
        const int b = qo & 3;
        const uint32_t n = (uint32_t)(qo >> 2);
        // corners; x-neighbours by warp shuffle, y-neighbours by a point-to-point hand-off
        // from the warp below.  Fixed order per node: ((i-1,j-1)+(i,j-1)) + ((i-1,j)+(i,j)).
        double B[3], Tt[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double G1 = F[4 * c + 0], Gx = F[4 * c + 1], Gy = F[4 * c + 2], Gxy = F[4 * c + 3];
          const double es = G1 - Gy, ed = Gx - Gxy, fs = G1 + Gy, fd = Gx + Gxy;
          const double c00 = es - ed, c10 = es + ed, c01 = fs - fd, c11 = fs + fd;
          const double c10l = __shfl_up_sync(0xffffffffu, c10, 1);  // from cell i-1
          const double c11l = __shfl_up_sync(0xffffffffu, c11, 1);
          B[c] = c10l + c00;   // node row cj,   cells (i-1,j), (i,j)
          Tt[c] = c11l + c01;  // node row cj+1, cells (i-1,j), (i,j)
        }
        // the warp above (higher id: scheduled first, so usually ahead) hands its B down;
        // this warp outputs node row cj+1 = Tt (own, lower cells) + B (cells above).
        if (ty >= 1) {
          if (n >= 1) mbar_wait_a(tew0 + 8u * TY * b, (n - 1) & 1);
          double* dst = tw0 + b * (TY * TX * 3);
          dst[0] = B[0]; dst[1] = B[1]; dst[2] = B[2];
          __syncwarp();
          if (tx == 0) mbar_arrive_a(tfw0 + 8u * TY * b);
        }
        if (ty < TY - 1) {
          mbar_wait_a(tfr0 + 8u * TY * b, n & 1);
          const double* src = tr0 + b * (TY * TX * 3);
          double v[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) v[c] = Tt[c] + src[c];
          __syncwarp();
          if (tx == 0) mbar_arrive_a(ter0 + 8u * TY * b);
          if (owner) {
            const bool bnode = bnode_xy || qo == qface0 || qo == qface1;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              double vv = v[c], xv = xsave[c];
              if (bnode) {
                if (!TM) {  // row path: boundary values are not staged
                  xv = xpb[c];
                  if (mode == 2) xv = fma(beta, ppb[c], xv);
                }
                vv = xv;
              }
              yp[c] = vv;
              if (mode == 2) pnb[c] = xv;
              if (mode >= 1) pq = fma(vv, xv, pq);
              if (mode == 3) rr2 = fma(xv, xv, rr2);
            }
          }
          if (mode == 2) { ppb += x.ppitch; pnb += x.ppitch; }
          yp += yo.ppitch;
          xpb += x.ppitch;
        }
      }
    }
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

// ---- two cell rows per thread (FEM_EL_CY = 2) -------------------------------
// One cell layer of the modal closed form: (bottom face fb, top face ft, lambda h/16, mu h/16)
// -> complete face F at the bottom plane (carried top face cb of the layer below + this layer's
// bottom face), cbo <- this layer's top face.  Same arithmetic as the loop body of elastic_kernel.
template <bool GLL>
__device__ __forceinline__ void elastic_layer(const Face* fb, const Face* ft, double L0, double M0,
                                              const double* cb, double* cbo, double* F) {
  const double ux = fb[0].x + ft[0].x, uy = fb[0].y + ft[0].y, uxy = fb[0].xy + ft[0].xy;
  const double uz = ft[0].s - fb[0].s, uxz = ft[0].x - fb[0].x, uyz = ft[0].y - fb[0].y, uxyz = ft[0].xy - fb[0].xy;
  const double vx = fb[1].x + ft[1].x, vy = fb[1].y + ft[1].y, vxy = fb[1].xy + ft[1].xy;
  const double vz = ft[1].s - fb[1].s, vxz = ft[1].x - fb[1].x, vyz = ft[1].y - fb[1].y, vxyz = ft[1].xy - fb[1].xy;
  const double wx = fb[2].x + ft[2].x, wy = fb[2].y + ft[2].y, wxy = fb[2].xy + ft[2].xy;
  const double wz = ft[2].s - fb[2].s, wxz = ft[2].x - fb[2].x, wyz = ft[2].y - fb[2].y, wxyz = ft[2].xy - fb[2].xy;
  const double M2 = M0 + M0;
  const double S0 = ux + vy + wz;
  const double LS0 = L0 * S0;
  const double gux = fma(M2, ux, LS0), gvy = fma(M2, vy, LS0), gwz = fma(M2, wz, LS0);
  const double tuv = M0 * (uy + vx), tuw = M0 * (uz + wx), tvw = M0 * (vz + wy);
  const double guy = tuv, gvx = tuv, guz = tuw, gwx = tuw, gvz = tvw, gwy = tvw;
  const double L1 = GLL ? L0 : L0 * (1.0 / 3.0), M1 = GLL ? M0 : M0 * (1.0 / 3.0);
  const double Sxi = vxy + wxz, Seta = uxy + wyz, Szeta = uxz + vyz;
  const double LSxi = L1 * Sxi, LSeta = L1 * Seta, LSzeta = L1 * Szeta;
  const double MB = GLL ? 3.0 * M0 : M0;
  const double guxy = fma(MB, uxy, LSeta), gwyz = fma(MB, wyz, LSeta);
  const double gvxy = fma(MB, vxy, LSxi), gwxz = fma(MB, wxz, LSxi);
  const double guxz = fma(MB, uxz, LSzeta), gvyz = fma(MB, vyz, LSzeta);
  const double T = uyz + vxz + wxy;
  const double guyz = M1 * (T + uyz), gvxz = M1 * (T + vxz), gwxy = M1 * (T + wxy);
  const double K3 = GLL ? fma(4.0, M0, L0) : fma(4.0, M0, L0) * (1.0 / 9.0);
  const double guxyz = K3 * uxyz, gvxyz = K3 * vxyz, gwxyz = K3 * wxyz;
  const double gx[3] = {gux, gvx, gwx}, gy[3] = {guy, gvy, gwy}, gxy[3] = {guxy, gvxy, gwxy};
  const double gz[3] = {guz, gvz, gwz}, gxz[3] = {guxz, gvxz, gwxz}, gyz[3] = {guyz, gvyz, gwyz};
  const double gxyz[3] = {guxyz, gvxyz, gwxyz};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    F[4 * c + 0] = cb[4 * c + 0] - gz[c];
    F[4 * c + 1] = cb[4 * c + 1] + (gx[c] - gxz[c]);
    F[4 * c + 2] = cb[4 * c + 2] + (gy[c] - gyz[c]);
    F[4 * c + 3] = cb[4 * c + 3] + (gxy[c] - gxyz[c]);
    cbo[4 * c + 0] = gz[c];
    cbo[4 * c + 1] = gx[c] + gxz[c];
    cbo[4 * c + 2] = gy[c] + gyz[c];
    cbo[4 * c + 3] = gxy[c] + gxyz[c];
  }
}

// Depth of elastic2_kernel's y hand-off ring: 4 planes when it fits in shared memory beside the
// plane ring (227 KB per CTA), else 2 (the 8-stage row-pair ring of fem_apply)
template <int TY, size_t RING>
constexpr int el2_handoff_depth() {
  constexpr size_t per = (size_t)TY * (32 * kEl2HW * sizeof(double) + 2 * sizeof(uint64_t));
  return (FEM_EL2_HD >= 16 && RING + 16 * per + 1024 <= 232448) ? 16
       : (FEM_EL2_HD >= 8 && RING + 8 * per + 1024 <= 232448) ? 8
       : (RING + 4 * per + 1024 <= 232448) ? 4 : 2;
}

// corner values of a complete face F (4 modes x 3 comps): c00, c10, c01, c11 per component
__device__ __forceinline__ void face_corners(const double* F, int c, double& c00, double& c10, double& c01,
                                             double& c11) {
  const double G1 = F[4 * c + 0], Gx = F[4 * c + 1], Gy = F[4 * c + 2], Gxy = F[4 * c + 3];
  const double es = G1 - Gy, ed = Gx - Gxy, fs = G1 + Gy, fd = Gx + Gxy;
  c00 = es - ed; c10 = es + ed; c01 = fs - fd; c11 = fs + fd;
}

// Thread (tx, ty) owns the two cells (i0-1+tx, j0-1+2ty) ("A") and (i0-1+tx, j0+2ty) ("B"): the
// node row between them (nA = j0+2ty) is summed in registers, the row above B (nB) with the
// bottom corners handed down by warp ty+1.  Per cell: 9 instead of 12 staged node values, one
// y hand-off per two cells, the x butterflies of the shared node row computed once.  Per node the
// summation order is the one of elastic_kernel: ((i-1,j-1)+(i,j-1)) + ((i-1,j)+(i,j)).
// Which CTAs a launch covers (GM template parameter of elastic2_kernel): 0 the whole xt x yt x zc
// grid (blockIdx = tile, tile, z-chunk); 1 the "interior" box [xa,xb] x [ya,yb] x [za,zb] of it
// -- CTAs whose staged region touches no Dirichlet face, run without any mask / identity-row
// logic; 2 its complement (the "shell"), 1-D grid, every CTA Dirichlet-aware.  1 and 2 are two
// separately register-allocated kernels (one kernel holding both marches spills), launched
// side by side on two streams and sharing one reduction (Reduce::boff / btot).
struct TileMap {
  int X, Y, Z;                    // tiles in x, y; z-chunks
  int xa, xb, ya, yb, za, zb;     // interior box (inclusive)
};
__device__ __forceinline__ void tile_of_block(int GM, const TileMap& m, int& bx, int& by, int& bz) {
  if (GM == 0) { bx = blockIdx.x; by = blockIdx.y; bz = blockIdx.z; return; }
  if (GM == 1) { bx = m.xa + blockIdx.x; by = m.ya + blockIdx.y; bz = m.za + blockIdx.z; return; }
  const int nxi = m.xb - m.xa + 1, nyi = m.yb - m.ya + 1, nzi = m.zb - m.za + 1;
  const int XY = m.X * m.Y;
  int L = blockIdx.x;
  const int nfull = (m.Z - nzi) * XY;  // z-chunks outside [za, zb]: whole xy layers
  if (L < nfull) {
    const int zz = L / XY, r = L - zz * XY;
    bz = zz < m.za ? zz : zz + nzi;
    by = r / m.X;
    bx = r - by * m.X;
    return;
  }
  L -= nfull;
  const int R = XY - nxi * nyi;  // ring of one z-chunk inside [za, zb]
  bz = m.za + L / R;
  int r = L % R;
  const int nrow = (m.Y - nyi) * m.X;  // tile rows outside [ya, yb]: whole rows
  if (r < nrow) {
    const int yy = r / m.X;
    by = yy < m.ya ? yy : yy + nyi;
    bx = r - yy * m.X;
    return;
  }
  r -= nrow;
  const int w = m.X - nxi;
  by = m.ya + r / w;
  const int xx = r % w;
  bx = xx < m.xa ? xx : xx + nxi;
}

template <bool TM, int MODE, int TY, int S, bool GLL, bool PAIR = false, int GM = 0>
__global__ void __launch_bounds__(32 * (TY + ((TM && kEl2Self) ? 0 : 1)), 1)
    elastic2_kernel(Grid g, PlaneSrc x, OutVec yo, const __grid_constant__ CUtensorMap umap,
                    TmaOrigin uorg, const __grid_constant__ CUtensorMap mmap, int64_t mat_layer0,
                    const __grid_constant__ CUtensorMap umap2, const double* pold, double* pnew,
                    int bc, int64_t kchunk, int64_t kspan, CgScalars* sc, Reduce red, const __grid_constant__ PeerMaps peer,
                    int txa, int tya, PairGeom pg, TileMap tmap) {
  constexpr int mode = MODE;
  constexpr int NU = (MODE == 2) ? 2 : 1;
  constexpr int TX = 32;
  // SELF: no producer warp -- consumer warp 0 (the bottom of the y hand-off chain, hence the last
  // warp through every plane) refills the slot of plane t with plane t+S right after reading t
  static_assert(TM, "elastic2_kernel: TMA path only (caller vectors use elastic_kernel)");
  constexpr bool SELF = TM && kEl2Self;
  constexpr int NT = TX * (TY + (SELF ? 0 : 1));
  constexpr int ROWS = 2 * TY + 1;  // node rows j0-1 .. j0+2TY-1
  constexpr int COLS = TX + 1;      // node cols i0-1 .. i0+TX-1
  constexpr int HW = kEl2HW;        // doubles per thread and y hand-off (3 corner sums)
  using Ring = PlaneRing<TM, ROWS, COLS, 3, S, kElMatRows, TX, NU, PAIR>;
  constexpr int HD = el2_handoff_depth<TY, Ring::BYTES + Ring::META>();  // y hand-off ring depth
  // The hand-off slot written for output plane q is rewritten for plane q + HD at the writer's
  // step q + HD + 2, which needs ring plane q + HD + 2, whose refill needs every warp to have
  // released plane q + HD + 2 - S (q + HD + 3 - S with the paired refills), i.e. the reader to
  // have finished its step q + HD + 1 - S >= q + 2 -- its read of plane q -- whenever
  // HD >= S + 1.  With HD >= S + 2 the "slot consumed" barriers are therefore redundant.
  constexpr bool NOEMPTY = SELF && FEM_EL2_NOEMPTY && HD >= S + 2;
  constexpr int TPART = HD * TY * TX * HW;
  static_assert(kElMatRows >= 2 * TY, "material box covers the tile's cell rows");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red_sh[32];
  Ring ring;
  double* tpart = reinterpret_cast<double*>(smem_raw + Ring::BYTES);  // [HD][TY][TX][HW]
  uint64_t* tfull = reinterpret_cast<uint64_t*>(tpart + TPART);        // [HD][TY]
  uint64_t* tempty = tfull + HD * TY;                                   // [HD][TY]
  ring.carve(smem_raw, reinterpret_cast<unsigned char*>(tempty + HD * TY));
  const uint32_t tfull_a = smem_u32(tfull), tempty_a = smem_u32(tempty);

  if (mode >= 1 && sc->done) return;
  // fused CG (mode 2): operator input p = r + beta p_old, beta = rr_new / rr (0 on the first step)
  const double beta = (mode == 2) ? (sc->first ? 0.0 : sc->rr_new / sc->rr) : 0.0;

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + TX * ty;
  int bx, by, bz;
  tile_of_block(GM, tmap, bx, by, bz);
  // output tile: nodes i0 .. i0+txa-1 (txa <= TX-1), j0 .. j0+tya-1 (tya <= 2TY-1)
  const int64_t i0 = (int64_t)bx * txa;
  const int64_t j0 = (int64_t)by * tya;
  const int64_t kb = g.k0 + (int64_t)bz * kchunk;
  const int64_t ke = min(g.k1, kb + kspan);
  const int64_t pfirst = kb - 1;
  if (tid < HD * TY) {
    mbar_init(&tfull[tid], 1);
    mbar_init(&tempty[tid], 1);
  }
  ring.init(tid, NT, TY);
  if (PAIR) ring.set_pair_tile(i0 - 1, j0 - 1, pg);
  const int tux = TM ? ring.set_tshift(i0 - 1, uorg) : 0, tuy = (int)(j0 - 1 - uorg.t_j0);
  const int tmx = (int)(2 * (i0 - 1)), tmy = (int)(j0 - 1);
  const int nplane = (int)(ke - pfirst + 1);  // planes kb-1 .. ke
  if (SELF && tid == 0) {  // prologue: the first S planes
    tma_prefetch_desc(&umap);
    if (MODE == 2) tma_prefetch_desc(&umap2);
    tma_prefetch_desc(&mmap);
    for (int t = 0; t < S && t < nplane; ++t)
      ring.issue_tm(t, pfirst + t, tux, tuy, tmx, tmy, uorg, &umap, &umap2, &mmap, mat_layer0, &peer);
  }

  double pq = 0.0, rr2 = 0.0;
  if (!SELF && ty == TY) {
    ring.produce(x, g, pfirst, ke, i0 - 1, j0 - 1, bc, tx, &umap, uorg, &mmap, mat_layer0, &umap2, 0, &peer);
  } else {
    const int64_t ci = i0 - 1 + tx, cj = j0 - 1 + 2 * ty;  // cell A = (ci, cj), cell B = (ci, cj+1)
    const double hs = g.h * (1.0 / 16.0);
    const int64_t nA = cj + 1, nB = cj + 2;  // node rows this thread outputs
    const bool colok = tx >= 1 && tx <= txa && ci <= g.nx;
    const bool ownA = colok && 2 * ty < tya && nA <= g.ny;
    const bool ownB = colok && 2 * ty + 1 < tya && nB <= g.ny;
    const bool own = ownA || ownB;  // (ownB implies nA is a mesh row too)
    double* yp = yo.y + (kb - g.k0) * yo.ppitch + (own ? nA * yo.rpitch + ci * 3 : 0);
    const int64_t xoff0 = (kb - g.k0) * x.ppitch + (own ? nA * x.rpitch + ci * 3 : 0);
    double* pnb = (mode == 2) ? pnew + xoff0 : nullptr;
    double* const tw0 = tpart + (ty * TX + tx) * HW;
    const double* const tr0 = tpart + ((ty + 1) * TX + tx) * HW;
    const uint32_t tfw0 = tfull_a + 8u * ty, tew0 = tempty_a + 8u * ty;
    const uint32_t tfr0 = tfull_a + 8u * (ty + 1), ter0 = tempty_a + 8u * (ty + 1);
    // Dirichlet box: only CTAs whose tile or z-chunk touches a box face need the mask P
    // and the identity rows; all others run the same march without that logic (CTA-uniform).
    // (fused CG, mode 2: one path -- the split costs that kernel its register headroom, measured
    // 1.32 -> 1.52 ms with spills, and gains nothing there)
    const bool edge = MODE == 2 || (bc && (i0 <= 1 || i0 + TX - 1 >= g.nx || j0 <= 1 ||
                                           j0 - 1 + 2 * TY >= g.ny || pfirst <= 0 || ke >= g.nz));

    auto march = [&](auto mk) {
      constexpr bool MK = decltype(mk)::value;
      const bool mc0 = MK && bc && (ci == 0 || ci == g.nx), mc1 = MK && bc && (ci + 1 == 0 || ci + 1 == g.nx);
      const bool mr0 = MK && bc && (cj == 0 || cj == g.ny), mr1 = MK && bc && (cj + 1 == 0 || cj + 1 == g.ny);
      const bool mr2 = MK && bc && (cj + 2 == 0 || cj + 2 == g.ny);
      const bool bnA_xy = MK && bc && (ci == 0 || ci == g.nx || nA == 0 || nA == g.ny);
      const bool bnB_xy = MK && bc && (ci == 0 || ci == g.nx || nB == 0 || nB == g.ny);
      // ZF: the mask-free march of the interior grid also covers CTAs whose z-chunk touches a
      // z face (their x/y tiles are interior): per plane a uniform check zeroes a face plane's
      // staged values and makes the face plane's outputs identity rows
      constexpr bool ZF = !MK && GM == 1 && FEM_EL2_ZFACE;
      constexpr bool MZ = MK || ZF;
      const int qface0 = (MZ && bc) ? (int)(0 - kb) : -1000000;
      const int qface1 = (MZ && bc) ? (int)(g.nz - kb) : -1000000;

      // loop state in two register sets (ping-pong: the z-march is unrolled by two, so nothing is
      // moved at the back edge): faces of cells A, B at a node plane, carried top faces, the node
      // values of rows nA, nB, and the material of the cell layer above the plane (x h/16)
      Face fA[2][3], fB[2][3];
      double cA[2][12], cB[2][12];
      double xA[2][3], xB[2][3];
      double LA[2], MA[2], LB[2], MB[2];
#pragma unroll
      for (int t = 0; t < 12; ++t) { cA[0][t] = 0.0; cB[0][t] = 0.0; }

      auto load_plane = [&](int t, Face* fA, Face* fB, double* xA, double* xB, double& LA, double& MA,
                            double& LB, double& MB) {
        const int slot = t % S;
        ring.wait(slot, (uint32_t)((t / S) & 1));
        if (PAIR) ring.set_pair_plane(pfirst + t);
        const double2 lmA = ring.mat(slot, 2 * ty, tx), lmB = ring.mat(slot, 2 * ty + 1, tx);
        const double* r0 = ring.row_ptr(slot, 2 * ty) + tx * 3;
        const double* r1 = ring.row_ptr(slot, 2 * ty + 1) + tx * 3;
        const double* r2 = ring.row_ptr(slot, 2 * ty + 2) + tx * 3;
        const int64_t pl = pfirst + t;
        const bool pface = MK && bc && (pl == 0 || pl == g.nz);
        const bool m00 = pface || mc0 || mr0, m10 = pface || mc1 || mr0;
        const bool m01 = pface || mc0 || mr1, m11 = pface || mc1 || mr1;
        const bool m02 = pface || mc0 || mr2, m12 = pface || mc1 || mr2;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double a00 = r0[c], a10 = r0[3 + c], a01 = r1[c], a11 = r1[3 + c], a02 = r2[c], a12 = r2[3 + c];
          if (mode == 2) {  // p = r + beta p_old (second box)
            const double* q0 = r0 + Ring::UDBL;
            const double* q1 = r1 + Ring::UDBL;
            const double* q2 = r2 + Ring::UDBL;
            a00 = fma(beta, q0[c], a00);
            a10 = fma(beta, q0[3 + c], a10);
            a01 = fma(beta, q1[c], a01);
            a11 = fma(beta, q1[3 + c], a11);
            a02 = fma(beta, q2[c], a02);
            a12 = fma(beta, q2[3 + c], a12);
          }
          xA[c] = a01;  // node (ci, nA), unmasked
          xB[c] = a02;  // node (ci, nB)
          if (ZF && bc && (pl == 0 || pl == g.nz)) {  // a z-face plane: all its nodes are masked
            a00 = 0.0; a10 = 0.0; a01 = 0.0; a11 = 0.0; a02 = 0.0; a12 = 0.0;
          }
          if (MK && bc && (m00 || m10 || m01 || m11 || m02 || m12)) {
            a00 = m00 ? 0.0 : a00;
            a10 = m10 ? 0.0 : a10;
            a01 = m01 ? 0.0 : a01;
            a11 = m11 ? 0.0 : a11;
            a02 = m02 ? 0.0 : a02;
            a12 = m12 ? 0.0 : a12;
          }
          // x butterflies per node row (the middle row is shared by the two faces)
          const double s0 = a00 + a10, d0 = a10 - a00, s1 = a01 + a11, d1 = a11 - a01;
          const double s2 = a02 + a12, d2 = a12 - a02;
          fA[c] = Face{s0 + s1, s1 - s0, d0 + d1, d1 - d0};
          fB[c] = Face{s1 + s2, s2 - s1, d1 + d2, d2 - d1};
        }
        ring.release(slot, tx);
        if (FEM_EL2_REFILL2) {
          // refill two slots every other plane (odd t: planes t-1+S and t+S) -- warp 0, the last
          // warp through every plane and hence the one pacing the CTA, pays the refill block
          // (wait, fence, expect-tx, 2-3 TMA issues) half as often
          if (SELF && ty == 0 && (t & 1) && t - 1 + S < nplane) {
            // (every warp releases plane t-1 before t, so waiting for t suffices; the wait on t-1
            // passes at once and keeps every barrier phase observed -- compute-sanitizer synccheck)
            ring.wait_released(t - 1);
            ring.wait_released(t);
            if (tx == 0) {
              if (FEM_REFILL_FENCE) fence_proxy_async();  // every warp's generic reads of the slots before the TMA writes
              ring.issue_tm(t - 1 + S, pfirst + t - 1 + S, tux, tuy, tmx, tmy, uorg, &umap, &umap2, &mmap, mat_layer0,
                            &peer);
              if (t + S < nplane)
                ring.issue_tm(t + S, pfirst + t + S, tux, tuy, tmx, tmy, uorg, &umap, &umap2, &mmap, mat_layer0, &peer);
            }
          }
        } else if (SELF && ty == 0 && t + S < nplane) {  // refill this slot with plane t+S
          ring.wait_released(t);
          if (tx == 0) {
            if (FEM_REFILL_FENCE) fence_proxy_async();  // every warp's generic reads of the slot before the TMA write
            ring.issue_tm(t + S, pfirst + t + S, tux, tuy, tmx, tmy, uorg, &umap, &umap2, &mmap, mat_layer0, &peer);
          }
        }
        LA = lmA.x * hs;
        MA = lmA.y * hs;
        LB = lmB.x * hs;
        MB = lmB.y * hs;
      };
      load_plane(0, fA[0], fB[0], xA[0], xB[0], LA[0], MA[0], LB[0], MB[0]);

      // node output (identity rows on the Dirichlet box) + the fused CG epilogue terms
      auto put = [&](double* yq, double* pq_new, const double* v, const double* xs, bool bnode) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double vv = v[c];
          const double xv = xs[c];
          if (MZ && bnode) vv = xv;
          yq[c] = vv;
          if (mode == 2) pq_new[c] = xv;
          if (mode >= 1) pq = fma(vv, xv, pq);
          if (mode == 3) rr2 = fma(xv, xv, rr2);
        }
      };

      // one step of the z-march: plane t arrives in set V; the cell layer between planes t-1 (set
      // U) and t is applied; node plane t-1 of the ring (global kb + t - 2) is completed and written
      auto step = [&](int t, auto uc) {
        constexpr int U = decltype(uc)::value, V = 1 - U;
        load_plane(t, fA[V], fB[V], xA[V], xB[V], LA[V], MA[V], LB[V], MB[V]);
        const double* xs_A = xA[U];  // node values at plane t-1 (= the output plane)
        const double* xs_B = xB[U];
        // per-node order ((i-1,j-1)+(i,j-1)) + ((i-1,j)+(i,j)), independent of tiles and slabs
        double BA[3], TA[3], vA[3], TB[3];
        {
          double FA[12];
          elastic_layer<GLL>(fA[U], fA[V], LA[U], MA[U], cA[U], cA[V], FA);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double a00, a10, a01, a11;
            face_corners(FA, c, a00, a10, a01, a11);
            const double a10l = __shfl_up_sync(0xffffffffu, a10, 1);  // from cell i-1
            const double a11l = __shfl_up_sync(0xffffffffu, a11, 1);
            BA[c] = a10l + a00;  // node row cj (cells row cj): to warp ty-1
            TA[c] = a11l + a01;  // node row nA, cells row cj
          }
        }
        {
          double FB[12];
          elastic_layer<GLL>(fB[U], fB[V], LB[U], MB[U], cB[U], cB[V], FB);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double b00, b10, b01, b11;
            face_corners(FB, c, b00, b10, b01, b11);
            const double b10l = __shfl_up_sync(0xffffffffu, b10, 1);
            const double b11l = __shfl_up_sync(0xffffffffu, b11, 1);
            vA[c] = TA[c] + (b10l + b00);  // node row nA: cells row cj, then row cj+1
            TB[c] = b11l + b01;            // node row nB, cells row cj+1
          }
        }
        if (t >= 2) {  // node plane q = kb + t - 2 is complete
          const int qo = t - 2, b = qo & (HD - 1);
          const uint32_t n = (uint32_t)qo / (uint32_t)HD;
          if (ty >= 1) {
            if (!NOEMPTY && n >= 1) mbar_wait_a(tew0 + 8u * TY * b, (n - 1) & 1);
            double* dst = tw0 + b * (TY * TX * HW);
            dst[0] = BA[0]; dst[1] = BA[1]; dst[2] = BA[2];
            __syncwarp();
            if (tx == 0) mbar_arrive_a(tfw0 + 8u * TY * b);
          }
          const bool qf = MZ && (qo == qface0 || qo == qface1);
          if (ownA) put(yp, pnb, vA, xs_A, bnA_xy || qf);
          if (ty < TY - 1) {
            mbar_wait_a(tfr0 + 8u * TY * b, n & 1);
            const double* src = tr0 + b * (TY * TX * HW);
            double v[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) v[c] = TB[c] + src[c];
            if (!NOEMPTY) {
              __syncwarp();
              if (tx == 0) mbar_arrive_a(ter0 + 8u * TY * b);
            }
            if (ownB) put(yp + yo.rpitch, pnb + x.rpitch, v, xs_B, bnB_xy || qf);
          }
          if (mode == 2) pnb += x.ppitch;
          yp += yo.ppitch;
        }
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
#pragma unroll 1
      for (int t = 1; t < nplane; t += 2) {
        step(t, I0{});
        if (t + 1 >= nplane) break;
        step(t + 1, I1{});
      }
    };
    if constexpr (GM == 1) march(std::false_type{});
    else if constexpr (GM == 2 || MODE == 2) march(std::true_type{});
    else if (edge) march(std::true_type{});
    else march(std::false_type{});
  }
  if (mode == 3) {
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

template <bool TM, int TY, int S, bool PAIR = false>
static cudaError_t launch_cfg2(const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps, int bc, int mode,
                               CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  constexpr int TX = 32;
  using Ring1 = PlaneRing<TM, 2 * TY + 1, TX + 1, 3, S, kElMatRows, TX, 1, PAIR>;
  using Ring2 = PlaneRing<TM, 2 * TY + 1, TX + 1, 3, S, kElMatRows, TX, (TM ? 2 : 1)>;
  constexpr int HD1 = el2_handoff_depth<TY, Ring1::BYTES + Ring1::META>();
  constexpr int HD2 = el2_handoff_depth<TY, Ring2::BYTES + Ring2::META>();
  const size_t smem = mode == 2 ? Ring2::BYTES + Ring2::META + (size_t)HD2 * TY * (TX * kEl2HW * sizeof(double) + 2 * sizeof(uint64_t))
                                : Ring1::BYTES + Ring1::META + (size_t)HD1 * TY * (TX * kEl2HW * sizeof(double) + 2 * sizeof(uint64_t));
  const bool gll = maps.quad == 1;
  if (mode == 3 && !TM) return cudaErrorInvalidValue;
  auto pick = [&](auto gl) {
    constexpr bool G = decltype(gl)::value;
    if constexpr (PAIR) return elastic2_kernel<TM, 0, TY, S, G, true>;  // fem_apply only
    else
      return mode == 3 ? elastic2_kernel<TM, (TM ? 3 : 1), TY, S, G>
           : mode == 2 ? elastic2_kernel<TM, (TM ? 2 : 1), TY, S, G>
           : mode == 1 ? elastic2_kernel<TM, 1, TY, S, G>
                       : elastic2_kernel<TM, 0, TY, S, G>;
  };
  auto kern = gll ? pick(std::true_type{}) : pick(std::false_type{});
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
  }
  int txa, tya;
  const int64_t xt = balanced_tiles(g.nx + 1, TX - 1, &txa);
  const int64_t yt = balanced_tiles(g.ny + 1, 2 * TY - 1, &tya);
  const TileMap tm0{(int)xt, (int)yt, 1, 0, 0, 0, 0, 0, 0};
  const int64_t nplanes = g.k1 - g.k0;
  // resident CTAs per SM at ~255 registers per thread: 65536 / (32 (TY [+1]) 255)
  constexpr int kRes = (TY + ((TM && kEl2Self) ? 0 : 1)) <= 4 ? 2 : 1;
  int64_t zc = (4LL * kRes * sm_count + xt * yt - 1) / (xt * yt);
  const int64_t minchunk = (xt * yt * (nplanes / 8) < sm_count) ? 2 : 8;
  zc = std::max<int64_t>(1, std::min<int64_t>(zc, nplanes / minchunk));
  int64_t kchunk = (nplanes + zc - 1) / zc;
  zc = (nplanes + kchunk - 1) / kchunk;
  if (minchunk > 2) {  // wave-quantisation aware chunking (1 resident CTA per SM)
    const WorkGrid w = make_workgrid((int)xt, (int)yt, nplanes, (int64_t)kRes * sm_count, minchunk, 4);
    zc = w.zc;
    kchunk = w.kchunk;
  }
  if (maps.kchunk_force > 0) {  // halo overlap: the caller's plane selection
    kchunk = maps.kchunk_force;
    zc = maps.zc_force;
  }
  const int64_t kspan = maps.kspan > 0 ? maps.kspan : kchunk;
  if (xt * yt * zc > kMaxCtas) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)xt, (unsigned)yt, (unsigned)zc), block(TX, TY + ((TM && kEl2Self) ? 0 : 1));
  CUtensorMap um, um2;
  if (TM) um = *maps.u; else std::memset(&um, 0, sizeof(um));
  if (TM && mode == 2) um2 = *maps.u2; else std::memset(&um2, 0, sizeof(um2));
  TmaOrigin org{maps.t_i0, maps.t_j0, maps.t_k0};
  PeerMaps pm;
  if (maps.peer && maps.peer->on) pm = *maps.peer; else { std::memset(&pm, 0, sizeof(pm)); pm.klo = pm.khi = -(int64_t(1) << 62); }
  const PairGeom pgeo = maps.pair ? *maps.pair : PairGeom{0, 0, 0};
  if constexpr (TM) {
    if (FEM_EL2_TWOGRID && maps.kchunk_force == 0) {
      // interior / edge grids (TileMap): per axis, the tiles whose staged region touches no
      // Dirichlet face (the kernel's own `edge` predicate, separable per axis)
      auto range = [](int64_t n, auto is_edge, int& lo, int& hi) {
        lo = 0;
        while (lo < n && is_edge(lo)) ++lo;
        hi = (int)n - 1;
        while (hi >= lo && is_edge(hi)) --hi;
      };
      int xa, xb, ya, yb, za, zb;
      range(xt, [&](int64_t b) { const int64_t i0 = b * txa; return bc && (i0 <= 1 || i0 + TX - 1 >= g.nx); }, xa, xb);
      range(yt, [&](int64_t b) { const int64_t j0 = b * tya; return bc && (j0 <= 1 || j0 - 1 + 2 * TY >= g.ny); }, ya, yb);
      range(zc, [&](int64_t b) {  // (FEM_EL2_ZFACE: the interior kernel handles the z faces)
        const int64_t kb = g.k0 + b * kchunk, ke = std::min(g.k1, kb + kspan);
        return !FEM_EL2_ZFACE && bc && (kb - 1 <= 0 || ke >= g.nz);
      }, za, zb);
      if (xa <= xb && ya <= yb && za <= zb) {
        const TileMap tm{(int)xt, (int)yt, (int)zc, xa, xb, ya, yb, za, zb};
        const int64_t n_in = (int64_t)(xb - xa + 1) * (yb - ya + 1) * (zb - za + 1);
        const int64_t n_all = xt * yt * zc, n_edge = n_all - n_in;
        auto pick2 = [&](auto gl, auto gm) {
          constexpr bool G = decltype(gl)::value;
          constexpr int M = decltype(gm)::value;
          if constexpr (PAIR) return elastic2_kernel<TM, 0, TY, S, G, true, M>;
          else
            return mode == 3 ? elastic2_kernel<TM, 3, TY, S, G, false, M>
                 : mode == 2 ? elastic2_kernel<TM, 2, TY, S, G, false, M>
                 : mode == 1 ? elastic2_kernel<TM, 1, TY, S, G, false, M>
                             : elastic2_kernel<TM, 0, TY, S, G, false, M>;
        };
        using GI = std::integral_constant<int, 1>;
        using GE = std::integral_constant<int, 2>;
        auto kin = gll ? pick2(std::true_type{}, GI{}) : pick2(std::false_type{}, GI{});
        auto ked = gll ? pick2(std::true_type{}, GE{}) : pick2(std::false_type{}, GE{});
        for (auto k : {kin, ked}) {
          const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(k), (int)smem);
          if (e != cudaSuccess) return e;
        }
        Reduce ri = red, re = red;
        ri.boff = 0;
        ri.btot = (int)n_all;
        re.boff = (int)n_in;
        re.btot = (int)n_all;
        const bool two = maps.aux && maps.ev_fork && maps.ev_join && n_edge > 0;
        cudaStream_t se = two ? maps.aux : s;
        if (two) {
          cudaError_t e = cudaEventRecord(maps.ev_fork, s);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(maps.aux, maps.ev_fork, 0);
          if (e != cudaSuccess) return e;
        }
        if (n_edge > 0) {  // the slower, Dirichlet-aware CTAs first
          ked<<<dim3((unsigned)n_edge), block, smem, se>>>(g, x, y, um, org, *maps.mat, maps.mat_layer0, um2, maps.pold,
                                                           maps.pnew, bc, kchunk, kspan, sc, re, pm, txa, tya, pgeo, tm);
          add_launches(1);
          const cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) return e;
        }
        kin<<<dim3((unsigned)(xb - xa + 1), (unsigned)(yb - ya + 1), (unsigned)(zb - za + 1)), block, smem, s>>>(
            g, x, y, um, org, *maps.mat, maps.mat_layer0, um2, maps.pold, maps.pnew, bc, kchunk, kspan, sc, ri, pm,
            txa, tya, pgeo, tm);
        add_launches(1);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess && two) {
          e = cudaEventRecord(maps.ev_join, maps.aux);
          if (e == cudaSuccess) e = cudaStreamWaitEvent(s, maps.ev_join, 0);
        }
        return e;
      }
    }
  }
  kern<<<grid, block, smem, s>>>(g, x, y, um, org, *maps.mat, maps.mat_layer0, um2, maps.pold, maps.pnew,
                                 bc, kchunk, kspan, sc, red, pm, txa, tya, pgeo, tm0);
  add_launches(1);
  return cudaGetLastError();
}

template <bool TM, int TY, int S>
static cudaError_t launch_cfg(const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps, int bc, int mode,
                              CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  constexpr int TX = 32;
  using Ring1 = PlaneRing<TM, TY + 1, TX + 1, 3, S, kElMatRows, TX, 1>;
  using Ring2 = PlaneRing<TM, TY + 1, TX + 1, 3, S, kElMatRows, TX, (TM ? 2 : 1)>;
  const size_t ring_bytes = mode == 2 ? Ring2::BYTES + Ring2::META : Ring1::BYTES + Ring1::META;
  const size_t smem = ring_bytes + 4 * TY * TX * 3 * sizeof(double) + 8 * TY * sizeof(uint64_t);
  const bool gll = maps.quad == 1;
  if (mode == 3 && !TM) return cudaErrorInvalidValue;  // single-reduction CG: tensor path only
  auto pick = [&](auto gl) {
    constexpr bool G = decltype(gl)::value;
    return mode == 3 ? elastic_kernel<TM, (TM ? 3 : 1), TY, S, G>
         : mode == 2 ? elastic_kernel<TM, (TM ? 2 : 1), TY, S, G>
         : mode == 1 ? elastic_kernel<TM, 1, TY, S, G>
                     : elastic_kernel<TM, 0, TY, S, G>;
  };
  auto kern = gll ? pick(std::true_type{}) : pick(std::false_type{});
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
  }
  int txa, tya;
  const int64_t xt = balanced_tiles(g.nx + 1, TX - 1, &txa);
  const int64_t yt = balanced_tiles(g.ny + 1, TY - 1, &tya);
  const int64_t nplanes = g.k1 - g.k0;
  int64_t zc = ((kElTY <= 7 ? 8LL : 4LL) * sm_count + xt * yt - 1) / (xt * yt);
  // chunks of >= 8 planes amortise the pipeline fill; a mesh too small to fill the GPU that
  // way takes chunks down to 2 planes (latency: the z-march is the serial part of a CTA)
  const int64_t minchunk = (xt * yt * (nplanes / 8) < sm_count) ? 2 : 8;
  zc = std::max<int64_t>(1, std::min<int64_t>(zc, nplanes / minchunk));
  int64_t kchunk = (nplanes + zc - 1) / zc;
  zc = (nplanes + kchunk - 1) / kchunk;
  if (minchunk > 2) {  // wave-quantisation aware chunking (1 resident CTAs per SM)
    const WorkGrid w = make_workgrid((int)xt, (int)yt, nplanes, 1LL * sm_count, minchunk, 4);
    zc = w.zc;
    kchunk = w.kchunk;
  }
  if (maps.kchunk_force > 0) {  // halo overlap: the caller's plane selection
    kchunk = maps.kchunk_force;
    zc = maps.zc_force;
  }
  const int64_t kspan = maps.kspan > 0 ? maps.kspan : kchunk;
  if (xt * yt * zc > kMaxCtas) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)xt, (unsigned)yt, (unsigned)zc), block(TX, TY + 1);
  CUtensorMap um, um2;
  if (TM) um = *maps.u; else std::memset(&um, 0, sizeof(um));
  if (TM && mode == 2) um2 = *maps.u2; else std::memset(&um2, 0, sizeof(um2));
  TmaOrigin org{maps.t_i0, maps.t_j0, maps.t_k0};
  PeerMaps pm;
  if (maps.peer && maps.peer->on) pm = *maps.peer; else { std::memset(&pm, 0, sizeof(pm)); pm.klo = pm.khi = -(int64_t(1) << 62); }
  kern<<<grid, block, smem, s>>>(g, x, y, um, org, *maps.mat, maps.mat_layer0, um2, maps.pold, maps.pnew,
                                 bc, kchunk, kspan, sc, red, pm, txa, tya);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_elastic(int bc, const Grid& g, PlaneSrc x, OutVec y, ApplyMaps maps, int mode,
                           CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  if (mode == 2 && (!maps.u || !maps.u2)) return cudaErrorInvalidValue;  // fused CG needs TMA maps
  if (mode == 3 && !maps.u) return cudaErrorInvalidValue;
  // CG vectors (tensor maps): two cell rows per thread; caller vectors (bulk-row staging, one copy
  // per ring row): one cell row per thread, 16 rows per copy batch (measured faster there)
  if (maps.pair) {  // caller vector with odd rows through a row-pair tensor (fem_apply)
    if (mode != 0 || !bc) return cudaErrorInvalidValue;
    return launch_cfg2<true, kEl2TY, FEM_EL2_S0, true>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  }
  if (kElCY == 2 && maps.u) {
    if (mode == 2) return launch_cfg2<true, kEl2TY, kEl2S>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    return launch_cfg2<true, kEl2TY, FEM_EL2_S0>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  }
  if (maps.u) {
    if (mode == 2) return launch_cfg<true, kElTY, 4>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
    return launch_cfg<true, kElTY, (kElTY <= 7 ? 4 : 8)>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
  }
  return launch_cfg<false, kElTY, 4>(g, x, y, maps, bc, mode, sc, red, s, sm_count);
}

}  // namespace fem
