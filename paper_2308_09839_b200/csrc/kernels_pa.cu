// kernels_pa.cu -- partial assembly of the elasticity operator on the uniform box (the paper's
// comparison method, "precomputing and storing ... all the values at quadrature
// points"; Table 3: 21 data values per quadrature point for isotropic elasticity).
//
// Stored per cell e and Gauss point q (setup, once per material): the 21 upper-triangle entries
// of D_q = w_q det J_q C_e, the isotropic constitutive matrix in Voigt order (xx, yy, zz, yz, xz,
// xy; engineering shears) with the quadrature weight and Jacobian folded in -- 1,344 B per cell,
// SoA [q][k][cell] so a warp's loads are coalesced.  On the box J^-1 = (2/h) I is a constant,
// so nothing else is stored (reading R21).  The apply (y = A_c u) per cell layer:
// gather u^e (node planes staged by the PlaneRing, like the matrix-free kernels), reference
// gradient at each Gauss point from the Hadamard (modal) coefficients of u^e, strain, sigma =
// D_q eps from the stored values, test contraction accumulated in the modal basis, then the same
// atomic-free scatter as elastic_kernel: bottom face added to the carried top face of the layer
// below, x neighbours by warp shuffle, y neighbours by an mbarrier hand-off between warps.
// The kernel reads the 1,344 B/cell of D whatever the material (that is the method's cost).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <type_traits>

#include "kernels_common.cuh"

namespace fem {

namespace {
struct FaceP {
  double s, y, x, xy;
};
__device__ __forceinline__ FaceP facep_fwd(double u00, double u10, double u01, double u11) {
  const double s0 = u00 + u10, d0 = u10 - u00, s1 = u01 + u11, d1 = u11 - u01;
  return FaceP{s0 + s1, s1 - s0, d0 + d1, d1 - d0};
}
constexpr int kPaTY = 7;  // consumer warps (cell rows) of pa21_kernel; + 1 producer warp
}  // namespace

// Upper-triangle index of (i, j), i <= j, in row-major order of a symmetric 6x6
__host__ __device__ constexpr int sym6(int i, int j) { return i * 6 - (i * (i - 1)) / 2 + (j - i); }

__global__ void pa21_setup_kernel(const double2* __restrict__ lm, int64_t ncells, double wdet,
                                  double* __restrict__ D) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncells; e += stride) {
    const double l = lm[e].x * wdet, m = lm[e].y * wdet;
    double d[21];
#pragma unroll
    for (int k = 0; k < 21; ++k) d[k] = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
      for (int j = i; j < 3; ++j) d[sym6(i, j)] = (i == j) ? l + 2.0 * m : l;
      d[sym6(i + 3, i + 3)] = m;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int k = 0; k < 21; ++k) D[(int64_t)(q * 21 + k) * ncells + e] = d[k];
  }
}

// One cell layer: faces (bottom fb, top ft) of u^e -> complete face F at the bottom plane
// (carried top face cb + this layer's bottom face), cbo <- this layer's top face.
template <bool GLL>
__device__ __forceinline__ void pa21_layer(const FaceP* fb, const FaceP* ft, const double* __restrict__ Dc,
                                           int64_t cstride, bool inbox, double inv4h, const double* cb,
                                           double* cbo, double* F) {
  // modal (Hadamard) coefficients A_m = sum_a u_a prod_{d in m} s_ad per component
  double A[3][7];  // x, y, z, xy, xz, yz, xyz
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    A[c][0] = fb[c].x + ft[c].x;
    A[c][1] = fb[c].y + ft[c].y;
    A[c][2] = ft[c].s - fb[c].s;
    A[c][3] = fb[c].xy + ft[c].xy;
    A[c][4] = ft[c].x - fb[c].x;
    A[c][5] = ft[c].y - fb[c].y;
    A[c][6] = ft[c].xy - fb[c].xy;
  }
  double B[3][7];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 7; ++m) B[c][m] = 0.0;
  const double gq = GLL ? 1.0 : 0.57735026918962576451;  // Gauss point 1/sqrt(3) (Lobatto: 1)
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double xi = (q & 1) ? gq : -gq, eta = (q & 2) ? gq : -gq, zeta = (q & 4) ? gq : -gq;
    // 8 x reference gradient G[c][d] = 8 du_c / dxi_d
    double G[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      G[c][0] = fma(eta * zeta, A[c][6], fma(zeta, A[c][4], fma(eta, A[c][3], A[c][0])));
      G[c][1] = fma(xi * zeta, A[c][6], fma(zeta, A[c][5], fma(xi, A[c][3], A[c][1])));
      G[c][2] = fma(xi * eta, A[c][6], fma(eta, A[c][5], fma(xi, A[c][4], A[c][2])));
    }
    // physical strain (J^-1 = 2/h I): eps = sym grad u, engineering shears, Voigt order
    double e[6];
    e[0] = G[0][0] * inv4h;
    e[1] = G[1][1] * inv4h;
    e[2] = G[2][2] * inv4h;
    e[3] = (G[1][2] + G[2][1]) * inv4h;
    e[4] = (G[0][2] + G[2][0]) * inv4h;
    e[5] = (G[0][1] + G[1][0]) * inv4h;
    // sigma = D_q eps with the 21 stored values (w_q det J_q folded in)
    double d[21];
#pragma unroll
    for (int k = 0; k < 21; ++k) d[k] = inbox ? __ldcs(Dc + (int64_t)(q * 21 + k) * cstride) : 0.0;
    double sg[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < 6; ++j) v = fma(d[i <= j ? sym6(i, j) : sym6(j, i)], e[j], v);
      sg[i] = v;
    }
    const double S[3][3] = {{sg[0], sg[5], sg[4]}, {sg[5], sg[1], sg[3]}, {sg[4], sg[3], sg[2]}};
    // test contraction sum_d sigma_cd dphi_a/dx_d in the modal basis of the test functions
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double r0 = S[c][0], r1 = S[c][1], r2 = S[c][2];
      B[c][0] += r0;
      B[c][1] += r1;
      B[c][2] += r2;
      B[c][3] = fma(eta, r0, fma(xi, r1, B[c][3]));
      B[c][4] = fma(zeta, r0, fma(xi, r2, B[c][4]));
      B[c][5] = fma(zeta, r1, fma(eta, r2, B[c][5]));
      B[c][6] = fma(eta * zeta, r0, fma(xi * zeta, r1, fma(xi * eta, r2, B[c][6])));
    }
  }
  // v_a = sum_m g_m prod_{d in m} s_ad with g_m = B_m / (4h); inverse z into the two faces
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double gx = B[c][0] * inv4h, gy = B[c][1] * inv4h, gz = B[c][2] * inv4h;
    const double gxy = B[c][3] * inv4h, gxz = B[c][4] * inv4h, gyz = B[c][5] * inv4h, gxyz = B[c][6] * inv4h;
    F[4 * c + 0] = cb[4 * c + 0] - gz;
    F[4 * c + 1] = cb[4 * c + 1] + (gx - gxz);
    F[4 * c + 2] = cb[4 * c + 2] + (gy - gyz);
    F[4 * c + 3] = cb[4 * c + 3] + (gxy - gxyz);
    cbo[4 * c + 0] = gz;
    cbo[4 * c + 1] = gx + gxz;
    cbo[4 * c + 2] = gy + gyz;
    cbo[4 * c + 3] = gxy + gxyz;
  }
}

// y = A_c u (mode 0) or + p.Ap (mode 1, CG) from the stored Gauss-point data D.  One cell per
// thread: lane = cell column, warp = cell row; TY consumer warps + 1 producer warp streaming the
// node planes (TMA tensor boxes on the CG vectors, bulk row copies on caller vectors).
template <bool TM, int MODE, int TY, int S, bool GLL>
__global__ void __launch_bounds__(32 * (TY + 1), 1)
    pa21_kernel(Grid g, PlaneSrc x, OutVec yo, const __grid_constant__ CUtensorMap umap, TmaOrigin uorg,
                const double* __restrict__ D, int bc, int64_t kchunk, int64_t kspan, CgScalars* sc, Reduce red,
                int txa, int tya) {
  constexpr int mode = MODE;
  constexpr int TX = 32;
  constexpr int NT = TX * (TY + 1);
  constexpr int ROWS = TY + 1;  // node rows j0-1 .. j0+TY-1
  constexpr int COLS = TX + 1;  // node cols i0-1 .. i0+TX-1
  constexpr int TPART = 4 * TY * TX * 3;
  using Ring = PlaneRing<TM, ROWS, COLS, 3, S>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double red_sh[32];
  Ring ring;
  double* tpart = reinterpret_cast<double*>(smem_raw + Ring::BYTES);  // [4][TY][TX][3]
  uint64_t* tfull = reinterpret_cast<uint64_t*>(tpart + TPART);        // [4][TY]
  uint64_t* tempty = tfull + 4 * TY;                                    // [4][TY]
  ring.carve(smem_raw, reinterpret_cast<unsigned char*>(tempty + 4 * TY));
  const uint32_t tfull_a = smem_u32(tfull), tempty_a = smem_u32(tempty);
  if (mode >= 1 && sc->done) return;

  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = tx + TX * ty;
  const int64_t i0 = (int64_t)blockIdx.x * txa;
  const int64_t j0 = (int64_t)blockIdx.y * tya;
  const int64_t kb = g.k0 + (int64_t)blockIdx.z * kchunk;
  const int64_t ke = min(g.k1, kb + kspan);
  const int64_t pfirst = kb - 1;  // planes kb-1 .. ke (cell layers kb-1 .. ke-1)
  if (tid < 4 * TY) {
    mbar_init(&tfull[tid], 1);
    mbar_init(&tempty[tid], 1);
  }
  ring.init(tid, NT, TY);
  if (TM) ring.set_tshift(i0 - 1, uorg);

  double pq = 0.0;
  if (ty == TY) {
    ring.produce(x, g, pfirst, ke, i0 - 1, j0 - 1, bc, tx, &umap, uorg, nullptr, 0);
  } else {
    const int64_t ci = i0 - 1 + tx, cj = j0 - 1 + ty;
    const double inv4h = 1.0 / (4.0 * g.h);
    const int64_t nj = cj + 1;  // node row this thread outputs (top corners of its cell)
    const bool mc0 = bc && (ci == 0 || ci == g.nx), mc1 = bc && (ci + 1 == 0 || ci + 1 == g.nx);
    const bool mr0 = bc && (cj == 0 || cj == g.ny), mr1 = bc && (cj + 1 == 0 || cj + 1 == g.ny);
    const bool owner = tx >= 1 && tx <= txa && ty < tya && ci <= g.nx && nj <= g.ny;
    const bool bnode_xy = bc && (ci == 0 || ci == g.nx || nj == 0 || nj == g.ny);
    const bool cin = ci >= 0 && ci < g.nx && cj >= 0 && cj < g.ny;  // a cell of the box (xy)
    const int64_t ncells = g.nx * g.ny * g.nz;
    double* yp = yo.y + (kb - g.k0) * yo.ppitch + (owner ? nj * yo.rpitch + ci * 3 : 0);
    const double* xpb = x.main + (kb - g.k0) * x.ppitch + (owner ? nj * x.rpitch + ci * 3 : 0);
    const int nplane = (int)(ke - pfirst + 1);
    const int qface0 = bc ? (int)(0 - kb) : -1000000;
    const int qface1 = bc ? (int)(g.nz - kb) : -1000000;
    double* const tw0 = tpart + (ty * TX + tx) * 3;
    const double* const tr0 = tpart + ((ty + 1) * TX + tx) * 3;
    const uint32_t tfw0 = tfull_a + 8u * ty, tew0 = tempty_a + 8u * ty;
    const uint32_t tfr0 = tfull_a + 8u * (ty + 1), ter0 = tempty_a + 8u * (ty + 1);

    FaceP fb[3];
    double cb[12];
    double xc[3];
#pragma unroll
    for (int t = 0; t < 12; ++t) cb[t] = 0.0;

    auto load_plane = [&](int t, FaceP* ft, double* xn) {
      const int slot = t % S;
      ring.wait(slot, (uint32_t)((t / S) & 1));
      const double* r0 = ring.row_ptr(slot, ty) + tx * 3;
      const double* r1 = ring.row_ptr(slot, ty + 1) + tx * 3;
      const int64_t pl = pfirst + t;
      const bool pface = TM && bc && (pl == 0 || pl == g.nz);
      const bool m00 = pface || mc0 || mr0, m10 = pface || mc1 || mr0;
      const bool m01 = pface || mc0 || mr1, m11 = pface || mc1 || mr1;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double a00 = r0[c], a10 = r0[3 + c], a01 = r1[c], a11 = r1[3 + c];
        xn[c] = a01;
        if (TM && bc && (m00 || m10 || m01 || m11)) {
          a00 = m00 ? 0.0 : a00;
          a10 = m10 ? 0.0 : a10;
          a01 = m01 ? 0.0 : a01;
          a11 = m11 ? 0.0 : a11;
        }
        ft[c] = facep_fwd(a00, a10, a01, a11);
      }
      ring.release(slot, tx);
    };
    load_plane(0, fb, xc);

#pragma unroll 1
    for (int t = 1; t < nplane; ++t) {
      FaceP ft[3];
      double xn[3];
      load_plane(t, ft, xn);
      const int64_t layer = pfirst + t - 1;  // cell layer between planes t-1 and t
      const bool inbox = cin && layer >= 0 && layer < g.nz;
      const double* Dc = D + (inbox ? (layer * g.ny + cj) * g.nx + ci : 0);
      double F[12], cbo[12];
      pa21_layer<GLL>(fb, ft, Dc, ncells, inbox, inv4h, cb, cbo, F);
      double xsave[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) { fb[c] = ft[c]; xsave[c] = xc[c]; xc[c] = xn[c]; }
#pragma unroll
      for (int k = 0; k < 12; ++k) cb[k] = cbo[k];
      if (t >= 2) {  // node plane kb + t - 2 is complete
        const int qo = t - 2;
        const int b = qo & 3;
        const uint32_t n = (uint32_t)(qo >> 2);
        double B[3], Tt[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double G1 = F[4 * c + 0], Gx = F[4 * c + 1], Gy = F[4 * c + 2], Gxy = F[4 * c + 3];
          const double es = G1 - Gy, ed = Gx - Gxy, fs = G1 + Gy, fd = Gx + Gxy;
          const double c00 = es - ed, c10 = es + ed, c01 = fs - fd, c11 = fs + fd;
          const double c10l = __shfl_up_sync(0xffffffffu, c10, 1);
          const double c11l = __shfl_up_sync(0xffffffffu, c11, 1);
          B[c] = c10l + c00;
          Tt[c] = c11l + c01;
        }
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
                if (!TM) xv = xpb[c];  // row path: boundary values are not staged
                vv = xv;
              }
              yp[c] = vv;
              if (mode >= 1) pq = fma(vv, xv, pq);
            }
          }
          yp += yo.ppitch;
          xpb += x.ppitch;
        }
      }
    }
  }
  if (mode >= 1) cg_apply_epilogue(pq, false, sc, red, red_sh);
}

int64_t pa21_doubles(int64_t ncells) { return ncells * 8 * 21; }

cudaError_t launch_pa21_setup(const double2* lm, int64_t ncells, double h, double* D, cudaStream_t s,
                              int sm_count) {
  const double wdet = h * h * h / 8.0;  // w_q = 1 (both 2-point rules), det J = (h/2)^3
  const int64_t want = (ncells + 255) / 256;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count * 8));
  pa21_setup_kernel<<<grid, 256, 0, s>>>(lm, ncells, wdet, D);
  add_launches(1);
  return cudaGetLastError();
}

template <bool TM, int S>
static cudaError_t pa21_launch_cfg(const Grid& g, PlaneSrc x, OutVec y, const CUtensorMap* umap, TmaOrigin org,
                                   const double* D, int bc, int quad, int mode, CgScalars* sc, Reduce red,
                                   cudaStream_t s, int sm_count) {
  constexpr int TX = 32, TY = kPaTY;
  using Ring = PlaneRing<TM, TY + 1, TX + 1, 3, S>;
  const size_t smem = Ring::BYTES + Ring::META + 4 * TY * TX * 3 * sizeof(double) + 8 * TY * sizeof(uint64_t);
  auto pick = [&](auto gl) {
    constexpr bool G = decltype(gl)::value;
    return mode == 1 ? pa21_kernel<TM, 1, TY, S, G> : pa21_kernel<TM, 0, TY, S, G>;
  };
  auto kern = quad == 1 ? pick(std::true_type{}) : pick(std::false_type{});
  {
    const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
  }
  int txa, tya;
  const int64_t xt = balanced_tiles(g.nx + 1, TX - 1, &txa);
  const int64_t yt = balanced_tiles(g.ny + 1, TY - 1, &tya);
  const int64_t nplanes = g.k1 - g.k0;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * (TY + 1), smem);
  const int64_t minchunk = (xt * yt * (nplanes / 8) < sm_count) ? 2 : 8;
  const WorkGrid w = make_workgrid((int)xt, (int)yt, nplanes, (int64_t)std::max(occ, 1) * sm_count, minchunk, 2);
  if (xt * yt * w.zc > kMaxCtas) return cudaErrorInvalidConfiguration;
  dim3 grid((unsigned)xt, (unsigned)yt, (unsigned)w.zc), block(TX, TY + 1);
  CUtensorMap um;
  if (TM) um = *umap; else std::memset(&um, 0, sizeof(um));
  kern<<<grid, block, smem, s>>>(g, x, y, um, org, D, bc, w.kchunk, w.kchunk, sc, red, txa, tya);
  add_launches(1);
  return cudaGetLastError();
}

// u planes staged by bulk row copies on every vector (the CG vectors included): the kernel is
// bound by the 1,344 B/cell of stored data, not by the u staging
cudaError_t launch_pa21_apply(int bc, int quad, const Grid& g, PlaneSrc x, OutVec y, const double* D, int mode,
                              CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  if (mode > 1) return cudaErrorInvalidValue;
  return pa21_launch_cfg<false, 4>(g, x, y, nullptr, TmaOrigin{0, 0, 0}, D, bc, quad, mode, sc, red, s, sm_count);
}

}  // namespace fem
