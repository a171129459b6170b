// kernels_hex.cu -- general (deformed) trilinear hexahedral meshes: Algorithm 1 as written
// (P:311-360): gather the cell's nodal coordinates and u^e through the explicit node map
// (Table 2 "node map", "read nodal position"), recompute J, det J, J^-1 at each of the 2x2x2
// Gauss points, form grad u, the stress (scaled by w_q det J), P = sigma J^-T and
// v_i += P grad^phi_i, and add v^e into v.  FP64.
//
// B200 form: one thread per cell, everything in registers.  The reference
// gradients are applied in the Hadamard ("modal") basis of the trilinear space -- the 8 nodal
// values of a field become 7 modal coefficients (23 adds), from which the derivative at each
// Gauss point is 3 adds -- and the test contraction is accumulated in the same basis and
// transformed back once per cell (22 adds per component).  J^-1 and det J are used through the
// cofactor matrix: det(J) J^-T = cof(J), so P w det J = sigma cof(J) and one reciprocal per
// point suffices.  Scatter: red.global.add.f64 into v (the paper's atomics; P:303 -- the
// result is exact up to the summation order), constrained nodes skipped and then overwritten
// by the identity rows y = x in a second kernel.
//
// Constants (derivation in DESIGN.md §5.5): with unnormalised modal sums c (c_m = sum_a u_a
// prod_{d in m} s_ad) the reference derivative is d_e u(q) = (1/8)[c_e + g s_d1 c_ed1 +
// g s_d2 c_ed2 + g^2 s_d1 s_d2 c_xyz] at q = g s_q, g = 1/sqrt(3).  J' = 8 J and G' = 8 grad^ u
// drop the 1/8 (grad u = G' J'^-1 is invariant), det J = det J' / 512, cof J = cof J' / 64,
// grad^ phi_a carries 1/8: v_a = (1/512) sum_q sum_e (sigma cof J')_{ce} s_ae prod(1 + ..g).
#include <algorithm>

#include <cub/cub.cuh>

#include "fem_internal.cuh"

namespace fem {

namespace {

constexpr double kG = 0.57735026918962576451;   // 1/sqrt(3): Gauss point
constexpr double kG2 = 1.0 / 3.0;               // g^2
constexpr double kInv512 = 1.0 / 512.0;

struct Modal {
  double x, y, z, xy, xz, yz, xyz;  // the constant mode is not needed (no gradient)
};

// forward transform of 8 corner values in bit order (bit 0: x, bit 1: y, bit 2: z)
__device__ __forceinline__ Modal hadamard(const double v[8]) {
  const double s0 = v[0] + v[1], d0 = v[1] - v[0], s1 = v[2] + v[3], d1 = v[3] - v[2];
  const double s2 = v[4] + v[5], d2 = v[5] - v[4], s3 = v[6] + v[7], d3 = v[7] - v[6];
  const double ss0 = s0 + s1, y0 = s1 - s0, x0 = d0 + d1, xy0 = d1 - d0;
  const double ss1 = s2 + s3, y1 = s3 - s2, x1 = d2 + d3, xy1 = d3 - d2;
  Modal m;
  m.x = x0 + x1; m.y = y0 + y1; m.xy = xy0 + xy1;
  m.z = ss1 - ss0; m.xz = x1 - x0; m.yz = y1 - y0; m.xyz = xy1 - xy0;
  return m;
}

// pre-scale the bilinear / trilinear coefficients by g, g^2 (Gauss point coordinates)
// (GLL: the 2-point Gauss-Lobatto points are the nodes, g = 1; reading R1)
template <bool GLL>
__device__ __forceinline__ void prescale(Modal& m) {
  constexpr double g = GLL ? 1.0 : kG, g2 = GLL ? 1.0 : kG2;
  m.xy *= g; m.xz *= g; m.yz *= g; m.xyz *= g2;
}

// reference gradient (x 8) of a field at the Gauss point with signs (sx, sy, sz)
template <int SX, int SY, int SZ>
__device__ __forceinline__ void dref(const Modal& m, double& dx, double& dy, double& dz) {
  dx = m.x + (SY * m.xy + (SZ * m.xz + (SY * SZ) * m.xyz));
  dy = m.y + (SX * m.xy + (SZ * m.yz + (SX * SZ) * m.xyz));
  dz = m.z + (SX * m.xz + (SY * m.yz + (SX * SY) * m.xyz));
}

// transposed accumulation of P_{c,.} at the Gauss point (SX, SY, SZ) into the modal sums
template <int SX, int SY, int SZ>
__device__ __forceinline__ void accum(Modal& a, double p0, double p1, double p2) {
  a.x += p0; a.y += p1; a.z += p2;
  a.xy += SY * p0 + SX * p1;
  a.xz += SZ * p0 + SX * p2;
  a.yz += SZ * p1 + SY * p2;
  a.xyz += (SY * SZ) * p0 + ((SX * SZ) * p1 + (SX * SY) * p2);
}

// inverse transform of the modal sums (constant mode 0) to the 8 corners, bit order
__device__ __forceinline__ void inverse(const Modal& m, double v[8]) {
  // z: A = x +- xz, B = y +- yz, C = xy +- xyz, D = +- z
  const double Am = m.x - m.xz, Ap = m.x + m.xz, Bm = m.y - m.yz, Bp = m.y + m.yz;
  const double Cm = m.xy - m.xyz, Cp = m.xy + m.xyz;
  // y: E = D +- B, F = A +- C   (z = -1: D = -z; z = +1: D = +z)
  const double Emm = -m.z - Bm, Emp = -m.z + Bm, Epm = m.z - Bp, Epp = m.z + Bp;
  const double Fmm = Am - Cm, Fmp = Am + Cm, Fpm = Ap - Cp, Fpp = Ap + Cp;
  // x: v = E +- F ; index = bx + 2 by + 4 bz
  v[0] = Emm - Fmm; v[1] = Emm + Fmm;
  v[2] = Emp - Fmp; v[3] = Emp + Fmp;
  v[4] = Epm - Fpm; v[5] = Epm + Fpm;
  v[6] = Epp - Fpp; v[7] = Epp + Fpp;
}

// one Gauss point: J' from the coordinate modes, cofactors, det; grad u, stress, P; transposed
// accumulation; energy (u^T A_e u contribution, modes >= 1)
template <int KIND, int C, int SX, int SY, int SZ>
__device__ __forceinline__ void gauss_point(const Modal& mx, const Modal& my, const Modal& mz,
                                            const Modal* mu, Modal* acc, double L, double M,
                                            double& energy) {
  double J[3][3];
  dref<SX, SY, SZ>(mx, J[0][0], J[0][1], J[0][2]);
  dref<SX, SY, SZ>(my, J[1][0], J[1][1], J[1][2]);
  dref<SX, SY, SZ>(mz, J[2][0], J[2][1], J[2][2]);
  double cf[3][3];  // cofactor matrix: det(J) J^-T
  cf[0][0] = fma(J[1][1], J[2][2], -J[1][2] * J[2][1]);
  cf[0][1] = fma(J[1][2], J[2][0], -J[1][0] * J[2][2]);
  cf[0][2] = fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
  cf[1][0] = fma(J[0][2], J[2][1], -J[0][1] * J[2][2]);
  cf[1][1] = fma(J[0][0], J[2][2], -J[0][2] * J[2][0]);
  cf[1][2] = fma(J[0][1], J[2][0], -J[0][0] * J[2][1]);
  cf[2][0] = fma(J[0][1], J[1][2], -J[0][2] * J[1][1]);
  cf[2][1] = fma(J[0][2], J[1][0], -J[0][0] * J[1][2]);
  cf[2][2] = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]);
  const double det = fma(J[0][0], cf[0][0], fma(J[0][1], cf[0][1], J[0][2] * cf[0][2]));
  const double rdet = __drcp_rn(det);
  // Gt[c][d] = det * d u_c / d x_d = sum_e G'[c][e] cf[d][e]
  double Gt[C][3];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double g0, g1, g2;
    dref<SX, SY, SZ>(mu[c], g0, g1, g2);
#pragma unroll
    for (int d = 0; d < 3; ++d) Gt[c][d] = fma(g0, cf[d][0], fma(g1, cf[d][1], g2 * cf[d][2]));
  }
  if (KIND == 2) {
    // sigma~ = det * sigma = lambda tr(Gt) I + mu (Gt + Gt^T)   (reading R4)
    const double tr = Gt[0][0] + Gt[1][1] + Gt[2][2];
    const double Lt = L * tr, M2 = M + M;
    const double s00 = fma(M2, Gt[0][0], Lt), s11 = fma(M2, Gt[1][1], Lt), s22 = fma(M2, Gt[2][2], Lt);
    const double e01 = Gt[0][1] + Gt[1][0], e02 = Gt[0][2] + Gt[2][0], e12 = Gt[1][2] + Gt[2][1];
    const double s01 = M * e01, s02 = M * e02, s12 = M * e12;
    energy = fma(rdet, fma(s00, Gt[0][0], fma(s11, Gt[1][1], fma(s22, Gt[2][2],
                 fma(s01, e01, fma(s02, e02, s12 * e12))))), energy);
    const double S[3][3] = {{s00 * rdet, s01 * rdet, s02 * rdet},
                            {0.0, s11 * rdet, s12 * rdet},
                            {0.0, 0.0, s22 * rdet}};
    auto sg = [&](int a, int b) { return a <= b ? S[a][b] : S[b][a]; };
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double p[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) p[e] = fma(sg(c, 0), cf[0][e], fma(sg(c, 1), cf[1][e], sg(c, 2) * cf[2][e]));
      accum<SX, SY, SZ>(acc[c], p[0], p[1], p[2]);
    }
  } else {
    // Laplace (scalar / per component): flux = grad u; P = grad u cof(J)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      energy = fma(rdet, fma(Gt[c][0], Gt[c][0], fma(Gt[c][1], Gt[c][1], Gt[c][2] * Gt[c][2])), energy);
      const double f0 = Gt[c][0] * rdet, f1 = Gt[c][1] * rdet, f2 = Gt[c][2] * rdet;
      double p[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) p[e] = fma(f0, cf[0][e], fma(f1, cf[1][e], f2 * cf[2][e]));
      accum<SX, SY, SZ>(acc[c], p[0], p[1], p[2]);
    }
  }
}

constexpr int kHexThreads = 128;

template <int KIND, int MODE, bool GLL>
__global__ void __launch_bounds__(kHexThreads, (KIND == 0) ? 3 : 2)
    hex_apply_kernel(const int4* __restrict__ cells, const double4* __restrict__ xyz,
                     const double2* __restrict__ lm, const double* __restrict__ u,
                     double* __restrict__ y, double* __restrict__ E, int64_t ncells, int bc, CgScalars* sc,
                     Reduce red) {
  constexpr int C = (KIND == 0) ? 1 : 3;
  __shared__ double red_sh[32];
  if (MODE >= 1 && sc->done) return;
  double energy = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncells; e += stride) {
    // gather (Alg. 1 line 1): node map -> coordinates and u^e (masked at constrained nodes)
    const int4 lo = cells[2 * e], hi = cells[2 * e + 1];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    int id[8];
    bool fix[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      fix[a] = bc && raw[a] < 0;  // Dirichlet node of an operator with bc (mask P)
      id[a] = raw[a] & 0x7fffffff;
    }
    Modal mx, my, mz;
    {
      double X[8], Y[8], Z[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const double4 p = xyz[id[a]];
        X[a] = p.x; Y[a] = p.y; Z[a] = p.z;
      }
      mx = hadamard(X); my = hadamard(Y); mz = hadamard(Z);
      prescale<GLL>(mx); prescale<GLL>(my); prescale<GLL>(mz);
    }
    Modal mu[C], acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double U[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) U[a] = fix[a] ? 0.0 : u[(int64_t)C * id[a] + c];
      mu[c] = hadamard(U);
      prescale<GLL>(mu[c]);
      acc[c] = Modal{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    }
    double L = 0.0, M = 0.0;
    if (KIND == 2) {
      const double2 v = lm[e];
      L = v.x; M = v.y;
    }
    double en = 0.0;
    // the 8 Gauss points (Alg. 1 "for each quadrature point q")
    gauss_point<KIND, C, -1, -1, -1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, +1, -1, -1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, -1, +1, -1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, +1, +1, -1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, -1, -1, +1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, +1, -1, +1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, -1, +1, +1>(mx, my, mz, mu, acc, L, M, en);
    gauss_point<KIND, C, +1, +1, +1>(mx, my, mz, mu, acc, L, M, en);
    energy += en;
    // back to nodes and scatter-add (Alg. 1 last line)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Modal& m = acc[c];
      m.x *= kInv512; m.y *= kInv512; m.z *= kInv512;
      constexpr double g = GLL ? 1.0 : kG, g2 = GLL ? 1.0 : kG2;
      m.xy *= g * kInv512; m.xz *= g * kInv512; m.yz *= g * kInv512; m.xyz *= g2 * kInv512;
      double v[8];
      inverse(m, v);
      if (E) {  // deterministic scatter: element outputs, summed per node by hex_gather_kernel
#pragma unroll
        for (int a = 0; a < 8; ++a) E[((int64_t)e * 8 + a) * C + c] = fix[a] ? 0.0 : v[a];
      } else {
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (!fix[a]) atomicAdd(y + (int64_t)C * id[a] + c, v[a]);
      }
    }
  }
  if (MODE >= 1) {  // p.Ap of the masked operator part: sum of the element energies
    double total;
    if (last_block_reduce(block_sum(energy * kInv512, red_sh), red, red_sh, &total)) sc->pq = total;
  }
}

// ---- software-pipelined variant (FEM_HEX_PREFETCH) ---------------------------
// Same per-cell arithmetic; a persistent grid (one CTA per resident slot) and a two-deep
// cp.async pipeline per thread: while cell e is computed, the node ids of cell e + 2 stride and
// the coordinates / u / material of cell e + stride (gathered through the ids already staged)
// travel into this thread's shared-memory staging area, so the gather latency (ncu: the top
// stall of the one-shot kernel, 1.97 warps per issue on long_scoreboard) overlaps the FP64 work.
__device__ __forceinline__ void hex_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void hex_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void hex_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void hex_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int C>
constexpr size_t hex_pf_smem(int T) {
  return (size_t)T * (8 * 32 + 8 * C * 8 + 4 * 16 + 16);
}

template <int KIND, int MODE, bool GLL>
__global__ void __launch_bounds__(kHexThreads, (KIND == 0) ? 3 : 2)
    hex_apply_pf_kernel(const int4* __restrict__ cells, const double4* __restrict__ xyz,
                        const double2* __restrict__ lm, const double* __restrict__ u,
                        double* __restrict__ y, double* __restrict__ E, int64_t ncells, int bc, CgScalars* sc,
                        Reduce red) {
  constexpr int C = (KIND == 0) ? 1 : 3;
  constexpr int T = kHexThreads;
  __shared__ double red_sh[32];
  extern __shared__ __align__(16) unsigned char hsm[];
  double4* sxyz = reinterpret_cast<double4*>(hsm);         // [8][T]
  double* su = reinterpret_cast<double*>(sxyz + 8 * T);    // [8 C][T]
  int4* sid = reinterpret_cast<int4*>(su + 8 * C * T);     // [2 slots][2][T]
  double2* slm = reinterpret_cast<double2*>(sid + 4 * T);  // [T]
  if (MODE >= 1 && sc->done) return;
  const int tid = threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * T;
  auto stage_ids = [&](int64_t c, int slot) {
    hex_cp16(&sid[(slot * 2 + 0) * T + tid], &cells[2 * c]);
    hex_cp16(&sid[(slot * 2 + 1) * T + tid], &cells[2 * c + 1]);
  };
  auto stage_cell = [&](int64_t c, int slot) {  // gathers through the ids staged in `slot`
    const int4 lo = sid[(slot * 2 + 0) * T + tid], hi = sid[(slot * 2 + 1) * T + tid];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int64_t n = raw[a] & 0x7fffffff;
      const double* src = reinterpret_cast<const double*>(xyz + n);
      hex_cp16(&sxyz[a * T + tid], src);
      hex_cp16(reinterpret_cast<double*>(&sxyz[a * T + tid]) + 2, src + 2);
#pragma unroll
      for (int k = 0; k < C; ++k) hex_cp8(&su[(a * C + k) * T + tid], u + (int64_t)C * n + k);
    }
    if (KIND == 2) hex_cp16(&slm[tid], &lm[c]);
  };
  double energy = 0.0;
  int64_t e = blockIdx.x * (int64_t)T + tid;
  if (e < ncells) stage_ids(e, 0);
  if (e + stride < ncells) stage_ids(e + stride, 1);
  hex_commit();
  hex_wait_all();
  if (e < ncells) stage_cell(e, 0);
  hex_commit();
  int slot = 0;
#pragma unroll 1
  for (; e < ncells; e += stride, slot ^= 1) {
    hex_wait_all();  // cell e's gathers and the ids of e + stride have landed
    const int4 lo = sid[(slot * 2 + 0) * T + tid], hi = sid[(slot * 2 + 1) * T + tid];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    int id[8];
    bool fix[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      fix[a] = bc && raw[a] < 0;
      id[a] = raw[a] & 0x7fffffff;
    }
    Modal mx, my, mz, mu[C], acc[C];
    {
      double X[8], Y[8], Z[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const double4 p = sxyz[a * T + tid];
        X[a] = p.x; Y[a] = p.y; Z[a] = p.z;
      }
      mx = hadamard(X); my = hadamard(Y); mz = hadamard(Z);
      prescale<GLL>(mx); prescale<GLL>(my); prescale<GLL>(mz);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double U[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) U[a] = fix[a] ? 0.0 : su[(a * C + c) * T + tid];
      mu[c] = hadamard(U);
      prescale<GLL>(mu[c]);
      acc[c] = Modal{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    }
    double L = 0.0, M = 0.0;
    if (KIND == 2) {
      const double2 v = slm[tid];
      L = v.x; M = v.y;
    }
    // the staged values are in registers now: refill the staging area for the next cell
    const int64_t en = e + stride;
    if (en < ncells) stage_cell(en, slot ^ 1);
    if (en + stride < ncells) stage_ids(en + stride, slot);
    hex_commit();
    double en_q = 0.0;
    gauss_point<KIND, C, -1, -1, -1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, +1, -1, -1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, -1, +1, -1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, +1, +1, -1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, -1, -1, +1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, +1, -1, +1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, -1, +1, +1>(mx, my, mz, mu, acc, L, M, en_q);
    gauss_point<KIND, C, +1, +1, +1>(mx, my, mz, mu, acc, L, M, en_q);
    energy += en_q;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Modal& m = acc[c];
      m.x *= kInv512; m.y *= kInv512; m.z *= kInv512;
      constexpr double g = GLL ? 1.0 : kG, g2 = GLL ? 1.0 : kG2;
      m.xy *= g * kInv512; m.xz *= g * kInv512; m.yz *= g * kInv512; m.xyz *= g2 * kInv512;
      double v[8];
      inverse(m, v);
      if (E) {  // deterministic scatter: element outputs, summed per node by hex_gather_kernel
#pragma unroll
        for (int a = 0; a < 8; ++a) E[((int64_t)e * 8 + a) * C + c] = fix[a] ? 0.0 : v[a];
      } else {
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (!fix[a]) atomicAdd(y + (int64_t)C * id[a] + c, v[a]);
      }
    }
  }
  hex_wait_all();
  if (MODE >= 1) {
    double total;
    if (last_block_reduce(block_sum(energy * kInv512, red_sh), red, red_sh, &total)) sc->pq = total;
  }
}

// identity rows of the constrained nodes: y = x; mode 1 adds sum x_b^2 to p.Ap
template <int MODE>
__global__ void __launch_bounds__(256) hex_dirichlet_kernel(const int32_t* __restrict__ nodes, int64_t nb, int C,
                                                            const double* __restrict__ x, double* __restrict__ y,
                                                            CgScalars* sc, Reduce red) {
  __shared__ double red_sh[32];
  if (MODE >= 1 && sc->done) return;
  double acc = 0.0;
  const int64_t n = nb * C;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += stride) {
    const int64_t i = (int64_t)nodes[t / C] * C + t % C;
    const double v = x[i];
    y[i] = v;
    acc = fma(v, v, acc);
  }
  if (MODE >= 1) {
    double total;
    if (last_block_reduce(block_sum(acc, red_sh), red, red_sh, &total)) sc->pq += total;
  }
}

// validation: node ids in range, det J > 0 at every Gauss point
__global__ void __launch_bounds__(256) hex_check_kernel(const int4* __restrict__ cells,
                                                        const double4* __restrict__ xyz, int64_t ncells,
                                                        int64_t nnodes, int rule, unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncells; e += stride) {
    const int4 lo = cells[2 * e], hi = cells[2 * e + 1];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    bool ok = true;
    double X[8], Y[8], Z[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int id = raw[a] & 0x7fffffff;
      ok = ok && id < nnodes;
      const double4 p = xyz[ok ? id : 0];
      X[a] = p.x; Y[a] = p.y; Z[a] = p.z;
    }
    if (!ok) {
      atomicAdd(&bad[0], 1ull);
      continue;
    }
    const Modal ux = hadamard(X), uy = hadamard(Y), uz = hadamard(Z);
    bool pos = true;
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // the 8 points of the rule: Gauss (0) or Gauss-Lobatto = nodes (1)
      Modal mx = ux, my = uy, mz = uz;
      if (rule == 0) { prescale<false>(mx); prescale<false>(my); prescale<false>(mz); }
      const double sx = (q & 1) ? 1.0 : -1.0, sy = (q & 2) ? 1.0 : -1.0, sz = (q & 4) ? 1.0 : -1.0;
      double J[3][3];
      const Modal* f[3] = {&mx, &my, &mz};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const Modal& m = *f[d];
        J[d][0] = m.x + sy * m.xy + sz * m.xz + sy * sz * m.xyz;
        J[d][1] = m.y + sx * m.xy + sz * m.yz + sx * sz * m.xyz;
        J[d][2] = m.z + sx * m.xz + sy * m.yz + sx * sy * m.xyz;
      }
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      pos = pos && det > 0.0 && isfinite(det);
    }
    if (!pos) atomicAdd(&bad[1], 1ull);
  }
}

// VTK corner order -> bit order (bit 0 x, bit 1 y, bit 2 z), Dirichlet flag in bit 31
__global__ void hex_pack_cells_kernel(const int32_t* __restrict__ vtk, const uint8_t* __restrict__ dir,
                                      int64_t ncells, int64_t nnodes, int* __restrict__ out,
                                      unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ncells * 8; t += stride) {
    const int64_t e = t >> 3;
    const int bx = (int)(t & 1), by = (int)((t >> 1) & 1), bz = (int)((t >> 2) & 1);
    const int vidx = 4 * bz + (by ? (bx ? 2 : 3) : bx);  // VTK index of this bit-order corner
    const int id = vtk[e * 8 + vidx];
    if (id < 0 || id >= nnodes) {
      atomicAdd(&bad[0], 1ull);
      out[t] = 0;
      continue;
    }
    out[t] = (dir && dir[id]) ? (int)((unsigned)id | 0x80000000u) : id;
  }
}

// ------------------------------------------------------------------------------------------
// Partial assembly (the paper's comparison method, Table 3): the geometry
// of every Gauss point is computed once and stored; the apply then reads it instead of
// recomputing J.  Stored per cell and point (SoA, [q][k][cell], coalesced):
//   Laplace:    D' = cof(J')^T cof(J') / det J'   (6 values, the paper's "6 per qpt")
//   elasticity: B  = cof(J') / sqrt(det J')         (9 values; the paper stores 21 with the
//               material folded in -- here lambda, mu stay per cell, 2 values)
// so that P' = G' D' (Laplace) or P' = sigma(G' B^T) B (elasticity) equal the matrix-free P'.
template <int KIND, bool GLL>
__global__ void __launch_bounds__(256) hex_pa_setup_kernel(const int4* __restrict__ cells,
                                                           const double4* __restrict__ xyz,
                                                           double* __restrict__ pa, int64_t ncells) {
  constexpr int K = (KIND == 2) ? 9 : 6;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncells; e += stride) {
    const int4 lo = cells[2 * e], hi = cells[2 * e + 1];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    double X[8], Y[8], Z[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const double4 p = xyz[raw[a] & 0x7fffffff];
      X[a] = p.x; Y[a] = p.y; Z[a] = p.z;
    }
    Modal mx = hadamard(X), my = hadamard(Y), mz = hadamard(Z);
    prescale<GLL>(mx); prescale<GLL>(my); prescale<GLL>(mz);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double sx = (q & 1) ? 1.0 : -1.0, sy = (q & 2) ? 1.0 : -1.0, sz = (q & 4) ? 1.0 : -1.0;
      double J[3][3];
      const Modal* f[3] = {&mx, &my, &mz};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const Modal& m = *f[d];
        J[d][0] = m.x + (sy * m.xy + (sz * m.xz + (sy * sz) * m.xyz));
        J[d][1] = m.y + (sx * m.xy + (sz * m.yz + (sx * sz) * m.xyz));
        J[d][2] = m.z + (sx * m.xz + (sy * m.yz + (sx * sy) * m.xyz));
      }
      double cf[3][3];
      cf[0][0] = fma(J[1][1], J[2][2], -J[1][2] * J[2][1]);
      cf[0][1] = fma(J[1][2], J[2][0], -J[1][0] * J[2][2]);
      cf[0][2] = fma(J[1][0], J[2][1], -J[1][1] * J[2][0]);
      cf[1][0] = fma(J[0][2], J[2][1], -J[0][1] * J[2][2]);
      cf[1][1] = fma(J[0][0], J[2][2], -J[0][2] * J[2][0]);
      cf[1][2] = fma(J[0][1], J[2][0], -J[0][0] * J[2][1]);
      cf[2][0] = fma(J[0][1], J[1][2], -J[0][2] * J[1][1]);
      cf[2][1] = fma(J[0][2], J[1][0], -J[0][0] * J[1][2]);
      cf[2][2] = fma(J[0][0], J[1][1], -J[0][1] * J[1][0]);
      const double det = fma(J[0][0], cf[0][0], fma(J[0][1], cf[0][1], J[0][2] * cf[0][2]));
      double* out = pa + (int64_t)q * K * ncells + e;
      if (KIND == 2) {
        const double rs = rsqrt(det);
#pragma unroll
        for (int d = 0; d < 3; ++d)
#pragma unroll
          for (int k = 0; k < 3; ++k) out[(3 * d + k) * ncells] = cf[d][k] * rs;
      } else {
        const double rd = 1.0 / det;
        // D'_{ef} = sum_d cf[d][e] cf[d][f] / det : (00, 01, 02, 11, 12, 22)
        const int E[6] = {0, 0, 0, 1, 1, 2}, Fi[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
        for (int k = 0; k < 6; ++k)
          out[k * ncells] =
              fma(cf[0][E[k]], cf[0][Fi[k]], fma(cf[1][E[k]], cf[1][Fi[k]], cf[2][E[k]] * cf[2][Fi[k]])) * rd;
      }
    }
  }
}

template <int KIND, int C, int SX, int SY, int SZ>
__device__ __forceinline__ void pa_point(const double* __restrict__ g, int64_t ncells, const Modal* mu,
                                         Modal* acc, double L, double M, double& energy) {
  if (KIND == 2) {
    double B[3][3];
#pragma unroll
    for (int k = 0; k < 9; ++k) B[k / 3][k % 3] = g[k * ncells];
    double Gt[3][3];  // G' B^T = sqrt(det J') grad u
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double g0, g1, g2;
      dref<SX, SY, SZ>(mu[c], g0, g1, g2);
#pragma unroll
      for (int d = 0; d < 3; ++d) Gt[c][d] = fma(g0, B[d][0], fma(g1, B[d][1], g2 * B[d][2]));
    }
    const double tr = Gt[0][0] + Gt[1][1] + Gt[2][2];
    const double Lt = L * tr, M2 = M + M;
    const double s00 = fma(M2, Gt[0][0], Lt), s11 = fma(M2, Gt[1][1], Lt), s22 = fma(M2, Gt[2][2], Lt);
    const double e01 = Gt[0][1] + Gt[1][0], e02 = Gt[0][2] + Gt[2][0], e12 = Gt[1][2] + Gt[2][1];
    const double s01 = M * e01, s02 = M * e02, s12 = M * e12;
    energy = fma(s00, Gt[0][0], fma(s11, Gt[1][1], fma(s22, Gt[2][2], fma(s01, e01, fma(s02, e02, fma(s12, e12, energy))))));
    const double S[3][3] = {{s00, s01, s02}, {s01, s11, s12}, {s02, s12, s22}};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double p[3];
#pragma unroll
      for (int e = 0; e < 3; ++e) p[e] = fma(S[c][0], B[0][e], fma(S[c][1], B[1][e], S[c][2] * B[2][e]));
      accum<SX, SY, SZ>(acc[c], p[0], p[1], p[2]);
    }
  } else {
    const double d00 = g[0], d01 = g[ncells], d02 = g[2 * ncells], d11 = g[3 * ncells],
                 d12 = g[4 * ncells], d22 = g[5 * ncells];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double g0, g1, g2;
      dref<SX, SY, SZ>(mu[c], g0, g1, g2);
      const double p0 = fma(d00, g0, fma(d01, g1, d02 * g2));
      const double p1 = fma(d01, g0, fma(d11, g1, d12 * g2));
      const double p2 = fma(d02, g0, fma(d12, g1, d22 * g2));
      energy = fma(g0, p0, fma(g1, p1, fma(g2, p2, energy)));
      accum<SX, SY, SZ>(acc[c], p0, p1, p2);
    }
  }
}

template <int KIND, int MODE, bool GLL>
__global__ void __launch_bounds__(128, (KIND == 0) ? 4 : 2)
    hex_pa_apply_kernel(const int4* __restrict__ cells, const double* __restrict__ pa,
                        const double2* __restrict__ lm, const double* __restrict__ u,
                        double* __restrict__ y, double* __restrict__ E, int64_t ncells, int bc, CgScalars* sc,
                        Reduce red) {
  constexpr int C = (KIND == 0) ? 1 : 3;
  constexpr int K = (KIND == 2) ? 9 : 6;
  __shared__ double red_sh[32];
  if (MODE >= 1 && sc->done) return;
  double energy = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ncells; e += stride) {
    const int4 lo = cells[2 * e], hi = cells[2 * e + 1];
    const int raw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    int id[8];
    bool fix[8];
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      fix[a] = bc && raw[a] < 0;
      id[a] = raw[a] & 0x7fffffff;
    }
    Modal mu[C], acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double U[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) U[a] = fix[a] ? 0.0 : u[(int64_t)C * id[a] + c];
      mu[c] = hadamard(U);
      prescale<GLL>(mu[c]);
      acc[c] = Modal{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    }
    double L = 0.0, M = 0.0;
    if (KIND == 2) {
      const double2 v = lm[e];
      L = v.x; M = v.y;
    }
    double en = 0.0;
    const double* g = pa + e;
    const int64_t qs = (int64_t)K * ncells;
    pa_point<KIND, C, -1, -1, -1>(g + 0 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, +1, -1, -1>(g + 1 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, -1, +1, -1>(g + 2 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, +1, +1, -1>(g + 3 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, -1, -1, +1>(g + 4 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, +1, -1, +1>(g + 5 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, -1, +1, +1>(g + 6 * qs, ncells, mu, acc, L, M, en);
    pa_point<KIND, C, +1, +1, +1>(g + 7 * qs, ncells, mu, acc, L, M, en);
    energy += en;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      Modal& m = acc[c];
      m.x *= kInv512; m.y *= kInv512; m.z *= kInv512;
      constexpr double g = GLL ? 1.0 : kG, g2 = GLL ? 1.0 : kG2;
      m.xy *= g * kInv512; m.xz *= g * kInv512; m.yz *= g * kInv512; m.xyz *= g2 * kInv512;
      double v[8];
      inverse(m, v);
      if (E) {  // deterministic scatter: element outputs, summed per node by hex_gather_kernel
#pragma unroll
        for (int a = 0; a < 8; ++a) E[((int64_t)e * 8 + a) * C + c] = fix[a] ? 0.0 : v[a];
      } else {
#pragma unroll
        for (int a = 0; a < 8; ++a)
          if (!fix[a]) atomicAdd(y + (int64_t)C * id[a] + c, v[a]);
      }
    }
  }
  if (MODE >= 1) {
    double total;
    if (last_block_reduce(block_sum(energy * kInv512, red_sh), red, red_sh, &total)) sc->pq = total;
  }
}

int grid_for(int64_t n, int threads, int sm_count, int per_sm) {
  const int64_t want = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count * per_sm));
}

}  // namespace

cudaError_t launch_hex_apply(int kind, int bc, int quad, const int4* cells, const double4* xyz, const double2* lm,
                             const double* x, double* y, double* E, int64_t ncells, int mode, CgScalars* sc,
                             Reduce red, cudaStream_t s, int sm_count) {
  if (ncells <= 0) return cudaSuccess;
  // measured: the pipelined kernel wins for the elasticity CG apply (2.87 ->
  // 2.67 ms at H1) but not for the plain elasticity apply (2.43 -> 2.49) nor the scalar kind
  if (kHexPrefetch && kind == 2 && mode >= 1) {  // persistent grid: one CTA per resident slot
    const int per_sm = kind == 0 ? 3 : 2;
    const int64_t want = (ncells + kHexThreads - 1) / kHexThreads;
    const int grid = (int)std::min<int64_t>(want, (int64_t)per_sm * sm_count);
    if (mode >= 1 && grid > red.capacity) return cudaErrorInvalidConfiguration;
#define PF_LAUNCH(K, M, G)                                                                               \
  {                                                                                                       \
    constexpr size_t sm = hex_pf_smem<(K == 0) ? 1 : 3>(kHexThreads);                                     \
    {                                                                                                     \
      const cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(hex_apply_pf_kernel<K, M, G>),  \
                                             (int)sm);                                                    \
      if (e != cudaSuccess) return e;                                                                     \
    }                                                                                                     \
    hex_apply_pf_kernel<K, M, G><<<grid, kHexThreads, sm, s>>>(cells, xyz, lm, x, y, E, ncells, bc, sc, red); \
  }
#define PF_LAUNCH2(K, M) { if (quad == 1) PF_LAUNCH(K, M, true) else PF_LAUNCH(K, M, false) }
    if (kind == 0) { if (mode) PF_LAUNCH2(0, 1) else PF_LAUNCH2(0, 0) }
    else if (kind == 1) { if (mode) PF_LAUNCH2(1, 1) else PF_LAUNCH2(1, 0) }
    else { if (mode) PF_LAUNCH2(2, 1) else PF_LAUNCH2(2, 0) }
#undef PF_LAUNCH2
#undef PF_LAUNCH
    add_launches(1);
    return cudaGetLastError();
  }
  const int grid = grid_for(ncells, kHexThreads, sm_count, 8);
  if (mode >= 1 && grid > red.capacity) return cudaErrorInvalidConfiguration;
#define HEX_LAUNCH(K, M, G) hex_apply_kernel<K, M, G><<<grid, kHexThreads, 0, s>>>(cells, xyz, lm, x, y, E, ncells, bc, sc, red)
#define HEX_LAUNCH2(K, M) { if (quad == 1) HEX_LAUNCH(K, M, true); else HEX_LAUNCH(K, M, false); }
  if (kind == 0) { if (mode) HEX_LAUNCH2(0, 1) else HEX_LAUNCH2(0, 0) }
  else if (kind == 1) { if (mode) HEX_LAUNCH2(1, 1) else HEX_LAUNCH2(1, 0) }
  else { if (mode) HEX_LAUNCH2(2, 1) else HEX_LAUNCH2(2, 0) }
#undef HEX_LAUNCH2
#undef HEX_LAUNCH
  add_launches(1);
  return cudaGetLastError();
}

int64_t hex_pa_doubles(int kind, int64_t ncells) { return (int64_t)8 * ((kind == 2) ? 9 : 6) * ncells; }

cudaError_t launch_hex_pa_setup(int kind, int quad, const int4* cells, const double4* xyz, double* pa,
                                int64_t ncells, cudaStream_t s, int sm_count) {
  const int grid = grid_for(ncells, 256, sm_count, 8);
  if (kind == 2) {
    if (quad == 1) hex_pa_setup_kernel<2, true><<<grid, 256, 0, s>>>(cells, xyz, pa, ncells);
    else hex_pa_setup_kernel<2, false><<<grid, 256, 0, s>>>(cells, xyz, pa, ncells);
  } else {
    if (quad == 1) hex_pa_setup_kernel<0, true><<<grid, 256, 0, s>>>(cells, xyz, pa, ncells);
    else hex_pa_setup_kernel<0, false><<<grid, 256, 0, s>>>(cells, xyz, pa, ncells);
  }
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hex_pa_apply(int kind, int bc, int quad, const int4* cells, const double* pa, const double2* lm,
                                const double* x, double* y, double* E, int64_t ncells, int mode, CgScalars* sc,
                                Reduce red, cudaStream_t s, int sm_count) {
  if (ncells <= 0) return cudaSuccess;
  const int grid = grid_for(ncells, 128, sm_count, 8);
  if (mode >= 1 && grid > red.capacity) return cudaErrorInvalidConfiguration;
#define PA_LAUNCH(K, M, G) hex_pa_apply_kernel<K, M, G><<<grid, 128, 0, s>>>(cells, pa, lm, x, y, E, ncells, bc, sc, red)
#define PA_LAUNCH2(K, M) { if (quad == 1) PA_LAUNCH(K, M, true); else PA_LAUNCH(K, M, false); }
  if (kind == 0) { if (mode) PA_LAUNCH2(0, 1) else PA_LAUNCH2(0, 0) }
  else if (kind == 1) { if (mode) PA_LAUNCH2(1, 1) else PA_LAUNCH2(1, 0) }
  else { if (mode) PA_LAUNCH2(2, 1) else PA_LAUNCH2(2, 0) }
#undef PA_LAUNCH2
#undef PA_LAUNCH
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hex_dirichlet(const int32_t* nodes, int64_t nb, int comps, const double* x, double* y,
                                 int mode, CgScalars* sc, Reduce red, cudaStream_t s, int sm_count) {
  if (nb <= 0) return cudaSuccess;
  const int grid = grid_for(nb * comps, 256, sm_count, 4);
  if (mode) hex_dirichlet_kernel<1><<<grid, 256, 0, s>>>(nodes, nb, comps, x, y, sc, red);
  else hex_dirichlet_kernel<0><<<grid, 256, 0, s>>>(nodes, nb, comps, x, y, sc, red);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hex_check(const int4* cells, const double4* xyz, int64_t ncells, int64_t nnodes, int rule,
                             unsigned long long* bad, cudaStream_t s, int sm_count) {
  hex_check_kernel<<<grid_for(ncells, 256, sm_count, 8), 256, 0, s>>>(cells, xyz, ncells, nnodes, rule, bad);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_hex_pack_cells(const int32_t* vtk, const uint8_t* dir, int64_t ncells, int64_t nnodes,
                                  int* out, unsigned long long* bad, cudaStream_t s, int sm_count) {
  hex_pack_cells_kernel<<<grid_for(ncells * 8, 256, sm_count, 8), 256, 0, s>>>(vtk, dir, ncells, nnodes, out, bad);
  add_launches(1);
  return cudaGetLastError();
}

// ---- deterministic scatter (option "deterministic") ---------------------------
// The apply kernels write every cell's 8 x C element outputs to E[cell][corner][comp]; one thread
// per node then sums the entries of its incident (cell, corner) pairs in ascending entry order
// (node -> entry CSR built once per mesh by a stable radix sort), so the result is independent of
// the launch configuration and of the run: no floating-point atomics.
template <int C>
__global__ void __launch_bounds__(256) hex_gather_kernel(const int32_t* __restrict__ off,
                                                         const int32_t* __restrict__ list,
                                                         const double* __restrict__ E, double* __restrict__ y,
                                                         int64_t nnodes) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nnodes; n += stride) {
    double acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    const int32_t b = off[n], e = off[n + 1];
    for (int32_t k = b; k < e; ++k) {
      const double* src = E + (int64_t)list[k] * C;
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] += src[c];
    }
#pragma unroll
    for (int c = 0; c < C; ++c) y[n * C + c] = acc[c];
  }
}

__global__ void hex_entry_keys_kernel(const int4* __restrict__ cells, int64_t ncells, int32_t* __restrict__ key,
                                      int32_t* __restrict__ val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncells * 8; i += stride) {
    const int* c = reinterpret_cast<const int*>(cells);
    key[i] = c[i] & 0x7fffffff;  // node of (cell i / 8, corner i % 8)
    val[i] = (int32_t)i;
  }
}

// off[n] = first sorted entry of node n (keys sorted ascending), off[nnodes] = n_entries; nodes
// without entries get an empty range
__global__ void hex_entry_offsets_kernel(const int32_t* __restrict__ key, int64_t n_entries, int64_t nnodes,
                                         int32_t* __restrict__ off) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n_entries; i += stride) {
    const int64_t prev = (i == 0) ? -1 : key[i - 1];
    const int64_t cur = (i == n_entries) ? nnodes : key[i];
    for (int64_t n = prev + 1; n <= cur; ++n) off[n] = (int32_t)i;
  }
}

cudaError_t launch_hex_node_csr(const int4* cells, int64_t ncells, int64_t nnodes, int32_t* off, int32_t* list,
                                int sm_count) {
  const int64_t n = ncells * 8;
  if (n > 0x7fffffffLL) return cudaErrorInvalidValue;
  int32_t *k0 = nullptr, *k1 = nullptr, *v0 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e = cudaMalloc(&k0, n * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&k1, n * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&v0, n * sizeof(int32_t));
  if (e == cudaSuccess) {
    hex_entry_keys_kernel<<<grid_for(n, 256, sm_count, 8), 256>>>(cells, ncells, k0, v0);
    add_launches(1);
    e = cudaGetLastError();
  }
  int end_bit = 1;
  while (end_bit < 31 && (int64_t(1) << end_bit) < nnodes) ++end_bit;
  if (e == cudaSuccess)  // stable LSD radix sort: equal nodes keep ascending entry order
    e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, k1, v0, list, (int)n, 0, end_bit);
  if (e == cudaSuccess) e = cudaMalloc(&tmp, tmp_bytes);
  if (e == cudaSuccess) e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, k1, v0, list, (int)n, 0, end_bit);
  if (e == cudaSuccess) {
    hex_entry_offsets_kernel<<<grid_for(n + 1, 256, sm_count, 8), 256>>>(k1, n, nnodes, off);
    add_launches(1);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaFree(k0); cudaFree(k1); cudaFree(v0); cudaFree(tmp);
  return e;
}

cudaError_t launch_hex_gather(int comps, const int32_t* off, const int32_t* list, const double* E, double* y,
                              int64_t nnodes, cudaStream_t s, int sm_count) {
  if (nnodes <= 0) return cudaSuccess;
  const int grid = grid_for(nnodes, 256, sm_count, 8);
  if (comps == 1) hex_gather_kernel<1><<<grid, 256, 0, s>>>(off, list, E, y, nnodes);
  else hex_gather_kernel<3><<<grid, 256, 0, s>>>(off, list, E, y, nnodes);
  add_launches(1);
  return cudaGetLastError();
}

}  // namespace fem
