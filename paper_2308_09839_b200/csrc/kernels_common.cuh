// kernels_common.cuh -- plane staging (cp.async ring) shared by the apply kernels.
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

// cp.async with zero-fill: copies 8 bytes when valid, else writes 8 zero bytes.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc, bool valid) {
  unsigned int d = (unsigned int)__cvta_generic_to_shared(smem_dst);
  int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(src_size)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Stage the halo tile of node plane k into smem:
//   rows j = jlo .. jlo+ROWS-1, columns i = ilo .. ilo+COLS-1, COMPS components per node,
//   smem layout dst[row * PITCH + col * COMPS + comp].
// Values outside the domain, and (bc == Dirichlet) on the box faces, are zero-filled:
// that is the mask P of y = P A P x + (I-P) x.
template <int ROWS, int COLS, int COMPS, int PITCH, int NT>
__device__ __forceinline__ void stage_plane(double* dst, const PlaneSrc& x, const Grid& g, int64_t k,
                                            int64_t ilo, int64_t jlo, int bc, int tid) {
  const double* base = plane_ptr(x, g, k, COMPS);
  const bool kface = (k == 0 || k == g.nz);
  constexpr int PER_ROW = COLS * COMPS;
  constexpr int TOTAL = ROWS * PER_ROW;
  const int64_t rowlen = g.nx + 1;
#pragma unroll 4
  for (int e = tid; e < TOTAL; e += NT) {
    const int r = e / PER_ROW;
    const int m = e - r * PER_ROW;
    const int col = m / COMPS;
    const int comp = m - col * COMPS;
    const int64_t i = ilo + col, j = jlo + r;
    bool valid = base != nullptr && i >= 0 && i <= g.nx && j >= 0 && j <= g.ny;
    if (bc) valid = valid && !(kface || i == 0 || i == g.nx || j == 0 || j == g.ny);
    const double* src = valid ? base + (j * rowlen + i) * COMPS + comp : x.main;
    cp_async8(dst + r * PITCH + m, src, valid);
  }
}

}  // namespace fem
