// kernels_csr.cu -- assembled-CSR baseline (Table 1; "performing a sparse matrix
// vector multiplication") built on the device from the same element matrices.
//
// Assembly: the paper adds element matrices into the sparse matrix by search +
// atomic add.  On the structured box the sparsity is the 27-point node stencil, so each row is
// produced by one thread that sums, for every neighbour column, the contributions of the cells
// shared by the two nodes (no search, no atomics, deterministic).  Dirichlet rows/columns are
// eliminated with a unit diagonal (A_c = P A P + (I - P)) and structurally dropped.
// Storage: int64 row offsets, int32 column indices, FP64 values (12 B / non-zero).
#include <cub/cub.cuh>

#include "fem_internal.cuh"

namespace fem {

// unit-cube element matrices (h = 1), corner index a = dx + 2 dy + 4 dz; set by fem_api.cu
__constant__ double c_K[64];
__constant__ double c_Kl[576];
__constant__ double c_Km[576];

cudaError_t upload_unit_matrices(const double* K, const double* Kl, const double* Km) {
  cudaError_t e = cudaMemcpyToSymbol(c_K, K, sizeof(double) * 64);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_Kl, Kl, sizeof(double) * 576);
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_Km, Km, sizeof(double) * 576);
  return e;
}

__device__ __forceinline__ bool on_face(const Grid& g, int64_t i, int64_t j, int64_t k) {
  return i == 0 || j == 0 || k == 0 || i == g.nx || j == g.ny || k == g.nz;
}

__global__ void csr_rowcount_kernel(int comps, int bc, Grid g, int64_t* __restrict__ cnt) {
  const int64_t nn = g.plane * (g.nz + 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nn; n += stride) {
    const int64_t i = n % (g.nx + 1), j = (n / (g.nx + 1)) % (g.ny + 1), k = n / g.plane;
    int64_t c = 0;
    if (bc && on_face(g, i, j, k)) {
      c = 1;
    } else {
      for (int dk = -1; dk <= 1; ++dk)
        for (int dj = -1; dj <= 1; ++dj)
          for (int di = -1; di <= 1; ++di) {
            const int64_t a = i + di, b = j + dj, d = k + dk;
            if (a < 0 || b < 0 || d < 0 || a > g.nx || b > g.ny || d > g.nz) continue;
            if (bc && on_face(g, a, b, d)) continue;
            c += comps;
          }
    }
    for (int q = 0; q < comps; ++q) cnt[n * comps + q + 1] = c;
  }
}

__global__ void csr_fill_kernel(int kind, int bc, Grid g, const double2* __restrict__ lm,
                                const int64_t* __restrict__ rowptr,
                                int32_t* __restrict__ col, double* __restrict__ val) {
  const int comps = kind == 0 ? 1 : 3;
  const int64_t nrows = g.plane * (g.nz + 1) * comps;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < nrows; row += stride) {
    const int64_t n = row / comps;
    const int kk = (int)(row - n * comps);
    const int64_t i = n % (g.nx + 1), j = (n / (g.nx + 1)) % (g.ny + 1), k = n / g.plane;
    int64_t w = rowptr[row];
    if (bc && on_face(g, i, j, k)) {
      col[w] = (int32_t)row;
      val[w] = 1.0;
      continue;
    }
    for (int dk = -1; dk <= 1; ++dk)
      for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di) {
          const int64_t a = i + di, b = j + dj, d = k + dk;
          if (a < 0 || b < 0 || d < 0 || a > g.nx || b > g.ny || d > g.nz) continue;
          if (bc && on_face(g, a, b, d)) continue;
          const int64_t m = a + (g.nx + 1) * (b + (g.ny + 1) * d);
          double v[3] = {0.0, 0.0, 0.0};
          // cells containing both nodes: ci in {i-1, i} and {a-1, a}, inside the box
          for (int64_t ck = max(k, d) - 1; ck <= min(k, d); ++ck) {
            if (ck < 0 || ck >= g.nz) continue;
            for (int64_t cj = max(j, b) - 1; cj <= min(j, b); ++cj) {
              if (cj < 0 || cj >= g.ny) continue;
              for (int64_t ci = max(i, a) - 1; ci <= min(i, a); ++ci) {
                if (ci < 0 || ci >= g.nx) continue;
                const int ra = (int)((i - ci) + 2 * (j - cj) + 4 * (k - ck));
                const int rb = (int)((a - ci) + 2 * (b - cj) + 4 * (d - ck));
                if (kind == 2) {
                  const int64_t e = ci + g.nx * (cj + g.ny * ck);
                  const double le = lm[e].x * g.h, me = lm[e].y * g.h;
                  for (int l = 0; l < 3; ++l) {
                    const int ix = (3 * ra + kk) * 24 + 3 * rb + l;
                    v[l] += le * c_Kl[ix] + me * c_Km[ix];
                  }
                } else {
                  v[0] += g.h * c_K[ra * 8 + rb];
                }
              }
            }
          }
          if (kind == 0) {
            col[w] = (int32_t)m;
            val[w] = v[0];
            ++w;
          } else {
            for (int l = 0; l < 3; ++l) {
              col[w] = (int32_t)(3 * m + l);
              val[w] = (kind == 1) ? (l == kk ? v[0] : 0.0) : v[l];
              ++w;
            }
          }
        }
  }
}

// y = A x; LPR lanes per row, shuffle reduction within the lane group.
template <int LPR>
__global__ void __launch_bounds__(256) csr_spmv_kernel(int64_t nrows, const int64_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ col,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y) {
  const int lane = threadIdx.x % LPR;
  const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / LPR; row < nrows;
       row += groups) {
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    double s = 0.0;
    for (int64_t t = b + lane; t < e; t += LPR) s = fma(__ldg(val + t), __ldg(x + __ldg(col + t)), s);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LPR);
    if (lane == 0) y[row] = s;
  }
}

cudaError_t launch_csr_rowcount(int comps, int bc, const Grid& g, int64_t* rowptr, cudaStream_t s) {
  const int64_t nn = g.plane * (g.nz + 1);
  cudaError_t e = cudaMemsetAsync(rowptr, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  csr_rowcount_kernel<<<(unsigned)std::min<int64_t>((nn + 255) / 256, 65535 * 8), 256, 0, s>>>(comps, bc, g, rowptr);
  add_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // inclusive scan of counts (rowptr[1..n]) -> offsets
  const int64_t nrows = nn * comps;
  size_t tmp = 0;
  e = cub::DeviceScan::InclusiveSum(nullptr, tmp, rowptr + 1, rowptr + 1, nrows, s);
  if (e != cudaSuccess) return e;
  void* buf = nullptr;
  e = cudaMallocAsync(&buf, tmp, s);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::InclusiveSum(buf, tmp, rowptr + 1, rowptr + 1, nrows, s);
  add_launches(1);
  cudaFreeAsync(buf, s);
  return e;
}

cudaError_t launch_csr_fill(int kind, int bc, const Grid& g, const double2* lm,
                            const int64_t* rowptr, int32_t* col, double* val, cudaStream_t s) {
  const int comps = kind == 0 ? 1 : 3;
  const int64_t nrows = g.plane * (g.nz + 1) * comps;
  csr_fill_kernel<<<(unsigned)std::min<int64_t>((nrows + 255) / 256, 65535 * 8), 256, 0, s>>>(
      kind, bc, g, lm, rowptr, col, val);
  add_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_csr_spmv(int comps, int64_t nrows, const int64_t* rowptr, const int32_t* col,
                            const double* val, const double* x, double* y, cudaStream_t s,
                            int sm_count) {
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nrows * (comps == 1 ? 8 : 16) + 255) / 256,
                                                                           (int64_t)sm_count * 32));
  if (comps == 1)
    csr_spmv_kernel<8><<<blocks, 256, 0, s>>>(nrows, rowptr, col, val, x, y);
  else
    csr_spmv_kernel<16><<<blocks, 256, 0, s>>>(nrows, rowptr, col, val, x, y);
  add_launches(1);
  return cudaGetLastError();
}

}  // namespace fem
