// Calibration microbenchmark: the apply kernels' plane pipeline (PlaneRing, TMA path) with the
// consumer arithmetic removed, on the C2 scalar (257^3 nodes) padded layout.  Separates the
// pipeline/memory ceiling from the consumer-compute ceiling.
//   mode 0: consumers wait/release only;  1: + one 8-B store per node;  2: + read 3 rows x 3 LDS
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2308_09839_b200/csrc -o ring_probe ring_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>

#include "kernels_common.cuh"

using namespace fem;
namespace fem {
void add_launches(int64_t) {}
}

template <int TY, int R, int S, int MODE>
__global__ void __launch_bounds__(32 * (TY + 1), 2)
    probe(Grid g, PlaneSrc x, double* y, int64_t ypitch, const __grid_constant__ CUtensorMap umap, TmaOrigin uorg,
          int64_t kchunk) {
  constexpr int TX = 32, ROWS = TY * R + 2, COLS = TX + 2;
  using Ring = PlaneRing<true, ROWS, COLS, 1, S>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Ring ring;
  ring.carve(smem_raw, smem_raw + Ring::BYTES);
  const int tx = threadIdx.x, ty = threadIdx.y, tid = tx + TX * ty;
  const int64_t i0 = (int64_t)blockIdx.x * TX, j0 = (int64_t)blockIdx.y * (TY * R);
  const int64_t kb = g.k0 + (int64_t)blockIdx.z * kchunk, ke = min(g.k1, kb + kchunk);
  ring.init(tid, 32 * (TY + 1), TY);
  ring.set_tshift(i0 - 1, uorg);
  if (ty == TY) {
    ring.produce(x, g, kb - 1, ke, i0 - 1, j0 - 1, 1, tx, &umap, uorg, nullptr, 0);
    return;
  }
  double acc = 0.0;
  double* yr = y + (j0 + ty * R) * (g.nx + 1) + i0 + tx;
  for (int64_t p = kb - 1; p <= ke; ++p) {
    const int t = (int)(p - (kb - 1)), slot = t & (S - 1);
    ring.wait(slot, (uint32_t)((t / S) & 1));
    if (MODE >= 2) {
#pragma unroll
      for (int rr = 0; rr < R + 2; ++rr) {
        const double* row = ring.row_ptr(slot, ty * R + rr) + tx;
        acc += row[0] + row[1] + row[2];
      }
    }
    ring.release(slot, tx);
    if (MODE >= 1 && p >= kb && p < ke && i0 + tx <= g.nx)
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (j0 + ty * R + r <= g.ny) yr[(p - g.k0) * ypitch + r * (g.nx + 1)] = acc;
  }
}

int main() {
  const int64_t n = 256, nn = n + 1;
  const int64_t rp = nn + 1, pp = rp * nn, lead = 1;  // padded layout (Dirichlet lead 1)
  double *xpl, *y;
  cudaMalloc(&xpl, (lead + (nn + 2) * pp + 1) * 8);
  cudaMalloc(&y, nn * nn * nn * 8);
  cudaMemset(xpl, 0, (lead + (nn + 2) * pp + 1) * 8);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap m;
  const double* base = xpl + lead + (1 - (-1)) * pp + 1 * rp + 1;
  cuuint64_t dims[3] = {(cuuint64_t)(n - 1), (cuuint64_t)(n - 1), (cuuint64_t)(n - 1)};
  cuuint64_t str[2] = {(cuuint64_t)rp * 8, (cuuint64_t)pp * 8};
  cuuint32_t box[3] = {36, 18, 1}, es[3] = {1, 1, 1};
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  Grid g{n, n, n, 1.0 / n, 0, nn, nn * nn};
  PlaneSrc xs{xpl + lead + pp, xpl + lead, nullptr, rp, pp};
  TmaOrigin org{1, 1, 1};
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, const char* name, size_t smem, int zc) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t kchunk = (nn + zc - 1) / zc;
    dim3 grid(9, 17, (unsigned)((nn + kchunk - 1) / kchunk)), block(32, 9);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      kern<<<grid, block, smem>>>(g, xs, y, nn * nn, m, org, kchunk);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"probe\": \"%s\", \"zc\": %d, \"us\": %.1f, \"eq_GBps_16B_per_node\": %.1f, \"err\": \"%s\"}\n", name, zc,
           best * 1e3, 16.0 * nn * nn * nn / (best * 1e6), cudaGetErrorString(cudaGetLastError()));
  };
  using R8 = PlaneRing<true, 18, 34, 1, 8>;
  const size_t smem8 = R8::BYTES + R8::META;
  for (int zc : {4, 8, 16}) {
    run(probe<8, 2, 8, 0>, "wait_release_only", smem8, zc);
    run(probe<8, 2, 8, 1>, "plus_store", smem8, zc);
    run(probe<8, 2, 8, 2>, "plus_lds_and_store", smem8, zc);
  }
  return 0;
}
