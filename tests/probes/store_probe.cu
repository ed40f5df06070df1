// Store-bandwidth probe: what write rate do different store shapes reach on this GPU?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o store_probe store_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef long long i64;

// (1) grid-stride, 8 B per lane, fully contiguous
__global__ void k_stride8(double* out, i64 n) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) out[i] = 1.5;
}
// (2) grid-stride, 16 B per lane
__global__ void k_stride16(double2* out, i64 n2) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n2; i += (i64)gridDim.x * blockDim.x)
    out[i] = make_double2(1.5, 2.5);
}
// (3) tile per CTA (contiguous 128 KB), warp w writes rows of `run` doubles starting at odd offsets
__global__ void k_tile_runs(double* out, i64 n, int tile, int run, int lanes) {
  const i64 t0 = (i64)blockIdx.x * tile;
  if (t0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups_per_warp = 32 / lanes;
  const int g = lane / lanes, sl = lane % lanes;
  const int nruns = tile / (run + 1);
  for (int r = warp * groups_per_warp + g; r < nruns; r += 8 * groups_per_warp) {
    double* dst = out + t0 + (i64)r * (run + 1) + 1;  // +1: misaligned start, one-double gap between runs
    for (int i = sl; i < run; i += lanes) dst[i] = 1.5 * i;
  }
}
// (4) like (3) but every value needs one shared-memory load and a multiply
__global__ void k_tile_runs_lds(double* out, i64 n, int tile, int run, int lanes) {
  __shared__ double w[1024];
  for (int t = threadIdx.x; t < 1024; t += blockDim.x) w[t] = 1.0 + t;
  __syncthreads();
  const i64 t0 = (i64)blockIdx.x * tile;
  if (t0 >= n) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int groups_per_warp = 32 / lanes;
  const int g = lane / lanes, sl = lane % lanes;
  const int nruns = tile / (run + 1);
  for (int r = warp * groups_per_warp + g; r < nruns; r += 8 * groups_per_warp) {
    double* dst = out + t0 + (i64)r * (run + 1) + 1;
    const double A = w[r & 1023];
    for (int i = sl; i < run; i += lanes) dst[i] = A * w[i & 1023];
  }
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const i64 n = (i64)1 << 27;  // 1 GiB of doubles
  double* out;
  cudaMalloc(&out, n * 8);
  auto rep = [&](const char* name, float ms) { printf("%-44s %8.3f ms  %8.1f GB/s\n", name, ms, n * 8 / ms / 1e6); };
  rep("memset", timeit([&] { cudaMemsetAsync(out, 0, n * 8); }));
  for (int grid : {148 * 8, 148 * 32}) {
    char nm[64];
    snprintf(nm, 64, "stride 8B/lane grid=%d", grid);
    rep(nm, timeit([&] { k_stride8<<<grid, 256>>>(out, n); }));
    snprintf(nm, 64, "stride 16B/lane grid=%d", grid);
    rep(nm, timeit([&] { k_stride16<<<grid, 256>>>((double2*)out, n / 2); }));
  }
  const int tile = 16384;
  for (int run : {15, 31, 67, 135, 250}) {
    for (int lanes : {32, 16, 8}) {
      char nm[64];
      snprintf(nm, 64, "tile runs=%d lanes=%d", run, lanes);
      rep(nm, timeit([&] { k_tile_runs<<<(unsigned)(n / tile), 256>>>(out, n, tile, run, lanes); }));
    }
  }
  for (int run : {67, 135}) {
    for (int lanes : {32, 16}) {
      char nm[64];
      snprintf(nm, 64, "tile runs+LDS+mul=%d lanes=%d", run, lanes);
      rep(nm, timeit([&] { k_tile_runs_lds<<<(unsigned)(n / tile), 256>>>(out, n, tile, run, lanes); }));
    }
  }
  return 0;
}
