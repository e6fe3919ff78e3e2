// Microbenchmark: mbarrier round trip "one thread signals -> a 256-thread group waits and
// answers -> the signalling warp waits for the answer", with the answer barrier counting
// all 256 threads (one arrive each) or 8 warps (__syncwarp, lane 0 arrives).  Cycles per
// round trip, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2505_16864_b200/csrc \
//        tests/native/bar_rt.cu -o tests/native/bar_rt && tests/native/bar_rt
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace tcb;

template <bool PER_WARP>
__global__ void __launch_bounds__(288) k_rt(int iters, unsigned long long* out) {
  __shared__ uint64_t sig, ans;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&sig, 1);
    ptx::mbar_init(&ans, PER_WARP ? 8 : 256);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (lane == 0) ptx::mbar_arrive(&sig);
      ptx::mbar_wait(&ans, i & 1);
    }
    if (lane == 0) out[blockIdx.x] = clock64() - t0;
  } else {
    for (int i = 0; i < iters; ++i) {
      ptx::mbar_wait(&sig, i & 1);
      if (PER_WARP) {
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ans);
      } else {
        ptx::mbar_arrive(&ans);
      }
    }
  }
}

template <bool PW>
void run(const char* name) {
  const int grid = 148, iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, grid * sizeof(unsigned long long));
  k_rt<PW><<<grid, 288>>>(iters, d);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid);
  cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  printf("%-34s %7.1f cycles per round trip\n", name, (double)mx / iters);
  cudaFree(d);
}

int main() {
  run<false>("256 per-thread arrivals");
  run<true>("8 per-warp arrivals (__syncwarp)");
  run<false>("256 per-thread arrivals");
  return 0;
}
