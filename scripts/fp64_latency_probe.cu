// fp64_latency_probe.cu -- microbenchmark of the FP64 pipe on sm_100a:
// dependent-chain latency of DFMA / DADD / DMUL / MUFU.RCP64H and DFMA
// throughput against the number of independent chains per warp and warps per
// SM (what the brick kernel's 'wait' stalls are made of).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64lat scripts/fp64_latency_probe.cu
//   /tmp/fp64lat
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void k_chain(double* out, double a, double b, long long* cyc) {
  double x = a + threadIdx.x * 1e-9;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    if (OP == 0) x = __fma_rn(x, a, b);
    if (OP == 1) x = __dadd_rn(x, b);
    if (OP == 2) x = __dmul_rn(x, a);
    if (OP == 3) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

// C independent DFMA chains per thread
template <int C>
__global__ void k_ilp(double* out, double a, double b, long long* cyc) {
  double x[C];
#pragma unroll
  for (int c = 0; c < C; ++c) x[c] = a + (threadIdx.x + c) * 1e-9;
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = __fma_rn(x[c], a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 1 << 16);
  long long h[1024];
  auto lat = [&](auto kern, const char* name) {
    kern<<<1, 32>>>(out, 0.999999, 1e-7, cyc);
    kern<<<1, 32>>>(out, 0.999999, 1e-7, cyc);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("latency %-10s %.2f cycles\n", name, (double)h[0] / ITERS);
  };
  lat(k_chain<0>, "DFMA");
  lat(k_chain<1>, "DADD");
  lat(k_chain<2>, "DMUL");
  lat(k_chain<3>, "RCP64H");
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  // throughput: DFMA lane-ops per cycle per SM for warps/SM x chains/warp
  auto thr = [&](auto kern, int C) {
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      kern<<<nsm, 32 * warps>>>(out, 0.999999, 1e-7, cyc);
      cudaEventRecord(e0);
      kern<<<nsm, 32 * warps>>>(out, 0.999999, 1e-7, cyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)ITERS * C * 32 * warps;   // per SM
      printf("chains/warp %d warps/SM %2d: %.1f DFMA lanes/clk/SM (clock64), %.2f TFMA/s device\n", C, warps,
             ops / (double)h[0], ops * nsm / (ms * 1e-3) / 1e12);
    }
  };
  thr(k_ilp<1>, 1);
  thr(k_ilp<2>, 2);
  thr(k_ilp<4>, 4);
  thr(k_ilp<8>, 8);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
