// grid_barrier_probe.cu -- cost of one grid-wide barrier on sm_100a for the
// persistent small-grid integration (hj_stage_generic.cuh k_stage_persist):
// the counter + generation barrier used there, per barrier, for several grid
// sizes, plus an L2 round trip (ld.global.cg of data another CTA just stored).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gbar scripts/grid_barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      atomicExch(&bar[0], 0u);
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (*(volatile unsigned*)&bar[1] == gen) {
      }
    }
    __threadfence();
  }
  ++gen;
  __syncthreads();
}

// variant: every CTA's thread 0 spins with ld.acquire instead of volatile
__global__ void k_bar(unsigned* bar, int iters, double* sink) {
  unsigned gen = 0;
  double acc = 0.0;
  for (int i = 0; i < iters; ++i) {
    grid_barrier(bar, gen);
    acc += 1.0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = acc;
}

// barrier + a dependent exchange: each thread stores a value, after the
// barrier reads its neighbour CTA's value through L2
__global__ void k_bar_xchg(unsigned* bar, int iters, double* buf) {
  unsigned gen = 0;
  const long long n = (long long)gridDim.x * blockDim.x;
  const long long me = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double v = (double)me;
  for (int i = 0; i < iters; ++i) {
    double* w = buf + (i & 1) * n;
    double* r = buf + ((i + 1) & 1) * n;
    w[me] = v;
    grid_barrier(bar, gen);
    v = __ldcg(r + (me + blockDim.x) % n) * 0.5 + 1.0;
  }
  buf[2 * n + me] = v;
}

int main() {
  unsigned* bar;
  double* buf;
  cudaMalloc(&bar, 8);
  cudaMalloc(&buf, (size_t)3 * 148 * 2048 * 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  for (int threads : {128, 256}) {
    for (int per_sm : {1, 2, 4, 5}) {
      const int blocks = nsm * per_sm;
      for (int xchg = 0; xchg < 2; ++xchg) {
        void* args_b[] = {&bar, (void*)&iters, &buf};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(bar, 0, 8);
          cudaEventRecord(e0);
          cudaError_t e = cudaLaunchCooperativeKernel(xchg ? (const void*)k_bar_xchg : (const void*)k_bar,
                                                      dim3(blocks), dim3(threads), args_b, 0, 0);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          if (e != cudaSuccess) {
            printf("launch failed: %s\n", cudaGetErrorString(e));
            break;
          }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          best = ms < best ? ms : best;
        }
        printf("threads %3d blocks %4d (%d/SM) %-12s: %.3f us per barrier\n", threads, blocks, per_sm,
               xchg ? "store+barrier+ldcg" : "barrier", best * 1e3 / iters);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
