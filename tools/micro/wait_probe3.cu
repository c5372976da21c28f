// Do waiting warps steal issue slots?  Warps 0..7 run a fixed ALU workload (8 independent FMA
// chains, issue-bound) and then arrive on mbarrier A; warps 8..15 wait for A with (0) nothing (they
// exit at once), (1) try_wait loop, (2) test_wait + nanosleep(1024), (3) test_wait + nanosleep(64),
// (4) bar.sync behind one try_wait poller.  Prints the workers' time.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool test_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P;\nmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  return ok;
}
__global__ void probe(int wmode, int iters, float* out, long long* dt) {
  __shared__ uint64_t barA;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(smem_u32(&barA)));
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp < 8) {
    long long t0 = clock64();
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 0.001f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], 0.9999f, 0.0001f);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&barA)) : "memory");
    if (threadIdx.x == 0) dt[blockIdx.x] = clock64() - t0;
  } else if (wmode == 1) {
    while (!try_wait(&barA, 0)) {}
  } else if (wmode == 2) {
    while (!test_wait(&barA, 0)) __nanosleep(1024);
  } else if (wmode == 3) {
    while (!test_wait(&barA, 0)) __nanosleep(64);
  } else if (wmode == 4) {
    if (warp == 8) while (!try_wait(&barA, 0)) {}
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
}
int main() {
  float* o; long long* dt;
  cudaMalloc(&o, 4 * 512); cudaMalloc(&dt, 8 * 148);
  const char* wn[] = {"no waiters", "try_wait", "test+nanosleep(1024)", "test+nanosleep(64)", "bar.sync behind 1 poller"};
  for (int w = 0; w < 5; ++w) {
    probe<<<148, 512>>>(w, 200000, o, dt);
    cudaError_t e = cudaDeviceSynchronize();
    long long d;
    cudaMemcpy(&d, dt, 8, cudaMemcpyDeviceToHost);
    printf("%-26s worker %8.1f us %s\n", wn[w], d / 1900.0, e ? cudaGetErrorString(e) : "");
    fflush(stdout);
  }
  return 0;
}
