// Idle-warp wait cost probe: warp 0 spins on clock64 for T cycles then arrives on an mbarrier;
// warps 1..7 wait for the phase with (mode 0) try_wait loop, (1) test_wait + nanosleep(1024),
// (2) try_wait with a 1 ms suspend hint, (3) test_wait + nanosleep(64); each counts its poll
// iterations.  Prints iterations per waiting warp per microsecond.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void probe(int mode, long long T, unsigned long long* iters, long long* dt) {
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  __syncthreads();
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    long long t0 = clock64();
    while (clock64() - t0 < T) {}
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
    if (threadIdx.x == 0) dt[blockIdx.x] = clock64() - t0;
  } else {
    unsigned long long n = 0;
    uint32_t ok = 0;
    while (!ok) {
      ++n;
      if (mode == 0) {
        asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
      } else if (mode == 2) {
        asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0, %2;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"(1000000u) : "memory");
      } else {
        asm volatile("{\n.reg .pred P;\nmbarrier.test_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.u32 %0,1,0,P;\n}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        if (!ok) { if (mode == 1) __nanosleep(1024); else if (mode == 3) __nanosleep(64); else if (mode == 4) __nanosleep(8192); }
      }
    }
    if ((threadIdx.x & 31) == 0) atomicAdd(iters, n);
  }
}
int main() {
  unsigned long long* it; long long* dt;
  cudaMalloc(&it, 8); cudaMalloc(&dt, 8 * 148);
  const long long T = 2000000;  // ~1 ms at 1.9 GHz
  const char* names[] = {"try_wait", "test+nanosleep(1024)", "try_wait(hint 1ms)", "test+nanosleep(64)", "test+nanosleep(8192)"};
  for (int mode = 0; mode < 5; ++mode) {
    cudaMemset(it, 0, 8);
    probe<<<148, 256>>>(mode, T, it, dt);
    cudaDeviceSynchronize();
    unsigned long long h; long long d;
    cudaMemcpy(&h, it, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&d, dt, 8, cudaMemcpyDeviceToHost);
    const double us = d / 1900.0;
    printf("%-24s polls per waiting warp per us: %8.2f  (worker %.0f us)\n", names[mode], h / (148.0 * 7) / us, us);
  }
  return 0;
}
