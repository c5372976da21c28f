// Idle-warp wait cost under background activity: warp 0 works for ~1 ms then arrives on mbarrier A;
// warps 1..3 generate "noise" (mode n: 0 none, 1 __syncwarp + ALU loop, 2 mbarrier arrive/wait on B,
// 3 1-D bulk copies global->shared completing on B, 4 bar.sync among the noise warps);
// warps 4..7 wait for A with (w: 0 try_wait, 1 test_wait + nanosleep(1024), 2 named-barrier block
// behind one try_wait poller).  Prints polls per waiting warp per microsecond.
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
__global__ void probe(int noise, int wmode, long long T, const uint8_t* src, unsigned long long* iters, long long* dt) {
  __shared__ uint64_t barA, barB;
  __shared__ volatile int stop;
  __shared__ __align__(128) uint8_t buf[3][4096];
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&barA)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&barB)));
    stop = 0;
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    long long t0 = clock64();
    while (clock64() - t0 < T) {}
    if (lane == 0) {
      stop = 1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&barA)) : "memory");
      dt[blockIdx.x] = clock64() - t0;
    }
  } else if (warp < 4) {
    uint32_t ph = 0, x = threadIdx.x;
    while (!stop) {
      if (noise == 1) {
        for (int i = 0; i < 64; ++i) { x = x * 1664525u + 1013904223u; __syncwarp(); }
      } else if (noise == 2 && warp == 1) {
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&barB)) : "memory");
        while (!try_wait(&barB, ph)) {}
        ph ^= 1;
      } else if (noise == 3 && warp == 1) {
        if (lane == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&barB)), "r"(4096u) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(buf[ph % 3])),
                       "l"(src + 4096 * (blockIdx.x % 64)), "r"(4096u), "r"(smem_u32(&barB)) : "memory");
        }
        while (!try_wait(&barB, ph)) {}
        ph ^= 1;
      } else if (noise == 4) {
        asm volatile("bar.sync 2, 96;" ::: "memory");
      }
    }
    if (threadIdx.x == 32) buf[0][0] = x;
  } else {
    unsigned long long n = 0;
    if (wmode == 0) {
      do { ++n; } while (!try_wait(&barA, 0));
    } else if (wmode == 1) {
      do { ++n; if (test_wait(&barA, 0)) break; __nanosleep(1024); } while (true);
    } else {
      if (warp == 4) { do { ++n; } while (!try_wait(&barA, 0)); }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (warp != 4) n = 1;
    }
    if (lane == 0) atomicAdd(iters, n);
  }
}
int main() {
  unsigned long long* it; long long* dt; uint8_t* src;
  cudaMalloc(&it, 8); cudaMalloc(&dt, 8 * 148); cudaMalloc(&src, 1 << 20);
  const long long T = 2000000;
  const char* nn[] = {"none", "syncwarp+alu", "mbar arrive/wait", "bulk copy + mbar", "bar.sync"};
  const char* wn[] = {"try_wait", "test+nanosleep(1024)", "bar.sync behind 1 poller"};
  for (int noise = 0; noise < 4; ++noise)
    for (int w = 0; w < 3; ++w) {
      cudaMemset(it, 0, 8);
      probe<<<148, 256>>>(noise, w, T, src, it, dt);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h; long long d;
      cudaMemcpy(&h, it, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&d, dt, 8, cudaMemcpyDeviceToHost);
      printf("noise %-18s wait %-26s polls/warp/us %9.3f %s\n", nn[noise], wn[w], h / (148.0 * 4) / (d / 1900.0),
             e ? cudaGetErrorString(e) : ""); fflush(stdout);
    }
  return 0;
}
