// Achievable DRAM rate of K4-T's access pattern without any conversion work: every CTA (one per
// SM) has W warps; each warp stages "units" of 16 row segments (random frame rows of a 2.83 GB
// pool, segment = 16-byte aligned span of 3w bytes, w log-uniform by octave in [32, 256) as in
// cfg2) with one 1-D bulk copy per segment into a ring of S slots (mbarrier per slot), waits for
// a unit, then recycles its slot.  Prints GB/s of segment bytes for several W / S.
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
extern __shared__ __align__(128) uint8_t smem[];
__global__ void gather(const uint8_t* pool, uint64_t pool_rows, uint32_t pitch, int units_per_warp, int slots,
                       int slot_bytes, unsigned long long* bytes_out, uint32_t wmin, const uint8_t* weights, int wchunks) {
  // optional weight stream (K4-T's B operand): the last warp bulk-copies wchunks 18 KB K-blocks of a
  // 3.5 MB L2-resident matrix through a 3-stage ring while the other warps gather
  const int nw_all = blockDim.x >> 5;
  if (wchunks > 0 && (threadIdx.x >> 5) == nw_all - 1) {
    uint64_t* wb = reinterpret_cast<uint64_t*>(smem) + 31 * 16;  // 3 barriers in warp 31's (unused) block
    uint8_t* wring = smem + 4096 + (nw_all - 1) * slots * slot_bytes;
    if ((threadIdx.x & 31) == 0) {
      for (int st = 0; st < 3; ++st) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&wb[st])));
      uint32_t wpar = 0;
      for (int k = 0; k < wchunks; ++k) {
        const int st = k % 3;
        if (k >= 3) {
          asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(smem_u32(&wb[st])), "r"((wpar >> st) & 1u) : "memory");
          wpar ^= 1u << st;
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&wb[st])), "r"(18432u) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(wring + st * 18432)),
                     "l"(weights + (k % 192) * 18432ull), "r"(18432u), "r"(smem_u32(&wb[st])) : "memory");
      }
      for (int st = 0; st < 3; ++st)
        asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(smem_u32(&wb[(wchunks + st) % 3])), "r"(((wpar >> ((wchunks + st) % 3)) & 1u)) : "memory");
    }
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = wchunks > 0 ? nw_all - 1 : nw_all;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* ring = smem + 4096 + warp * slots * slot_bytes;  // [32 warps x 16 mbarriers][rings]
  if (lane == 0)
    for (int s = 0; s < slots; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp * 16 + s])));
  __syncwarp();
  unsigned long long tot = 0;
  uint32_t par = 0;
  auto seg = [&](int u, uint32_t& off, uint32_t& len, uint64_t& row) {
    const uint32_t h = hash32((blockIdx.x * nw + warp) * 1000003u + u * 131u + lane);
    const uint32_t oct = h % 3, w = (wmin << oct) + ((h >> 8) % (wmin << oct));
    const uint32_t x0 = (h >> 16) % (1280u - w);
    off = (3u * x0) & ~15u;
    len = ((3u * (x0 + w) + 15u) & ~15u) - off;
    row = (static_cast<uint64_t>(hash32(h ^ 0x9e3779b9u)) * 7919u) % pool_rows;
  };
  auto stage = [&](int u, int s) {
    uint32_t off, len; uint64_t row;
    seg(u, off, len, row);
    if (lane >= 16) len = 0;
    uint32_t incl = len;
    for (int d = 1; d < 32; d <<= 1) { uint32_t v = __shfl_up_sync(0xffffffffu, incl, d); if (lane >= d) incl += v; }
    if (incl > static_cast<uint32_t>(slot_bytes)) {  // keep the unit inside its slot (rare large units)
      const uint32_t start = incl - len;
      len = start >= static_cast<uint32_t>(slot_bytes) ? 0u : ((static_cast<uint32_t>(slot_bytes) - start) & ~15u);
      incl = start + len;
    }
    const uint32_t total = __reduce_add_sync(0xffffffffu, len);  // bytes actually copied
    const uint32_t bar = smem_u32(&bars[warp * 16 + s]);
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(total) : "memory");
    __syncwarp();
    if (len) {
      const uint32_t dst = smem_u32(ring + s * slot_bytes + (incl - len));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(pool + row * pitch + off), "r"(len), "r"(bar) : "memory");
    }
    return total;
  };
  // all S slots in flight: stage unit u + S after unit u has landed (its slot is then free)
  for (int u = 0; u < slots && u < units_per_warp; ++u) tot += stage(u, u);
  for (int u = 0; u < units_per_warp; ++u) {
    const int s = u % slots;
    const uint32_t bar = smem_u32(&bars[warp * 16 + s]);
    asm volatile("{\n.reg .pred P;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W%=;\n}" ::"r"(bar), "r"((par >> s) & 1u) : "memory");
    par ^= 1u << s;
    __syncwarp();
    if (u + slots < units_per_warp) tot += stage(u + slots, s);
  }
  if (lane == 0) atomicAdd(bytes_out, tot);
}
int main() {
  const uint32_t H = 720, W = 1280, pitch = 3 * W;
  const uint64_t frames = 1024, rows = frames * H;
  uint8_t* pool; cudaMalloc(&pool, rows * pitch);
  cudaMemset(pool, 1, rows * pitch);
  unsigned long long* b; cudaMalloc(&b, 8);
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  const int slot_bytes = 6144;  // cfg2's units average ~5.6 KB (K4-T packs them into 22 KB rings)
  uint8_t* wts; cudaMalloc(&wts, 192 * 18432);
  cudaMemset(wts, 2, 192 * 18432);
  // {gather warps, slots, w_min, weight stream}: the weight warp streams 3.5 MB per 128 x 64 crop rows
  // of gathered tuples, as K4-T does for the fused pair (192 K-blocks of 18 KB per 128-tuple tile)
  int cfgs[][4] = {{8, 3, 32, 0}, {8, 3, 32, 1}, {8, 2, 32, 1}, {16, 2, 32, 0}, {16, 2, 32, 1}};
  for (auto& c : cfgs) {
    const int wpc = c[0], slots = c[1];
    const uint32_t wmin = c[2];
    const bool wstream = c[3] != 0;
    const size_t sm = 4096 + (size_t)(wpc + (wstream ? 1 : 0)) * slots * slot_bytes + (wstream ? 3 * 18432 : 0);
    if (sm > 232448) { printf("W %d S %d: smem %zu too big\n", wpc, slots, sm); continue; }
    const int units = 4000;
    cudaMemset(b, 0, 8);
    // units are crop rows of 16 tuples; per 128 tuples x 64 rows (= 512 units) the tile streams 192 K-blocks
    const int threads = (wpc + (wstream ? 1 : 0)) * 32;
    gather<<<148, threads, sm>>>(pool, rows, pitch, 200, slots, slot_bytes, b, wmin, wts, wstream ? 200 * wpc * 192 / 512 : 0);  // warm
    cudaMemset(b, 0, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    gather<<<148, threads, sm>>>(pool, rows, pitch, units, slots, slot_bytes, b, wmin, wts, wstream ? units * wpc * 192 / 512 : 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hb; cudaMemcpy(&hb, b, 8, cudaMemcpyDeviceToHost);
    const double copies = 148.0 * wpc * units * 16;
    printf("%s w >= %2u W %2d S %d: %.1f GB/s of segment bytes (%.2f GB in %.2f ms), %.1f M copies/ms/SM %s\n", wstream ? "+weights" : "        ", wmin, wpc, slots,
           hb / (ms * 1e6), hb / 1e9, ms, copies / ms / 148 / 1e6,
           err ? cudaGetErrorString(err) : "");
    fflush(stdout);
  }
  return 0;
}
