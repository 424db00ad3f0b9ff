// TMEM load latency / throughput microbenchmark (debug aid): nvcc -gencode arch=compute_100a,code=sm_100a
// -o /tmp/tmem_bench scripts/tmem_bench.cu && /tmp/tmem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void ldwait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// nw warps; each does `iters` rounds of `per` x32 loads (64*per... columns) then one wait
__global__ void bench(int nw, int iters, int per, long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0, r[32];
  long long t0 = clock64();
  if (warp < nw) {
    for (int i = 0; i < iters; i++) {
      for (int j = 0; j < per; j++) {
        ld32(base + (uint32_t)(32 * ((j + warp / 4 * per) & 15)), r);
        acc += r[0] ^ r[31];
      }
      ldwait();
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0 && warp < nw) out[warp] = t1 - t0;
  sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}

int main() {
  long long* out; uint32_t* sink;
  cudaMalloc(&out, 64 * 8); cudaMalloc(&sink, 1024 * 4);
  for (int nw : {1, 4, 8}) for (int per : {1, 2, 4}) {
    const int iters = 200;
    bench<<<1, 32 * (nw < 4 ? 4 : nw)>>>(nw, iters, per, out, sink);
    bench<<<1, 32 * (nw < 4 ? 4 : nw)>>>(nw, iters, per, out, sink);
    long long h[8] = {0};
    cudaMemcpy(h, out, 8 * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int w = 0; w < nw; w++) mx = h[w] > mx ? h[w] : mx;
    printf("warps %d, %d x32 loads per wait: %.1f cycles per round (%.1f per load), err=%s\n", nw, per,
           (double)mx / iters, (double)mx / iters / per, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
