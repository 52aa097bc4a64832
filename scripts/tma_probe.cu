// tma_probe.cu -- micro-benchmark of 1-D bulk async copies (cp.async.bulk) on
// one B200: read-only streaming (TMA loads into a shared-memory ring) and
// streaming copy (TMA load + TMA store of every row), by request size, ring
// depth and resident CTAs per SM; plus the LDG/STG float4 copy for reference.
// Decides the staging granularity of the tile kernel.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/tma_probe scripts/tma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                   su32(b)),
               "r"(par)
               : "memory");
}
__device__ __forceinline__ void ld_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void st_bulk(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
               : "memory");
}

// rows: independent streams (each `len` bytes long, row r at src + r*len);
// a tile = rb bytes of every row.  mode 0: loads only; 1: load + store.
__global__ void probe(const char* src, char* dst, long long len, int rows, int rb, int S, int mode, int issuers) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  unsigned char* ring = sm + 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long tiles = len / rb;
  const long long mine = blockIdx.x < tiles ? (tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mb_init(&full[s], issuers);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto c0 = [&](long long i) { return (blockIdx.x + i * gridDim.x) * (long long)rb; };
  auto load = [&](long long i) {
    const int s = int(i % S);
    int k = 0;
    for (int r = warp; r < rows; r += issuers) ++k;
    mb_expect(&full[s], uint32_t(rb) * k);
    for (int r = warp; r < rows; r += issuers)
      ld_bulk(ring + (size_t(s) * rows + r) * rb, src + r * len + c0(i), rb, &full[s]);
  };
  const bool issuer = lane == 0 && warp < issuers;
  // read: S tiles in flight, stage refilled right after it is consumed;
  // copy: S-1 loaded ahead, a stage is refilled once its store left smem
  if (issuer)
    for (int i = 0; i < (mode ? S - 1 : S) && i < mine; ++i) load(i);
  for (long long i = 0; i < mine; ++i) {
    const int s = int(i % S);
    mb_wait(&full[s], uint32_t((i / S) & 1));
    __syncthreads();
    if (issuer) {
      if (mode) {
        for (int r = warp; r < rows; r += issuers) st_bulk(dst + r * len + c0(i), ring + (size_t(s) * rows + r) * rb, rb);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (i + S - 1 < mine) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          load(i + S - 1);
        }
      } else if (i + S < mine) {
        load(i + S);
      }
    }
  }
  if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void ldg_copy(const float4* src, float4* dst, long long n4) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x)
    dst[q] = src[q];
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const long long total = 8LL << 30;  // bytes per side
  char *src, *dst;
  cudaMalloc(&src, total);
  cudaMalloc(&dst, total);
  cudaMemset(src, 1, total);
  cudaMemset(dst, 0, total);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  {
    const long long n4 = total / 16;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ldg_copy<<<sms * 8, 256>>>(reinterpret_cast<float4*>(src), reinterpret_cast<float4*>(dst), n4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg_copy float4 GB/s(r+w) %.0f\n", 2.0 * total / ms / 1e6);
  }
  const int rbs[] = {512, 1024, 2048, 4096, 8192};
  for (int mode = 0; mode < 2; ++mode)
    for (int rows : {8, 32})
      for (int rb : rbs)
        for (int S : {3, 4, 6})
          for (int issuers : {1, 4}) {
            const size_t smem = 128 + size_t(S) * rows * rb;
            if (smem > 227 * 1024) continue;
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, probe, 128, smem);
            if (occ < 1) continue;
            const long long len = total / rows / rb * rb;
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
              cudaEventRecord(a);
              probe<<<sms * occ, 128, smem>>>(src, dst, len, rows, rb, S, mode, issuers);
              cudaEventRecord(b);
              cudaEventSynchronize(b);
              float ms;
              cudaEventElapsedTime(&ms, a, b);
              best = ms < best ? ms : best;
            }
            cudaError_t e = cudaGetLastError();
            const double bytes = double(len) * rows * (mode ? 2 : 1);
            printf("mode=%s rows=%d rb=%d S=%d issuers=%d occ=%d smem=%zuK GB/s %.0f %s\n", mode ? "copy" : "read", rows,
                   rb, S, issuers, occ, smem / 1024, bytes / best / 1e6, e ? cudaGetErrorString(e) : "");
          }
  return 0;
}
