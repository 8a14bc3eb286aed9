// atomics_bench.cu — sm_100a microbenchmark of shared-memory vote primitives.
// Decides the K1 vote strategy per L by measurement:
// throughput of ATOMS.ADD / ATOMS.POPC.INC / LDS+STS under the address
// patterns a GLCM vote produces. Prints one JSON object.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

constexpr int kT = 1024;
constexpr int kIters = 4096;

enum Mode {
  M_LANE_PRIVATE_INC = 0,   // [cell][lane] layout, add 1           (COPIES32 on noise)
  M_LANE_PRIVATE_ADDN,      // same, add variable n
  M_RANDOM_64K_INC,         // random word in 128 KB (L=256 packed / L=181 u32)
  M_RANDOM_64K_RET,         // same, with return value consumed (PACKED16 spill check)
  M_RANDOM_4K_INC,          // random word in 16 KB (L=64, R=1)
  M_SAME_ADDR_INC,          // all lanes of a warp on one word (smooth hot cell, R=1)
  M_SAME_ADDR_ADDN,         // same, variable increment
  M_LDS_STS_PRIVATE,        // non-atomic RMW, lane-private
  M_RANDOM_8WAY,            // COPIES8 layout: random cell*8 + lane%8 over 16K words
  M_RANDOM_8WAY_RET,        // same, returning (what a drain check would need)
  M_PACKED_16WAY_RET,       // L=64 candidate: 16 copies of packed u16 pairs, word*16 + lane%16, returning
  // The modes above draw addresses from a per-thread LCG whose 32 lanes form an
  // arithmetic progression: banks are quasi-random (2.48 wavefronts per warp
  // ATOMS instead of 3.53 for independent cells). The hashed modes below pass
  // the LCG state through murmur3's finaliser so every lane's word is
  // independent, like a noise image's GLCM cells.
  M_HASH_128KB_INC,         // random word in 128 KB, hashed (L=256 PACKED16 on noise)
  M_HASH_128KB_RET,         // same, returning (the PACKED16 drain check)
  M_HASH_8WAY_INC,          // COPIES8 layout, hashed cells (L=64 on noise)
  M_HASH_16WAY_RET,         // 16 copies of packed u16 pairs, hashed cells, returning
  M_HASH_16WAY_INC,         // same, non-returning (the L=64 16-copy layout's atomic ceiling)
  M_HASH_16WAY_PAIRBANK,    // 16 copies, each owning 2 banks (lanes l, l+16), hashed cells, non-returning
  M_NMODES
};
const char* kNames[] = {"lane_private_inc", "lane_private_addn", "random_128KB_inc", "random_128KB_ret",
                        "random_16KB_inc", "same_addr_inc", "same_addr_addn", "lds_sts_private",
                        "copies8_random", "copies8_random_ret", "packed16x16_random_ret",
                        "hashed_128KB_inc", "hashed_128KB_ret", "hashed_copies8_inc", "hashed_packed16x16_ret",
                        "hashed_packed16x16_inc", "hashed_16copies_2banks_inc"};

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  return h ^ (h >> 16);
}

template <int mode>
__global__ void __launch_bounds__(kT, 1) bench(unsigned long long* cycles, uint32_t* sink) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < 32768; i += kT) s[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t acc = 0;
  uint32_t h = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
  const unsigned long long t0 = clock64();
#pragma unroll 8
  for (int k = 0; k < kIters; ++k) {
    h = h * 1664525u + 1013904223u;  // LCG, 1 IMAD
    const uint32_t r = h >> 9;
    switch (mode) {  // compile-time
      case M_LANE_PRIVATE_INC: atomicAdd(&s[((r & 1023) << 5) | lane], 1u); break;
      case M_LANE_PRIVATE_ADDN: atomicAdd(&s[((r & 1023) << 5) | lane], (h & 7) + 1); break;
      case M_RANDOM_64K_INC: atomicAdd(&s[r & 32767], 1u); break;
      case M_RANDOM_64K_RET: acc += atomicAdd(&s[r & 32767], 1u << ((h >> 3) & 16)); break;
      case M_RANDOM_4K_INC: atomicAdd(&s[r & 4095], 1u); break;
      case M_SAME_ADDR_INC: atomicAdd(&s[(warp << 5) | (k & 31)], 1u); break;
      case M_SAME_ADDR_ADDN: atomicAdd(&s[(warp << 5) | (k & 31)], (lane & 3) + 1); break;
      case M_LDS_STS_PRIVATE: {
        volatile uint32_t* v = s;
        const uint32_t a = ((r & 1023) << 5) | lane;
        v[a] = v[a] + 1;
        break;
      }
      case M_RANDOM_8WAY: atomicAdd(&s[((r & 4095) << 3) | (lane & 7)], 1u); break;
      case M_RANDOM_8WAY_RET: acc |= atomicAdd(&s[((r & 4095) << 3) | (lane & 7)], 1u); break;
      case M_PACKED_16WAY_RET:
        acc |= atomicAdd(&s[((r & 2047) << 4) | (lane & 15)], 1u << ((h >> 3) & 16));
        break;
      case M_HASH_128KB_INC: atomicAdd(&s[fmix32(h) & 32767], 1u); break;
      case M_HASH_128KB_RET: {
        const uint32_t x = fmix32(h);
        acc |= atomicAdd(&s[x & 32767], 1u << ((x >> 15) & 16));
        break;
      }
      case M_HASH_8WAY_INC: atomicAdd(&s[((fmix32(h) & 4095) << 3) | (lane & 7)], 1u); break;
      case M_HASH_16WAY_INC: {
        const uint32_t x = fmix32(h);
        atomicAdd(&s[((x & 2047) << 4) | (lane & 15)], 1u << ((x >> 11) & 16));
        break;
      }
      case M_HASH_16WAY_PAIRBANK: {  // word (row, bank 2k + bit): lanes l, l+16 share banks 2k, 2k+1
        const uint32_t x = fmix32(h);
        atomicAdd(&s[((x & 1023) << 5) | ((lane & 15) << 1) | ((x >> 10) & 1)], 1u << ((x >> 11) & 16));
        break;
      }
      case M_HASH_16WAY_RET: {
        const uint32_t x = fmix32(h);
        acc |= atomicAdd(&s[((x & 2047) << 4) | (lane & 15)], 1u << ((x >> 11) & 16));
        break;
      }
    }
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
  if (acc == 0x12345678u) sink[0] = acc + s[lane];
}

// Distributed shared memory: a 2-CTA cluster, each CTA votes random words of
// a 128 KB histogram half; `remote_pct` of the votes go to the peer CTA.
template <int remote_pct>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kT, 1) dsmem_bench(unsigned long long* cycles) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < 32768; i += kT) s[i] = 0;
  uint32_t rank, peer_base, local_base;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  local_base = static_cast<uint32_t>(__cvta_generic_to_shared(s));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_base) : "r"(local_base), "r"(rank ^ 1));
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t h = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
  const unsigned long long t0 = clock64();
#pragma unroll 8
  for (int k = 0; k < kIters; ++k) {
    h = h * 1664525u + 1013904223u;
    const uint32_t r = h >> 9;
    const bool remote = ((h >> 2) % 100u) < (uint32_t)remote_pct;
    const uint32_t addr = (remote ? peer_base : local_base) + ((r & 32767u) << 2);
    asm volatile("red.shared::cluster.add.u32 [%0], 1;" ::"r"(addr) : "memory");
  }
  const unsigned long long t1 = clock64();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
}

// Global (L2) atomics: red.global.add.u32 on random words of a region that is
// either private per CTA (`priv` words each) or shared by all CTAs.
template <bool shared_region>
__global__ void __launch_bounds__(kT, 1) gbench(unsigned long long* cycles, uint32_t* g, uint32_t words) {
  uint32_t h = threadIdx.x * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
  uint32_t* base = shared_region ? g : g + (size_t)blockIdx.x * words;
  const unsigned long long t0 = clock64();
#pragma unroll 8
  for (int k = 0; k < kIters / 4; ++k) {
    h = h * 1664525u + 1013904223u;
    const uint32_t r = (h >> 7) ^ (h >> 19);
    asm volatile("red.global.add.u32 [%0], 1;" ::"l"(base + (r % words)) : "memory");
  }
  const unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cycles, t1 - t0);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 64);
  using K = void (*)(unsigned long long*, uint32_t*);
  K ks[M_NMODES] = {bench<0>, bench<1>, bench<2>, bench<3>, bench<4>, bench<5>, bench<6>, bench<7>,
                    bench<8>, bench<9>, bench<10>, bench<11>, bench<12>, bench<13>, bench<14>, bench<15>, bench<16>};
  for (auto k : ks) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("{\"sms\": %d, \"clock_khz\": %d, \"modes\": {", sms, clk);
  for (int m = 0; m < M_NMODES; ++m) {
    for (int rep = 0; rep < 2; ++rep) {  // first rep = warm-up
      cudaMemset(cyc, 0, 8);
      cudaEventRecord(a);
      ks[m]<<<sms, kT, 131072>>>(cyc, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)sms * kT * kIters;
    printf("%s\"%s\": {\"ms\": %.4f, \"Gops_s\": %.1f, \"ops_per_clk_per_sm\": %.3f, \"sm_mhz_est\": %.0f}",
           m ? ", " : "", kNames[m], ms, ops / ms / 1e6, (double)kT * kIters / (double)c, c / (ms * 1e3));
  }
  using D = void (*)(unsigned long long*);
  D ds[3] = {dsmem_bench<0>, dsmem_bench<50>, dsmem_bench<100>};
  const char* dn[3] = {"dsmem_red_0pct_remote", "dsmem_red_50pct_remote", "dsmem_red_100pct_remote"};
  for (int m = 0; m < 3; ++m) {
    cudaFuncSetAttribute(ds[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(cyc, 0, 8);
      cudaEventRecord(a);
      ds[m]<<<sms, kT, 131072>>>(cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double ops = (double)sms * kT * kIters;
    printf(", \"%s\": {\"ms\": %.4f, \"Gops_s\": %.1f, \"ops_per_clk_per_sm\": %.3f}", dn[m], ms, ops / ms / 1e6,
           (double)kT * kIters / (double)c);
  }
  {
    uint32_t* g;
    const uint32_t words = 8192;
    cudaMalloc(&g, (size_t)sms * words * 4);
    using G = void (*)(unsigned long long*, uint32_t*, uint32_t);
    G gs[2] = {gbench<false>, gbench<true>};
    const char* gn[2] = {"l2_red_private_8K", "l2_red_shared_8K"};
    for (int m = 0; m < 2; ++m) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(cyc, 0, 8);
        cudaEventRecord(a);
        gs[m]<<<sms, kT>>>(cyc, g, words);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = (double)sms * kT * (kIters / 4);
      printf(", \"%s\": {\"ms\": %.4f, \"Gops_s\": %.1f}", gn[m], ms, ops / ms / 1e6);
    }
  }
  printf("}, \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
