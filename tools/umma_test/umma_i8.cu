// Standalone check of the tcgen05 kind::i8 path (descriptors, TMEM, ld layout) before it goes into
// the MAC kernel: D[M=128][N] = sum_k A[m][k] (s8) * B[n][k] (u8), K = 64 (two MMAs), vs CPU.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__device__ __forceinline__ uint32_t idesc_i8(int m, int n) {
  uint32_t d = 0;
  d |= 2u << 4;                   // D format S32
  d |= 1u << 7;                   // A signed 8-bit
  d |= 0u << 10;                  // B unsigned 8-bit
  d |= (uint32_t)(n >> 3) << 17;  // N
  d |= (uint32_t)(m >> 4) << 24;  // M
  return d;                       // A, B K-major
}

// K-major no-swizzle canonical layout for a rows x 32-byte slice: [row/8][kchunk(2)][row%8][16 B]
__device__ __forceinline__ int kmaj_off(int row, int kbyte) {
  return (row >> 3) * 256 + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15);
}

__global__ void __launch_bounds__(128) k_umma(const int8_t* A, const uint8_t* B, int32_t* D) {
  __shared__ __align__(1024) uint8_t sA[K / 32][M * 32];
  __shared__ __align__(1024) uint8_t sB[K / 32][N * 32];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < M * K; e += 128) {
    const int m = e / K, k = e % K;
    sA[k / 32][kmaj_off(m, k % 32)] = (uint8_t)A[e];
  }
  for (int e = tid; e < N * K; e += 128) {
    const int n = e / K, k = e % K;
    sB[k / 32][kmaj_off(n, k % 32)] = B[e];
  }
  if (warp == 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, N);
    for (int ks = 0; ks < K / 32; ks++) {
      const uint64_t da = smem_desc((uint32_t)__cvta_generic_to_shared(&sA[ks][0]), 128, 256);
      const uint64_t db = smem_desc((uint32_t)__cvta_generic_to_shared(&sB[ks][0]), 128, 256);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
  }
  {  // wait for the MMAs
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(mb), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // each warp reads its 32 lanes (rows 32w..32w+31), N columns, 32-bit
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; j++) D[(warp * 32 + (tid & 31)) * N + c0 + j] = (int32_t)r[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

int main() {
  int8_t hA[M * K];
  uint8_t hB[N * K];
  int32_t hD[M * N], ref[M * N];
  srand(7);
  for (int i = 0; i < M * K; i++) hA[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * K; i++) hB[i] = (uint8_t)(rand() % 256);
  for (int m = 0; m < M; m++)
    for (int n = 0; n < N; n++) {
      int32_t s = 0;
      for (int k = 0; k < K; k++) s += (int32_t)hA[m * K + k] * (int32_t)hB[n * K + k];
      ref[m * N + n] = s;
    }
  int8_t* dA;
  uint8_t* dB;
  int32_t* dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, sizeof hD);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, sizeof hD);
  k_umma<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M * N; i++)
    if (hD[i] != ref[i]) {
      if (bad < 5) printf("mismatch at m=%d n=%d: got %d want %d\n", i / N, i % N, hD[i], ref[i]);
      bad++;
    }
  printf("umma_i8: %d mismatches of %d\n", bad, M * N);
  return bad != 0;
}
