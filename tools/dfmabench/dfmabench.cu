// FP64-pipe microbenchmark for the MAC kernel design: DFMA throughput vs
// resident warps per SM and independent accumulators per thread, with and without the
// consume-loop's shared-memory operand loads (8 weights + 2 (hi,lo) columns per k).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define ITERS 2048

template <int NACC>
__global__ void k_dfma(double* out, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NACC; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; i++) s += acc[i];
  if (s == 1.2345) out[0] = s;
}

// consume-loop shape: per k, 4 LDS.128 broadcast weights + 2 LDS.128 columns, 32 DFMA
__global__ void k_consume(double* out) {
  __shared__ double2 W[64][4];
  __shared__ double2 X[32][64];
  for (int i = threadIdx.x; i < 64 * 4; i += blockDim.x) W[i / 4][i % 4] = make_double2(i, i + 1);
  for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) X[i / 64][i % 64] = make_double2(i, 2 * i);
  __syncthreads();
  double ah[8][2], al[8][2];
#pragma unroll
  for (int r = 0; r < 8; r++) ah[r][0] = ah[r][1] = al[r][0] = al[r][1] = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < ITERS / 16; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int kk = (it + k) & 63;
      double w[8];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        double2 t = W[kk][r];
        w[2 * r] = t.x;
        w[2 * r + 1] = t.y;
      }
      double2 x0 = X[kk & 31][lane], x1 = X[kk & 31][lane + 32];
#pragma unroll
      for (int r = 0; r < 8; r++) {
        ah[r][0] = fma(w[r], x0.x, ah[r][0]);
        al[r][0] = fma(w[r], x0.y, al[r][0]);
        ah[r][1] = fma(w[r], x1.x, ah[r][1]);
        al[r][1] = fma(w[r], x1.y, al[r][1]);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < 8; r++) s += ah[r][0] + ah[r][1] + al[r][0] + al[r][1];
  if (s == 1.2345) out[0] = s;
}


// TM x TN register tile: per k, TM/2 LDS.128 broadcast weights + TN LDS.128 (hi, lo) columns
template <int TM, int TN>
__global__ void k_tile(double* out) {
  __shared__ double2 W[16][TM / 2];
  __shared__ double2 X[16][32 * TN];
  for (int i = threadIdx.x; i < 16 * TM / 2; i += blockDim.x) W[i / (TM / 2)][i % (TM / 2)] = make_double2(i, i + 1);
  for (int i = threadIdx.x; i < 16 * 32 * TN; i += blockDim.x) X[i / (32 * TN)][i % (32 * TN)] = make_double2(i, 2 * i);
  __syncthreads();
  double ah[TM][TN], al[TM][TN];
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int n = 0; n < TN; n++) ah[r][n] = al[r][n] = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < ITERS / 16; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
      const int kk = (it + k) & 15;
      double w[TM];
#pragma unroll
      for (int r = 0; r < TM / 2; r++) {
        double2 t = W[kk][r];
        w[2 * r] = t.x;
        w[2 * r + 1] = t.y;
      }
      double2 x[TN];
#pragma unroll
      for (int n = 0; n < TN; n++) x[n] = X[kk][lane + 32 * n];
#pragma unroll
      for (int r = 0; r < TM; r++)
#pragma unroll
        for (int n = 0; n < TN; n++) {
          ah[r][n] = fma(w[r], x[n].x, ah[r][n]);
          al[r][n] = fma(w[r], x[n].y, al[r][n]);
        }
    }
  }
  double s = 0;
#pragma unroll
  for (int r = 0; r < TM; r++)
#pragma unroll
    for (int n = 0; n < TN; n++) s += ah[r][n] + al[r][n];
  if (s == 1.2345) out[0] = s;
}

template <class F>
static void run(const char* name, F launch, double dfma_per_thread, int blocks, int threads) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 2; r++) launch();
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; r++) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double ops = (double)blocks * threads * dfma_per_thread * reps;
  double per_clk_sm = ops / (ms * 1e-3) / 148.0 / (clk_khz * 1e3);
  printf("%-34s blocks=%5d threads=%4d  %.2f TDFMA/s  %.1f DFMA/clk/SM (at %d MHz attr)\n", name, blocks, threads,
         ops / (ms * 1e-3) / 1e12, per_clk_sm, clk_khz / 1000);
}

int main() {
  double* o;
  cudaMalloc(&o, 8);
  for (int cps : {1, 2, 4, 8}) {
    for (int thr : {128, 256}) {
      int blocks = 148 * cps;
      char nm[64];
      snprintf(nm, sizeof nm, "dfma acc=8 warps/SM=%d", cps * thr / 32);
      run(nm, [&] { k_dfma<8><<<blocks, thr>>>(o, 1.0000001, 0.5); }, 8.0 * ITERS, blocks, thr);
      snprintf(nm, sizeof nm, "dfma acc=32 warps/SM=%d", cps * thr / 32);
      run(nm, [&] { k_dfma<32><<<blocks, thr>>>(o, 1.0000001, 0.5); }, 32.0 * ITERS, blocks, thr);
    }
  }
  for (int cps : {1, 2, 3, 4}) {
    for (int thr : {128, 256}) {
      int blocks = 148 * cps;
      char nm[64];
      snprintf(nm, sizeof nm, "consume warps/SM=%d", cps * thr / 32);
      run(nm, [&] { k_consume<<<blocks, thr>>>(o); }, 32.0 * ITERS, blocks, thr);
    }
  }
  for (int cps : {1, 2}) {
    int blocks = 148 * cps;
    run("tile 8x2 256thr", [&] { k_tile<8, 2><<<blocks, 256>>>(o); }, 32.0 * ITERS, blocks, 256);
    run("tile 8x4 256thr", [&] { k_tile<8, 4><<<blocks, 256>>>(o); }, 64.0 * ITERS, blocks, 256);
    run("tile 16x2 256thr", [&] { k_tile<16, 2><<<blocks, 256>>>(o); }, 64.0 * ITERS, blocks, 256);
    run("tile 8x4 128thr", [&] { k_tile<8, 4><<<blocks, 128>>>(o); }, 64.0 * ITERS, blocks, 128);
    run("tile 4x4 256thr", [&] { k_tile<4, 4><<<blocks, 256>>>(o); }, 32.0 * ITERS, blocks, 256);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
