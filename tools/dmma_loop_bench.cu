// Microbenchmark: DMMA issue efficiency of the stage kernel's consumer k-loop shape
// (N = 4: 80-row X blocks, 5 n-tiles, units = n-tile pairs + odd tail) with operands in
// shared memory, no producers, no barriers.  Reports FP64 TFLOP/s of useful+padded MMA work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_loop_bench dmma_loop_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}

constexpr int ROWS = 80, XS = 108 + 60 + 12, KS4 = 42, NTL = 5;

template <int NPAIR, int NSING, int CWARPS>
__device__ void consumer(const double* sX, const double* sOp, int cw, int s0, int reps, double* out) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  int mtp[NPAIR > 0 ? NPAIR : 1], ntp[NPAIR > 0 ? NPAIR : 1], mts[NSING > 0 ? NSING : 1];
  for (int k = 0; k < NPAIR; ++k) { int p = cw + k * CWARPS; mtp[k] = p / 2; ntp[k] = 2 * (p % 2); }
  for (int k = 0; k < NSING; ++k) mts[k] = s0 + k * CWARPS;
  constexpr int NSLOT = 2 * NPAIR + NSING;
  double acc[NSLOT][4];
  for (int u = 0; u < NSLOT; ++u) acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0;
  for (int r = 0; r < reps; ++r) {
#pragma unroll 4
    for (int ks = 0; ks < KS4; ++ks) {
      const double* ob = sOp + ks * NTL * 32;
#pragma unroll
      for (int k = 0; k < NPAIR; ++k) {
        const double* xa = sX + (mtp[k] * 16 + g) * XS + t4 + ks * 4;
        const double a0 = xa[0], a1 = xa[8 * XS];
        const double2 b = *reinterpret_cast<const double2*>(ob + ntp[k] * 32 + 2 * lane);
        dmma_16x8x4(acc[2 * k], a0, a1, b.x);
        dmma_16x8x4(acc[2 * k + 1], a0, a1, b.y);
      }
#pragma unroll
      for (int k = 0; k < NSING; ++k) {
        const double* xa = sX + (mts[k] * 16 + g) * XS + t4 + ks * 4;
        const double a0 = xa[0], a1 = xa[8 * XS];
        dmma_16x8x4(acc[2 * NPAIR + k], a0, a1, ob[(NTL - 1) * 32 + lane]);
      }
    }
  }
  double s = 0;
  for (int u = 0; u < NSLOT; ++u) s += acc[u][0] + acc[u][1] + acc[u][2] + acc[u][3];
  if (s == 1234.5) out[0] = s;
}

__global__ void __launch_bounds__(512, 1) kern(int reps, double* out) {
  extern __shared__ double sm[];
  double* sX = sm;
  double* sOp = sX + ROWS * XS;
  for (int i = threadIdx.x; i < ROWS * XS + KS4 * NTL * 32; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp < 8) return;  // "producers" idle
  const int cw = warp - 8;
  // N=4 unit assignment of the stage kernel: P = 10 pair units, 5 singles
  const int cp = 10 > cw ? (10 - 1 - cw) / 8 + 1 : 0;
  const int s0 = ((cw - 10 % 8) % 8 + 8) % 8;
  const int cs = 5 > s0 ? (5 - 1 - s0) / 8 + 1 : 0;
  if (cp == 2 && cs == 0) consumer<2, 0, 8>(sX, sOp, cw, s0, reps, out);
  else if (cp == 1 && cs == 1) consumer<1, 1, 8>(sX, sOp, cw, s0, reps, out);
  else consumer<1, 0, 8>(sX, sOp, cw, s0, reps, out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t smem = (ROWS * XS + KS4 * NTL * 32) * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* out;
  cudaMalloc(&out, 8);
  int reps = 200;
  kern<<<sms, 512, smem>>>(reps, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<sms, 512, smem>>>(reps, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double flops = 2.0 * 80 * 40 * 168 * reps * (double)sms;   // padded tile MMA work
  printf("consumer k-loop: %.3f ms, %.2f TFLOP/s (padded), err=%s\n", ms, flops / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
