// FP64 throughput microbenchmark for B200 (sm_100a): DFMA vs legacy DMMA
// (mma.sync .f64) shapes, plus a fragment-layout self-check for every shape
// the DG kernels use. Standalone: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------- DFMA
template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------- DMMA
__device__ __forceinline__ void mma_m8n8k4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k4(double (&d)[4], const double (&a)[2], double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a[0]), "d"(a[1]), "d"(b));
}
__device__ __forceinline__ void mma_m16n8k8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma_m16n8k16(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
               "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int ACC>
__global__ void dmma_loop(double* out, int iters) {
  int lane = threadIdx.x & 31;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (lane + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * (lane - i);
  double d[ACC][4];
#pragma unroll
  for (int c = 0; c < ACC; ++c)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[c][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < ACC; ++c) {
      if (SHAPE == 0) {
        double dd[2] = {d[c][0], d[c][1]};
        mma_m8n8k4(dd, a[0], b[0]);
        d[c][0] = dd[0]; d[c][1] = dd[1];
      } else if (SHAPE == 1) {
        double aa[2] = {a[0], a[1]};
        mma_m16n8k4(d[c], aa, b[0]);
      } else if (SHAPE == 2) {
        double aa[4] = {a[0], a[1], a[2], a[3]};
        double bb[2] = {b[0], b[1]};
        mma_m16n8k8(d[c], aa, bb);
      } else {
        mma_m16n8k16(d[c], a, b);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < ACC; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.678) out[0] = s;
}

// ---------------------------------------------------------------- layout check
// A is row-major MxK, B is KxN (stored row-major here), D = A*B MxN.
// Assumed fragment layouts (g = lane>>2, t = lane&3):
//   m8n8k4 : a0=A[g][t]; b0=B[t][g]; d0,d1=D[g][2t+{0,1}]
//   m16n8kK: a(2j)=A[g][t+4j], a(2j+1)=A[g+8][t+4j]; b(j)=B[t+4j][g];
//            d0,d1=D[g][2t+{0,1}], d2,d3=D[g+8][2t+{0,1}]
template <int SHAPE>
__global__ void layout_kernel(const double* A, const double* B, double* D) {
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  if (SHAPE == 0) {
    double d[2] = {0, 0};
    mma_m8n8k4(d, A[g * 4 + t], B[t * 8 + g]);
    D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1];
    return;
  }
  constexpr int K = SHAPE == 1 ? 4 : SHAPE == 2 ? 8 : 16;
  double a[8] = {0}, b[4] = {0}, d[4] = {0, 0, 0, 0};
  for (int j = 0; j < K / 4; ++j) {
    a[2 * j] = A[g * K + t + 4 * j];
    a[2 * j + 1] = A[(g + 8) * K + t + 4 * j];
    b[j] = B[(t + 4 * j) * 8 + g];
  }
  if (SHAPE == 1) { double aa[2] = {a[0], a[1]}; mma_m16n8k4(d, aa, b[0]); }
  if (SHAPE == 2) { double aa[4] = {a[0], a[1], a[2], a[3]}; double bb[2] = {b[0], b[1]}; mma_m16n8k8(d, aa, bb); }
  if (SHAPE == 3) { mma_m16n8k16(d, a, b); }
  D[g * 8 + 2 * t] = d[0]; D[g * 8 + 2 * t + 1] = d[1];
  D[(g + 8) * 8 + 2 * t] = d[2]; D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

template <int SHAPE>
bool check_layout() {
  const int M = SHAPE == 0 ? 8 : 16, N = 8, K = SHAPE == 0 ? 4 : SHAPE == 1 ? 4 : SHAPE == 2 ? 8 : 16;
  std::vector<double> A(M * K), B(K * N), D(M * N), R(M * N, 0.0);
  for (int i = 0; i < M * K; ++i) A[i] = (i * 7 % 13) - 6 + 0.25 * i;
  for (int i = 0; i < K * N; ++i) B[i] = (i * 5 % 11) - 5 + 0.125 * i;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) R[m * N + n] += A[m * K + k] * B[k * N + n];
  double *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dD, D.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  layout_kernel<SHAPE><<<1, 32>>>(dA, dB, dD);
  CK(cudaGetLastError());
  CK(cudaMemcpy(D.data(), dD, D.size() * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(D[i] - R[i]));
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  printf("layout shape %d (m%dn%dk%d): max err %.3e %s\n", SHAPE, M, N, K, err, err < 1e-9 ? "OK" : "MISMATCH");
  return err < 1e-9;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  printf("device %s, SMs %d, clock %d MHz, smem/block optin %zu\n", p.name, p.multiProcessorCount,
         clk_khz / 1000, p.sharedMemPerBlockOptin);
  check_layout<0>(); check_layout<1>(); check_layout<2>(); check_layout<3>();
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  // DFMA
  for (int bpsm : {2, 4, 8}) {
    int iters = 4096, threads = 256, blocks = sms * bpsm;
    dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e0));
    dfma_loop<8><<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    printf("DFMA  blocks/SM %d: %.2f TFLOP/s (%.3f ms)\n", bpsm, flops / ms / 1e9, ms);
  }
  // DMMA
  const char* names[4] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
  const double fma_per[4] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8, 16 * 8 * 16};
  for (int shape = 0; shape < 4; ++shape) {
    for (int wpsm : {4, 8, 16}) {
      int iters = 2048, threads = 128, blocks = sms * wpsm / 4;
      auto launch = [&]() {
        if (shape == 0) dmma_loop<0, 4><<<blocks, threads>>>(out, iters);
        if (shape == 1) dmma_loop<1, 4><<<blocks, threads>>>(out, iters);
        if (shape == 2) dmma_loop<2, 4><<<blocks, threads>>>(out, iters);
        if (shape == 3) dmma_loop<3, 4><<<blocks, threads>>>(out, iters);
      };
      launch();
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * fma_per[shape] * 4 * iters * (double)(threads / 32) * blocks;
      printf("DMMA %-9s warps/SM %2d: %.2f TFLOP/s (%.3f ms)\n", names[shape], wpsm, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
