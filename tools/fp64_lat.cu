// FP64 pipe micro-benchmarks on one SM (sm_100a): DFMA / DMMA / MUFU.RCP64H latency, and how a
// DFMA chain in one warp fares while another warp on the same SMSP streams DMMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_lat tools/fp64_lat.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

constexpr int ITER = 2048;
#ifndef B_FULL
#define B_FULL 0
#endif

// role: 0 idle, 1 dependent DFMA chain, 2 DMMA stream (8 independent accumulators),
//       3 DFMA with ILP 8, 4 dependent DMMA chain, 5 dependent rcp.approx chain
__device__ void run(int role, double x, double* out, long long* cyc) {
  long long t0 = clock64();
  double r = x;
  if (role == 1) {
    for (int i = 0; i < ITER; ++i) r = fma(r, 0.999999, 1e-9);
  } else if (role == 2) {
    double acc[8][2] = {};
    for (int i = 0; i < ITER / 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(acc[k], x, 1.0001 + (B_FULL ? 0.123456789012345 * k + 1e-7 * threadIdx.x : 0.0));
    for (int k = 0; k < 8; ++k) r += acc[k][0] + acc[k][1];
  } else if (role == 3) {
    double v[8];
    for (int k = 0; k < 8; ++k) v[k] = x + k;
    for (int i = 0; i < ITER / 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = fma(v[k], 0.999999, 1e-9);
    for (int k = 0; k < 8; ++k) r += v[k];
  } else if (role == 4) {
    double acc[2] = {x, x};
    for (int i = 0; i < ITER / 8; ++i) dmma(acc, acc[0] * 1e-30, 1.0);
    r = acc[0] + acc[1];
  } else if (role == 6) {
    double acc[4][2] = {};
    for (int i = 0; i < ITER / 4; ++i)
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(acc[k], x, 1.0001);
    for (int k = 0; k < 4; ++k) r += acc[k][0] + acc[k][1];
  } else if (role == 5) {
    for (int i = 0; i < ITER / 8; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;\n" : "+d"(r));
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
  out[threadIdx.x] = r;
}

__global__ void bench(const int* roles, double x, double* out, long long* cyc) {
  run(roles[threadIdx.x >> 5], x, out, cyc);
}

__global__ void bench_all(int role, double x, double* out, long long* cyc) {
  run(role, x, out + blockIdx.x * blockDim.x, cyc + blockIdx.x * (blockDim.x / 32));
}

int main(int argc, char** argv) {
  if (argc > 1) {   // full-GPU mode: fp64_lat <grid> <warps per CTA> <role>
    const int grid = atoi(argv[1]), nw = atoi(argv[2]), role = atoi(argv[3]);
    double* out;
    long long* cyc;
    cudaMalloc(&out, size_t(grid) * nw * 32 * sizeof(double));
    cudaMalloc(&cyc, size_t(grid) * nw * sizeof(long long));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double x = argc > 4 ? atof(argv[4]) : 1.0;
    bench_all<<<grid, 32 * nw>>>(role, x, out, cyc);
    cudaEventRecord(a);
    bench_all<<<grid, 32 * nw>>>(role, x, out, cyc);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long* h = new long long[size_t(grid) * nw];
    cudaMemcpy(h, cyc, size_t(grid) * nw * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid * nw; ++i) avg += h[i];
    avg /= grid * nw;
    const double ops = (role <= 3 || role == 6) ? ITER : ITER / 8;
    const double fma_per = (role == 2 || role == 4 || role == 6) ? 256.0 : 32.0;
    printf("grid %d x %d warps role %d: %.3f ms, avg %.2f cyc/op per warp, %.2f TFLOP/s\n", grid, nw, role, ms,
           avg / ops, 2.0 * fma_per * ops * grid * nw / (ms * 1e-3) / 1e12);
    return 0;
  }
  int* droles;
  double* dout;
  long long* dcyc;
  cudaMalloc(&droles, 32 * sizeof(int));
  cudaMalloc(&dout, 1024 * sizeof(double));
  cudaMalloc(&dcyc, 32 * sizeof(long long));
  struct Case { const char* name; int nw; int roles[8]; };
  // warps w and w+4 share SMSP w % 4
  Case cases[] = {
      {"DFMA chain alone (w0)", 1, {1}},
      {"DFMA ILP8 alone (w0)", 1, {3}},
      {"DMMA chain alone (w0)", 1, {4}},
      {"DMMA stream alone (w0)", 1, {2}},
      {"rcp.approx chain alone (w0)", 1, {5}},
      {"w0 DMMA stream + w4 DFMA chain", 8, {2, 0, 0, 0, 1, 0, 0, 0}},
      {"w0 DFMA chain + w4 DMMA stream", 8, {1, 0, 0, 0, 2, 0, 0, 0}},
      {"w0 DMMA stream + w4 DFMA ILP8", 8, {2, 0, 0, 0, 3, 0, 0, 0}},
      {"w0 DFMA ILP8 + w4 DMMA stream", 8, {3, 0, 0, 0, 2, 0, 0, 0}},
      {"w0 DMMA stream + w4 DMMA stream", 8, {2, 0, 0, 0, 2, 0, 0, 0}},
      {"w0 DMMA stream + w1 DFMA ILP8", 8, {2, 3, 0, 0, 0, 0, 0, 0}},
      {"w0 DMMA stream + w1 DFMA chain", 8, {2, 1, 0, 0, 0, 0, 0, 0}},
      {"w0..w3 DMMA stream", 8, {2, 2, 2, 2, 0, 0, 0, 0}},
      {"w0 DMMA + w1..w3 DFMA ILP8", 8, {2, 3, 3, 3, 0, 0, 0, 0}},
      {"w0..w3 DFMA ILP8", 8, {3, 3, 3, 3, 0, 0, 0, 0}},
      {"w0..w7 DFMA ILP8", 8, {3, 3, 3, 3, 3, 3, 3, 3}},
      {"w0 DMMA + w1..w7 DFMA ILP8", 8, {2, 3, 3, 3, 3, 3, 3, 3}},
      {"w0 DMMA ILP4 stream alone", 1, {6}},
  };
  for (auto& c : cases) {
    int roles[32] = {0};
    for (int i = 0; i < c.nw; ++i) roles[i] = c.roles[i];
    cudaMemcpy(droles, roles, sizeof(roles), cudaMemcpyHostToDevice);
    long long cyc[32];
    for (int rep = 0; rep < 2; ++rep) bench<<<1, 32 * c.nw>>>(droles, 1.0, dout, dcyc);
    cudaDeviceSynchronize();
    cudaMemcpy(cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost);
    printf("%-34s", c.name);
    for (int i = 0; i < c.nw; ++i) {
      if (!roles[i]) continue;
      const double ops = (roles[i] <= 3 || roles[i] == 6) ? ITER : ITER / 8;
      printf("  w%d role%d %.2f cyc/op", i, roles[i], cyc[i] / ops);
    }
    printf("\n");
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
