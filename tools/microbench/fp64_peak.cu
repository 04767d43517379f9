// FP64 roofline denominators for B200 (MEASURED_PEAKS.json has none):
// DFMA issue rate and mma.sync f64 (DMMA) rates for each legal shape.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_dfma(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed + threadIdx.x * 1e-9 + i;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_m8n8k4(double* out, double seed) {
  double c[4][2];
  for (int i = 0; i < 4; i++) c[i][0] = c[i][1] = 0;
  double a = seed + threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_m16n8k4(double* out, double seed) {
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  double a0 = seed + threadIdx.x, a1 = a0 * 0.5, b = 1.0 - 1e-9 * threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_m16n8k8(double* out, double seed) {
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  double a0 = seed + threadIdx.x, a1 = a0 * 0.5, a2 = a0 * 0.25, a3 = a0 * 0.125;
  double b0 = 1.0 - 1e-9 * threadIdx.x, b1 = b0 * 0.5;
  for (int it = 0; it < ITERS / 2; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

__global__ void k_m16n8k16(double* out, double seed) {
  double c[4][4];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = seed + threadIdx.x + i;
  for (int i = 0; i < 4; i++) b[i] = 1.0 - 1e-9 * (threadIdx.x + i);
  for (int it = 0; it < ITERS / 4; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
void run(const char* name, F kern, double flops_per_thread, int blocks_per_sm, int threads) {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * blocks_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) kern<<<blocks, threads>>>(out, 1.0);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; r++) kern<<<blocks, threads>>>(out, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double tf = flops_per_thread * blocks * threads * reps / (ms * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", name, blocks_per_sm, threads, tf);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  cudaFree(out);
}

int main() {
  for (int bps : {2, 4, 8}) {
    run("dfma", k_dfma, 2.0 * 8 * ITERS, bps, 256);
    // per warp: 4 mma * ITERS * (8*8*4*2 flops); per thread = /32
    run("dmma_m8n8k4", k_m8n8k4, 4.0 * ITERS * 512 / 32, bps, 256);
    run("dmma_m16n8k4", k_m16n8k4, 4.0 * ITERS * 1024 / 32, bps, 256);
    run("dmma_m16n8k8", k_m16n8k8, 4.0 * (ITERS / 2) * 2048 / 32, bps, 256);
    run("dmma_m16n8k16", k_m16n8k16, 4.0 * (ITERS / 4) * 4096 / 32, bps, 256);
  }
  return 0;
}
