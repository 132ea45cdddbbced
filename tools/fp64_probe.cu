// fp64 pipe probe: DADD/DMUL/DFMA throughput, DDIV throughput and latency,
// DSETP throughput (one B200, CUDA events).  Calibrates the fp64 compute roof
// quoted in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void thr(double* out, double a, double b, int iters) {
  double x0 = threadIdx.x * 1e-3 + 1.0, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int it = 0; it < iters; ++it) {
#define STEP(x)                                  \
  if (OP == 0) x = x + a;                        \
  if (OP == 1) x = x * a;                        \
  if (OP == 2) x = fma(x, a, b);                 \
  if (OP == 3) x = b / x;                        \
  if (OP == 4) x = (x > b) ? x * a : x + a;
    STEP(x0) STEP(x1) STEP(x2) STEP(x3) STEP(x4) STEP(x5) STEP(x6) STEP(x7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void lat_div(double* out, double b, int iters) {
  double x = threadIdx.x * 1e-3 + 1.5;
  for (int it = 0; it < iters; ++it) x = b / (x + 1.0);
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}
__global__ void lat_add(double* out, double b, int iters) {
  double x = threadIdx.x * 1e-3 + 1.5;
  for (int it = 0; it < iters; ++it) x = x * b + 1.0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"dadd", "dmul", "dfma", "ddiv", "dsetp+sel"};
  const int iters = 4096;
  for (int op = 0; op < 5; ++op) {
    auto run = [&]() {
      dim3 g(sms * 8), b(256);
      switch (op) {
        case 0: thr<0><<<g, b>>>(out, 1.0000001, 0.5, iters); break;
        case 1: thr<1><<<g, b>>>(out, 1.0000001, 0.5, iters); break;
        case 2: thr<2><<<g, b>>>(out, 1.0000001, 0.5, iters); break;
        case 3: thr<3><<<g, b>>>(out, 1.0000001, 0.5, iters / 8); break;
        case 4: thr<4><<<g, b>>>(out, 1.0000001, 0.5, iters); break;
      }
    };
    run();
    cudaEventRecord(e0);
    run();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)sms * 8 * 256 * 8 * (op == 3 ? iters / 8 : iters);
    printf("%-10s %8.3f ms  %8.2f Gop/s  %6.2f op/clk/SM @1.965GHz\n", names[op], ms, n / ms / 1e6,
           n / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int l = 0; l < 2; ++l) {
    cudaEventRecord(e0);
    if (l == 0) lat_div<<<1, 32>>>(out, 0.7, 10000); else lat_add<<<1, 32>>>(out, 0.7, 10000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s latency: %.1f cycles/iter\n", l == 0 ? "add+ddiv" : "mul+add", ms * 1e-3 / 10000 * 1.965e9);
  }
  return 0;
}
