// pipe_probe.cu -- issue cost of the packed FP32 instruction forms on B200.
// Each kernel runs 8 independent chains per thread of one instruction form;
// the result is lane-operations per clock per SM (FFMA2 = 2 per lane).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_probe tools/pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
#define BODY(expr)                                                       \
  for (int i = 0; i < iters; ++i) {                                      \
    _Pragma("unroll") for (int r = 0; r < 8; ++r) {                      \
      _Pragma("unroll") for (int k = 0; k < CH; ++k) { expr; }           \
    }                                                                    \
  }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

template <int FORM>
__global__ void k_probe(float *out, int iters, float a, float b) {
  float2 x[CH], y[CH], z[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    x[k] = f2(threadIdx.x * 1e-3f + k, k * 0.5f);
    y[k] = f2(a + k * 1e-6f, a - k * 1e-6f);
    z[k] = f2(b + k * 1e-6f, b - k * 2e-6f);
  }
  const float2 A = f2(a, a * 0.999f), B = f2(b, b * 1.001f);
  float s1 = a, s2 = b;
  if (FORM == 0) BODY(x[k] = __ffma2_rn(x[k], A, B))                      // packed, invariant regs
  if (FORM == 1) BODY(x[k] = __ffma2_rn(x[k], y[k], z[k]))                // packed, 3 distinct regs
  if (FORM == 2) BODY(x[k] = __ffma2_rn(x[k], f2(s1, s1), z[k]))          // one scalar-broadcast operand
  if (FORM == 3) BODY(x[k] = __ffma2_rn(x[k], f2(0.9999f, 0.9999f), z[k]))  // immediate multiplier
  if (FORM == 4) BODY(x[k] = __fmul2_rn(x[k], y[k]))                      // FMUL2
  if (FORM == 5) BODY(x[k] = __fadd2_rn(x[k], y[k]))                      // FADD2
  if (FORM == 6) BODY(x[k] = __fmul2_rn(x[k], f2(s1, s1)))                // FMUL2 scalar operand
  if (FORM == 7) BODY(x[k].x = fmaf(x[k].x, y[k].x, z[k].x))              // scalar FFMA 3-reg
  if (FORM == 8) BODY(x[k].x = fmaf(x[k].x, 0.9999f, z[k].x))             // scalar FFMA imm
  if (FORM == 9) BODY(x[k].x = x[k].x * y[k].x)                           // scalar FMUL
  if (FORM == 10) BODY(x[k] = __ffma2_rn(f2(s1, s1), y[k], x[k]))         // broadcast in slot a
  if (FORM == 11) BODY(x[k] = __ffma2_rn(x[k], y[k], f2(s2, s2)))         // broadcast addend
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += x[k].x + x[k].y + y[k].x + z[k].y;
  if (s == 1234.5f) out[0] = s;
}

template <int FORM>
static void run(const char *name, int lanes_per_op, int sms) {
  float *out;
  cudaMalloc(&out, 4);
  const int iters = 2048, blocks = sms * 8, threads = 256;
  k_probe<FORM><<<blocks, threads>>>(out, 16, 1.0001f, 0.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_probe<FORM><<<blocks, threads>>>(out, iters, 1.0001f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int khz;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double ops = (double)blocks * threads * iters * 8 * CH * lanes_per_op;
  const double clk = ms * 1e-3 * khz * 1e3;
  printf("%-34s %8.3f ms  %7.1f lane-ops/clk/SM (at %d MHz)\n", name, ms, ops / clk / sms, khz / 1000);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("FFMA2 x,A,B (invariant)", 2, sms);
  run<1>("FFMA2 x,y,z (3 distinct)", 2, sms);
  run<2>("FFMA2 x,s.F32,z", 2, sms);
  run<3>("FFMA2 x,imm,z", 2, sms);
  run<4>("FMUL2 x,y", 2, sms);
  run<5>("FADD2 x,y", 2, sms);
  run<6>("FMUL2 x,s.F32", 2, sms);
  run<7>("FFMA x,y,z", 1, sms);
  run<8>("FFMA x,imm,z", 1, sms);
  run<9>("FMUL x,y", 1, sms);
  run<10>("FFMA2 s.F32,y,x", 2, sms);
  run<11>("FFMA2 x,y,s.F32", 2, sms);
  return 0;
}
