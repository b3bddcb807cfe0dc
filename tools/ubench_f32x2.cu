// Microbenchmark: issue throughput of scalar FP32 (FFMA/FADD) vs the sm_100 packed FP32x2
// instructions (FFMA2/FADD2/FMUL2), the whole loop in PTX so that no register moves pollute the
// count -- decides whether the line-FFT engine is rewritten on f32x2.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ubench_f32x2.cu -o build/ubench_f32x2
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 4096;
#define BODY8(OP) OP(0) OP(1) OP(2) OP(3) OP(4) OP(5) OP(6) OP(7)
#define S_FFMA(i) "fma.rn.f32 a" #i ", a" #i ", b, c;\n"
#define S_FADD(i) "add.rn.f32 a" #i ", a" #i ", b;\n"
#define S_FFMA2(i) "fma.rn.f32x2 d" #i ", d" #i ", e, f;\n"
#define S_FADD2(i) "add.rn.f32x2 d" #i ", d" #i ", e;\n"
#define S_FMUL2(i) "mul.rn.f32x2 d" #i ", d" #i ", e;\n"
#define S_MIX(i) "add.rn.f32x2 d" #i ", d" #i ", e;\nadd.rn.f32 a" #i ", a" #i ", b;\n"
#define KERNEL(NAME, OPS, PER)                                                                          \
  __global__ void NAME(float* out, float x) {                                                           \
    float r;                                                                                            \
    asm volatile(                                                                                       \
        "{\n.reg .f32 a0,a1,a2,a3,a4,a5,a6,a7,b,c;\n.reg .b64 d0,d1,d2,d3,d4,d5,d6,d7,e,f;\n"            \
        ".reg .pred p;\n.reg .u32 i;\n"                                                                 \
        "mov.f32 a0,%1; add.f32 a1,%1,0f3F800000; add.f32 a2,a1,0f3F800000; add.f32 a3,a2,0f3F800000; add.f32 a4,a3,0f3F800000; add.f32 a5,a4,0f3F800000;\n"  \
        "add.f32 a6,a5,0f3F800000; add.f32 a7,a6,0f3F800000; mov.f32 b,%1; mov.f32 c,a3;\n"                                   \
        "mov.b64 d0,{a0,a1}; mov.b64 d1,{a1,a2}; mov.b64 d2,{a2,a3}; mov.b64 d3,{a3,a4}; mov.b64 d4,{a4,a5}; mov.b64 d5,{a5,a6};\n" \
        "mov.b64 d6,{a6,a7}; mov.b64 d7,{a7,a0}; mov.b64 e,{b,c}; mov.b64 f,{c,b};\n"                                   \
        "mov.u32 i,0;\n"                                                                                \
        "LOOP:\n" OPS OPS OPS OPS                                                                       \
        "add.u32 i,i,1;\nsetp.lt.u32 p,i,%2;\n@p bra LOOP;\n"                                          \
        "add.f32 a0,a0,a1; add.f32 a0,a0,a2; add.f32 a0,a0,a3; add.f32 a0,a0,a4; add.f32 a0,a0,a5;\n"  \
        "add.f32 a0,a0,a6; add.f32 a0,a0,a7;\n"                                                         \
        "{.reg .f32 u,v; mov.b64 {u,v},d0; add.f32 a0,a0,u; add.f32 a0,a0,v; mov.b64 {u,v},d1; add.f32 a0,a0,u;\n" \
        "add.f32 a0,a0,v; mov.b64 {u,v},d2; add.f32 a0,a0,u; add.f32 a0,a0,v; mov.b64 {u,v},d3; add.f32 a0,a0,u;\n" \
        "add.f32 a0,a0,v; mov.b64 {u,v},d4; add.f32 a0,a0,u; add.f32 a0,a0,v; mov.b64 {u,v},d5; add.f32 a0,a0,u;\n" \
        "add.f32 a0,a0,v; mov.b64 {u,v},d6; add.f32 a0,a0,u; add.f32 a0,a0,v; mov.b64 {u,v},d7; add.f32 a0,a0,u;\n" \
        "add.f32 a0,a0,v;}\n"                                                                            \
        "mov.f32 %0,a0;\n}\n"                                                                           \
        : "=f"(r)                                                                                       \
        : "f"(x), "n"(IT));                                                                             \
    if (r == 1234.5f) out[0] = r;                                                                       \
  }
KERNEL(k_ffma, BODY8(S_FFMA), 32)
KERNEL(k_fadd, BODY8(S_FADD), 32)
KERNEL(k_ffma2, BODY8(S_FFMA2), 32)
KERNEL(k_fadd2, BODY8(S_FADD2), 32)
KERNEL(k_fmul2, BODY8(S_FMUL2), 32)
KERNEL(k_mix, BODY8(S_MIX), 64)

int main() {
  float* o;
  cudaMalloc(&o, 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[] = {"FFMA", "FADD", "FFMA2", "FADD2", "FMUL2", "FADD2+FADD"};
  void (*ks[])(float*, float) = {k_ffma, k_fadd, k_ffma2, k_fadd2, k_fmul2, k_mix};
  const int per[] = {32, 32, 32, 32, 32, 64};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int threads = 32 * warps, blocks = sms * 2;
    for (int v = 0; v < 6; ++v) {
      ks[v]<<<blocks, threads>>>(o, 1.0f);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) ks[v]<<<blocks, threads>>>(o, 1.0f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double inst = 5.0 * blocks * warps * (double)IT * per[v];
      printf("warps/SM %3d  %-11s %.3f ms  warp-inst/clk/SM (at %d MHz) = %.3f\n", 2 * warps, names[v], ms / 5,
             clk / 1000, inst / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
