// sm_100a kernels of the per-probe multislice gradient chain (arXiv 2205.06327, Alg. 1 step 6,
// P:14; Eq. 1-2; multislice G) and its helpers.
//
// Design:
//  * Each pass is a batch of N independent 1-D complex transforms ("lines") held in registers:
//    N = P*Q, one line per Q threads, thread q holds elements q + Q*k (k < P).  A line FFT is a
//    four-step P x Q Stockham transform: in-register DFT_P, twiddle W_N^{qk} (table rounded from
//    double), one padded shared-memory exchange, in-register DFT_Q.  Input and output share the
//    same distribution, so FFT -> pointwise -> IFFT needs no reordering.
//  * The propagator H is separable (H = H_1(u) H_1(v)), so one slice's propagation is a row
//    pass (FFT.H_1.IFFT) and a column pass.  Slices alternate the axis they start on, so every
//    pass is "finish the previous slice's propagation along my axis, transmit by t_s (stash
//    phi_s), start the next propagation along my axis" and writes its output transposed.
//    2S+1 passes per probe instead of 4S-1 (DESIGN.md §Pass schedule).
//  * V_k, AccBuf_k and the stash store slice s in the layout of the pass that touches it
//    (even slices [y][x], odd slices [x][y]), so every HBM access is along a contiguous line.
//  * Scatter-add / SGD (Alg. 1 steps 7-8) are fused into the backward pass: each voxel of
//    win ^ R_k has exactly one writer per probe, probes are stream-ordered -> deterministic,
//    no atomics.
#include <cuda_runtime.h>
#include <cstdint>
#include "internal.h"
#include "twiddle32.h"


namespace ptycho {

// ------------------------------------------------------------------------------------------
// complex helpers.  sm_100 packed FP32x2 (FADD2 / FMUL2 / FFMA2): one instruction updates both
// halves of a complex64, and the operand modifiers of the packed forms (broadcast .F32, swap
// .LO_HI, half negation .NP) absorb the swaps and sign flips of complex arithmetic, so a complex
// add is 1 instruction (scalar: 2), a complex multiply 2 (scalar: 4) and a radix-4 butterfly 8
// (scalar: 16).  The FP32 pipe time is the same (measured: FFMA2 issues at half the FFMA rate,
// tools/ubench_f32x2.cu), but the passes are issue-bound, so the saved issue
// slots are what counts.  Rounding is that of the scalar forms (each half is one RN add / mul /
// fused multiply-add).  PTYCHO_SCALAR_FP builds the scalar arithmetic for A/B runs.
// ------------------------------------------------------------------------------------------
#ifndef PTYCHO_SCALAR_FP
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 csub_i(float2 a, float2 b) {  // a - i b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(1.f, -1.f), a);
}
__device__ __forceinline__ float2 cadd_i(float2 a, float2 b) {  // a + i b
  return __ffma2_rn(make_float2(b.y, b.x), make_float2(-1.f, 1.f), a);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {  // a*b = b.x a + b.y (-a.y, a.x)
  return __ffma2_rn(make_float2(a.y, a.x), make_float2(-b.y, b.y), __fmul2_rn(make_float2(b.x, b.x), a));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b) = b.x a + b.y (a.y, -a.x)
  return __ffma2_rn(make_float2(a.y, a.x), make_float2(b.y, -b.y), __fmul2_rn(make_float2(b.x, b.x), a));
}
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 csub_i(float2 a, float2 b) { return make_float2(a.x + b.y, a.y - b.x); }
__device__ __forceinline__ float2 cadd_i(float2 a, float2 b) { return make_float2(a.x - b.y, a.y + b.x); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
#endif

template <int P> struct Log2 { static constexpr int v = 1 + Log2<P / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

__host__ __device__ constexpr int brev(int i, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
  return r;
}

// a * exp(-+ 2 pi i m / 32); m is a compile-time constant after unrolling.
template <bool INV>
__device__ __forceinline__ float2 twmul32(float2 a, int m) {
  m &= 31;
  if (m == 0) return a;
  if (m == 16) return make_float2(-a.x, -a.y);
  if (m == 8) return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
  if (m == 24) return INV ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
  const float c = tw_cos32(m), s = tw_sin32(m);
  return INV ? cmul(a, make_float2(c, s)) : cmul(a, make_float2(c, -s));
}

// In-register forward DFT of size P in {2,4,8,16,32}, natural order in and out, unnormalised
// (exp(-2 pi i jk/P)).  Mixed radix: P = A*B with A = 4 (A = 2 for P = 2, 8): B-point DFTs on
// the A decimated subsequences, twiddles W_P^{n1 k2} (compile-time, rounded from double; the
// trivial ones are exact sign/swaps), then A-point DFTs.  All indices are compile-time, so the
// sub-arrays are register renames.
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  const float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}
__device__ __forceinline__ void dft4(float2& a, float2& b, float2& c, float2& d) {
  const float2 t0 = cadd(a, c), t1 = csub(a, c), t2 = cadd(b, d), t3 = csub(b, d);
  a = cadd(t0, t2);
  c = csub(t0, t2);
  b = csub_i(t1, t3);
  d = cadd_i(t1, t3);
}

template <int P> struct DftReg {
  static constexpr int A = (P == 8) ? 2 : 4, B = P / A;
  __device__ __forceinline__ static void run(float2 (&x)[P]) {
    float2 y[A][B];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) {
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) y[n1][n2] = x[n1 + A * n2];
      DftReg<B>::run(y[n1]);
#pragma unroll
      for (int k2 = 1; k2 < B; ++k2) y[n1][k2] = twmul32<false>(y[n1][k2], n1 * k2 * (32 / P));
    }
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) {
      float2 z[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) z[n1] = y[n1][k2];
      DftReg<A>::run(z);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) x[k2 + B * k1] = z[k1];
    }
  }
};
template <> struct DftReg<2> {
  __device__ __forceinline__ static void run(float2 (&x)[2]) { dft2(x[0], x[1]); }
};
template <> struct DftReg<4> {
  __device__ __forceinline__ static void run(float2 (&x)[4]) { dft4(x[0], x[1], x[2], x[3]); }
};

// exp(i x) for the transmission t = exp(i sigma V): Cephes minimax polynomials on |x| <= pi/4
// (about 1 ulp, no range reduction -- sigma V is a small phase for any physical potential),
// sincospi with its exact reduction otherwise.  The choice is made ONCE per pointwise step for the
// whole warp (small_phases: one vote over every element the warp's threads hold), so the unrolled
// step loops are branch-free and their elements interleave (a per-element vote split every
// element into its own basic block).  A branch-free Cody-Waite-reduced variant measured slower
// (2x4 tiles -1 %, lone chain -2.3 %, profiles/round2/ab_tma.txt).
template <bool FAST>
__device__ __forceinline__ void sincos_t(float x, float* sn, float* cs) {
  if (FAST) {
    const float z = x * x;
    *sn = fmaf(fmaf(fmaf(-1.9515295891e-4f, z, 8.3321608736e-3f), z, -1.6666654611e-1f), z * x, x);
    *cs = fmaf(fmaf(fmaf(2.443315711809948e-5f, z, -1.388731625493765e-3f), z, 4.166664568298827e-2f), z * z,
               fmaf(-0.5f, z, 1.0f));
  } else {
    sincospif(x * 0.318309886183790672f, sn, cs);
  }
}
// |sigma v| <= pi/4 for every v[idx(k)], k < P, of every thread of the warp (rounding of sigma*v is
// monotone in |v|, so the max decides exactly what the per-element test did)
template <int P, typename Idx>
__device__ __forceinline__ bool small_phases(const float* v, float sigma, Idx idx) {
  float m = 0.f;
#pragma unroll
  for (int k = 0; k < P; ++k) m = fmaxf(m, fabsf(v[idx(k)]));
  return __all_sync(0xffffffffu, fabsf(sigma * m) <= 0.785398163f);
}
template <bool B> struct Bool { static constexpr bool value = B; };

// ------------------------------------------------------------------------------------------
// FFT engines.  A line of N complex values is held by T threads, E = N/T elements each.
// Distribution D0 (natural): thread t holds element t + T*k in register k.  dit() computes the
// unnormalised forward DFT taking D0 to an engine-specific distribution D1; dif() computes the
// same DFT taking D1 to D0.  idx(dist, t, k) = natural index of register k.  The pass kernel
// alternates dit, dif, dit, dif, so FFT -> pointwise -> FFT never needs a reordering pass.
// ------------------------------------------------------------------------------------------

// Four-step P x P (N = 64, 256): T = P threads, D1 == D0; tw[k*P + q] = W_N^{qk}.
template <int P>
struct EngFour {
  static constexpr int N = P * P, T = P, E = P;
  // exchange buffer per line (float2): rows padded to P + 2 (16-B aligned rows) -- the column
  // writes (STS.64) and the row reads (LDS.128, 8 threads per phase at a 4-bank stride) are both
  // bank-conflict free
  static constexpr int LD = P + 2;
  static constexpr int EX = P * LD;
  static constexpr int TW = N;            // twiddle table (float2)
  __device__ __forceinline__ static int idx(int, int t, int k) { return t + T * k; }
  __device__ __forceinline__ static void sync_line(int) { __syncwarp(); }
  // transpose of the P x P block held by the line's P threads (thread q: column q -> row q)
  __device__ __forceinline__ static void exchange(float2 (&x)[E], float2* __restrict__ ex, int q) {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < P; ++k) ex[k * LD + q] = x[k];
    __syncwarp();
    const float4* row = (const float4*)(ex + q * LD);
#pragma unroll
    for (int n = 0; n < P / 2; ++n) {
      const float4 v = row[n];
      x[2 * n] = make_float2(v.x, v.y);
      x[2 * n + 1] = make_float2(v.z, v.w);
    }
    __syncwarp();
  }
  // the same transpose through a real-valued buffer of half the size (rows padded to P + 4 floats:
  // STS.32 column writes and LDS.128 row reads conflict-free), real parts then imaginary parts --
  // for the 3-CTA/SM backward build, where shared memory is the occupancy limit
  static constexpr int LDH = P + 4;
  static constexpr int EXH = P * LDH;  // floats
  __device__ __forceinline__ static void exchange_half(float2 (&x)[E], float* __restrict__ exf, int q) {
    const float4* row = (const float4*)(exf + q * LDH);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < P; ++k) exf[k * LDH + q] = x[k].x;
    __syncwarp();
#pragma unroll
    for (int n = 0; n < P / 4; ++n) {
      const float4 v = row[n];
      x[4 * n].x = v.x;
      x[4 * n + 1].x = v.y;
      x[4 * n + 2].x = v.z;
      x[4 * n + 3].x = v.w;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < P; ++k) exf[k * LDH + q] = x[k].y;
    __syncwarp();
#pragma unroll
    for (int n = 0; n < P / 4; ++n) {
      const float4 v = row[n];
      x[4 * n].y = v.x;
      x[4 * n + 1].y = v.y;
      x[4 * n + 2].y = v.z;
      x[4 * n + 3].y = v.w;
    }
    __syncwarp();
  }
  __device__ __forceinline__ static void fft_rh(float2 (&x)[E], float* __restrict__ exf, int q,
                                               const float2 (&twr)[P]) {
    DftReg<P>::run(x);
#pragma unroll
    for (int k = 1; k < P; ++k) x[k] = cmul(x[k], twr[k]);
    exchange_half(x, exf, q);
    DftReg<P>::run(x);
  }
  __device__ __forceinline__ static void fft(float2 (&x)[E], float2* __restrict__ ex, int q,
                                            const float2* __restrict__ tw) {
    DftReg<P>::run(x);
#pragma unroll
    for (int k = 1; k < P; ++k) x[k] = cmul(x[k], tw[k * P + q]);
    exchange(x, ex, q);
    DftReg<P>::run(x);
  }
  // same transform with the thread's P twiddles W_N^{qk} held in registers (loaded once per pass)
  __device__ __forceinline__ static void fft_r(float2 (&x)[E], float2* __restrict__ ex, int q,
                                              const float2 (&twr)[P]) {
#ifdef PTYCHO_EXPERIMENT_NO_FFT
    return;  // timing experiment only: everything but the transforms
#endif
    DftReg<P>::run(x);
#pragma unroll
    for (int k = 1; k < P; ++k) x[k] = cmul(x[k], twr[k]);
    exchange(x, ex, q);
    DftReg<P>::run(x);
  }
  __device__ __forceinline__ static void dit(float2 (&x)[E], float2* ex, int t, const float2* tw, int) {
    fft(x, ex, t, tw);
  }
  __device__ __forceinline__ static void dif(float2 (&x)[E], float2* ex, int t, const float2* tw, int) {
    fft(x, ex, t, tw);
  }
  static void fill(float2* tw) {
    for (int k = 0; k < P; ++k)
      for (int q = 0; q < P; ++q) {
        const double th = -2.0 * 3.14159265358979323846 * (double)(q * k) / (double)N;
        tw[k * P + q] = make_float2((float)cos(th), (float)sin(th));
      }
  }
};

// N = 1024 = 16 * 16 * 4 with T = 64 threads per line (E = 16): twice the warps of a 32 x 32
// four-step and half the registers.  With n = t + 64p, t = a + 4b and k = k1 + 16c + 256d:
//   W^{nk} = W16^{p k1} . W1024^{t k1} . W16^{b c} . W64^{a c} . W4^{a d}
// DIT: DFT16 over p | x W1024^{t k1} | exchange | DFT16 over b | x W64^{ac} | exchange | 4 DFT4 over a.
// DIF runs the mirror stages.  D1: thread t = 4 k1 + g holds k = k1 + 64 g + 16 r + 256 d in
// register d + 4r.  Exchange layouts are XOR-swizzled so that both the writing and the reading
// pattern of each exchange are shared-memory-bank-conflict free (one 8 KB buffer per line).
struct Eng1024 {
  static constexpr int N = 1024, T = 64, E = 16;
  static constexpr int EX = 1024;
  static constexpr int T2 = 1024;         // W64^{ac} at tw[T2 + 17a + c]
  static constexpr int TW = 1024 + 72;
  __device__ __forceinline__ static int e1(int k1, int t) { return k1 * 64 + (t ^ ((k1 & 3) << 2)); }
  __device__ __forceinline__ static int e2(int k1, int a, int c) {
    return k1 * 64 + 16 * a + ((((c >> 2) ^ a) << 2) | ((c & 3) ^ (k1 & 3)));
  }
  __device__ __forceinline__ static int idx(int dist, int t, int k) {
    return dist ? (t >> 2) + 64 * (t & 3) + 16 * (k >> 2) + 256 * (k & 3) : t + 64 * k;
  }
  __device__ __forceinline__ static void sync_line(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }

  __device__ __forceinline__ static void dit(float2 (&x)[16], float2* __restrict__ ex, int t,
                                            const float2* __restrict__ tw, int bid) {
    DftReg<16>::run(x);  // over p -> k1
#pragma unroll
    for (int k1 = 1; k1 < 16; ++k1) x[k1] = cmul(x[k1], tw[e1(k1, t)]);
    sync_line(bid);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) ex[e1(k1, t)] = x[k1];
    sync_line(bid);
    const int k1u = t >> 2, a = t & 3;
#pragma unroll
    for (int b = 0; b < 16; ++b) x[b] = ex[e1(k1u, a + 4 * b)];
    DftReg<16>::run(x);  // over b -> c
#pragma unroll
    for (int c = 1; c < 16; ++c) x[c] = cmul(x[c], tw[T2 + 17 * a + c]);
    sync_line(bid);
#pragma unroll
    for (int c = 0; c < 16; ++c) ex[e2(k1u, a, c)] = x[c];
    sync_line(bid);
    const int g = t & 3;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int aa = 0; aa < 4; ++aa) x[aa + 4 * r] = ex[e2(k1u, aa, 4 * g + r)];
#pragma unroll
    for (int r = 0; r < 4; ++r) dft4(x[4 * r], x[4 * r + 1], x[4 * r + 2], x[4 * r + 3]);  // over a -> d
  }

  __device__ __forceinline__ static void dif(float2 (&x)[16], float2* __restrict__ ex, int t,
                                            const float2* __restrict__ tw, int bid) {
    const int k1w = t >> 2, g = t & 3;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      dft4(x[4 * r], x[4 * r + 1], x[4 * r + 2], x[4 * r + 3]);  // over d -> a
#pragma unroll
      for (int aa = 1; aa < 4; ++aa) x[aa + 4 * r] = cmul(x[aa + 4 * r], tw[T2 + 17 * aa + 4 * g + r]);
    }
    sync_line(bid);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int aa = 0; aa < 4; ++aa) ex[e2(k1w, aa, 4 * g + r)] = x[aa + 4 * r];
    sync_line(bid);
    const int a = t & 3;
#pragma unroll
    for (int c = 0; c < 16; ++c) x[c] = ex[e2(k1w, a, c)];
    DftReg<16>::run(x);  // over c -> b
#pragma unroll
    for (int b = 0; b < 16; ++b) x[b] = cmul(x[b], tw[e1(k1w, a + 4 * b)]);
    sync_line(bid);
#pragma unroll
    for (int b = 0; b < 16; ++b) ex[e1(k1w, a + 4 * b)] = x[b];
    sync_line(bid);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) x[k1] = ex[e1(k1, t)];
    DftReg<16>::run(x);  // over k1 -> p
  }

  static void fill(float2* tw) {
    const double pi2 = 2.0 * 3.14159265358979323846;
    for (int i = 0; i < TW; ++i) tw[i] = make_float2(0.f, 0.f);
    for (int k1 = 0; k1 < 16; ++k1)
      for (int t = 0; t < 64; ++t) {
        const double th = -pi2 * (double)(t * k1) / 1024.0;
        tw[k1 * 64 + (t ^ ((k1 & 3) << 2))] = make_float2((float)cos(th), (float)sin(th));
      }
    for (int a = 0; a < 4; ++a)
      for (int c = 0; c < 16; ++c) {
        const double th = -pi2 * (double)(a * c) / 64.0;
        tw[T2 + 17 * a + c] = make_float2((float)cos(th), (float)sin(th));
      }
  }
};

template <int N> struct EngOf;
template <int N> struct EngThreads { static constexpr int v = N == 64 ? 8 : (N == 256 ? 16 : 32); };
#ifdef PTYCHO_ENG1024_3STAGE
template <> struct EngThreads<1024> { static constexpr int v = 64; };
#endif
template <> struct EngOf<64> { using type = EngFour<8>; };
template <> struct EngOf<256> { using type = EngFour<16>; };
// The 16x16x4 / 64-thread engine doubles the warps but measured slower on B200 (two exchanges
// per transform saturate the shared-memory pipe: 22.9 us vs 20.6 us per backward pass, ncu
// profiles/round1.md); the 32 x 32 four-step is used.  Eng1024 stays selectable for experiments.
#ifdef PTYCHO_ENG1024_3STAGE
template <> struct EngOf<1024> { using type = Eng1024; };
#else
template <> struct EngOf<1024> { using type = EngFour<32>; };
#endif

size_t twiddle_table_size(int n) {
  switch (n) {
    case 64: return EngFour<8>::TW;
    case 256: return EngFour<16>::TW;
    case 1024: return EngOf<1024>::type::TW;
    default: return 0;
  }
}

void fill_twiddles(int n, float2* tw) {
  switch (n) {
    case 64: EngFour<8>::fill(tw); break;
    case 256: EngFour<16>::fill(tw); break;
    case 1024: EngOf<1024>::type::fill(tw); break;
    default: break;
  }
}

// ------------------------------------------------------------------------------------------
// pass kernel
// ------------------------------------------------------------------------------------------
// Pointwise steps between forward-DFT calls (F).  With F^-1 = conj o F o conj (unnormalised,
// 1/N folded into H):
//   propagation  P  = F^-1 (H/N) F       ->  F ; y <- conj(H/N) conj(y) ; F ; result = conj(z)
//   adjoint      P^H = F^-1 conj(H)/N F  ->  F ; y <- (H/N) conj(y)      ; F ; result = conj(z)
// so after the second F of a propagation the register value is the conjugate of the true field
// ("conj pending"); the next step folds that conjugation in.
// Unroll factor of the rolled pointwise steps (TRANSMIT / GRAD / RECON), see S_GRAD: round 1 (per-
// element sincos votes) 4 > 8; with one vote per step the loops are branch-free and 8 measured
// +0.6 % (8 tiles) / +0.5 % (lone chain) over 4 (profiles/round2/ab_unroll.txt).
#ifndef PTYCHO_STEP_UNROLL
#define PTYCHO_STEP_UNROLL 8
#endif
constexpr int kStepUnroll = PTYCHO_STEP_UNROLL;
#ifndef PTYCHO_PREF_UNROLL
#define PTYCHO_PREF_UNROLL 8
#endif
#ifndef PTYCHO_STORE_UNROLL
#define PTYCHO_STORE_UNROLL 4
#endif
constexpr int kPrefUnroll = PTYCHO_PREF_UNROLL;    // V / AccBuf row prefetch loop
constexpr int kStoreUnroll = PTYCHO_STORE_UNROLL;  // transposed-store loop

enum Step : int {
  S_NONE = 0,
  S_HC_FWD,      // y <- conj(H) conj(y)            (inside P)
  S_HC_ADJ,      // y <- H conj(y)                  (inside P^H)
  S_CONJ,        // y <- conj(y)                    (start an inverse transform of a true field)
  S_TRANSMIT,    // psi = conj(y) [cp] or y ; phi = t_s psi ; stash phi ; y <- phi
  S_RESID,       // X = y ; loss ; chi = r X/(|X| N) ; y <- conj(chi)   (start of the 2-D inverse)
  S_SIMUL,       // |X| -> measurement store
  S_GRAD,        // chi_phi = conj(y) ; g ; AccBuf/V update ; y <- conj(t) chi_phi
  S_RECON,       // phi_s = conj(y) -> stash ring ; y <- conj(t_s) phi_s   (stash-free adjoint)
  S_RECON_T,     // y <- conj(t_s) y  (true phi_{S-1} from the stash)
};

// Per pass kind: steps before each F call, the step after the last F, and whether the stored
// field is "conj pending".
struct Plan {
  int nf;          // number of forward DFT calls
  int pre[4];      // step applied before F call i
  int post;        // step after the last F
  bool store_conj; // stored value = conj(register)
  bool transmit_cp;// S_TRANSMIT input is conj pending
};

__host__ __device__ constexpr Plan plan_of(int kind) {
  switch (kind) {
    case K_FWD_FIRST_PROP: return {2, {S_TRANSMIT, S_HC_FWD, 0, 0}, S_NONE, true, false};
    case K_FWD_FIRST_FFT: return {1, {S_TRANSMIT, 0, 0, 0}, S_NONE, false, false};
    case K_FWD_MID: return {4, {S_NONE, S_HC_FWD, S_TRANSMIT, S_HC_FWD}, S_NONE, true, true};
    case K_FWD_LAST: return {3, {S_NONE, S_HC_FWD, S_TRANSMIT, 0}, S_NONE, false, true};
    case K_TURN: return {2, {S_NONE, S_RESID, 0, 0}, S_NONE, true, false};
    case K_SIMULATE: return {1, {S_NONE, 0, 0, 0}, S_SIMUL, false, false};
    case K_BWD_LAST_PROP: return {3, {S_CONJ, S_GRAD, S_HC_ADJ, 0}, S_NONE, true, false};
    case K_BWD_LAST_END: return {1, {S_CONJ, 0, 0, 0}, S_GRAD, false, false};
    case K_BWD_MID: return {4, {S_NONE, S_HC_ADJ, S_GRAD, S_HC_ADJ}, S_NONE, true, false};
    case K_BWD_END: return {2, {S_NONE, S_HC_ADJ, 0, 0}, S_GRAD, false, false};
    case K_EXIT_COMPLETE: return {2, {S_NONE, S_HC_FWD, 0, 0}, S_NONE, true, false};
    // the phi chain mirrors the chi chain pass for pass (same P^H, same conj(t_s)): psi_s =
    // conj(t_s) phi_s and phi_{s-1} = P^H psi_s (P unitary, |t_s| = 1; App. A)
    case K_RECON_FIRST: return {2, {S_RECON_T, S_HC_ADJ, 0, 0}, S_NONE, true, false};
    case K_RECON_MID: return {4, {S_NONE, S_HC_ADJ, S_RECON, S_HC_ADJ}, S_NONE, true, false};
    case K_RECON_END: return {2, {S_NONE, S_HC_ADJ, 0, 0}, S_RECON, false, false};
    default: return {0, {0, 0, 0, 0}, 0, false, false};
  }
}

__host__ __device__ constexpr bool has_step(const Plan& p, int st) {
  return p.post == st || (p.nf > 0 && p.pre[0] == st) || (p.nf > 1 && p.pre[1] == st) ||
         (p.nf > 2 && p.pre[2] == st) || (p.nf > 3 && p.pre[3] == st);
}

__host__ __device__ constexpr bool kind_transmit(int k) {
  return k == K_FWD_FIRST_PROP || k == K_FWD_FIRST_FFT || k == K_FWD_MID || k == K_FWD_LAST;
}
__host__ __device__ constexpr bool kind_grad(int k) {
  return k == K_BWD_LAST_PROP || k == K_BWD_LAST_END || k == K_BWD_MID || k == K_BWD_END;
}
__host__ __device__ constexpr bool kind_recon(int k) {
  return k == K_RECON_FIRST || k == K_RECON_MID || k == K_RECON_END;
}
__host__ __device__ constexpr bool kind_first(int k) { return k == K_FWD_FIRST_PROP || k == K_FWD_FIRST_FFT; }
__host__ __device__ constexpr int kind_store(int k) {
  return k == K_SIMULATE || k == K_BWD_LAST_END || k == K_BWD_END || k == K_RECON_END
             ? 0
             : (k == K_EXIT_COMPLETE ? 2 : 1);
}

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async4(void* sm, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sm)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sm, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm)), "l"(g) : "memory");
}
// Streaming data (V / AccBuf rows, the stash, measurement rows) is touched once per pass and not
// again until a much later pass; it is marked evict-first in L2 so that it does not push out the
// wavefield ping-pong buffers the next pass reads (PTYCHO_NO_L2_HINTS: plain accesses).  Measured:
// lone chain +0.6 %, 8 tiles neutral (profiles/round1.md).
__device__ __forceinline__ unsigned long long l2_stream_policy() {
  unsigned long long p = 0;
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ void cp_async4s(void* sm, const void* g, unsigned long long pol) {
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_u32(sm)), "l"(g), "l"(pol)
               : "memory");
#else
  cp_async4(sm, g);
#endif
}
__device__ __forceinline__ void cp_async16s(void* sm, const void* g, unsigned long long pol) {
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(sm)), "l"(g), "l"(pol)
               : "memory");
#else
  cp_async16(sm, g);
#endif
}
__device__ __forceinline__ void st_stream(float* p, float v, unsigned long long pol) {
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
__device__ __forceinline__ void st_stream(float2* p, float2 v, unsigned long long pol) {
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol) : "memory");
#else
  *p = v;
#endif
}
// AccBuf_k[p] += g (Alg. 1 step 7) as a fire-and-forget L2 reduction: one writer per voxel per
// probe and probes are stream-ordered, so the result is fl(AccBuf + g) exactly as a read-modify-
// write -- without the prefetch of the AccBuf row (4 KB of shared memory per line at N = 1024) and
// without the load latency
__device__ __forceinline__ void red_add_stream(float* p, float v, unsigned long long pol) {
#ifndef PTYCHO_NO_L2_HINTS
  asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(v), "l"(pol) : "memory");
#else
  atomicAdd(p, v);
#endif
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---- TMA (cp.async.bulk.tensor) and bulk copies with an mbarrier (one per CTA, used once)
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE;\n"
      " bra LAB_WAIT;\n DONE:\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int x, int y, int z,
                                          unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(z),
      "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, unsigned bytes, unsigned long long pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}


// ---- thread-block clusters (cluster_chain_kernel)
__device__ __forceinline__ void st_cluster_v4(const void* local_smem, unsigned rank, float4 v) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local_smem)), "r"(rank));
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w) : "memory");
}
__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// every CTA of the cluster has finished the pass: its DSMEM stores and global V / AccBuf / stash
// writes are visible (release / acquire at cluster scope; the cluster-scope fence also invalidates
// L1, so the next pass's L1-allocating cp.async reads of V / AccBuf are not stale)
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}

// Location of this line inside R_k for slice parity ax.
struct LineLoc {
  long long row;  // offset of (line, pos=0) in the slice, valid only if ok
  int pos0;       // tile-local coordinate of window position 0 along the line
  int plim;       // extent along the line
  bool ok;        // line inside R_k
};

__device__ __forceinline__ LineLoc line_loc(const PassArgs& a, int ax, int line, int wy0, int wx0) {
  LineLoc L;
  if (ax == 0) {  // line = window row, position = window column; slice stored [eh][pitch0]
    const int ty = wy0 + line - a.ey0;
    L.ok = (unsigned)ty < (unsigned)a.eh;
    L.row = (long long)ty * a.pitch0;
    L.pos0 = wx0 - a.ex0;
    L.plim = a.ew;
  } else {        // line = window column, position = window row; slice stored [ew][pitch1]
    const int tx = wx0 + line - a.ex0;
    L.ok = (unsigned)tx < (unsigned)a.ew;
    L.row = (long long)tx * a.pitch1;
    L.pos0 = wy0 - a.ey0;
    L.plim = a.eh;
  }
  return L;
}

// Shared-memory carve-up of a pass CTA.  HALF: the half-size exchange buffer (EngFour only).
template <int N, int KIND, bool HALF = false>
struct Smem {
  using ENG = typename EngOf<N>::type;
  static constexpr int L = LINES_PER_CTA;
  static constexpr bool TW_REG = (ENG::T * ENG::T == N);               // twiddles in registers
  static constexpr size_t tw = 0;                                    // twiddles (engine layout)
  static constexpr size_t ht = tw + (TW_REG ? 0 : (size_t)ENG::TW * 8);  // H_1/N, m = 0..N/2
  static constexpr size_t bar = ht + (N / 2 + 2) * 8;                // mbarrier of the TMA prefetch
  static constexpr size_t red = bar + 8;                             // TURN: per-warp loss partials
  static constexpr size_t lines = (red + 64 + 127) / 128 * 128;      // per-line buffers, 128-B aligned (TMA)
  static constexpr size_t ex_b = HALF ? ((size_t)ENG::T * (ENG::T + 4) * 4 + 127) / 128 * 128
                                      : (size_t)ENG::EX * 8;          // exchange buffer per line
  static constexpr size_t st_b = kind_grad(KIND) ? (size_t)N * 8 : 0;  // stash prefetch per line
  // V / AccBuf rows: N floats + the 4-float tail of the 16-B aligned TMA superset (rounded to
  // 128 B so that every TMA destination stays 128-B aligned)
  static constexpr size_t v_b =
      (kind_transmit(KIND) || kind_grad(KIND) || kind_recon(KIND) || KIND == K_TURN) ? (size_t)N * 4 + 128 : 0;
#ifdef PTYCHO_ACC_RMW
  static constexpr size_t acc_b = kind_grad(KIND) ? (size_t)N * 4 + 128 : 0;  // AccBuf prefetch per line
#else
  static constexpr size_t acc_b = 0;  // AccBuf += g by red.global.add: no prefetch, no buffer
#endif
  static constexpr size_t per_line = ex_b + st_b + v_b + acc_b;
  static constexpr size_t stage_b = (size_t)N * (L + 1) * 8;         // transposed-store staging
  static constexpr size_t total = lines + (per_line * L > stage_b ? per_line * L : stage_b);
  // the pass kernels have no static shared memory, so the dynamic window starts at shared offset 0
  // (declared 128-B aligned): every offset above is an immediate, no run-time pointer alignment
  static constexpr size_t alloc = total;
};
#ifndef PTYCHO_TMA_BOX
#define PTYCHO_TMA_BOX 256
#endif
__host__ __device__ constexpr int tma_box(int n) { return n < PTYCHO_TMA_BOX ? n : PTYCHO_TMA_BOX; }

// The body of one pass for one group of LINES_PER_CTA lines (grp).  PERSIST = false: a
// standalone kernel in a CUDA-graph/PDL chain (tables loaded here, probe from *desc, input read
// after griddepcontrol.wait).  PERSIST = true: one step of chain_kernel (tables and twiddles
// already resident, probe passed in, input written by other CTAs before the grid barrier, read
// through L2).
// CL = true: one step of cluster_chain_kernel -- the CTA holds N/16 lines of a 16-CTA cluster as
// groups of LINES_PER_CTA lines (tid = thread index inside the group, smem = the group's region);
// the pass input is read from the CTA's own shared memory (cin: its N/16 lines) and the transposed
// output is written straight into the owning CTA's shared memory over DSMEM (cout).
template <int N, int KIND, bool PERSIST, bool TWG = false, bool CL = false, bool HALF = false>
__device__ __forceinline__ void pass_body(const PassArgs& a, const int grp, int4 pd,
                                          const float2 (&twr)[EngOf<N>::type::T * EngOf<N>::type::T == N
                                                                  ? EngOf<N>::type::E : 1],
                                          unsigned char* smem, const CUtensorMap* tmV = nullptr,
                                          const CUtensorMap* tmA = nullptr, const float2* cin = nullptr,
                                          float2* cout = nullptr) {
  using ENG = typename EngOf<N>::type;
  constexpr int P = ENG::E, Q = ENG::T, L = LINES_PER_CTA;
  constexpr Plan PL = plan_of(KIND);
  using SM = Smem<N, KIND, HALF>;
  float2* tw = (float2*)(smem + SM::tw);
  float2* ht = (float2*)(smem + SM::ht);
  const int tid = CL ? (int)(threadIdx.x % (L * Q)) : (int)threadIdx.x;
  const int lw = tid / Q, q = tid % Q;
  const int bid = 1 + lw;  // named barrier of this line (engines with T > 32)
  const unsigned long long pol = l2_stream_policy();
  const int line = grp * L + lw;
  unsigned char* lbase = smem + SM::lines + lw * SM::per_line;
  float2* ex = (float2*)lbase;
  float2* pst = (float2*)(lbase + SM::ex_b);                // prefetched stash row (GRAD)
  float* pv = (float*)(lbase + SM::ex_b + SM::st_b);        // prefetched V row / amplitude row
  float* pacc = (float*)(lbase + SM::ex_b + SM::st_b + SM::v_b);  // prefetched AccBuf row (GRAD)
  // TWG: twiddles read from the global table through L1 at every transform (no registers, no
  // shared memory) -- the 4-CTA/SM forward build
  constexpr bool TW_REG = (ENG::T * ENG::T == N) && !TWG;
  if constexpr (PERSIST) __syncthreads();  // the previous step's staging reads of smem are done

  // ---- before the grid dependency: tables, and prefetches of data written >= 2 kernels ago
  // tables: asynchronous copies (no register round trip); waited for with the other prefetches
  if constexpr (!PERSIST) {
    if constexpr (!TW_REG && !TWG)
      for (int e = tid; e < ENG::TW / 2; e += L * Q) cp_async16((float4*)tw + e, (const float4*)a.wtab + e);
    for (int e = tid; e < N / 4 + 1; e += L * Q) cp_async16((float4*)ht + e, (const float4*)a.htab + e);
  }
  cp_async_commit();  // group 1: tables
  constexpr bool FIRST = kind_first(KIND);
  // probe descriptor written >= 2 kernels ago (by the previous probe's last pass)
  if constexpr (!PERSIST && !FIRST) pd = *a.desc;
  if constexpr (!PERSIST && FIRST) {
    griddep_wait();
    griddep_launch();
    pd = *a.desc;
  }
  if (pd.x < 0) {  // inactive batch slot (CTA-uniform; no barrier has been passed)
    cp_async_wait_all();  // the table copies must land before the CTA's shared memory is released
    return;
  }
  const int i = pd.x, wy0 = pd.y, wx0 = pd.z;
  const int ax = a.s & 1;
  LineLoc LL = line_loc(a, ax, line, wy0, wx0);
  // TMA path (standalone pass kernels): one thread loads every line's V / AccBuf row segment as
  // 1-D boxes of the 3-D tensor maps -- out-of-bounds = zero fill: the zero-extension of reading
  // #12 with no bounds code -- and the stash / |y| rows as bulk copies, all on one mbarrier.  A box
  // must start on a 16-B boundary of the row (a misaligned start faults), so the boxes cover the
  // aligned superset [pos0 & ~3, (pos0 & ~3) + N + 4) (N / min(N, 256) main boxes + one 4-float
  // tail box) and the consumers read the row at a shift of pos0 & 3.  The updated V / AccBuf words
  // go back with masked st.global (a TMA store of the superset would also rewrite up to 3 voxels
  // outside win ^ R_k, which a concurrent batch slot may own).  The persistent chain keeps
  // per-element cp.async.
#ifdef PTYCHO_NO_TMA
  constexpr bool TMA = false;  // A/B build: per-element cp.async prefetch
#else
  constexpr bool TMA = !PERSIST;
#endif
  constexpr int BOX = tma_box(N), NBOX = N / BOX;
  constexpr bool NEED_V = kind_transmit(KIND) || kind_grad(KIND) || kind_recon(KIND);
#ifdef PTYCHO_STASH_STG
  constexpr bool STASH_BULK = false;
#else
  constexpr bool STASH_BULK = TMA && ENG::T * ENG::T == N;  // stash row written by one bulk copy
#endif
  unsigned long long* mbar = (unsigned long long*)(smem + SM::bar);
  const int xal = LL.pos0 & ~3;                       // 16-B aligned start of the superset
  auto lidx_of = [&](int ln) { return ax == 0 ? wy0 + ln - a.ey0 : wx0 + ln - a.ex0; };
  const int dsh = (TMA && NEED_V) ? (LL.pos0 & 3) : 0;  // shift of window position 0 in pv / pacc
  if constexpr (TMA) {
    // the first thread of every line issues its own line's copies (L issuers in parallel; one
    // issuer for the whole CTA kept the other warps waiting at the next __syncthreads)
    if (tid == 0) {
      mbar_init(mbar, L);
      fence_proxy_async();
    }
    __syncthreads();
    if (q == 0) {
      constexpr unsigned row = 4u * N + 16u;
      constexpr unsigned per = (NEED_V ? row : 0u) + (kind_grad(KIND) ? 8u * N : 0u) + (KIND == K_TURN ? 4u * N : 0u);
      const unsigned acc_bytes = (kind_grad(KIND) && SM::acc_b && !a.no_acc) ? row : 0u;
      mbar_expect_tx(mbar, per + acc_bytes);
      const int li = lidx_of(line);
      unsigned char* lb = smem + SM::lines + lw * SM::per_line;
      if constexpr (NEED_V) {
        unsigned char* d = lb + SM::ex_b + SM::st_b;
#pragma unroll
        for (int b = 0; b < NBOX; ++b) tma_load3(d + b * BOX * 4, tmV, xal + b * BOX, li, a.s >> 1, mbar, pol);
        tma_load3(d + N * 4, tmV + 4, xal + N, li, a.s >> 1, mbar, pol);  // 4-float tail box
      }
      if constexpr (kind_grad(KIND)) {
        if (SM::acc_b && !a.no_acc) {
          unsigned char* d = lb + SM::ex_b + SM::st_b + SM::v_b;
#pragma unroll
          for (int b = 0; b < NBOX; ++b) tma_load3(d + b * BOX * 4, tmA, xal + b * BOX, li, a.s >> 1, mbar, pol);
          tma_load3(d + N * 4, tmA + 4, xal + N, li, a.s >> 1, mbar, pol);
        }
        bulk_load(lb + SM::ex_b, a.stash + (size_t)a.stash_s * N * N + (size_t)line * N, 8u * N, mbar, pol);
      }
      if constexpr (KIND == K_TURN) bulk_load(lb + SM::ex_b + SM::st_b, a.amp + (size_t)i * N * N + (size_t)line * N, 4u * N, mbar, pol);
    }
  }
  if constexpr (!TMA && (kind_transmit(KIND) || kind_grad(KIND) || kind_recon(KIND))) {
    const long long so = (long long)a.s * a.slice_stride + LL.row;
    const float* vrow = a.V + so;
    const float* arow = a.acc + so;
#pragma unroll kPrefUnroll
    for (int k = 0; k < P; ++k) {
      const int j = q + Q * k, p = LL.pos0 + j;
      if (LL.ok && (unsigned)p < (unsigned)LL.plim) {
        cp_async4s(pv + j, vrow + p, pol);
        if constexpr (kind_grad(KIND) && SM::acc_b > 0) {
          if (!a.no_acc) cp_async4s(pacc + j, arow + p, pol);
        }
      } else {
        pv[j] = 0.f;
        if constexpr (kind_grad(KIND) && SM::acc_b > 0) pacc[j] = 0.f;
      }
    }
  }
  if constexpr (!TMA && kind_grad(KIND)) {
    const float4* src = (const float4*)(a.stash + (size_t)a.stash_s * N * N + (size_t)line * N);
    float4* dst = (float4*)pst;
#pragma unroll 4
    for (int c = q; c < N / 2; c += Q) cp_async16s(dst + c, src + c, pol);
  }
  if constexpr (!TMA && KIND == K_TURN) {
    const float4* src = (const float4*)(a.amp + (size_t)i * N * N + (size_t)line * N);
    float4* dst = (float4*)pv;
#pragma unroll 4
    for (int c = q; c < N / 4; c += Q) cp_async16s(dst + c, src + c, pol);
  }
  cp_async_commit();
  // the row prefetches have landed (all threads; before any read of pst / pv / pacc)
  auto prefetch_wait = [&]() {
    if constexpr (TMA) mbar_wait(mbar, 0);
    else cp_async_wait_all();
  };
  pv += dsh;    // window position j of the V / AccBuf rows (TMA superset: shifted by pos0 & 3)
  pacc += dsh;
  float2 x[P];
  if constexpr (FIRST) {
    const float2* src = a.probe + (size_t)line * N + q;
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = src[Q * k];
  } else if constexpr (!PERSIST) {
    griddep_wait();
    griddep_launch();
    const float2* src = (KIND == K_RECON_FIRST ? a.stash + (size_t)a.stash_s * N * N : a.in) + (size_t)line * N + q;
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = src[Q * k];
  } else if constexpr (CL) {
    const float2* src = cin + (size_t)(line % (N / 16)) * N + q;  // written over DSMEM by the cluster
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = src[Q * k];
  } else {
    const float2* src = a.in + (size_t)line * N + q;  // written by other SMs last step: bypass L1
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = __ldcg(src + Q * k);
  }
  if constexpr (TMA) cp_async_wait_all();  // tables landed (the TMA rows are tracked by the mbarrier)
  else asm volatile("cp.async.wait_group 1;" ::: "memory");  // tables landed (row prefetches may not have)
  __syncthreads();

  float part = 0.f;  // loss partial (RESID)
  // dist: distribution of the registers when the step runs (0 = natural D0, 1 = engine's D1)
  auto step = [&](int st, int dist) {
    if ((has_step(PL, S_HC_FWD) && st == S_HC_FWD) || (has_step(PL, S_HC_ADJ) && st == S_HC_ADJ)) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        // H_1 depends on m_u^2 only: look up min(u, N - u)
        int m;
        if constexpr (ENG::T * ENG::T == N) {  // four-step, D1 == D0: u = q + Qk
          m = k < P / 2 ? q + Q * k : Q * (P - k) - q;
        } else {
          const int u = ENG::idx(dist, q, k);
          m = u <= N / 2 ? u : N - u;
        }
        const float2 h = ht[m];
        const float2 y = x[k];
        // conj(H) conj(y) = h.x conj(y) - h.y (y.y, y.x) ;  H conj(y) = h.x conj(y) + h.y (y.y, y.x)
#ifndef PTYCHO_SCALAR_FP
        const float hy = st == S_HC_FWD ? -h.y : h.y;
        x[k] = __ffma2_rn(make_float2(y.y, y.x), make_float2(hy, hy), __fmul2_rn(make_float2(y.x, -y.y), make_float2(h.x, h.x)));
#else
        if (st == S_HC_FWD) x[k] = make_float2(h.x * y.x - h.y * y.y, -(h.x * y.y + h.y * y.x));
        else x[k] = make_float2(h.x * y.x + h.y * y.y, h.y * y.x - h.x * y.y);
#endif
      }
    } else if (has_step(PL, S_CONJ) && st == S_CONJ) {
#pragma unroll
      for (int k = 0; k < P; ++k) x[k].y = -x[k].y;
    } else if (has_step(PL, S_TRANSMIT) && st == S_TRANSMIT) {
      // phi_s = exp(i sigma V_s[win ^ R_k]) psi_s  (t = 1 outside R_k, reading #12); stash phi_s
      prefetch_wait();
      float2* stp = a.stash + (size_t)a.stash_s * N * N + (size_t)line * N + q;
      const bool keep = a.stash_store != 0;  // stash-free: only phi_{S-1} is kept
#ifndef PTYCHO_UNROLLED_STEPS
      float2* xs = ex + q;  // rolled through the idle exchange buffer (instruction-cache footprint)
#pragma unroll
      for (int k = 0; k < P; ++k) xs[Q * k] = x[k];
#ifdef PTYCHO_DEBUG_CHECKS
      {  // the V row prefetched before griddepcontrol.wait (TMA) equals V in L2 now: no stale read
        const float* vr = a.V + (long long)a.s * a.slice_stride + LL.row;
        for (int k = 0; k < P; ++k) {
          const int p = LL.pos0 + q + Q * k;
          if (LL.ok && (unsigned)p < (unsigned)LL.plim && __ldcg(vr + p) != pv[q + Q * k]) atomicOr(a.dbg, 8u);
        }
      }
#endif
      auto body = [&](auto fast) {
#pragma unroll kStepUnroll
        for (int k = 0; k < P; ++k) {
          const float v = pv[q + Q * k];
          float sn, cs;
          sincos_t<decltype(fast)::value>(a.sigma * v, &sn, &cs);
          float2 y = xs[Q * k];
          if (PL.transmit_cp) y.y = -y.y;
          const float2 phi = cmul(y, make_float2(cs, sn));
          xs[Q * k] = phi;
          if (!STASH_BULK && keep) st_stream(stp + Q * k, phi, pol);
        }
      };
      if (small_phases<P>(pv, a.sigma, [&](int k) { return q + Q * k; })) body(Bool<true>());
      else body(Bool<false>());
      if constexpr (STASH_BULK) {
        // the rolled buffer holds phi_s of this line in natural order = the stash row: one 8N-byte
        // bulk copy (cp.async.bulk shared -> global) instead of N / Q stores per thread
        if (keep) {
          fence_proxy_async();
          ENG::sync_line(bid);
          if (q == 0) {
            bulk_store(stp - q, ex, 8u * N, pol);
            bulk_commit();
          }
        }
      }
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = xs[Q * k];
      if constexpr (STASH_BULK) {
        if (keep && q == 0) bulk_wait_read();  // the next exchange overwrites the buffer
        ENG::sync_line(bid);
      }
#else
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const float v = pv[q + Q * k];
        float sn, cs;
        sincos_t<false>(a.sigma * v, &sn, &cs);
        float2 y = x[k];
        if (PL.transmit_cp) y.y = -y.y;
        x[k] = cmul(y, make_float2(cs, sn));
        if (keep) stp[Q * k] = x[k];
      }
#endif
    } else if (has_step(PL, S_RESID) && st == S_RESID) {
      // X = raw 2-D DFT (N x true F phi_{S-1}); |Psi| = |X|/N (App. A: |H| = 1)
      prefetch_wait();
      ENG::sync_line(bid);
      const float invn = 1.0f / (float)N;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const float m = sqrtf(x[k].x * x[k].x + x[k].y * x[k].y);
        const float mag = m * invn;
        const float r = mag - pv[ENG::idx(dist, q, k)];
        part += r * r;
        // chi_Psi = r Psi/|Psi| (0 where |Psi| <= thr, reading #30), /N for the two unnormalised
        // inverse line transforms; conjugated to start the inverse as conj o F o conj.
        const float sc = (mag > a.thr) ? r * invn / m : 0.f;
        x[k] = make_float2(x[k].x * sc, -x[k].y * sc);
      }
    } else if (has_step(PL, S_SIMUL) && st == S_SIMUL) {
      const float invn = 1.0f / (float)N;
      float* am = a.amp + (size_t)i * N * N + (size_t)line * N;
#pragma unroll
      for (int k = 0; k < P; ++k) am[ENG::idx(dist, q, k)] = sqrtf(x[k].x * x[k].x + x[k].y * x[k].y) * invn;
    } else if ((has_step(PL, S_RECON) && st == S_RECON) || (has_step(PL, S_RECON_T) && st == S_RECON_T)) {
      // stash-free adjoint: phi_s (conj pending after P^H, or true from the stash) -> stash ring
      // slot; psi_s = conj(t_s) phi_s with t_s from the pre-update V (the gradient pass of slice
      // s runs after this one).  Rolled through the idle exchange buffer like S_GRAD.
      prefetch_wait();
      ENG::sync_line(bid);
      float2* stp = a.stash + (size_t)a.stash_s * N * N + (size_t)line * N;
      const bool pending = (st == S_RECON);
      float2* xs = ex;
#pragma unroll
      for (int k = 0; k < P; ++k) xs[ENG::idx(dist, q, k)] = x[k];
      auto body = [&](auto fast) {
#pragma unroll kStepUnroll
        for (int k = 0; k < P; ++k) {
          const int j = ENG::idx(dist, q, k);
          float2 phi = xs[j];
          if (pending) {
            phi.y = -phi.y;
            st_stream(stp + j, phi, pol);
          }
          float sn, cs;
          sincos_t<decltype(fast)::value>(a.sigma * pv[j], &sn, &cs);
          xs[j] = cmulc(phi, make_float2(cs, sn));
        }
      };
      if (small_phases<P>(pv, a.sigma, [&](int k) { return ENG::idx(dist, q, k); })) body(Bool<true>());
      else body(Bool<false>());
#pragma unroll
      for (int k = 0; k < P; ++k) x[k] = xs[ENG::idx(dist, q, k)];
    } else if (has_step(PL, S_GRAD) && st == S_GRAD) {
      // chi_phi = conj(y).  g_s = 2 sigma Im(chi conj(phi_s)) (App. A); on win ^ R_k:
      // AccBuf += g (Alg. 1 step 7), V -= alpha g (step 8); chi <- conj(t_s) chi with t_s from
      // the PRE-update V.
      const long long so = (long long)a.s * a.slice_stride + LL.row;
      float* vrow = a.V + so;
      float* arow = a.acc + so;
      prefetch_wait();
      ENG::sync_line(bid);
      const float two_sigma = 2.0f * a.sigma;
      const bool exporting = a.gexport != nullptr;  // debug: write g instead of updating
      float* gexp = exporting ? a.gexport + (size_t)a.s * N * N : nullptr;
      const int lim = LL.ok ? LL.plim : 0;
#ifndef PTYCHO_UNROLLED_STEPS
      // Rolled over the line through the (idle) exchange buffer: the unrolled body was ~13 KB of
      // SASS, and the pass loop (transform + steps) then overflowed the 32 KB instruction cache.
      // Each thread only touches its own positions, so no synchronisation is needed.
      float2* xs = ex;
      // HALF (3-CTA/SM backward build): the exchange buffer holds half a line of complex values,
      // so the line is rolled through it in two halves of the thread's elements
      constexpr int NH = HALF ? 2 : 1, KH = P / NH;
#ifdef PTYCHO_DEBUG_CHECKS
      {  // V / AccBuf / stash rows prefetched before griddepcontrol.wait equal their L2 values now
        const float2* sr = a.stash + (size_t)a.stash_s * N * N + (size_t)line * N;
        for (int k = 0; k < P; ++k) {
          const int j = ENG::idx(dist, q, k);
          const int p = LL.pos0 + j;
          if ((unsigned)p < (unsigned)lim) {
            if (__ldcg(vrow + p) != pv[j]) atomicOr(a.dbg, 1u);
            if (SM::acc_b && !a.no_acc && __ldcg(arow + p) != pacc[j]) atomicOr(a.dbg, 2u);
          }
          const float2 sg = __ldcg(sr + j);
          if (sg.x != pst[j].x || sg.y != pst[j].y) atomicOr(a.dbg, 4u);
        }
      }
#endif
      const bool fast_phase = small_phases<P>(pv, a.sigma, [&](int k) { return ENG::idx(dist, q, k); });
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int kb = h * KH, jb = HALF ? ENG::idx(dist, 0, kb) : 0;  // EngFour: j = q + Q k
#pragma unroll
        for (int k = kb; k < kb + KH; ++k) xs[ENG::idx(dist, q, k) - jb] = x[k];
        auto body = [&](auto fast) {
#pragma unroll kStepUnroll
          for (int k = kb; k < kb + KH; ++k) {
            const int j = ENG::idx(dist, q, k);
            const int p = LL.pos0 + j;
            const float2 ph = pst[j];
            const float2 y = xs[j - jb];
            const float2 chi = make_float2(y.x, -y.y);
            const float g = two_sigma * (chi.y * ph.x - chi.x * ph.y);
            const float v = pv[j];
            if (!exporting && (unsigned)p < (unsigned)lim) {
              if constexpr (SM::acc_b > 0) {
                if (!a.no_acc) st_stream(arow + p, pacc[j] + g, pol);
              } else {
                if (!a.no_acc) red_add_stream(arow + p, g, pol);
              }
              st_stream(vrow + p, v - a.alpha * g, pol);
            }
            if (exporting) gexp[ax == 0 ? (size_t)line * N + j : (size_t)j * N + line] = g;  // debug: g itself
            float sn, cs;
            sincos_t<decltype(fast)::value>(a.sigma * v, &sn, &cs);
            xs[j - jb] = cmulc(chi, make_float2(cs, sn));
          }
        };
        if (fast_phase) body(Bool<true>());
        else body(Bool<false>());
#pragma unroll
        for (int k = kb; k < kb + KH; ++k) x[k] = xs[ENG::idx(dist, q, k) - jb];
      }
#else
#pragma unroll
      for (int k = 0; k < P; ++k) {
        if ((k & 7) == 0) asm volatile("" ::: "memory");
        const int j = ENG::idx(dist, q, k);
        const int p = LL.pos0 + j;
        const float2 ph = pst[j];
        const float2 chi = make_float2(x[k].x, -x[k].y);
        const float g = two_sigma * (chi.y * ph.x - chi.x * ph.y);
        const float v = pv[j];
        if (!exporting && (unsigned)p < (unsigned)lim) {
          if (!a.no_acc) red_add_stream(arow + p, g, pol);
          vrow[p] = v - a.alpha * g;
        }
        if (exporting) gexp[ax == 0 ? (size_t)line * N + j : (size_t)j * N + line] = g;
        float sn, cs;
        sincos_t<false>(a.sigma * v, &sn, &cs);
        x[k] = cmulc(chi, make_float2(cs, sn));
      }
#endif

    }
  };

#pragma unroll 1
  for (int f = 0; f < PL.nf; ++f) {
    int st = PL.pre[0];
    if (f == 1) st = PL.pre[1];
    if (f == 2) st = PL.pre[2];
    if (f == 3) st = PL.pre[3];
    step(st, f & 1);
    if constexpr (HALF) {
      ENG::fft_rh(x, (float*)ex, q, twr);
    } else if constexpr (TW_REG) {
      ENG::fft_r(x, ex, q, twr);
    } else {
      const float2* twp = TWG ? a.wtab : tw;
      if (f & 1) ENG::dif(x, ex, q, twp, bid);
      else ENG::dit(x, ex, q, twp, bid);
    }
  }
  step(PL.post, PL.nf & 1);
  constexpr int DIST_OUT = PL.nf & 1;

  if constexpr (KIND == K_TURN) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    float* red = (float*)(smem + SM::red);  // LINES_PER_CTA * Q / 32 <= 16 floats
    static_assert(LINES_PER_CTA * Q / 32 + 1 <= 16, "red");
    if ((tid & 31) == 0) red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < (L * Q + 31) / 32; ++w) tot += (double)red[w];
      a.loss_part[grp] += tot;
    }
  }

  if constexpr (PL.store_conj) {
#pragma unroll
    for (int k = 0; k < P; ++k) x[k].y = -x[k].y;
  }
  constexpr int STORE = kind_store(KIND);
  if constexpr (STORE == 1) {
    // out[j][line]: stage the CTA's L = 4 lines as 32-B rows [j][4] (element l stored at
    // l ^ ((j >> 2) & 3): conflict-free column writes), then write 16-B chunks of each output
    // row segment (L consecutive complex64 = one 32-B sector).
    static_assert(L == 4, "staging assumes 4 lines per CTA");
    __syncthreads();
    float2* stg = (float2*)(smem + SM::lines);
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = ENG::idx(DIST_OUT, q, k);
      stg[j * 4 + (lw ^ ((j >> 2) & 3))] = x[k];
    }
    __syncthreads();
    float2* dst = a.out + (size_t)grp * L;
#pragma unroll kStoreUnroll
    for (int e = tid; e < N * 2; e += L * Q) {
      const int j = e >> 1, c = e & 1, sw = (j >> 2) & 3;
      float4 v = *(const float4*)(stg + j * 4 + 2 * c);
      if (sw & 1) v = make_float4(v.z, v.w, v.x, v.y);
      if constexpr (CL) {  // next pass's line j lives in cluster CTA j / (N/16), row j % (N/16)
        const float2* loc = cout + (size_t)(j % (N / 16)) * N + grp * L + 2 * (c ^ (sw >> 1));
        st_cluster_v4(loc, (unsigned)(j / (N / 16)), v);
      } else {
        *(float4*)(dst + (size_t)j * N + 2 * (c ^ (sw >> 1))) = v;
      }
    }
  }
  if constexpr (STORE == 2) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = ENG::idx(DIST_OUT, q, k);
      const size_t o = a.natural_transposed ? (size_t)j * N + line : (size_t)line * N + j;
      a.natural_out[o] = x[k];
    }
  }

  if constexpr (STASH_BULK && kind_transmit(KIND)) {
    if (q == 0 && a.stash_store) bulk_wait();  // the stash row is in global memory before the CTA retires
  }
  if (!PERSIST && a.advance) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(a.done, 1u);
      if (prev == gridDim.x - 1) {  // every CTA has read *desc: advance to the next probe
        *a.done = 0u;
        const int nx = pd.x + 1 < a.n_probes ? pd.x + 1 : pd.x;
        const int2 c = a.centers[nx];
        *a.desc = make_int4(pd.x + 1, c.x - N / 2, c.y - N / 2, 0);
        __threadfence();
      }
    }
  }
}

// MINB: CTAs per SM the register allocation must allow.  2: the single-chain-latency build
// (a probe chain alone on the GPU: 2.67 ms/probe at N = 1024, S = 100); 3: forward passes at
// <= 168 registers leave room for CTAs of other tiles' chains (2 chains +4 %, 8 tiles +6 %
// probes/s, but a lone chain runs 12 % slower).  The host picks per context (api.cu).  Backward
// passes always use 2 (they spill at 168).  Both builds execute the same arithmetic.
// HALF_BWD (opt-in, -DPTYCHO_BWD3=1): backward passes of the multi-chain build (MINB >= 3) at
// N = 1024 at 3 CTAs/SM -- half-size exchange buffer (exchange_half), AccBuf by red.global.add and
// the gradient step rolled in two halves bring the CTA to 72 KB of shared memory and 168
// registers.  Bit-identical, but measured 2 % slower than 2 CTAs/SM (548 vs 560 probe-loc/s,
// profiles/round2/ab_bwd3.txt): the extra warps do not pay for the second exchange round and
// the register cap.
#ifndef PTYCHO_BWD3
#define PTYCHO_BWD3 0
#endif
template <int N, int KIND, int MINB>
__host__ __device__ constexpr bool half_bwd() {
  return PTYCHO_BWD3 && kind_grad(KIND) && MINB >= 3 && N == 1024 && EngOf<N>::type::T * EngOf<N>::type::T == N;
}
template <int N, int KIND, int MINB>
__global__ void __launch_bounds__(LINES_PER_CTA * EngThreads<N>::v,
                                  kind_grad(KIND) ? (half_bwd<N, KIND, MINB>() ? 3 : 2) : MINB)
pass_kernel(const PassArgs a) {
  using ENG = typename EngOf<N>::type;
  constexpr int P = ENG::E, Q = ENG::T;
  constexpr bool HB = half_bwd<N, KIND, MINB>();
  constexpr bool TWG = MINB >= 4 && !kind_grad(KIND) && ENG::T * ENG::T == N;
  constexpr bool TW_REG = (ENG::T * ENG::T == N) && !TWG;
  extern __shared__ __align__(128) unsigned char smem[];
  const int q = threadIdx.x % Q;
  // four-step engines keep the thread's twiddles in registers (no shared-memory table)
  float2 twr[ENG::T * ENG::T == N ? P : 1];
  if constexpr (TW_REG) {
#pragma unroll
    for (int k = 0; k < P; ++k) twr[k] = __ldg(a.wtab + k * Q + q);
  }
  // batched schedule: CTA block b of N/L lines serves batch slot b (its own stash, wavefields,
  // probe descriptor and loss partials)
  constexpr int groups = N / LINES_PER_CTA;
  const int b = blockIdx.x / groups, grp = blockIdx.x - b * groups;
  if (b == 0) {
    pass_body<N, KIND, false, TWG, false, HB>(a, grp, make_int4(0, 0, 0, 0), twr, smem, a.tmV, a.tmA);
  } else {
    PassArgs ab = a;
    ab.stash += b * a.stash_slot;
    ab.in += b * a.wf_slot;
    ab.out += b * a.wf_slot;
    ab.desc += b;
    ab.loss_part += b * groups;
    pass_body<N, KIND, false, TWG, false, HB>(ab, grp, make_int4(0, 0, 0, 0), twr, smem, a.tmV, a.tmA);
  }
}

// ------------------------------------------------------------------------------------------
// Persistent chain kernel: the probe chains of a pass segment for all local tiles in one
// cooperative launch.  Every grid step runs one pass index (all tiles in lockstep), the CTAs
// sweep the (tile, line group) items statically, and a grid barrier separates the steps (the
// next pass reads the transposed wavefield every CTA wrote).  The barrier's gpu-scope fence
// also invalidates L1 (CCTL.IVALL), so V/AccBuf rows written by other SMs are never read stale.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    const unsigned long long t0 = globaltimer();
    while (ld_acquire(bar) < target) {
      __nanosleep(32);
      if (globaltimer() - t0 > 20000000000ull) __trap();  // 20 s: never hang the device
    }
    __threadfence();
  }
  __syncthreads();
}

__host__ __device__ constexpr int chain_kind(int p, int S) {
  return S == 1 ? (p == 0 ? K_FWD_FIRST_FFT : (p == 1 ? K_TURN : K_BWD_LAST_END))
                : (p == 0 ? K_FWD_FIRST_PROP
                          : (p < S - 1 ? K_FWD_MID
                                       : (p == S - 1 ? K_FWD_LAST
                                                     : (p == S ? K_TURN
                                                               : (p == S + 1 ? K_BWD_LAST_PROP
                                                                             : (p < 2 * S ? K_BWD_MID : K_BWD_END))))));
}
__host__ __device__ constexpr int chain_slice(int p, int S) { return p < S ? p : (p == S ? S : 2 * S - p); }

template <int N>
__global__ void __launch_bounds__(LINES_PER_CTA * EngThreads<N>::v, 2) chain_kernel(const ChainArgs c) {
  using ENG = typename EngOf<N>::type;
  constexpr int P = ENG::E, Q = ENG::T, L = LINES_PER_CTA;
  constexpr bool TW_REG = (ENG::T * ENG::T == N);
  extern __shared__ __align__(128) unsigned char smem[];
  const int q = threadIdx.x % Q;
  float2 twr[TW_REG ? P : 1];
  if constexpr (TW_REG) {
#pragma unroll
    for (int k = 0; k < P; ++k) twr[k] = __ldg(c.t[0].wtab + k * Q + q);
  } else {
    for (int e = threadIdx.x; e < ENG::TW; e += L * Q) ((float2*)smem)[e] = c.t[0].wtab[e];
  }
  {  // H_1/N table (same offset for every pass kind)
    float2* ht = (float2*)(smem + Smem<N, K_FWD_MID>::ht);
    for (int e = threadIdx.x; e <= N / 2; e += L * Q) ht[e] = c.t[0].htab[e];
  }
  const int S = c.S, groups = N / L, items = c.ntiles * groups;
  unsigned target = 0;
  for (int j = 0; j < c.maxn; ++j) {
    for (int pp = 0; pp < 2 * S + 1; ++pp) {
      const int kind = chain_kind(pp, S), sl = chain_slice(pp, S);
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        const int tl = it / groups, grp = it - tl * groups;
        if (j >= c.count[tl]) continue;  // block-uniform
        PassArgs a = c.t[tl];
        a.s = sl;
        a.stash_s = sl;
        a.stash_store = 1;
        a.in = pp == 0 ? a.probe : c.wf[tl][pp & 1];
        a.out = c.wf[tl][(pp + 1) & 1];
        const int pi = c.first + j;
        const int2 ctr = a.centers[pi];
        const int4 pd = make_int4(pi, ctr.x - N / 2, ctr.y - N / 2, 0);
        switch (kind) {
          case K_FWD_FIRST_PROP: pass_body<N, K_FWD_FIRST_PROP, true>(a, grp, pd, twr, smem); break;
          case K_FWD_FIRST_FFT: pass_body<N, K_FWD_FIRST_FFT, true>(a, grp, pd, twr, smem); break;
          case K_FWD_MID: pass_body<N, K_FWD_MID, true>(a, grp, pd, twr, smem); break;
          case K_FWD_LAST: pass_body<N, K_FWD_LAST, true>(a, grp, pd, twr, smem); break;
          case K_TURN: pass_body<N, K_TURN, true>(a, grp, pd, twr, smem); break;
          case K_BWD_LAST_PROP: pass_body<N, K_BWD_LAST_PROP, true>(a, grp, pd, twr, smem); break;
          case K_BWD_LAST_END: pass_body<N, K_BWD_LAST_END, true>(a, grp, pd, twr, smem); break;
          case K_BWD_MID: pass_body<N, K_BWD_MID, true>(a, grp, pd, twr, smem); break;
          default: pass_body<N, K_BWD_END, true>(a, grp, pd, twr, smem); break;
        }
      }
      target += gridDim.x;
      grid_barrier(c.bar, target);
    }
  }
}

template <int N>
__host__ __device__ constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
template <int N>
__host__ __device__ constexpr size_t chain_smem_max() {
  return cmax<N>(cmax<N>(cmax<N>(Smem<N, K_FWD_FIRST_PROP>::alloc, Smem<N, K_FWD_FIRST_FFT>::alloc),
                         cmax<N>(Smem<N, K_FWD_MID>::alloc, Smem<N, K_FWD_LAST>::alloc)),
                 cmax<N>(cmax<N>(Smem<N, K_TURN>::alloc, Smem<N, K_BWD_LAST_PROP>::alloc),
                         cmax<N>(cmax<N>(Smem<N, K_BWD_LAST_END>::alloc, Smem<N, K_BWD_MID>::alloc),
                                 Smem<N, K_BWD_END>::alloc)));
}
template <int N>
static size_t chain_smem() {
  size_t m = 0;
  const size_t v[] = {Smem<N, K_FWD_FIRST_PROP>::alloc, Smem<N, K_FWD_FIRST_FFT>::alloc, Smem<N, K_FWD_MID>::alloc,
                      Smem<N, K_FWD_LAST>::alloc,       Smem<N, K_TURN>::alloc,          Smem<N, K_BWD_LAST_PROP>::alloc,
                      Smem<N, K_BWD_LAST_END>::alloc,   Smem<N, K_BWD_MID>::alloc,       Smem<N, K_BWD_END>::alloc};
  for (size_t x : v) m = x > m ? x : m;
  return m;
}

template <int N>
static cudaError_t launch_chain_n(const ChainArgs& c, cudaStream_t stream) {
  auto kern = chain_kernel<N>;
  const size_t smem = chain_smem<N>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = LINES_PER_CTA * EngThreads<N>::v;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem);
  if (e != cudaSuccess) return e;
  if (per < 1) return cudaErrorCooperativeLaunchTooLarge;
  int grid = per * sms;
  const int items = c.ntiles * (N / LINES_PER_CTA);
  if (grid > items) grid = items;
  void* args[] = {(void*)&c};
  return cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(threads), args, smem, stream);
}

cudaError_t launch_chain(int n, const ChainArgs& c, cudaStream_t stream) {
  switch (n) {
    case 64: return launch_chain_n<64>(c, stream);
    case 256: return launch_chain_n<256>(c, stream);
    case 1024: return launch_chain_n<1024>(c, stream);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------
// Cluster-resident chain for N <= 256 (SURVEY §7 phase 7): one 16-CTA cluster per tile runs the
// whole probe chain of a pass segment in one launch.  The N x N wavefield never leaves the
// cluster: CTA r holds lines [r N/16, (r+1) N/16) in shared memory (double buffered), each pass
// writes its transposed output straight into the owning CTA's buffer over DSMEM, and a cluster
// barrier replaces the kernel boundary of the graph + PDL chain (whose launch / prologue /
// grid-completion latency dominates the small passes: 3.9 us per N = 256 pass).  The arithmetic
// of every pass is pass_body's, so results are bit-identical to the standalone chain.
// ------------------------------------------------------------------------------------------
template <int N>
struct ClusterLayout {
  static constexpr int LPC = N / 16;                    // lines per CTA
  static constexpr int G = LPC / LINES_PER_CTA;         // pass_body groups per CTA
  static constexpr int TPG = LINES_PER_CTA * EngThreads<N>::v;
  static constexpr size_t wbuf = (size_t)LPC * N * 8;   // one wavefield buffer (bytes)
  static constexpr size_t group = (chain_smem_max<N>() + 127) / 128 * 128;
  static constexpr size_t total = 2 * wbuf + G * group;
};

template <int N>
__global__ void __launch_bounds__(ClusterLayout<N>::G * ClusterLayout<N>::TPG, 1) cluster_chain_kernel(const ChainArgs c) {
  using CLY = ClusterLayout<N>;
  using ENG = typename EngOf<N>::type;
  constexpr int P = ENG::E, Q = ENG::T;
  static_assert(ENG::T * ENG::T == N, "four-step engine (twiddles in registers)");
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned rank = cluster_ctarank();
  const int tl = blockIdx.x / 16;
  const int g = threadIdx.x / CLY::TPG, tid = threadIdx.x % CLY::TPG, q = tid % Q;
  unsigned char* gsm = smem + 2 * CLY::wbuf + g * CLY::group;
  float2* wb[2] = {(float2*)smem, (float2*)(smem + CLY::wbuf)};
  const PassArgs& a0 = c.t[tl];
  float2 twr[P];
#pragma unroll
  for (int k = 0; k < P; ++k) twr[k] = __ldg(a0.wtab + k * Q + q);
  {
    float2* ht = (float2*)(gsm + Smem<N, K_FWD_MID>::ht);
    for (int e = tid; e <= N / 2; e += CLY::TPG) ht[e] = a0.htab[e];
  }
  __syncthreads();
  PassArgs a = a0;
  const int S = c.S, cnt = c.count[tl];
  const int grp = (int)rank * CLY::G + g;
  for (int j = 0; j < cnt; ++j) {
    const int pi = c.first + j;
    const int2 ctr = a.centers[pi];
    const int4 pd = make_int4(pi, ctr.x - N / 2, ctr.y - N / 2, 0);
    for (int pp = 0; pp < 2 * S + 1; ++pp) {
      const int kind = chain_kind(pp, S), sl = chain_slice(pp, S);
      a.s = sl;
      a.stash_s = sl;
      a.stash_store = 1;
      const float2* cin = wb[pp & 1];
      float2* cout = wb[(pp + 1) & 1];
      switch (kind) {
        case K_FWD_FIRST_PROP: pass_body<N, K_FWD_FIRST_PROP, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_FWD_FIRST_FFT: pass_body<N, K_FWD_FIRST_FFT, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_FWD_MID: pass_body<N, K_FWD_MID, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_FWD_LAST: pass_body<N, K_FWD_LAST, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_TURN: pass_body<N, K_TURN, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_BWD_LAST_PROP: pass_body<N, K_BWD_LAST_PROP, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_BWD_LAST_END: pass_body<N, K_BWD_LAST_END, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        case K_BWD_MID: pass_body<N, K_BWD_MID, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
        default: pass_body<N, K_BWD_END, true, false, true>(a, grp, pd, twr, gsm, nullptr, nullptr, cin, cout); break;
      }
      cluster_sync_all();
    }
  }
}

template <int N>
static cudaError_t launch_cluster_n(const ChainArgs& c, cudaStream_t stream) {
  using CLY = ClusterLayout<N>;
  auto kern = cluster_chain_kernel<N>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CLY::total);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16 * c.ntiles);
  cfg.blockDim = dim3(CLY::G * CLY::TPG);
  cfg.dynamicSmemBytes = CLY::total;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 16;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, c);
}

cudaError_t launch_cluster(int n, const ChainArgs& c, cudaStream_t stream) {
  switch (n) {
    case 64: return launch_cluster_n<64>(c, stream);
    case 256: return launch_cluster_n<256>(c, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int N, int KIND, int MINB>
static cudaError_t launch_one(const PassArgs& a, cudaStream_t stream, bool pdl) {
  auto kern = pass_kernel<N, KIND, MINB>;
  const size_t smem = Smem<N, KIND, half_bwd<N, KIND, MINB>()>::alloc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((N / LINES_PER_CTA) * (a.batch > 1 ? a.batch : 1));
  cfg.blockDim = dim3(LINES_PER_CTA * EngOf<N>::type::T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int N, int MINB>
static cudaError_t launch_pass_nm(PassKind kind, const PassArgs& a, cudaStream_t s, bool pdl) {
  switch (kind) {
    case K_FWD_FIRST_PROP: return launch_one<N, K_FWD_FIRST_PROP, MINB>(a, s, pdl);
    case K_FWD_FIRST_FFT: return launch_one<N, K_FWD_FIRST_FFT, MINB>(a, s, pdl);
    case K_FWD_MID: return launch_one<N, K_FWD_MID, MINB>(a, s, pdl);
    case K_FWD_LAST: return launch_one<N, K_FWD_LAST, MINB>(a, s, pdl);
    case K_TURN: return launch_one<N, K_TURN, MINB>(a, s, pdl);
    case K_SIMULATE: return launch_one<N, K_SIMULATE, MINB>(a, s, pdl);
    case K_BWD_LAST_PROP: return launch_one<N, K_BWD_LAST_PROP, (MINB >= 3 ? 3 : 2)>(a, s, pdl);
    case K_BWD_LAST_END: return launch_one<N, K_BWD_LAST_END, (MINB >= 3 ? 3 : 2)>(a, s, pdl);
    case K_BWD_MID: return launch_one<N, K_BWD_MID, (MINB >= 3 ? 3 : 2)>(a, s, pdl);
    case K_BWD_END: return launch_one<N, K_BWD_END, (MINB >= 3 ? 3 : 2)>(a, s, pdl);
    case K_EXIT_COMPLETE: return launch_one<N, K_EXIT_COMPLETE, MINB>(a, s, pdl);
    case K_RECON_FIRST: return launch_one<N, K_RECON_FIRST, MINB>(a, s, pdl);
    case K_RECON_MID: return launch_one<N, K_RECON_MID, MINB>(a, s, pdl);
    case K_RECON_END: return launch_one<N, K_RECON_END, MINB>(a, s, pdl);
    default: return cudaErrorInvalidValue;
  }
}

template <int N>
static cudaError_t launch_pass_n(PassKind kind, const PassArgs& a, cudaStream_t s, bool pdl) {
#ifndef PTYCHO_FWD_MINB
#define PTYCHO_FWD_MINB 3
#endif
  return a.high_occupancy ? launch_pass_nm<N, PTYCHO_FWD_MINB>(kind, a, s, pdl) : launch_pass_nm<N, 2>(kind, a, s, pdl);
}

cudaError_t launch_pass(int n, PassKind kind, const PassArgs& a, cudaStream_t stream, bool pdl) {
  switch (n) {
    case 64: return launch_pass_n<64>(kind, a, stream, pdl);
    case 256: return launch_pass_n<256>(kind, a, stream, pdl);
    case 1024: return launch_pass_n<1024>(kind, a, stream, pdl);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------------------------
// Region / elementwise helpers (APPP passes, accumulated step, layout transforms)
// ------------------------------------------------------------------------------------------

// dst[z][r][c] (op)= src[z][r][c], strided rows; grid (ceil(cols/128), rows, nslices)
// Each thread moves COPY_U elements of one row (loads first, then the stores: COPY_U independent
// loads in flight per thread -- what a peer (NVLink) source needs to approach link bandwidth).
constexpr int COPY_U = 4;
__global__ void __launch_bounds__(256) copy2d_kernel(float* __restrict__ dst, long long dld, long long dss,
                                                     const float* __restrict__ src, long long sld, long long sss,
                                                     int rows, int cols, int op) {
  const int r = blockIdx.y;
  const long long z = blockIdx.z;
  float* d = dst + z * dss + (long long)r * dld;
  const float* s = src + z * sss + (long long)r * sld;
  const int c0 = blockIdx.x * (256 * COPY_U) + threadIdx.x;
  float v[COPY_U];
#pragma unroll
  for (int u = 0; u < COPY_U; ++u) {
    const int c = c0 + 256 * u;
    v[u] = c < cols ? s[c] : 0.f;
  }
#pragma unroll
  for (int u = 0; u < COPY_U; ++u) {
    const int c = c0 + 256 * u;
    if (c < cols) {
      if (op == 0) d[c] = v[u];
      else d[c] += v[u];
    }
  }
}

// The same with 16-B accesses (rows 16-B aligned, pitches multiples of 4 floats): 4x fewer
// requests -- what matters when src is a peer's AccBuf read over NVLink (APPP P2P transport);
// the row tail (cols % 4) is moved by the first CTA of the row.
__global__ void __launch_bounds__(256) copy2d_v4_kernel(float* __restrict__ dst, long long dld, long long dss,
                                                        const float* __restrict__ src, long long sld, long long sss,
                                                        int rows, int cols, int op) {
  const int r = blockIdx.y;
  const long long z = blockIdx.z;
  float* d = dst + z * dss + (long long)r * dld;
  const float* s = src + z * sss + (long long)r * sld;
  const int c4 = cols >> 2;
  const int i0 = blockIdx.x * (256 * COPY_U) + threadIdx.x;
  float4 v[COPY_U];
#pragma unroll
  for (int u = 0; u < COPY_U; ++u) {
    const int i = i0 + 256 * u;
    v[u] = i < c4 ? ((const float4*)s)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < COPY_U; ++u) {
    const int i = i0 + 256 * u;
    if (i < c4) {
      float4* dp = (float4*)d + i;
      if (op == 0) {
        *dp = v[u];
      } else {
        float4 o = *dp;
        o.x += v[u].x;
        o.y += v[u].y;
        o.z += v[u].z;
        o.w += v[u].w;
        *dp = o;
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < (cols & 3)) {
    const int c = (c4 << 2) + threadIdx.x;
    if (op == 0) d[c] = s[c];
    else d[c] += s[c];
  }
}

cudaError_t launch_copy2d(float* dst, long long dld, long long dss, const float* src, long long sld,
                          long long sss, int rows, int cols, int nslices, int op, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0 || nslices <= 0) return cudaSuccess;
  const bool v4 = (((uintptr_t)dst | (uintptr_t)src) & 15) == 0 && ((dld | sld | dss | sss) & 3) == 0 && cols >= 4;
  if (v4) {
    for (int z0 = 0; z0 < nslices; z0 += 65535) {
      const int nz = nslices - z0 < 65535 ? nslices - z0 : 65535;
      for (int r0 = 0; r0 < rows; r0 += 65535) {
        const int nr = rows - r0 < 65535 ? rows - r0 : 65535;
        dim3 grid(((cols >> 2) + 256 * COPY_U - 1) / (256 * COPY_U), nr, nz);
        copy2d_v4_kernel<<<grid, 256, 0, stream>>>(dst + z0 * dss + (long long)r0 * dld, dld, dss,
                                                   src + z0 * sss + (long long)r0 * sld, sld, sss, nr, cols, op);
      }
    }
    return cudaGetLastError();
  }
  for (int z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = nslices - z0 < 65535 ? nslices - z0 : 65535;
    for (int r0 = 0; r0 < rows; r0 += 65535) {
      const int nr = rows - r0 < 65535 ? rows - r0 : 65535;
      dim3 grid((cols + 256 * COPY_U - 1) / (256 * COPY_U), nr, nz);
      copy2d_kernel<<<grid, 256, 0, stream>>>(dst + z0 * dss + (long long)r0 * dld, dld, dss,
                                              src + z0 * sss + (long long)r0 * sld, sld, sss, nr, cols, op);
    }
  }
  return cudaGetLastError();
}

// dst[z][r][c] (op)= src[z][c][r]; dst has rows x cols.  32x32 tiles through shared memory.
__global__ void transpose2d_kernel(float* __restrict__ dst, long long dld, long long dss,
                                   const float* __restrict__ src, long long sld, long long sss, int rows,
                                   int cols, int op) {
  __shared__ float t[32][33];
  const long long z = blockIdx.z;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const float* s = src + z * sss;
  float* d = dst + z * dss;
  // read src rows c0.. (src[c][r]) coalesced along r
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (c < cols && r < rows) t[k][threadIdx.x] = s[(long long)c * sld + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) {
      const float v = t[threadIdx.x][k];
      if (op == 0) d[(long long)r * dld + c] = v;
      else d[(long long)r * dld + c] += v;
    }
  }
}

cudaError_t launch_transpose2d(float* dst, long long dld, long long dss, const float* src, long long sld,
                               long long sss, int rows, int cols, int nslices, int op, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0 || nslices <= 0) return cudaSuccess;
  for (int z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = nslices - z0 < 65535 ? nslices - z0 : 65535;
    dim3 grid((cols + 31) / 32, (rows + 31) / 32, nz);
    transpose2d_kernel<<<grid, dim3(32, 8), 0, stream>>>(dst + z0 * dss, dld, dss, src + z0 * sss, sld, sss,
                                                          rows, cols, op);
  }
  return cudaGetLastError();
}

// Alg. 1 steps 14-16: V -= alpha_acc * AccBuf ; AccBuf = 0 (float4, grid-stride)
__global__ void acc_step_kernel(float4* __restrict__ v, float4* __restrict__ acc, long long n4, float alpha) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 a = acc[i], x = v[i];
    x.x -= alpha * a.x;
    x.y -= alpha * a.y;
    x.z -= alpha * a.z;
    x.w -= alpha * a.w;
    v[i] = x;
    acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

cudaError_t launch_acc_step(float* V, float* acc, long long n, float alpha, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const long long n4 = n / 4;  // n is a multiple of 32 (slice_stride padding)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long blocks = (n4 + 255) / 256;
  if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
  acc_step_kernel<<<(unsigned)blocks, 256, 0, stream>>>((float4*)V, (float4*)acc, n4, alpha);
  return cudaGetLastError();
}

// measurement store: out[c][a][b] = f(src[c][.][.]) with optional ifftshift, sqrt, transpose
__global__ void amp_load_kernel(float* __restrict__ dst, const float* __restrict__ src, int n, int shift,
                                int intensity, int transpose) {
  const long long c = blockIdx.y;
  const int a = blockIdx.x;  // output row
  const float* s = src + c * n * n;
  float* d = dst + c * n * n + (long long)a * n;
  for (int b = threadIdx.x; b < n; b += blockDim.x) {
    int ky = transpose ? b : a, kx = transpose ? a : b;  // output (a,b) <- natural (ky,kx)
    if (shift) {
      ky = (ky + n / 2) & (n - 1);
      kx = (kx + n / 2) & (n - 1);
    }
    float v = s[(long long)ky * n + kx];
    if (intensity) v = sqrtf(fmaxf(v, 0.f));
    d[b] = v;
  }
}

cudaError_t launch_amp_load(float* dst, const float* src, int count, int n, int shift, int intensity,
                            int transpose, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  for (int c0 = 0; c0 < count; c0 += 65535) {
    const int nc = count - c0 < 65535 ? count - c0 : 65535;
    amp_load_kernel<<<dim3(n, nc), 256, 0, stream>>>(dst + (long long)c0 * n * n, src + (long long)c0 * n * n, n,
                                                     shift, intensity, transpose);
  }
  return cudaGetLastError();
}

__global__ void set_batch_kernel(int4* desc, const int2* centers, const int* list, int cnt, int batch, int n) {
  const int b = threadIdx.x;
  if (b >= batch) return;
  if (b < cnt) {
    const int v = list[b];
    const int2 c = centers[v];
    desc[b] = make_int4(v, c.x - n / 2, c.y - n / 2, 0);
  } else {
    desc[b] = make_int4(-1, 0, 0, 0);
  }
}

cudaError_t launch_set_batch(int4* desc, const int2* centers, const int* list, int cnt, int batch, int n,
                             cudaStream_t stream) {
  set_batch_kernel<<<1, ((batch + 31) / 32) * 32, 0, stream>>>(desc, centers, list, cnt, batch, n);
  return cudaGetLastError();
}

__global__ void set_desc_kernel(int4* desc, const int2* centers, int v, int nk, int n) {
  const int j = v < nk ? v : (nk > 0 ? nk - 1 : 0);
  const int2 c = centers[j];
  *desc = make_int4(v, c.x - n / 2, c.y - n / 2, 0);
}

cudaError_t launch_set_desc(int4* desc, const int2* centers, int v, int nk, int n, cudaStream_t stream) {
  set_desc_kernel<<<1, 1, 0, stream>>>(desc, centers, v, nk, n);
  return cudaGetLastError();
}

__global__ void fill_kernel(float* p, long long n, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

cudaError_t launch_fill(float* p, long long n, float v, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  fill_kernel<<<(unsigned)blocks, 256, 0, stream>>>(p, n, v);
  return cudaGetLastError();
}

// Host -> device upload through the device alias of pinned host memory (PCIe reads by a few
// CTAs, 64 B per thread in flight): the asynchronous measurement load uses it instead of copy-engine
// copies, whose completion events the chains' cross-stream waits observe late (DESIGN.md §8 e2e).
__global__ void __launch_bounds__(1024) upload_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                                      long long n4) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}

cudaError_t launch_upload(float* dst, const float* src, long long n, int ctas, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  upload_kernel<<<ctas, 1024, 0, stream>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst),
                                           n / 4);
  return cudaGetLastError();
}

// deterministic fixed-order sum of the per-CTA loss partials
__global__ void sum_double_kernel(const double* parts, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += parts[i];
    *out = t;
  }
}

cudaError_t launch_sum_double(const double* parts, int n, double* out, cudaStream_t stream) {
  sum_double_kernel<<<1, 32, 0, stream>>>(parts, n, out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// APPP peer-to-peer transport (SURVEY §8(e) "fused"): the receiver's copy kernel reads the
// sender's AccBuf region straight from peer memory over NVLink (CUDA IPC mapping) and adds or
// copies it in place -- no pack, no staging buffer, no NCCL.  One flag pair per hop orders the
// two ranks: READY (sender -> receiver: the region is final) and DONE (receiver -> sender: the
// region has been read, the sender may overwrite it).  Flags carry the APPP call's epoch, so they
// never need resetting.  System-scope release/acquire.  A wait that exceeds timeout_ns (0 = no
// limit; PTYCHO_P2P_TIMEOUT_S, default 600 s) does not trap: it raises *err (pinned host memory,
// mapped) and returns, the host reports PTYCHO_ECUDA at its next synchronisation point, and the
// peer's context stays usable (a trap poisons the context of a rank that merely waited
// for a straggler).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const unsigned* flag, unsigned epoch, unsigned long long timeout_ns,
                                           unsigned* err) {
  const unsigned long long t0 = globaltimer();
  while ((int)(ld_acquire_sys(flag) - epoch) < 0) {
    __nanosleep(64);
    if (timeout_ns && globaltimer() - t0 > timeout_ns) {
      if (err) atomicExch_system(err, 1u);
      return;
    }
  }
}

// sender: publish "region final" to the receiver, then wait until the receiver has read it
__global__ void p2p_signal_kernel(unsigned* remote_ready, unsigned epoch, const unsigned* local_done,
                                  unsigned long long timeout_ns, unsigned* err) {
  __threadfence_system();  // AccBuf writes of the preceding kernels (stream order) before READY
  st_release_sys(remote_ready, epoch);
  spin_until(local_done, epoch, timeout_ns, err);
}
// receiver: wait for READY (the copy kernel that follows on the stream then reads peer memory)
__global__ void p2p_wait_kernel(const unsigned* local_ready, unsigned epoch, unsigned long long timeout_ns,
                                unsigned* err) {
  spin_until(local_ready, epoch, timeout_ns, err);
}
// receiver: after the copy kernel, tell the sender its region may be overwritten
__global__ void p2p_post_kernel(unsigned* remote_done, unsigned epoch) {
  __threadfence_system();
  st_release_sys(remote_done, epoch);
}

cudaError_t launch_p2p_signal(unsigned* remote_ready, unsigned epoch, const unsigned* local_done,
                              unsigned long long timeout_ns, unsigned* err, cudaStream_t s) {
  p2p_signal_kernel<<<1, 1, 0, s>>>(remote_ready, epoch, local_done, timeout_ns, err);
  return cudaGetLastError();
}
cudaError_t launch_p2p_wait(const unsigned* local_ready, unsigned epoch, unsigned long long timeout_ns,
                            unsigned* err, cudaStream_t s) {
  p2p_wait_kernel<<<1, 1, 0, s>>>(local_ready, epoch, timeout_ns, err);
  return cudaGetLastError();
}
cudaError_t launch_p2p_post(unsigned* remote_done, unsigned epoch, cudaStream_t s) {
  p2p_post_kernel<<<1, 1, 0, s>>>(remote_done, epoch);
  return cudaGetLastError();
}

}  // namespace ptycho
