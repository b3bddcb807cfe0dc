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
// complex helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

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
  if (INV) return make_float2(a.x * c - a.y * s, a.x * s + a.y * c);
  return make_float2(a.x * c + a.y * s, a.y * c - a.x * s);
}

// In-register DFT of size P (<= 32), natural order in and out (radix-2 DIT on a compile-time
// bit-reversed register permutation).  Forward: exp(-2 pi i jk/P), unnormalised.
template <int P, bool INV>
__device__ __forceinline__ void dft_reg(float2 (&x)[P]) {
  constexpr int LOG = Log2<P>::v;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const int j = brev(i, LOG);
    if (j > i) {
      const float2 t = x[i];
      x[i] = x[j];
      x[j] = t;
    }
  }
#pragma unroll
  for (int half = 1; half < P; half <<= 1) {
#pragma unroll
    for (int i = 0; i < P; i += 2 * half) {
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const float2 b = twmul32<INV>(x[i + k + half], k * (32 / (2 * half)));
        const float2 a = x[i + k];
        x[i + k] = cadd(a, b);
        x[i + k + half] = csub(a, b);
      }
    }
  }
}

template <int N> struct Geo;
template <> struct Geo<64> { static constexpr int P = 8, Q = 8; };
template <> struct Geo<256> { static constexpr int P = 16, Q = 16; };
template <> struct Geo<1024> { static constexpr int P = 32, Q = 32; };

// Unnormalised N-point DFT of one line; thread q holds x[q + Q*k] in and X[q + Q*k] out.
// ex: this line's exchange buffer P x (Q+1) float2.
template <int N, bool INV>
__device__ __forceinline__ void line_fft(float2 (&x)[Geo<N>::P], float2* __restrict__ ex, int q,
                                         const float2* __restrict__ wtab) {
  constexpr int P = Geo<N>::P, Q = Geo<N>::Q;
  dft_reg<P, INV>(x);
#pragma unroll
  for (int k = 1; k < P; ++k) {
    const float2 w = __ldg(wtab + q * k);
    x[k] = INV ? cmulc(x[k], w) : cmul(x[k], w);
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < P; ++k) ex[k * (Q + 1) + q] = x[k];
  __syncwarp();
#pragma unroll
  for (int n = 0; n < Q; ++n) x[n] = ex[q * (Q + 1) + n];
  dft_reg<Q, INV>(x);
}

// 1-D Fresnel propagation along the line: IFFT(H_1/N . FFT(x)) (ADJ: conj(H_1)).
template <int N, bool ADJ>
__device__ __forceinline__ void line_prop(float2 (&x)[Geo<N>::P], float2* __restrict__ ex, int q,
                                          const float2* __restrict__ wtab, const float2* __restrict__ htab) {
  constexpr int P = Geo<N>::P, Q = Geo<N>::Q;
  line_fft<N, false>(x, ex, q, wtab);
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const float2 h = __ldg(htab + q + Q * k);
    x[k] = ADJ ? cmulc(x[k], h) : cmul(x[k], h);
  }
  line_fft<N, true>(x, ex, q, wtab);
}

enum : int { OP_NONE = 0, OP_PROPF, OP_PROPA, OP_FFT, OP_IFFT };
enum : int { MID_NONE = 0, MID_TRANSMIT, MID_RESID, MID_SIMUL, MID_GRAD };
enum : int { ST_NONE = 0, ST_TRANS, ST_NATURAL };

template <int N, int OP>
__device__ __forceinline__ void apply_op(float2 (&x)[Geo<N>::P], float2* ex, int q, const PassArgs& a) {
  if constexpr (OP == OP_PROPF) line_prop<N, false>(x, ex, q, a.wtab, a.htab);
  if constexpr (OP == OP_PROPA) line_prop<N, true>(x, ex, q, a.wtab, a.htab);
  if constexpr (OP == OP_FFT) line_fft<N, false>(x, ex, q, a.wtab);
  if constexpr (OP == OP_IFFT) line_fft<N, true>(x, ex, q, a.wtab);
}

__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Location of this line inside R_k for slice parity ax: row pointer offset and valid range of
// the position coordinate.
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

template <int N, bool PROBE_IN, int PRE, int MID, int POST, int STORE>
__global__ void __launch_bounds__(LINES_PER_CTA * Geo<N>::Q)
pass_kernel(const PassArgs a) {
  constexpr int P = Geo<N>::P, Q = Geo<N>::Q, L = LINES_PER_CTA;
  extern __shared__ float2 smem[];
  griddep_wait();
  griddep_launch();

  const int lw = threadIdx.x / Q, q = threadIdx.x % Q;
  const int line = blockIdx.x * L + lw;
  const int i = *a.cursor;
  const int2 ctr = a.centers[i];
  const int wy0 = ctr.x - N / 2, wx0 = ctr.y - N / 2;
  float2* ex = smem + lw * P * (Q + 1);

  float2 x[P];
  {
    const float2* src = (PROBE_IN ? a.probe : a.in) + (size_t)line * N + q;
#pragma unroll
    for (int k = 0; k < P; ++k) x[k] = src[Q * k];
  }

  apply_op<N, PRE>(x, ex, q, a);

  if constexpr (MID == MID_TRANSMIT) {
    // phi_s = exp(i sigma V_s[win ^ R_k]) psi_s  (t = 1 outside R_k, reading #12); stash phi_s.
    const int ax = a.s & 1;
    const LineLoc LL = line_loc(a, ax, line, wy0, wx0);
    const float* vrow = a.V + (long long)a.s * a.slice_stride + LL.row;
    float2* st = a.stash + (size_t)a.s * N * N + (size_t)line * N + q;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int p = LL.pos0 + q + Q * k;
      const float v = (LL.ok && (unsigned)p < (unsigned)LL.plim) ? vrow[p] : 0.f;
      float sn, cs;
      sincosf(a.sigma * v, &sn, &cs);
      x[k] = cmul(x[k], make_float2(cs, sn));
      st[Q * k] = x[k];
    }
  }

  if constexpr (MID == MID_RESID || MID == MID_SIMUL) {
    // X = raw 2-D DFT (N x true F phi_{S-1}); |Psi| = |X|/N (App. A: |H| = 1).
    const float invn = 1.0f / (float)N;
    float* am = a.amp + (size_t)i * N * N + (size_t)line * N + q;
    float part = 0.f;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const float m = sqrtf(x[k].x * x[k].x + x[k].y * x[k].y);
      const float mag = m * invn;
      if constexpr (MID == MID_SIMUL) {
        am[Q * k] = mag;
      } else {
        const float r = mag - am[Q * k];
        part += r * r;
        // chi_Psi = r Psi/|Psi| (0 where |Psi| <= thr, reading #30), times 1/N for the two
        // unnormalised inverse line transforms that complete the unitary 2-D inverse.
        const float sc = (mag > a.thr) ? r * invn / m : 0.f;
        x[k] = make_float2(x[k].x * sc, x[k].y * sc);
      }
    }
    if constexpr (MID == MID_RESID) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      __shared__ float red[LINES_PER_CTA * Q / 32 + 1];
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += (double)red[w];
        a.loss_part[blockIdx.x] += tot;
      }
    }
  }

  if constexpr (MID == MID_GRAD) {
    // chi holds chi_phi_s.  g_s = 2 sigma Im(chi conj(phi_s)) (App. A);  on win ^ R_k:
    // AccBuf += g (Alg. 1 step 7), V -= alpha g (step 8); then chi <- conj(t_s) chi with t_s
    // from the PRE-update V.
    const int ax = a.s & 1;
    const LineLoc LL = line_loc(a, ax, line, wy0, wx0);
    const long long so = (long long)a.s * a.slice_stride + LL.row;
    float* vrow = a.V + so;
    float* arow = a.acc + so;
    const float2* st = a.stash + (size_t)a.s * N * N + (size_t)line * N + q;
    const float two_sigma = 2.0f * a.sigma;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = q + Q * k;
      const int p = LL.pos0 + j;
      const bool ok = LL.ok && (unsigned)p < (unsigned)LL.plim;
      const float2 ph = st[Q * k];
      const float g = two_sigma * (x[k].y * ph.x - x[k].x * ph.y);
      float v = 0.f;
      if (ok) v = vrow[p];
      if (a.gexport != nullptr) {
        const size_t o = (size_t)a.s * N * N + (ax == 0 ? (size_t)line * N + j : (size_t)j * N + line);
        a.gexport[o] = g;
      } else if (ok) {
        arow[p] += g;
        vrow[p] = v - a.alpha * g;
      }
      float sn, cs;
      sincosf(a.sigma * v, &sn, &cs);
      x[k] = cmulc(x[k], make_float2(cs, sn));
    }
  }

  apply_op<N, POST>(x, ex, q, a);

  if constexpr (STORE == ST_TRANS) {
    // out[j][line]: stage the CTA's L lines, then write L consecutive complex per output row.
    __syncthreads();
    float2* stg = smem;
#pragma unroll
    for (int k = 0; k < P; ++k) stg[(q + Q * k) * (L + 1) + lw] = x[k];
    __syncthreads();
    float2* dst = a.out + (size_t)blockIdx.x * L;
#pragma unroll 4
    for (int e = threadIdx.x; e < N * L; e += L * Q) {
      const int j = e / L, l = e - j * L;
      dst[(size_t)j * N + l] = stg[j * (L + 1) + l];
    }
  }
  if constexpr (STORE == ST_NATURAL) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const int j = q + Q * k;
      const size_t o = a.natural_transposed ? (size_t)j * N + line : (size_t)line * N + j;
      a.natural_out[o] = x[k];
    }
  }

  if (a.advance) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(a.done, 1u);
      if (prev == gridDim.x - 1) {
        *a.done = 0u;
        atomicAdd(a.cursor, 1);
        __threadfence();
      }
    }
  }
}

template <int N>
static size_t pass_smem() {
  constexpr int P = Geo<N>::P, Q = Geo<N>::Q, L = LINES_PER_CTA;
  const size_t ex = (size_t)L * P * (Q + 1) * sizeof(float2);
  const size_t st = (size_t)N * (L + 1) * sizeof(float2);
  return ex > st ? ex : st;
}

template <int N, bool PROBE_IN, int PRE, int MID, int POST, int STORE>
static cudaError_t launch_one(const PassArgs& a, cudaStream_t stream, bool pdl) {
  auto kern = pass_kernel<N, PROBE_IN, PRE, MID, POST, STORE>;
  const size_t smem = pass_smem<N>();
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N / LINES_PER_CTA);
  cfg.blockDim = dim3(LINES_PER_CTA * Geo<N>::Q);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int N>
static cudaError_t launch_pass_n(PassKind kind, const PassArgs& a, cudaStream_t s, bool pdl) {
  switch (kind) {
    case K_FWD_FIRST_PROP: return launch_one<N, true, OP_NONE, MID_TRANSMIT, OP_PROPF, ST_TRANS>(a, s, pdl);
    case K_FWD_FIRST_FFT: return launch_one<N, true, OP_NONE, MID_TRANSMIT, OP_FFT, ST_TRANS>(a, s, pdl);
    case K_FWD_MID: return launch_one<N, false, OP_PROPF, MID_TRANSMIT, OP_PROPF, ST_TRANS>(a, s, pdl);
    case K_FWD_LAST: return launch_one<N, false, OP_PROPF, MID_TRANSMIT, OP_FFT, ST_TRANS>(a, s, pdl);
    case K_TURN: return launch_one<N, false, OP_FFT, MID_RESID, OP_IFFT, ST_TRANS>(a, s, pdl);
    case K_SIMULATE: return launch_one<N, false, OP_FFT, MID_SIMUL, OP_NONE, ST_NONE>(a, s, pdl);
    case K_BWD_LAST_PROP: return launch_one<N, false, OP_IFFT, MID_GRAD, OP_PROPA, ST_TRANS>(a, s, pdl);
    case K_BWD_LAST_END: return launch_one<N, false, OP_IFFT, MID_GRAD, OP_NONE, ST_NONE>(a, s, pdl);
    case K_BWD_MID: return launch_one<N, false, OP_PROPA, MID_GRAD, OP_PROPA, ST_TRANS>(a, s, pdl);
    case K_BWD_END: return launch_one<N, false, OP_PROPA, MID_GRAD, OP_NONE, ST_NONE>(a, s, pdl);
    case K_EXIT_COMPLETE: return launch_one<N, false, OP_PROPF, MID_NONE, OP_NONE, ST_NATURAL>(a, s, pdl);
    default: return cudaErrorInvalidValue;
  }
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
__global__ void copy2d_kernel(float* __restrict__ dst, long long dld, long long dss,
                              const float* __restrict__ src, long long sld, long long sss, int rows, int cols,
                              int op) {
  const int r = blockIdx.y;
  const long long z = blockIdx.z;
  float* d = dst + z * dss + (long long)r * dld;
  const float* s = src + z * sss + (long long)r * sld;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += gridDim.x * blockDim.x) {
    if (op == 0) d[c] = s[c];
    else d[c] += s[c];
  }
}

cudaError_t launch_copy2d(float* dst, long long dld, long long dss, const float* src, long long sld,
                          long long sss, int rows, int cols, int nslices, int op, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0 || nslices <= 0) return cudaSuccess;
  for (int z0 = 0; z0 < nslices; z0 += 65535) {
    const int nz = nslices - z0 < 65535 ? nslices - z0 : 65535;
    for (int r0 = 0; r0 < rows; r0 += 65535) {
      const int nr = rows - r0 < 65535 ? rows - r0 : 65535;
      dim3 grid((cols + 255) / 256 < 8 ? (cols + 255) / 256 : 8, nr, nz);
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

}  // namespace ptycho
