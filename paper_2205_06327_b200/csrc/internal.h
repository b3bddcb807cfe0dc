// Internal declarations shared by api.cu (host orchestration) and kernels.cu (sm_100a kernels).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda.h>  // CUtensorMap (TMA descriptors of V_k / AccBuf_k)
#include <cuda_runtime.h>

namespace ptycho {

// Lines (1-D transforms) handled by one CTA in a pass kernel.  The transposed store writes
// LINES_PER_CTA consecutive complex64 (= 32 B, one L2 sector) per output row.
constexpr int LINES_PER_CTA = 4;

// Everything a pass kernel needs; passed by value (baked into the per-probe CUDA graph, the
// probe itself is read from *desc on the device).
struct PassArgs {
  float* V;                 // V_k, slice s at V + s*slice_stride; layout L_{s&1}
  float* acc;               // AccBuf_k, same layout as V
  long long slice_stride;   // floats per slice
  int pitch0, pitch1;       // row pitch of even slices ([eh][pitch0]) and odd slices ([ew][pitch1])
  int ey0, ex0, eh, ew;     // R_k in global coordinates
  float2* stash;            // phi_s, [S][N][N] in layout L_{s&1} (stash-free: a ring of 2 slices)
  const float2* in;         // wavefield in (line-major in this pass's layout)
  float2* out;              // wavefield out (written transposed)
  const float2* probe;      // p, [N][N] natural
  float* amp;               // measurement store [n_k][N][N], layout L_{S&1}, DC at [0][0]
  const int2* centers;      // (cy, cx) of the tile's probes, local order
  int4* desc;               // current probe {local index, window y0, window x0, 0} (device)
  unsigned* done;           // block-completion counter for the cursor advance
  double* loss_part;        // per-CTA loss partial sums
  const float2* wtab;       // engine twiddle table (fill_twiddles; rounded from double)
  const float2* htab;       // H_1[u]/N = exp(-i pi c m_u^2/N^2)/N (rounded from double)
  float* gexport;           // debug: gradient out [S][N][N] natural (GRAD passes) or nullptr
  float2* natural_out;      // debug: exit wave out [N][N] natural
  float sigma, alpha, thr;  // t = exp(i sigma V); per-probe step; |Psi| threshold (true scale)
  float sigma_pi;           // sigma / pi (t = sincospi(sigma_pi V), rounded from double)
  int s;                    // slice index of this pass (TRANSMIT / GRAD / RECON)
  int stash_s;              // stash slice of this pass (s, or s & 1 in the stash-free ring)
  int stash_store;          // TRANSMIT writes phi_s to the stash (0: stash-free, s < S-1)
  int advance;              // last block advances *desc to the next probe when done
  int n_probes;             // probes of this tile (desc stops at the last one)
  int natural_transposed;   // debug store: lines are columns (1) or rows (0)
  int high_occupancy;       // forward passes built for 3 CTAs/SM (many concurrent tile chains)
  int batch;                // probes processed side by side (batched schedule; 1 = sequential)
  long long stash_slot;     // float2 between the stashes of consecutive batch slots
  long long wf_slot;        // float2 between the wavefields of consecutive batch slots
  int no_acc;               // HVE baseline: per-probe SGD only, AccBuf neither read nor written
  // TMA descriptors of V_k and AccBuf_k for this pass's slice parity (3-D: position along the
  // line, line, slice/2; box = min(N, 256) positions of one line; out-of-bounds = zero fill on
  // load, clipped on store -- exactly the zero-extension of reading #12 and the win ^ R_k mask).
  // Device copies in the workspace (64-B aligned, written once by set_workspace); unused by the
  // persistent chain.
  const CUtensorMap* tmV;
  const CUtensorMap* tmA;
  unsigned* dbg;            // PTYCHO_DEBUG_CHECKS builds: ordering / staleness error bits (else unused)
};

enum PassKind : int {
  K_FWD_FIRST_PROP = 0,   // probe in; t_0; stash; P            ; store^T
  K_FWD_FIRST_FFT,        // probe in; t_0; stash; FFT          ; store^T  (S == 1)
  K_FWD_MID,              // P ; t_s ; stash ; P                 ; store^T
  K_FWD_LAST,             // P ; t_s ; stash ; FFT               ; store^T
  K_TURN,                 // FFT ; residual/loss/chi ; IFFT      ; store^T
  K_SIMULATE,             // FFT ; write |X| to the measurement store
  K_BWD_LAST_PROP,        // IFFT ; grad/update ; P^H            ; store^T  (s = S-1 > 0)
  K_BWD_LAST_END,         // IFFT ; grad/update                  (S == 1)
  K_BWD_MID,              // P^H ; grad/update ; P^H             ; store^T
  K_BWD_END,              // P^H ; grad/update                   (s = 0)
  K_EXIT_COMPLETE,        // P ; natural store (debug exit wave)
  // stash-free adjoint (PTYCHO_F_STASH_FREE): phi_s = P^H(conj(t_{s+1}) phi_{s+1})
  // is recomputed by a second adjoint chain running one slice ahead of the gradient chain.
  K_RECON_FIRST,          // stash phi_{S-1} in; conj(t_{S-1}) ; P^H      ; store^T
  K_RECON_MID,            // P^H ; phi_s -> stash ring ; conj(t_s) ; P^H ; store^T
  K_RECON_END,            // P^H ; phi_0 -> stash ring
  K_COUNT
};

// Persistent chain kernel (cooperative launch): probes [first, first + count[t]) of every local
// tile t, all tiles in lockstep, grid barrier between passes.
constexpr int MAX_CHAIN_TILES = 16;
struct ChainArgs {
  PassArgs t[MAX_CHAIN_TILES];         // per tile (s / in / out / advance are set per step)
  float2* wf[MAX_CHAIN_TILES][2];      // wavefield ping-pong per tile
  int count[MAX_CHAIN_TILES];          // probes of this segment per tile
  int ntiles, first, maxn, S;
  unsigned* bar;                       // grid-barrier counter (zeroed before the launch)
};
cudaError_t launch_chain(int n, const ChainArgs& c, cudaStream_t stream);
// Cluster-resident chain (N = 64, 256): one 16-CTA cluster per tile, the wavefield in DSMEM,
// probes [first, first + count[t]) of tile t; in / out / bar of ChainArgs unused.
cudaError_t launch_cluster(int n, const ChainArgs& c, cudaStream_t stream);

// Launch one pass kernel (with programmatic dependent launch on `stream`).
cudaError_t launch_pass(int n, PassKind kind, const PassArgs& a, cudaStream_t stream, bool pdl);

// Region ops on per-slice alternating layouts.  dst/src are 2-D strided float arrays.
//   op 0: dst = src ; op 1: dst += src
cudaError_t launch_copy2d(float* dst, long long dld, long long dss, const float* src, long long sld,
                          long long sss, int rows, int cols, int nslices, int op, cudaStream_t stream);
// dst[r][c] (op)= src[c][r]  (transposing copy), slices as above
cudaError_t launch_transpose2d(float* dst, long long dld, long long dss, const float* src, long long sld,
                               long long sss, int rows, int cols, int nslices, int op, cudaStream_t stream);
// V -= alpha*acc ; acc = 0  over n floats
cudaError_t launch_acc_step(float* V, float* acc, long long n, float alpha, cudaStream_t stream);
// measurement store: dst[c][.][.] from src[c][N][N] with ifftshift / sqrt / transpose options
cudaError_t launch_amp_load(float* dst, const float* src, int count, int n, int shift, int intensity,
                            int transpose, cudaStream_t stream);
// twiddle table of the FFT engine for window n (layout private to kernels.cu)
size_t twiddle_table_size(int n);
void fill_twiddles(int n, float2* tw);
// desc[b] = probe list[b] for b < cnt, inactive (-1) for cnt <= b < batch
cudaError_t launch_set_batch(int4* desc, const int2* centers, const int* list, int cnt, int batch, int n,
                             cudaStream_t stream);
// *desc = probe v of the tile (v clamped to [0, nk))
cudaError_t launch_set_desc(int4* desc, const int2* centers, int v, int nk, int n, cudaStream_t stream);
cudaError_t launch_fill(float* p, long long n, float v, cudaStream_t stream);
// dst[0, n) = src[0, n): src the device alias of pinned host memory, both 16-B aligned, n % 4 == 0
cudaError_t launch_upload(float* dst, const float* src, long long n, int ctas, cudaStream_t stream);
cudaError_t launch_sum_double(const double* parts, int n, double* out, cudaStream_t stream);
// APPP peer-to-peer transport: flag kernels (one thread each; see kernels.cu)
// timeout_ns = 0: wait without limit; otherwise a timed-out wait sets *err (host-mapped) and returns
cudaError_t launch_p2p_signal(unsigned* remote_ready, unsigned epoch, const unsigned* local_done,
                              unsigned long long timeout_ns, unsigned* err, cudaStream_t s);
cudaError_t launch_p2p_wait(const unsigned* local_ready, unsigned epoch, unsigned long long timeout_ns,
                            unsigned* err, cudaStream_t s);
cudaError_t launch_p2p_post(unsigned* remote_done, unsigned epoch, cudaStream_t s);

}  // namespace ptycho
