/*
 * ptycho.h -- C ABI of the B200-native gradient-decomposition ptychography hot path
 * (arXiv 2205.06327, "Image Gradient Decomposition for Parallel and Memory-Efficient
 * Ptychographic Reconstruction").
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation / algorithm named),
 * reading #k = DESIGN.md §Readings row k (how a silent or ambiguous passage is read).
 *
 * The calls follow the paper's problem statement (§Math Formulation, Eq. 1):
 * inputs are the diffraction amplitudes |y_i|, the probe p, the probe locations and an
 * initial volume V; the output is V.  Alg. 1 is driven by
 *     forward_grad (steps 5-8) -> appp_passes (steps 10-13) -> step (steps 14-16)
 * once per pass segment, and stitch (step 20) at the end.
 *
 * Conventions that hold for every call:
 *  - Every function returns a ptycho_status and never aborts; on error a message is
 *    available from ptycho_last_error(ctx) until the next call on that context.
 *    ECUDA / ENCCL leave the context unusable (destroy it).
 *  - The library never allocates device memory itself: the caller provides ONE device
 *    workspace (ptycho_workspace_bytes / ptycho_set_workspace) that the library carves
 *    into V_k, AccBuf_k, stash, wavefields, measurement store and tables.  The library
 *    borrows it until destroy and never frees it.  Host arrays are copied during the call.
 *  - All work is enqueued on the CUDA stream given to ptycho_create (asynchronous),
 *    except: calls with a non-NULL double* output and the debug_* calls synchronize;
 *    appp_passes / stitch / set_tiles are collective over all ranks when nranks > 1
 *    (every rank calls them the same number of times in the same order).
 *  - Coordinates are voxels; rects are int32[4] = {y0, x0, y1, x1}, half-open.
 *  - Complex data are interleaved float pairs (complex64).
 */
#ifndef PTYCHO_H
#define PTYCHO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ptycho_ctx_s* ptycho_ctx;

typedef enum {
  PTYCHO_OK = 0,
  PTYCHO_EARG = 1,    /* bad argument or config (N not in {64,256,1024}, T < 0, NULL ptr, ...) */
  PTYCHO_ESHAPE = 2,  /* buffer size inconsistent with the geometry                              */
  PTYCHO_ESTATE = 3,  /* call order violated (see "Call order" below)                            */
  PTYCHO_EHALO = 4,   /* PTYCHO_F_EXACT_WINDOW set and a window (clipped to the object) is not  */
                      /* covered by its tile's extended rect R_k (reading #12/#13)               */
  PTYCHO_ECUDA = 5,   /* CUDA runtime error (context unusable)                                    */
  PTYCHO_ENCCL = 6,   /* NCCL error (context unusable)                                            */
  PTYCHO_ENOMEM = 7   /* workspace smaller than ptycho_workspace_bytes                           */
} ptycho_status;

/* ptycho_config.flags */
#define PTYCHO_F_EXACT_WINDOW 1 /* require halo >= window reach (exact multi-tile == single tile) */
#define PTYCHO_F_STASH_FREE 2   /* stash-free adjoint: keep phi_{S-1} only and     */
                                /* recompute phi_s = P^H(conj(t_{s+1}) phi_{s+1}) during the backward */
                                /* (P unitary, |t| = 1; App. A).  Stash 2 N^2 instead of S N^2        */
                                /* complex64 per tile; S more passes per probe.  Same gradient up to  */
                                /* fp32 rounding of the recomputation.                                */

/* ptycho_load_measurements layout_flags */
#define PTYCHO_AMP_DC_CENTERED 1 /* input has DC at (N/2,N/2): ifftshift once at load           */
#define PTYCHO_AMP_INTENSITY 2   /* input is |y|^2: take the square root at load                 */
#define PTYCHO_AMP_ASYNC 4       /* host input, no layout change needed (no DC_CENTERED/INTENSITY, */
                                 /* S even): return once the copies are enqueued.  They go straight */
                                 /* into the stores on a copy stream in chunks of 8 probes, and each */
                                 /* probe chain waits only for its own chunk, so the transfer        */
                                 /* overlaps the gradient passes.  Pinned input with a device alias  */
                                 /* (cudaHostAlloc, torch pin_memory) is read by 8-CTA upload kernels */
                                 /* over PCIe; other host memory by copy-engine copies.  The host     */
                                 /* buffer must stay valid and unchanged until ptycho_synchronize.   */
                                 /* Otherwise the flag is ignored (synchronous).  Measured on B200,  */
                                 /* LT-small: the 17.4 GB upload costs the iteration +50-80 ms (upload */
                                 /* kernels) vs +265-300 ms (copy engine) vs +330 ms (synchronous).  */

typedef struct {
  int32_t n;         /* N: probe window = detector side; 64, 256 or 1024                          */
  int32_t slices;    /* S >= 1 ("a stack of 2D image slices")                              */
  int32_t height;    /* object H (voxels)                                                          */
  int32_t width;     /* object W (voxels)                                                          */
  float sigma;       /* interaction constant: transmission t_s = exp(i sigma V_s) (reading #2)     */
  float prop_c;      /* Fresnel coefficient c: H[u,v] = exp(-i pi c (m_u^2+m_v^2)/N^2) (reading #3) */
  float alpha;       /* per-probe step, Alg. 1 step 8                                       */
  float alpha_acc;   /* accumulated step, Alg. 1 step 15; reading #19 uses alpha_acc=alpha */
  float tau;         /* chi = 0 where |Psi| <= tau*||p||_2/N (reading #30); 1e-4 by default        */
  int32_t pass_period; /* T in local probes (Alg. 1 step 9; reading #17); 0 = once/iteration */
  int32_t flags;     /* PTYCHO_F_*                                                                 */
} ptycho_config;

/* ---------------------------------------------------------------------------------------------
 * Lifecycle.   Call order:  create -> set_tiles -> set_scan -> set_workspace -> set_probe ->
 *              load_measurements (any number) -> set_volume -> { forward_grad, appp_passes,
 *              step } per segment (or iterate) -> stitch -> destroy.  Other orders: ESTATE.
 * ------------------------------------------------------------------------------------------- */

/* Validate cfg and bind to CUDA device `device`; `cuda_stream` (cudaStream_t, NULL = legacy
 * default stream) is the stream all work is ordered on.  Builds the twiddle and propagator
 * tables on the host (double, rounded to float). */
ptycho_status ptycho_create(const ptycho_config* cfg, int device, void* cuda_stream, ptycho_ctx* out);

/* Free the library-owned objects (streams, events, graphs, NCCL communicator).  Never frees
 * the workspace. */
ptycho_status ptycho_destroy(ptycho_ctx ctx);

/* Message of the last failing call on ctx (ctx may be NULL for create errors).  Valid until
 * the next call on the same context. */
const char* ptycho_last_error(ptycho_ctx ctx);

/* Fill out[0..bytes) with a fresh NCCL unique id (128 bytes) for set_tiles.  Rank 0 calls it
 * and broadcasts the bytes (e.g. torch.distributed). */
ptycho_status ptycho_nccl_unique_id(void* out, size_t bytes);

/* Lateral tile grid (§Image Gradient Decomposition; Fig. forward_backward):
 * R x C tiles, tile k = r*C + c, interiors split uniformly with the remainder in the last row /
 * column (reading #14), extended rect R_k = interior dilated by `halo`, clipped to the object.
 * tile_owner[k] is the rank that owns tile k (NULL: every tile on this rank -- "virtual tiles").
 * When nranks > 1, nccl_id (128 bytes from ptycho_nccl_unique_id on rank 0) creates the NCCL
 * communicator used by the APPP P2P chains; collective. */
ptycho_status ptycho_set_tiles(ptycho_ctx ctx, int32_t rows, int32_t cols, int32_t halo,
                               const int32_t* tile_owner, const void* nccl_id, int32_t rank,
                               int32_t nranks);

/* Halo Voxel Exchange baseline (the paper's comparison system; "two extra rows
 * of probe locations ... halo width of 890 Picometers"), instead of set_tiles.
 * Same grid and R_k = interior dilated by `halo`; set_scan assigns to tile k EVERY probe whose
 * centre lies in its interior dilated by `margin` px (own + extra rows: margin = rows x scan
 * step), so a probe may sit on several tiles (local_probes lists the duplicates).  iterate =
 * one per-probe SGD sweep per tile (steps 6, 8; no AccBuf, passes or accumulated step), then the
 * copy-paste: every halo voxel is REPLACED by the tile whose interior holds it.
 * appp_passes = the exchange alone; step is ESTATE; cross-rank messages use NCCL.  A halo wider
 * than the adjacent interiors (the paper's "NA") is EHALO.  Collective like set_tiles. */
ptycho_status ptycho_set_tiles_hve(ptycho_ctx ctx, int32_t rows, int32_t cols, int32_t halo, int32_t margin,
                                   const int32_t* tile_owner, const void* nccl_id, int32_t rank,
                                   int32_t nranks);

/* Host-only geometry (no context, no GPU): rects[8*k .. 8*k+8) = {ext y0,x0,y1,x1, interior
 * y0,x0,y1,x1} of tile k = r*C + c for the grid set_tiles would build (same code). */
ptycho_status ptycho_tile_geometry(int32_t height, int32_t width, int32_t rows, int32_t cols, int32_t halo,
                                   int32_t* rects);

/* Host-only APPP schedule (no context, no GPU): the hop list appp_passes executes, in the global
 * order every rank follows.  hops_out[7*i ..] = {src tile, dst tile, y0, y1, x0, x1, add (1 = ADD,
 * forward passes; 0 = REPLACE, backward passes)}; hops_out may be NULL to query *count.
 * 2(R-1)C + 2(C-1)R hops (some may have empty regions when extended rects do not meet). */
ptycho_status ptycho_appp_schedule(int32_t height, int32_t width, int32_t rows, int32_t cols, int32_t halo,
                                   int32_t* hops_out, int32_t max_hops, int32_t* count);

/* Probe locations (raster order): host int32 [n_probes][2] = (cy, cx), global
 * order = acquisition time order.  Windows are N x N with top-left (cy-N/2, cx-N/2)
 * (reading #10); windows past the object edge are legal (V = 0 there, reading #12).  Probes
 * are assigned to tiles by centre containment in the half-open interior (reading #15); each
 * tile processes its probes in ascending global index (reading #16).  A centre outside the
 * object is EARG; with PTYCHO_F_EXACT_WINDOW an uncovered window is EHALO. */
ptycho_status ptycho_set_scan(ptycho_ctx ctx, const int32_t* centers_yx, int64_t n_probes);

/* Global probe ids owned by this rank, in local order (my tiles in increasing tile index, each
 * tile's probes ascending).  ids may be NULL to query *count only. */
ptycho_status ptycho_local_probes(ptycho_ctx ctx, int64_t* ids, int64_t* count);

/* Number of probes assigned to tile `tile` (any tile, owned or not). */
ptycho_status ptycho_tile_probe_count(ptycho_ctx ctx, int32_t tile, int64_t* count);

/* Rects of tile `tile`: ext = R_k, interior = the non-halo part (both may be NULL). */
ptycho_status ptycho_tile_rect(ptycho_ctx ctx, int32_t tile, int32_t ext[4], int32_t interior[4]);

/* Opt-in batched schedule (north_star item 3; the sequential per-probe update of Alg. 1 steps
 * 5-8, is the default): within each pass segment a tile's probes are grouped into rounds
 * -- round(i) = 1 + the largest round of an earlier probe whose window (clipped to R_k) overlaps
 * window i -- and each round's probes (ascending) run side by side in batches of <= max_batch
 * (1..64).  Every voxel sees the same ordered sequence of updates as in the sequential schedule,
 * so V_k and AccBuf_k are bit-identical to it (the reported loss may differ in rounding: its
 * partial sums are grouped per batch slot).  Costs max_batch x (stash + wavefields) of workspace.
 * Call after set_scan and before set_workspace. */
ptycho_status ptycho_set_schedule(ptycho_ctx ctx, int32_t batched, int32_t max_batch);

/* Bytes of device workspace this rank needs (after set_tiles and set_scan). */
ptycho_status ptycho_workspace_bytes(ptycho_ctx ctx, size_t* bytes);

/* Hand the device workspace to the library (>= workspace_bytes, 256-byte aligned).  Uploads
 * tables and centres, zeroes V_k and AccBuf_k (Alg. 1 step 2). */
ptycho_status ptycho_set_workspace(ptycho_ctx ctx, void* workspace_dev, size_t bytes);

/* Probe p (reading #9: one shared probe, integer-shifted): complex64 [N][N], beam axis at
 * (N/2, N/2).  on_device != 0: probe_c64 is a device pointer. */
ptycho_status ptycho_set_probe(ptycho_ctx ctx, const void* probe_c64, int on_device);

/* Diffraction amplitudes |y_i| (reading #6) for local probes [first_local,
 * first_local+count) in local order: float32 [count][N][N], DC at [0][0] unless
 * PTYCHO_AMP_DC_CENTERED; intensities if PTYCHO_AMP_INTENSITY.  on_device selects host/device. */
ptycho_status ptycho_load_measurements(ptycho_ctx ctx, const float* amp, int on_device,
                                       int64_t first_local, int64_t count, int32_t layout_flags);

/* Inverse of load_measurements: copy the stored amplitudes of local probes [first_local,
 * first_local+count) to host float32 [count][N][N], DC at [0][0] (e.g. after
 * simulate_measurements).  Synchronizes. */
ptycho_status ptycho_read_measurements(ptycho_ctx ctx, float* amp_out, int64_t first_local, int64_t count);

/* Alg. 1 step 3: every local tile receives V on R_k from the global volume
 * float32 [S][H][W] (host or device); V == NULL sets V_0 = 0.  AccBuf_k is zeroed. */
ptycho_status ptycho_set_volume(ptycho_ctx ctx, const float* volume, int on_device);

/* Synthetic-data plumbing: replace the measurement store of every local probe
 * by |G(p_i, V_k)| computed by the forward path from the current V_k. */
ptycho_status ptycho_simulate_measurements(ptycho_ctx ctx);

/* ---------------------------------------------------------------------------------------------
 * The hot path.
 * ------------------------------------------------------------------------------------------- */

/* Alg. 1 steps 5-8: for every local tile, for its local probes
 * [first, first+count) (clipped to the tile's count), sequentially in local order:
 *   g = d f_i / d V_k  (multislice forward G, amplitude residual, adjoint; Eq. 1-2)
 *   AccBuf_k[win ^ R_k] += g ;  V_k[win ^ R_k] -= alpha g  (t_s from the pre-update V).
 * Tiles run concurrently on internal streams.  loss_out (nullable): sum_i f_i over the probes
 * processed on this rank (synchronizes). */
ptycho_status ptycho_forward_grad(ptycho_ctx ctx, int64_t first, int64_t count, double* loss_out);

/* Alg. 1 steps 10-13 (Fig. forward_backward; APPP P:33-57): vertical
 * forward (ADD chains down tile columns), vertical backward (REPLACE chains up), horizontal
 * forward / backward over the full extended height (reading #21), on AccBuf.  Rank-local
 * tile pairs are device copies; cross-rank hops use the transport below, issued by every rank in
 * one global hop order with no barrier (a rank proceeds to its horizontal hops as soon as its
 * vertical ones are done: cross-direction pipelining).  Collective. */
ptycho_status ptycho_appp_passes(ptycho_ctx ctx);

/* Transport of cross-rank APPP hops.  PTYCHO_APPP_P2P: the receiving rank's copy
 * kernel reads the sender's AccBuf region in place over NVLink (CUDA IPC mapping of the sender's
 * workspace, exchanged once over the NCCL communicator) and adds / copies it into its own AccBuf;
 * a READY / DONE flag pair per hop (system-scope release/acquire) replaces the send/recv
 * handshake -- no pack, no staging buffer.  PTYCHO_APPP_NCCL: pack + ncclSend / ncclRecv +
 * unpack.  PTYCHO_APPP_AUTO (default; env PTYCHO_APPP_TRANSPORT=nccl|p2p overrides): P2P when
 * every rank can map every peer, else NCCL.  The choice is made collectively at the first APPP
 * call and is the same on every rank; set it before that call (ESTATE after).  Requesting P2P
 * where it is unavailable makes that first APPP call fail with ECUDA.  Results are bit-identical
 * for both transports (same ADD order). */
#define PTYCHO_APPP_AUTO 0
#define PTYCHO_APPP_NCCL 1
#define PTYCHO_APPP_P2P 2
ptycho_status ptycho_set_appp_transport(ptycho_ctx ctx, int32_t mode);
/* Active transport (PTYCHO_APPP_NCCL / _P2P), or PTYCHO_APPP_AUTO before the first APPP call. */
ptycho_status ptycho_appp_transport(ptycho_ctx ctx, int32_t* mode);

/* Alg. 1 steps 14-16: V_k -= alpha_acc * AccBuf_k ; AccBuf_k = 0. */
ptycho_status ptycho_step(ptycho_ctx ctx);

/* One iteration ("a cycle through all the probe locations"): for each pass segment
 * j (passes after local probes T, 2T, ... and a flush at the end, reading #17):
 * forward_grad(jT, T); appp_passes; step.  loss_out (nullable) = F(V) summed over ALL ranks'
 * probes of this sweep (a 1-double NCCL all-reduce when nranks > 1). */
ptycho_status ptycho_iterate(ptycho_ctx ctx, double* loss_out);

/* Alg. 1 step 20: interiors of every tile written to V_out float32 [S][H][W] on rank
 * `root` (host or device per out_on_device; other ranks may pass NULL).  Collective. */
ptycho_status ptycho_stitch(ptycho_ctx ctx, float* V_out, int out_on_device, int32_t root);

/* Block the host until all work enqueued by this context has finished. */
ptycho_status ptycho_synchronize(ptycho_ctx ctx);

/* Number of kernels this context has launched so far (all streams, including graph nodes). */
ptycho_status ptycho_kernel_launches(ptycho_ctx ctx, int64_t* count);

/* Measurement export (bench.py roofline): run the pass chain of local probes [first, first+count)
 * of local tile `tile` (real work: V_k and AccBuf_k are updated exactly as by forward_grad) with
 * direct launches bracketed by CUDA events on the tile's stream, and return per pass kind
 * (0..13, see PassKind in csrc/internal.h: 2 = forward middle pass, 8 = backward middle pass,
 * 11..13 = stash-free recomputation passes) the summed kernel time in ms and the number of
 * launches.  ms_out / launches_out: [14].
 * Synchronizes. */
ptycho_status ptycho_profile_chain(ptycho_ctx ctx, int32_t tile, int64_t first, int64_t count, double* ms_out,
                                   int64_t* launches_out);

/* Measurement export (bench.py breakdown; SURVEY §8(d) "how it will be timed" item 5, mirroring
 * the paper's runtime breakdown): run ONE iteration exactly as ptycho_iterate (real work,
 * same results) but with the APPP slab pipelining off, so the phases are serial on this rank, and
 * return in ms_out[8], measured with CUDA events on the context stream:
 *   [0] total, [1] compute (probe chains of all local tiles, all segments),
 *   [2] wait (P2P transport, receiving side: time in the READY waits, i.e. waiting for a peer to
 *       finish the region; 0 for the NCCL transport, whose receive time is in [3]),
 *   [3] comm (the rest of the APPP span: hop copies over NVLink / NCCL, local hops),
 *   [4] accumulated step (Alg. 1 steps 14-16),
 *   [5] sender hold (P2P, sending side: READY -> DONE spins = the peer's lateness + its copy of
 *       the region), [6] receiving side: time of the copy kernels pulling peer AccBuf regions over
 *       NVLink, [7] the bytes they pulled ([7] / [6] = the link rate).  Collective; synchronizes. */
ptycho_status ptycho_profile_iteration(ptycho_ctx ctx, double* ms_out);

/* Ordering checks (compute-sanitizer is not available on this pool): a library
 * built with -DPTYCHO_DEBUG_CHECKS (lib/libptycho_debug.so) re-reads, after griddepcontrol.wait,
 * every V / AccBuf / stash word a pass prefetched BEFORE the grid dependency resolved and ORs a bit
 * into an error word on any mismatch: 1 V (gradient pass), 2 AccBuf, 4 stash, 8 V (forward pass).
 * Synchronizes, returns and clears the bits; *checks_built = 0 for the product library (bits 0). */
ptycho_status ptycho_debug_errors(ptycho_ctx ctx, uint32_t* bits, int32_t* checks_built);

/* ---------------------------------------------------------------------------------------------
 * Debug exports (same library; used by the parity tests).  All synchronize; host buffers.
 * ------------------------------------------------------------------------------------------- */

/* Copy V_k (which = 0) or AccBuf_k (which = 1) of local tile `tile` to / from a host float32
 * array [S][ext_h][ext_w] in natural (y, x) order. */
ptycho_status ptycho_debug_read_tile(ptycho_ctx ctx, int32_t tile, int32_t which, float* out);
ptycho_status ptycho_debug_write_tile(ptycho_ctx ctx, int32_t tile, int32_t which, const float* in);

/* Full-window gradient d f_i/d V_k [S][N][N] (natural window order, before the R_k mask) and
 * f_i of local probe `probe` (index into the tile's own list) of tile `tile` at the current
 * V_k, without updating V_k or AccBuf_k.  Same kernels as forward_grad. */
ptycho_status ptycho_debug_probe_grad(ptycho_ctx ctx, int32_t tile, int64_t probe, float* grad_out,
                                      double* loss_out);

/* SURVEY §8(b) forms of the two exports above, by GLOBAL probe id (the tile of this rank that
 * holds it is looked up; EARG if none): output pointers may be host or device memory
 * (cudaMemcpyDefault). */
ptycho_status ptycho_probe_grad(ptycho_ctx ctx, int64_t probe, float* g_out, double* loss_out);
ptycho_status ptycho_probe_exitwave(ptycho_ctx ctx, int64_t probe, void* psi_out);

/* Literal exit wave psi_S (propagated after the last slice, reading #5), complex64 [N][N]
 * natural window order, of probe `probe` of tile `tile` at the current V_k. */
ptycho_status ptycho_debug_exit_wave(ptycho_ctx ctx, int32_t tile, int64_t probe, void* psi_out);

#ifdef __cplusplus
}
#endif
#endif /* PTYCHO_H */
