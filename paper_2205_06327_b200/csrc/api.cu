// Host side of the C ABI (include/ptycho.h): geometry, workspace carving, per-probe pass
// schedule (CUDA graph per tile), APPP hop schedule (device copies / NCCL P2P), stitch.
//
// Paper anchors: Alg. 1, §Image Gradient Decomposition, §Forward and
// Backward Accumulated Gradients Pass, APPP.
#include <cuda.h>  // driver types for cuMemGetAddressRange (resolved through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "ptycho.h"

using namespace ptycho;

namespace {

struct Hop {       // one APPP message: dst (op)= src on region [y0,y1) x [x0,x1), all slices
  int src, dst;
  int y0, y1, x0, x1;
  int add;         // 1 = ADD (forward passes), 0 = REPLACE (backward passes)
  int vol = 0;     // 0: AccBuf (APPP); 1: V (HVE copy-paste exchange)
};

struct Tile {
  int k = 0, r = 0, c = 0, owner = 0;
  int iy0 = 0, ix0 = 0, iy1 = 0, ix1 = 0;  // interior
  int ey0 = 0, ex0 = 0, ey1 = 0, ex1 = 0;  // extended rect R_k
  int eh = 0, ew = 0;
  int pitch0 = 0, pitch1 = 0;
  long long slice_stride = 0;
  std::vector<int64_t> probes;  // global ids, ascending
  // device state (local tiles only)
  float* V = nullptr;
  float* acc = nullptr;
  float2* stash = nullptr;
  float2* wf[2] = {nullptr, nullptr};
  float2* wfr[2] = {nullptr, nullptr};  // phi-chain wavefields (PTYCHO_F_STASH_FREE)
  float* amp = nullptr;
  int2* centers = nullptr;
  int4* desc = nullptr;
  unsigned* done = nullptr;
  double* loss_part = nullptr;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev = nullptr;
  cudaGraphExec_t graph = nullptr;
  std::vector<cudaEvent_t> slab_ev;  // APPP slab pipelining (segment_pipelined)
  // batched schedule
  int* order = nullptr;                  // device: probe lists of the current batches
  cudaGraphExec_t graph_b = nullptr;     // chain over `batch` slots, no cursor advance
  int64_t bfirst = -1, bcount = -1;      // cached batches for local probes [bfirst, bfirst+bcount)
  std::vector<std::vector<int>> batches;
  // asynchronous measurement loads (PTYCHO_AMP_ASYNC): chunk [begin, ...) of the tile's store is
  // complete when ev fires; chains wait only for the chunk holding their probe
  struct AmpChunk {
    int64_t begin;
    cudaEvent_t ev;
  };
  CUtensorMap* tm_dev = nullptr;  // TMA descriptors, device copies: [V 0, V 1, A 0, A 1] main box, + 4 tail box
  std::vector<AmpChunk> amp_pend;
  size_t amp_cur = 0;
  std::vector<cudaEvent_t> amp_pool;
  cudaEvent_t amp_free = nullptr;  // the tile stream's readers of the store are done
};

constexpr size_t ALIGN = 256;

// phi_s stash slices per batch slot: all S, or the 2-slice ring of the stash-free adjoint
static bool stash_free(const ptycho_config& c) { return (c.flags & PTYCHO_F_STASH_FREE) && c.slices > 1; }
static size_t stash_slices(const ptycho_config& c) { return stash_free(c) ? 2 : (size_t)c.slices; }
size_t align_up(size_t x, size_t a = ALIGN) { return (x + a - 1) / a * a; }

}  // namespace

struct ptycho_ctx_s {
  ptycho_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // tiles
  bool tiles_set = false;
  int R = 0, C = 0, halo = 0, rank = 0, nranks = 1;
  std::vector<Tile> tiles;
  std::vector<int> local;  // local tile indices, increasing
  std::vector<Hop> hops;
  ncclComm_t comm = nullptr;
  // scan
  bool scan_set = false;
  std::vector<int32_t> centers;
  // workspace
  bool ws_set = false;
  char* ws = nullptr;
  size_t ws_bytes = 0;
  float2* wtab = nullptr;
  float2* htab = nullptr;
  float2* probe = nullptr;
  double* dscratch = nullptr;
  int* iscratch = nullptr;
  float* staging = nullptr;
  size_t staging_floats = 0;
  float* debug = nullptr;
  size_t debug_floats = 0;
  float* sendbuf = nullptr;
  float* recvbuf = nullptr;
  size_t msg_floats = 0;
  bool probe_set = false;
  double probe_norm = 1.0;
  std::vector<float2> h_wtab, h_htab;
  long long launches = 0;
  cudaEvent_t ev_fork = nullptr;
  bool use_graph = true;
  bool use_pdl = true;
  bool debug_sync = false;  // PTYCHO_DEBUG_SYNC: synchronize after every direct pass launch
  int slab = 0;  // slices per APPP slab in ptycho_iterate (0 = passes after the whole segment)
  bool persist = false;  // run probe chains in the persistent cooperative chain kernel
  bool cluster = false;  // N <= 256: cluster-resident probe chains (wavefield in DSMEM)
  bool hve = false;      // Halo Voxel Exchange baseline (ptycho_set_tiles_hve)
  int hve_margin = 0;    // HVE probe-assignment margin (pixels)
  bool batched = false;  // opt-in batched schedule (non-overlapping windows side by side)
  int batch = 1;         // batch slots per tile
  // APPP transport between ranks (decided, collectively, at the first APPP call)
  int transport_req = PTYCHO_APPP_AUTO;
  int transport = PTYCHO_APPP_NCCL;
  bool transport_set = false;
  unsigned* flags = nullptr;  // [2][hops] READY / DONE epochs (P2P transport), in the workspace
  unsigned epoch = 0;         // APPP calls so far (identical on every rank)
  std::vector<char*> peer_ws;                   // [rank] peer workspace mapped into this process
  std::vector<void*> peer_map;                  // opened IPC mappings (closed at destroy)
  std::vector<long long> peer_flags;            // [rank] flags offset in that rank's workspace
  std::vector<std::vector<long long>> peer_acc; // [rank][tile] AccBuf offset (-1: not owned)
  cudaStream_t copy_stream = nullptr;           // asynchronous measurement loads
  cudaEvent_t ev_copy = nullptr;
  unsigned* p2p_err = nullptr;                  // pinned, mapped: a P2P flag wait timed out
  unsigned* p2p_err_dev = nullptr;
  unsigned long long p2p_timeout_ns = 600ull * 1000000000ull;
  std::vector<cudaEvent_t>* wait_ev = nullptr;    // ptycho_profile_iteration: events around P2P waits
  std::vector<cudaEvent_t>* signal_ev = nullptr;  // ... and around the senders' READY -> DONE spins
  std::vector<cudaEvent_t>* copy_ev = nullptr;    // ... and around the receivers' NVLink pulls
  double copy_bytes = 0.0;
};

static thread_local std::string g_create_err;
static ptycho_status check_p2p(ptycho_ctx ctx);

static ptycho_status fail(ptycho_ctx ctx, ptycho_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  else g_create_err = buf;
  return st;
}

#define CK(expr)                                                                                  \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess) return fail(ctx, PTYCHO_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define NK(expr)                                                                                  \
  do {                                                                                            \
    ncclResult_t r_ = (expr);                                                                     \
    if (r_ != ncclSuccess) return fail(ctx, PTYCHO_ENCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)
#define PASS(expr)                                                                                \
  do {                                                                                            \
    ptycho_status s_ = (expr);                                                                    \
    if (s_ != PTYCHO_OK) return s_;                                                               \
  } while (0)


// ------------------------------------------------------------------------------------------
// tiny device helpers launched from here
// ------------------------------------------------------------------------------------------

// ------------------------------------------------------------------------------------------
// lifecycle
// ------------------------------------------------------------------------------------------
extern "C" ptycho_status ptycho_create(const ptycho_config* cfg, int device, void* cuda_stream, ptycho_ctx* out) {
  ptycho_ctx ctx = nullptr;
  if (!cfg || !out) return fail(ctx, PTYCHO_EARG, "cfg and out must be non-NULL");
  if (cfg->n != 64 && cfg->n != 256 && cfg->n != 1024)
    return fail(ctx, PTYCHO_EARG, "n = %d: supported windows are 64, 256, 1024", cfg->n);
  if (cfg->slices < 1 || cfg->height < 1 || cfg->width < 1)
    return fail(ctx, PTYCHO_EARG, "slices/height/width must be >= 1");
  if (cfg->pass_period < 0) return fail(ctx, PTYCHO_EARG, "pass_period T must be >= 0");
  if (!(cfg->tau >= 0.f)) return fail(ctx, PTYCHO_EARG, "tau must be >= 0");
  if (cfg->flags & ~(PTYCHO_F_EXACT_WINDOW | PTYCHO_F_STASH_FREE))
    return fail(ctx, PTYCHO_EARG, "unknown flags 0x%x", (unsigned)cfg->flags);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return fail(ctx, PTYCHO_ECUDA, "CUDA device %d not available", device);
  ctx = new ptycho_ctx_s();
  ctx->cfg = *cfg;
  ctx->device = device;
  ctx->stream = (cudaStream_t)cuda_stream;
  if (const char* e = getenv("PTYCHO_NO_GRAPH")) ctx->use_graph = atoi(e) == 0;
  if (const char* e = getenv("PTYCHO_NO_PDL")) ctx->use_pdl = atoi(e) == 0;
  if (const char* e = getenv("PTYCHO_DEBUG_SYNC")) ctx->debug_sync = atoi(e) != 0;
  // APPP slab size: ~S/10 slices (>= 1); PTYCHO_SLAB overrides, 0 disables the pipelining
  ctx->slab = std::max(1, (cfg->slices + 9) / 10);
  if (const char* e = getenv("PTYCHO_SLAB")) ctx->slab = std::max(0, atoi(e));
  if (const char* e = getenv("PTYCHO_PERSIST")) ctx->persist = atoi(e) != 0;
  if (cfg->flags & PTYCHO_F_STASH_FREE) ctx->persist = false;  // the chain kernel keeps a full stash
  // Opt-in (PTYCHO_CLUSTER=1), N <= 256: one 16-CTA cluster per tile runs a whole segment's probe
  // chains with the wavefield in DSMEM.  Bit-identical to the graph + PDL chain but measured 2x
  // slower (small 3152 vs 6307 probe-loc/s): a cluster holds at most 16 CTAs, so each SM carries 4x
  // the lines of a standalone pass (profiles/round2/cluster_chain.txt).  Not with the stash-free
  // ring or the persistent kernel.
  ctx->cluster = false;
  if (const char* e = getenv("PTYCHO_CLUSTER"))
    ctx->cluster = atoi(e) != 0 && (cfg->n == 64 || cfg->n == 256) && !(cfg->flags & PTYCHO_F_STASH_FREE) &&
                   !ctx->persist;
  if (const char* e = getenv("PTYCHO_P2P_TIMEOUT_S")) ctx->p2p_timeout_ns = (unsigned long long)(atof(e) * 1e9);
  if (const char* e = getenv("PTYCHO_APPP_TRANSPORT")) {
    if (!strcmp(e, "nccl")) ctx->transport_req = PTYCHO_APPP_NCCL;
    else if (!strcmp(e, "p2p")) ctx->transport_req = PTYCHO_APPP_P2P;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    fail(nullptr, PTYCHO_ECUDA, "cuda init: %s", cudaGetErrorString(e));
    delete ctx;
    return PTYCHO_ECUDA;
  }
  // tables in double, rounded to float: W_N^k and H_1[u]/N (reading #3, #4)
  const int n = cfg->n;
  ctx->h_wtab.resize(twiddle_table_size(n));
  fill_twiddles(n, ctx->h_wtab.data());
  ctx->h_htab.resize(n);
  for (int k = 0; k < n; ++k) {
    const double m = (k < n / 2) ? (double)k : (double)(k - n);
    const double ph = -M_PI * (double)cfg->prop_c * m * m / ((double)n * (double)n);
    ctx->h_htab[k] = make_float2((float)(std::cos(ph) / n), (float)(std::sin(ph) / n));
  }
  *out = ctx;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_destroy(ptycho_ctx ctx) {
  if (!ctx) return PTYCHO_OK;
  cudaSetDevice(ctx->device);
  // Drain every stream the library queued work on before any handle goes away (the caller frees
  // the workspace right after).  Peers that mapped this workspace are done with it as well: a
  // sender's stream cannot pass its READY/DONE hop before the receiver has posted DONE.
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (int k : ctx->local)
    if (ctx->tiles[k].stream) cudaStreamSynchronize(ctx->tiles[k].stream);
  if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
  if (ctx->p2p_err) cudaFreeHost(ctx->p2p_err);
  for (auto& t : ctx->tiles) {
    if (t.graph) cudaGraphExecDestroy(t.graph);
    if (t.graph_b) cudaGraphExecDestroy(t.graph_b);
    if (t.stream && t.own_stream) cudaStreamDestroy(t.stream);
    if (t.ev) cudaEventDestroy(t.ev);
    for (cudaEvent_t e : t.slab_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : t.amp_pool) cudaEventDestroy(e);
    if (t.amp_free) cudaEventDestroy(t.amp_free);
  }
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->ev_copy) cudaEventDestroy(ctx->ev_copy);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  for (void* m : ctx->peer_map) cudaIpcCloseMemHandle(m);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  delete ctx;
  return PTYCHO_OK;
}

extern "C" const char* ptycho_last_error(ptycho_ctx ctx) {
  return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

extern "C" ptycho_status ptycho_nccl_unique_id(void* out, size_t bytes) {
  ptycho_ctx ctx = nullptr;
  if (!out || bytes < sizeof(ncclUniqueId)) return fail(ctx, PTYCHO_EARG, "need %zu bytes", sizeof(ncclUniqueId));
  ncclUniqueId id;
  NK(ncclGetUniqueId(&id));
  memcpy(out, &id, sizeof id);
  return PTYCHO_OK;
}

// ------------------------------------------------------------------------------------------
// geometry (readings #13-#16, #21)
// ------------------------------------------------------------------------------------------
static void split(int extent, int parts, int p, int* a, int* b) {
  const int base = extent / parts;
  *a = p * base;
  *b = (p == parts - 1) ? extent : (p + 1) * base;
}

// APPP hop list in the global order every rank follows (Fig. forward_backward a-d):
// vertical forward (ADD down each tile column), vertical backward (REPLACE up), horizontal forward
// and backward along each tile row over the full extended height Y_r (reading #21).
static void build_hops(const std::vector<Tile>& tiles, int rows, int cols, std::vector<Hop>& hops) {
  auto T = [&](int r, int c) -> const Tile& { return tiles[r * cols + c]; };
  hops.clear();
  for (int c = 0; c < cols; ++c)
    for (int r = 0; r + 1 < rows; ++r) {
      const Tile &a = T(r, c), &b = T(r + 1, c);
      hops.push_back({a.k, b.k, std::max(a.ey0, b.ey0), std::min(a.ey1, b.ey1), a.ex0, a.ex1, 1});
    }
  for (int c = 0; c < cols; ++c)
    for (int r = rows - 1; r >= 1; --r) {
      const Tile &a = T(r, c), &b = T(r - 1, c);
      hops.push_back({a.k, b.k, std::max(a.ey0, b.ey0), std::min(a.ey1, b.ey1), a.ex0, a.ex1, 0});
    }
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c + 1 < cols; ++c) {
      const Tile &a = T(r, c), &b = T(r, c + 1);
      hops.push_back({a.k, b.k, a.ey0, a.ey1, std::max(a.ex0, b.ex0), std::min(a.ex1, b.ex1), 1});
    }
  for (int r = 0; r < rows; ++r)
    for (int c = cols - 1; c >= 1; --c) {
      const Tile &a = T(r, c), &b = T(r, c - 1);
      hops.push_back({a.k, b.k, a.ey0, a.ey1, std::max(a.ex0, b.ex0), std::min(a.ex1, b.ex1), 0});
    }
}

// Tile rects (readings #13, #14): uniform split, remainder to the last row /
// column, extended rect = interior dilated by halo and clipped to the object.
static void build_tiles(int height, int width, int rows, int cols, int halo, std::vector<Tile>& tiles) {
  tiles.assign(rows * cols, Tile());
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      Tile& t = tiles[r * cols + c];
      t.k = r * cols + c;
      t.r = r;
      t.c = c;
      split(height, rows, r, &t.iy0, &t.iy1);
      split(width, cols, c, &t.ix0, &t.ix1);
      t.ey0 = std::max(0, t.iy0 - halo);
      t.ex0 = std::max(0, t.ix0 - halo);
      t.ey1 = std::min(height, t.iy1 + halo);
      t.ex1 = std::min(width, t.ix1 + halo);
      t.eh = t.ey1 - t.ey0;
      t.ew = t.ex1 - t.ex0;
      t.pitch0 = (t.ew + 31) / 32 * 32;
      t.pitch1 = (t.eh + 31) / 32 * 32;
      const long long a = (long long)t.eh * t.pitch0, b = (long long)t.ew * t.pitch1;
      t.slice_stride = (std::max(a, b) + 31) / 32 * 32;
    }
}

static bool grid_ok(int height, int width, int rows, int cols, int halo) {
  return rows >= 1 && cols >= 1 && rows <= height && cols <= width && halo >= 0;
}

extern "C" ptycho_status ptycho_tile_geometry(int32_t height, int32_t width, int32_t rows, int32_t cols,
                                              int32_t halo, int32_t* rects) {
  ptycho_ctx ctx = nullptr;
  if (!grid_ok(height, width, rows, cols, halo) || !rects) return fail(ctx, PTYCHO_EARG, "bad grid");
  std::vector<Tile> tiles;
  build_tiles(height, width, rows, cols, halo, tiles);
  for (const Tile& t : tiles) {
    int32_t* o = rects + 8 * t.k;
    o[0] = t.ey0; o[1] = t.ex0; o[2] = t.ey1; o[3] = t.ex1;
    o[4] = t.iy0; o[5] = t.ix0; o[6] = t.iy1; o[7] = t.ix1;
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_appp_schedule(int32_t height, int32_t width, int32_t rows, int32_t cols,
                                              int32_t halo, int32_t* hops_out, int32_t max_hops,
                                              int32_t* count) {
  ptycho_ctx ctx = nullptr;
  if (!grid_ok(height, width, rows, cols, halo) || !count) return fail(ctx, PTYCHO_EARG, "bad grid");
  std::vector<Tile> tiles;
  std::vector<Hop> hops;
  build_tiles(height, width, rows, cols, halo, tiles);
  build_hops(tiles, rows, cols, hops);
  *count = (int32_t)hops.size();
  if (hops_out) {
    if (max_hops < (int32_t)hops.size()) return fail(ctx, PTYCHO_EARG, "max_hops < %zu", hops.size());
    for (size_t i = 0; i < hops.size(); ++i) {
      const Hop& h = hops[i];
      int32_t* o = hops_out + 7 * i;
      o[0] = h.src; o[1] = h.dst; o[2] = h.y0; o[3] = h.y1; o[4] = h.x0; o[5] = h.x1; o[6] = h.add;
    }
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_tiles(ptycho_ctx ctx, int32_t rows, int32_t cols, int32_t halo,
                                          const int32_t* tile_owner, const void* nccl_id, int32_t rank,
                                          int32_t nranks) {
  if (!ctx) return PTYCHO_EARG;
  if (ctx->tiles_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles already called");
  const auto& cfg = ctx->cfg;
  if (!grid_ok(cfg.height, cfg.width, rows, cols, halo))
    return fail(ctx, PTYCHO_EARG, "bad grid %dx%d halo %d for object %dx%d", rows, cols, halo, cfg.height, cfg.width);
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, PTYCHO_EARG, "bad rank %d / %d", rank, nranks);
  if (nranks > 1 && !nccl_id) return fail(ctx, PTYCHO_EARG, "nccl_id required when nranks > 1");
  ctx->R = rows;
  ctx->C = cols;
  ctx->halo = halo;
  ctx->rank = rank;
  ctx->nranks = nranks;
  build_tiles(cfg.height, cfg.width, rows, cols, halo, ctx->tiles);
  for (Tile& t : ctx->tiles) {
    t.owner = tile_owner ? tile_owner[t.k] : rank;
    if (t.owner < 0 || t.owner >= nranks) return fail(ctx, PTYCHO_EARG, "tile_owner[%d] = %d", t.k, t.owner);
    if (t.owner == rank) ctx->local.push_back(t.k);
  }
  build_hops(ctx->tiles, rows, cols, ctx->hops);
  CK(cudaSetDevice(ctx->device));
  // At most G = 4 tile chains in flight (PTYCHO_TILE_STREAMS overrides): local tile i uses the
  // stream of local tile i % G.  Each chain's live wavefields are 16 MiB (N = 1024); 4 of them
  // stay in the 126 MB L2 next to the streaming traffic, 8 do not -- LT-small on one B200 with
  // 8 virtual tiles: G = 3..5 452 probe-loc/s, G = 6 439, G = 8 439 (profiles/round1.md).
  int groups = std::min<int>((int)ctx->local.size(), 4);
  if (const char* e = getenv("PTYCHO_TILE_STREAMS")) groups = std::max(1, std::min((int)ctx->local.size(), atoi(e)));
  for (size_t i = 0; i < ctx->local.size(); ++i) {
    Tile& t = ctx->tiles[ctx->local[i]];
    if ((int)i < groups) {
      CK(cudaStreamCreateWithFlags(&t.stream, cudaStreamNonBlocking));
      t.own_stream = true;
    } else {
      t.stream = ctx->tiles[ctx->local[i % groups]].stream;
    }
    CK(cudaEventCreateWithFlags(&t.ev, cudaEventDisableTiming));
  }
  if (nranks > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    NK(ncclCommInitRank(&ctx->comm, nranks, id, rank));
  }
  ctx->tiles_set = true;
  return PTYCHO_OK;
}

// HVE baseline: GD's grid and halo rects, no APPP hops; set_scan assigns duplicates and
// builds the copy-paste list.  Cross-rank exchange messages go over NCCL.
extern "C" ptycho_status ptycho_set_tiles_hve(ptycho_ctx ctx, int32_t rows, int32_t cols, int32_t halo,
                                              int32_t margin, const int32_t* tile_owner, const void* nccl_id,
                                              int32_t rank, int32_t nranks) {
  if (!ctx) return PTYCHO_EARG;
  if (margin < 0) return fail(ctx, PTYCHO_EARG, "margin %d < 0", margin);
  PASS(ptycho_set_tiles(ctx, rows, cols, halo, tile_owner, nccl_id, rank, nranks));
  ctx->hve = true;
  ctx->hve_margin = margin;
  ctx->hops.clear();
  ctx->transport_req = PTYCHO_APPP_NCCL;
  // TileTooSmall: each halo must lie inside the adjacent tiles' interiors
  for (const Tile& t : ctx->tiles) {
    const Tile& up = ctx->tiles[std::max(0, t.r - 1) * cols + t.c];
    const Tile& dn = ctx->tiles[std::min(rows - 1, t.r + 1) * cols + t.c];
    const Tile& lf = ctx->tiles[t.r * cols + std::max(0, t.c - 1)];
    const Tile& rt = ctx->tiles[t.r * cols + std::min(cols - 1, t.c + 1)];
    if (t.ey0 < up.iy0 || t.ey1 > dn.iy1 || t.ex0 < lf.ix0 || t.ex1 > rt.ix1)
      return fail(ctx, PTYCHO_EHALO, "HVE: tile %d's halo %d reaches past its neighbours' interiors (tile too small)",
                  t.k, halo);
  }
  // copy-paste list: tile j's halo voxels inside tile k's interior <- tile k (every pair, k != j)
  for (const Tile& j : ctx->tiles)
    for (const Tile& k : ctx->tiles) {
      if (k.k == j.k) continue;
      Hop h{k.k, j.k, std::max(j.ey0, k.iy0), std::min(j.ey1, k.iy1), std::max(j.ex0, k.ix0), std::min(j.ex1, k.ix1), 0};
      h.vol = 1;
      if (h.y0 < h.y1 && h.x0 < h.x1) ctx->hops.push_back(h);
    }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_scan(ptycho_ctx ctx, const int32_t* centers_yx, int64_t n_probes) {
  if (!ctx) return PTYCHO_EARG;
  if (!ctx->tiles_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles must precede set_scan");
  if (ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_scan already called");
  if (n_probes < 0 || (n_probes > 0 && !centers_yx)) return fail(ctx, PTYCHO_EARG, "bad scan");
  const auto& cfg = ctx->cfg;
  const int n = cfg.n;
  ctx->centers.assign(centers_yx, centers_yx + 2 * n_probes);
  for (int64_t i = 0; i < n_probes; ++i) {
    const int cy = centers_yx[2 * i], cx = centers_yx[2 * i + 1];
    if (cy < 0 || cy >= cfg.height || cx < 0 || cx >= cfg.width)
      return fail(ctx, PTYCHO_EARG, "probe %lld centre (%d,%d) outside the %dx%d object", (long long)i, cy, cx,
                  cfg.height, cfg.width);
    if (ctx->hve) {  // every tile whose interior dilated by the margin holds the centre
      const int m = ctx->hve_margin;
      for (Tile& t : ctx->tiles)
        if (cy >= t.iy0 - m && cy < t.iy1 + m && cx >= t.ix0 - m && cx < t.ix1 + m) t.probes.push_back(i);
      continue;
    }
    // centre containment in half-open interiors (reading #15): row/column by the uniform split
    const int base_y = cfg.height / ctx->R, base_x = cfg.width / ctx->C;
    const int r = std::min(cy / base_y, ctx->R - 1), c = std::min(cx / base_x, ctx->C - 1);
    Tile& t = ctx->tiles[r * ctx->C + c];
    if (cfg.flags & PTYCHO_F_EXACT_WINDOW) {
      const int wy0 = std::max(cy - n / 2, 0), wy1 = std::min(cy - n / 2 + n, cfg.height);
      const int wx0 = std::max(cx - n / 2, 0), wx1 = std::min(cx - n / 2 + n, cfg.width);
      if (wy0 < t.ey0 || wy1 > t.ey1 || wx0 < t.ex0 || wx1 > t.ex1)
        return fail(ctx, PTYCHO_EHALO, "probe %lld window not covered by tile %d's extended rect (halo %d < %d)",
                    (long long)i, t.k, ctx->halo, n / 2);
    }
    t.probes.push_back(i);
  }
  ctx->scan_set = true;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_local_probes(ptycho_ctx ctx, int64_t* ids, int64_t* count) {
  if (!ctx || !count) return PTYCHO_EARG;
  if (!ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_scan first");
  int64_t m = 0;
  for (int k : ctx->local)
    for (int64_t g : ctx->tiles[k].probes) {
      if (ids) ids[m] = g;
      ++m;
    }
  *count = m;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_tile_probe_count(ptycho_ctx ctx, int32_t tile, int64_t* count) {
  if (!ctx || !count) return PTYCHO_EARG;
  if (!ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_scan first");
  if (tile < 0 || tile >= (int)ctx->tiles.size()) return fail(ctx, PTYCHO_EARG, "bad tile %d", tile);
  *count = (int64_t)ctx->tiles[tile].probes.size();
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_tile_rect(ptycho_ctx ctx, int32_t tile, int32_t ext[4], int32_t interior[4]) {
  if (!ctx) return PTYCHO_EARG;
  if (!ctx->tiles_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles first");
  if (tile < 0 || tile >= (int)ctx->tiles.size()) return fail(ctx, PTYCHO_EARG, "bad tile %d", tile);
  const Tile& t = ctx->tiles[tile];
  if (ext) {
    ext[0] = t.ey0; ext[1] = t.ex0; ext[2] = t.ey1; ext[3] = t.ex1;
  }
  if (interior) {
    interior[0] = t.iy0; interior[1] = t.ix0; interior[2] = t.iy1; interior[3] = t.ix1;
  }
  return PTYCHO_OK;
}

// ------------------------------------------------------------------------------------------
// workspace
// ------------------------------------------------------------------------------------------
static size_t plan_workspace(ptycho_ctx ctx, bool carve) {
  const auto& cfg = ctx->cfg;
  const size_t n = cfg.n, n2 = n * n, S = cfg.slices;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* p = carve ? ctx->ws + off : nullptr;
    off = align_up(off + bytes);
    return p;
  };
  ctx->wtab = (float2*)take(ctx->h_wtab.size() * sizeof(float2));
  ctx->htab = (float2*)take(n * sizeof(float2));
  ctx->probe = (float2*)take(n2 * sizeof(float2));
  ctx->dscratch = (double*)take(64 * sizeof(double));
  ctx->iscratch = (int*)take(64 * sizeof(int));
  ctx->staging_floats = std::max<size_t>((size_t)cfg.height * cfg.width, 8 * n2);
  ctx->staging = (float*)take(ctx->staging_floats * sizeof(float));
  ctx->debug_floats = std::max<size_t>(S, 2) * n2;
  ctx->debug = (float*)take(ctx->debug_floats * sizeof(float));
  if (ctx->nranks > 1) {
    size_t mx = 0;
    for (const Hop& h : ctx->hops) {
      const size_t area = (size_t)std::max(0, h.y1 - h.y0) * std::max(0, h.x1 - h.x0);
      mx = std::max(mx, area);
    }
    for (const Tile& t : ctx->tiles) mx = std::max(mx, (size_t)(t.iy1 - t.iy0) * (t.ix1 - t.ix0));
    // messages are slabs of whole slices, at least one slice, at most ~64 MB
    ctx->msg_floats = std::max(mx, (size_t)(16u << 20));
    ctx->sendbuf = (float*)take(ctx->msg_floats * sizeof(float));
    ctx->recvbuf = (float*)take(ctx->msg_floats * sizeof(float));
    ctx->flags = (unsigned*)take(2 * std::max<size_t>(ctx->hops.size(), 1) * sizeof(unsigned));
  }
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const size_t vol = (size_t)t.slice_stride * S;
    t.V = (float*)take(vol * sizeof(float));
    t.acc = ctx->hve ? nullptr : (float*)take(vol * sizeof(float));  // HVE keeps no AccBuf
    const size_t B = (size_t)ctx->batch;
    t.stash = (float2*)take(B * stash_slices(cfg) * n2 * sizeof(float2));
    t.wf[0] = (float2*)take(B * n2 * sizeof(float2));
    t.wf[1] = (float2*)take(B * n2 * sizeof(float2));
    if (stash_free(cfg)) {
      t.wfr[0] = (float2*)take(B * n2 * sizeof(float2));
      t.wfr[1] = (float2*)take(B * n2 * sizeof(float2));
    }
    t.order = (int*)take(std::max<size_t>(t.probes.size(), 1) * sizeof(int));
    t.amp = (float*)take(std::max<size_t>(t.probes.size(), 1) * n2 * sizeof(float));
    t.centers = (int2*)take(std::max<size_t>(t.probes.size(), 1) * sizeof(int2));
    t.desc = (int4*)take(B * sizeof(int4));
    t.tm_dev = (CUtensorMap*)take(8 * sizeof(CUtensorMap));
    t.done = (unsigned*)take(sizeof(unsigned));
    t.loss_part = (double*)take(B * (n / LINES_PER_CTA) * sizeof(double));
  }
  return off;
}

extern "C" ptycho_status ptycho_workspace_bytes(ptycho_ctx ctx, size_t* bytes) {
  if (!ctx || !bytes) return PTYCHO_EARG;
  if (!ctx->tiles_set || !ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles and set_scan first");
  *bytes = plan_workspace(ctx, false);
  return PTYCHO_OK;
}

static ptycho_status zero_tiles(ptycho_ctx ctx, bool v, bool a) {
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const size_t vol = (size_t)t.slice_stride * ctx->cfg.slices;
    if (v) CK(cudaMemsetAsync(t.V, 0, vol * sizeof(float), ctx->stream));
    if (a && t.acc) CK(cudaMemsetAsync(t.acc, 0, vol * sizeof(float), ctx->stream));
  }
  return PTYCHO_OK;
}

// TMA descriptors: slice parity p of a tile buffer as a 3-D tensor
// {position along the line, line, slice / 2} with the layout's row pitch and 2 slice strides;
// box = one line segment of min(N, 256) floats.  OOB: zero fill (loads) / clipped (stores).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static ptycho_status make_tensor_maps(ptycho_ctx ctx, const Tile& t, float* buf, CUtensorMap out[2], int box0) {
  static EncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        !encode)
      return fail(ctx, PTYCHO_ECUDA, "cuTensorMapEncodeTiled unavailable");
  }
  const int S = ctx->cfg.slices, n = ctx->cfg.n;
  const cuuint32_t box[3] = {(cuuint32_t)box0, 1, 1}, es[3] = {1, 1, 1};
  (void)n;
  for (int par = 0; par < 2; ++par) {
    const cuuint64_t nz = (cuuint64_t)std::max(1, par == 0 ? (S + 1) / 2 : S / 2);
    const cuuint64_t dims[3] = {(cuuint64_t)(par == 0 ? t.ew : t.eh), (cuuint64_t)(par == 0 ? t.eh : t.ew), nz};
    const cuuint64_t strides[2] = {(cuuint64_t)(par == 0 ? t.pitch0 : t.pitch1) * 4, (cuuint64_t)t.slice_stride * 8};
    float* base = buf + (par == 0 ? 0 : (S > 1 ? t.slice_stride : 0));
    const CUresult r = encode(&out[par], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(ctx, PTYCHO_ECUDA, "cuTensorMapEncodeTiled(tile %d, parity %d): error %d", t.k, par, (int)r);
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_workspace(ptycho_ctx ctx, void* workspace_dev, size_t bytes) {
  if (!ctx) return PTYCHO_EARG;
  if (!ctx->tiles_set || !ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles and set_scan first");
  if (ctx->ws_set) return fail(ctx, PTYCHO_ESTATE, "set_workspace already called");
  if (!workspace_dev || ((uintptr_t)workspace_dev % ALIGN)) return fail(ctx, PTYCHO_EARG, "workspace must be 256-B aligned");
  const size_t need = plan_workspace(ctx, false);
  if (bytes < need) return fail(ctx, PTYCHO_ENOMEM, "workspace %zu B < required %zu B", bytes, need);
  CK(cudaSetDevice(ctx->device));
  ctx->ws = (char*)workspace_dev;
  ctx->ws_bytes = bytes;
  plan_workspace(ctx, true);
  const size_t n = ctx->cfg.n;
  CK(cudaMemcpyAsync(ctx->wtab, ctx->h_wtab.data(), ctx->h_wtab.size() * sizeof(float2), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(ctx->htab, ctx->h_htab.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
#ifndef PTYCHO_TMA_BOX
#define PTYCHO_TMA_BOX 256
#endif
    // main box = min(N, 256) floats (kernels.cu tma_box), tail box = 4 floats (16 B); AccBuf maps
    // alias V's in HVE contexts (no AccBuf, never dereferenced)
    CUtensorMap h[8];
    const int bmain = std::min((int)n, PTYCHO_TMA_BOX);
    PASS(make_tensor_maps(ctx, t, t.V, h + 0, bmain));
    PASS(make_tensor_maps(ctx, t, t.acc ? t.acc : t.V, h + 2, bmain));
    PASS(make_tensor_maps(ctx, t, t.V, h + 4, 4));
    PASS(make_tensor_maps(ctx, t, t.acc ? t.acc : t.V, h + 6, 4));
    CK(cudaMemcpy(t.tm_dev, h, sizeof h, cudaMemcpyHostToDevice));
    std::vector<int2> hc(std::max<size_t>(t.probes.size(), 1), make_int2(0, 0));
    for (size_t j = 0; j < t.probes.size(); ++j)
      hc[j] = make_int2(ctx->centers[2 * t.probes[j]], ctx->centers[2 * t.probes[j] + 1]);
    CK(cudaMemcpyAsync(t.centers, hc.data(), hc.size() * sizeof(int2), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(t.desc, 0, ctx->batch * sizeof(int4), ctx->stream));
    CK(cudaMemsetAsync(t.done, 0, sizeof(unsigned), ctx->stream));
    CK(cudaMemsetAsync(t.loss_part, 0, ctx->batch * (n / LINES_PER_CTA) * sizeof(double), ctx->stream));
    CK(cudaMemsetAsync(t.amp, 0, std::max<size_t>(t.probes.size(), 1) * n * n * sizeof(float), ctx->stream));
  }
  CK(cudaMemsetAsync(ctx->iscratch, 0, 64 * sizeof(int), ctx->stream));
  PASS(zero_tiles(ctx, true, true));
  if (ctx->flags) CK(cudaMemsetAsync(ctx->flags, 0, 2 * std::max<size_t>(ctx->hops.size(), 1) * sizeof(unsigned),
                                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // host vectors above go out of scope
  ctx->ws_set = true;
  return PTYCHO_OK;
}

static ptycho_status need_ws(ptycho_ctx ctx) {
  if (!ctx) return PTYCHO_EARG;
  if (!ctx->ws_set) return fail(ctx, PTYCHO_ESTATE, "set_workspace first");
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_probe(ptycho_ctx ctx, const void* probe_c64, int on_device) {
  PASS(need_ws(ctx));
  if (!probe_c64) return fail(ctx, PTYCHO_EARG, "probe is NULL");
  const size_t n2 = (size_t)ctx->cfg.n * ctx->cfg.n;
  CK(cudaSetDevice(ctx->device));
  std::vector<float2> h(n2);
  if (on_device) CK(cudaMemcpy(h.data(), probe_c64, n2 * sizeof(float2), cudaMemcpyDeviceToHost));
  else memcpy(h.data(), probe_c64, n2 * sizeof(float2));
  double nrm = 0.0;
  for (auto& v : h) nrm += (double)v.x * v.x + (double)v.y * v.y;
  ctx->probe_norm = std::sqrt(nrm);
  CK(cudaMemcpyAsync(ctx->probe, h.data(), n2 * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->probe_set = true;
  return PTYCHO_OK;
}

// Asynchronous host load straight into the measurement stores (no staging, no layout change): on
// the copy stream, after every earlier reader of the stores; one event per chunk of probes.
static ptycho_status load_async(ptycho_ctx ctx, const float* amp, int64_t first_local, int64_t count) {
  const size_t n2 = (size_t)ctx->cfg.n * ctx->cfg.n;
  if (!ctx->copy_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_copy, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(ctx->ev_copy, ctx->stream));  // e.g. set_workspace's clearing of the stores
  CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_copy, 0));
  int64_t chunk = 8;  // probes per event (32 MiB at N = 1024)
  if (const char* e = getenv("PTYCHO_AMP_CHUNK")) chunk = std::max(1, atoi(e));
  // pinned host input with a device alias: upload kernels on the copy stream (events of a compute
  // stream), else copy-engine copies (PTYCHO_AMP_CE=1 forces them)
  const float* amp_dev = nullptr;
  {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, amp) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer &&
        ((uintptr_t)at.devicePointer & 15) == 0 && !getenv("PTYCHO_AMP_CE"))
      amp_dev = (const float*)at.devicePointer;
    cudaGetLastError();
  }
  int up_ctas = 8;
  if (const char* e = getenv("PTYCHO_AMP_UPLOAD_CTAS")) up_ctas = std::max(1, atoi(e));
  struct Range {
    Tile* t;
    int64_t g, lo, hi;
  };
  std::vector<Range> rs;
  int64_t g = 0;
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t nk = (int64_t)t.probes.size();
    const int64_t lo = std::max(first_local, g), hi = std::min(first_local + count, g + nk);
    if (lo < hi) {
      // chunks of an earlier load not yet consumed: later chains wait for all of them
      while (t.amp_cur < t.amp_pend.size()) CK(cudaStreamWaitEvent(t.stream, t.amp_pend[t.amp_cur++].ev, 0));
      t.amp_pend.clear();
      t.amp_cur = 0;
      if (!t.amp_free) CK(cudaEventCreateWithFlags(&t.amp_free, cudaEventDisableTiming));
      CK(cudaEventRecord(t.amp_free, t.stream));  // chains still reading the store finish first
      CK(cudaStreamWaitEvent(ctx->copy_stream, t.amp_free, 0));
      rs.push_back({&t, g, lo, hi});
    }
    g += nk;
  }
  // round-robin over the tiles (the tiles' chains run concurrently and consume in probe order)
  for (size_t ne = 0;; ++ne) {
    bool any = false;
    for (Range& r : rs) {
      const int64_t p = r.lo + (int64_t)ne * chunk;
      if (p >= r.hi) continue;
      any = true;
      Tile& t = *r.t;
      const int64_t m = std::min(chunk, r.hi - p);
      if (amp_dev) {
        CK(launch_upload(t.amp + (size_t)(p - r.g) * n2, amp_dev + (size_t)(p - first_local) * n2,
                         (long long)m * (long long)n2, up_ctas, ctx->copy_stream));
        ++ctx->launches;
      } else {
        CK(cudaMemcpyAsync(t.amp + (size_t)(p - r.g) * n2, amp + (size_t)(p - first_local) * n2,
                           (size_t)m * n2 * sizeof(float), cudaMemcpyHostToDevice, ctx->copy_stream));
      }
      if (ne == t.amp_pool.size()) {
        t.amp_pool.push_back(nullptr);
        CK(cudaEventCreateWithFlags(&t.amp_pool.back(), cudaEventDisableTiming));
      }
      CK(cudaEventRecord(t.amp_pool[ne], ctx->copy_stream));
      t.amp_pend.push_back({p - r.g, t.amp_pool[ne]});
    }
    if (!any) break;
  }
  return PTYCHO_OK;
}

// Stream st waits for the pending asynchronous chunks of tile t that hold probes <= upto.
static ptycho_status amp_wait(ptycho_ctx ctx, Tile& t, int64_t upto, cudaStream_t st) {
  while (t.amp_cur < t.amp_pend.size() && t.amp_pend[t.amp_cur].begin <= upto)
    CK(cudaStreamWaitEvent(st, t.amp_pend[t.amp_cur++].ev, 0));
  if (t.amp_cur == t.amp_pend.size()) {
    t.amp_pend.clear();
    t.amp_cur = 0;
  }
  return PTYCHO_OK;
}

// Stream st waits for every pending asynchronous chunk of every local tile.
static ptycho_status amp_settle(ptycho_ctx ctx, cudaStream_t st) {
  for (int k : ctx->local) PASS(amp_wait(ctx, ctx->tiles[k], INT64_MAX, st));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_load_measurements(ptycho_ctx ctx, const float* amp, int on_device,
                                                  int64_t first_local, int64_t count, int32_t layout_flags) {
  PASS(need_ws(ctx));
  int64_t nloc = 0;
  for (int k : ctx->local) nloc += (int64_t)ctx->tiles[k].probes.size();
  if (count < 0 || first_local < 0 || first_local + count > nloc)
    return fail(ctx, PTYCHO_EARG, "range [%lld, %lld) outside the %lld local probes", (long long)first_local,
                (long long)(first_local + count), (long long)nloc);
  if (count == 0) return PTYCHO_OK;
  if (!amp) return fail(ctx, PTYCHO_EARG, "amp is NULL");
  CK(cudaSetDevice(ctx->device));
  const int n = ctx->cfg.n;
  const size_t n2 = (size_t)n * n;
  const int shift = (layout_flags & PTYCHO_AMP_DC_CENTERED) ? 1 : 0;
  const int inten = (layout_flags & PTYCHO_AMP_INTENSITY) ? 1 : 0;
  const int transpose = ctx->cfg.slices & 1;  // store in the turnaround pass's layout L_{S&1}
  if ((layout_flags & PTYCHO_AMP_ASYNC) && !on_device && !shift && !inten && !transpose)
    return load_async(ctx, amp, first_local, count);
  PASS(amp_settle(ctx, ctx->stream));  // earlier asynchronous copies land before this load
  const int64_t chunk = (int64_t)(ctx->staging_floats / n2);
  int64_t g = 0;  // local index of the first probe of the current tile
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t nk = (int64_t)t.probes.size();
    const int64_t lo = std::max(first_local, g), hi = std::min(first_local + count, g + nk);
    for (int64_t p = lo; p < hi;) {
      const int64_t m = on_device ? (hi - p) : std::min(chunk, hi - p);
      const float* src = amp + (size_t)(p - first_local) * n2;
      if (!on_device) {
        CK(cudaMemcpyAsync(ctx->staging, src, (size_t)m * n2 * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        src = ctx->staging;
      }
      CK(launch_amp_load(t.amp + (size_t)(p - g) * n2, src, (int)m, n, shift, inten, transpose, ctx->stream));
      ++ctx->launches;
      p += m;
    }
    g += nk;
  }
  if (!on_device) CK(cudaStreamSynchronize(ctx->stream));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_read_measurements(ptycho_ctx ctx, float* amp_out, int64_t first_local,
                                                  int64_t count) {
  PASS(need_ws(ctx));
  int64_t nloc = 0;
  for (int k : ctx->local) nloc += (int64_t)ctx->tiles[k].probes.size();
  if (count < 0 || first_local < 0 || first_local + count > nloc) return fail(ctx, PTYCHO_EARG, "bad range");
  if (count == 0) return PTYCHO_OK;
  if (!amp_out) return fail(ctx, PTYCHO_EARG, "amp_out is NULL");
  CK(cudaSetDevice(ctx->device));
  if (ctx->copy_stream) CK(cudaStreamSynchronize(ctx->copy_stream));
  for (int k : ctx->local) CK(cudaStreamSynchronize(ctx->tiles[k].stream));
  const int n = ctx->cfg.n;
  const size_t n2 = (size_t)n * n;
  const int64_t chunk = (int64_t)(ctx->staging_floats / n2);
  int64_t g = 0;
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t nk = (int64_t)t.probes.size();
    const int64_t lo = std::max(first_local, g), hi = std::min(first_local + count, g + nk);
    for (int64_t p = lo; p < hi;) {
      const int64_t m = std::min(chunk, hi - p);
      CK(launch_amp_load(ctx->staging, t.amp + (size_t)(p - g) * n2, (int)m, n, 0, 0, ctx->cfg.slices & 1, ctx->stream));
      ++ctx->launches;
      CK(cudaMemcpyAsync(amp_out + (size_t)(p - first_local) * n2, ctx->staging, (size_t)m * n2 * sizeof(float),
                         cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      p += m;
    }
    g += nk;
  }
  return PTYCHO_OK;
}

// slice pointers / region helpers for the alternating per-slice layout
struct SliceView {
  float* base;       // first element of the region in the first slice of this parity
  long long ld;      // row pitch
  long long ss;      // stride between slices of this parity (2 * slice_stride)
  int rows, cols, nslices;
};

// Region [y0,y1)x[x0,x1) of the slices s in [z0, z1) with s % 2 == parity.
static SliceView region_view(const Tile& t, float* buf, int parity, int z0, int z1, int y0, int y1, int x0,
                             int x1) {
  SliceView v;
  v.ss = 2 * t.slice_stride;
  const int s0 = z0 + (((z0 & 1) != parity) ? 1 : 0);
  v.nslices = s0 < z1 ? (z1 - s0 + 1) / 2 : 0;
  const long long sb = (long long)s0 * t.slice_stride;
  if (parity == 0) {
    v.base = buf + sb + (long long)(y0 - t.ey0) * t.pitch0 + (x0 - t.ex0);
    v.ld = t.pitch0;
    v.rows = y1 - y0;
    v.cols = x1 - x0;
  } else {
    v.base = buf + sb + (long long)(x0 - t.ex0) * t.pitch1 + (y0 - t.ey0);
    v.ld = t.pitch1;
    v.rows = x1 - x0;
    v.cols = y1 - y0;
  }
  return v;
}

// global slice [H][W] (row pitch W) <-> tile slice s on the rect [y0,y1)x[x0,x1)
static ptycho_status global_to_tile(ptycho_ctx ctx, const Tile& t, float* buf, int s, const float* g, int y0, int y1,
                                    int x0, int x1) {
  const int W = ctx->cfg.width;
  float* sl = buf + (long long)s * t.slice_stride;
  const float* gp = g + (long long)y0 * W + x0;
  if ((s & 1) == 0) {
    CK(launch_copy2d(sl + (long long)(y0 - t.ey0) * t.pitch0 + (x0 - t.ex0), t.pitch0, 0, gp, W, 0, y1 - y0, x1 - x0,
                     1, 0, ctx->stream));
  } else {  // tile[x][y] = g[y][x]
    CK(launch_transpose2d(sl + (long long)(x0 - t.ex0) * t.pitch1 + (y0 - t.ey0), t.pitch1, 0, gp, W, 0, x1 - x0,
                          y1 - y0, 1, 0, ctx->stream));
  }
  ++ctx->launches;
  return PTYCHO_OK;
}

static ptycho_status tile_to_global(ptycho_ctx ctx, const Tile& t, const float* buf, int s, float* g, int y0, int y1,
                                    int x0, int x1) {
  const int W = ctx->cfg.width;
  const float* sl = buf + (long long)s * t.slice_stride;
  float* gp = g + (long long)y0 * W + x0;
  if ((s & 1) == 0) {
    CK(launch_copy2d(gp, W, 0, sl + (long long)(y0 - t.ey0) * t.pitch0 + (x0 - t.ex0), t.pitch0, 0, y1 - y0, x1 - x0,
                     1, 0, ctx->stream));
  } else {  // g[y][x] = tile[x][y]
    CK(launch_transpose2d(gp, W, 0, sl + (long long)(x0 - t.ex0) * t.pitch1 + (y0 - t.ey0), t.pitch1, 0, y1 - y0,
                          x1 - x0, 1, 0, ctx->stream));
  }
  ++ctx->launches;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_volume(ptycho_ctx ctx, const float* volume, int on_device) {
  PASS(need_ws(ctx));
  CK(cudaSetDevice(ctx->device));
  const auto& cfg = ctx->cfg;
  PASS(zero_tiles(ctx, true, true));
  if (!volume) return PTYCHO_OK;  // V_0 = 0
  const size_t hw = (size_t)cfg.height * cfg.width;
  for (int s = 0; s < cfg.slices; ++s) {
    const float* g = volume + (size_t)s * hw;
    if (!on_device) {
      CK(cudaMemcpyAsync(ctx->staging, g, hw * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
      g = ctx->staging;
    }
    for (int k : ctx->local) {
      const Tile& t = ctx->tiles[k];
      PASS(global_to_tile(ctx, t, t.V, s, g, t.ey0, t.ey1, t.ex0, t.ex1));
    }
    if (!on_device) CK(cudaStreamSynchronize(ctx->stream));
  }
  return PTYCHO_OK;
}

// ------------------------------------------------------------------------------------------
// the per-probe pass chain (DESIGN.md §Pass schedule): 2S+1 kernels
// ------------------------------------------------------------------------------------------
enum ChainMode { CHAIN_GRAD = 0, CHAIN_SIMULATE, CHAIN_DEBUG_GRAD, CHAIN_DEBUG_EXIT, CHAIN_BATCH };

static PassArgs base_args(ptycho_ctx ctx, const Tile& t) {
  PassArgs a{};
  a.V = t.V;
  a.acc = t.acc;
  a.slice_stride = t.slice_stride;
  a.pitch0 = t.pitch0;
  a.pitch1 = t.pitch1;
  a.ey0 = t.ey0;
  a.ex0 = t.ex0;
  a.eh = t.eh;
  a.ew = t.ew;
  a.stash = t.stash;
  a.probe = ctx->probe;
  a.amp = t.amp;
  a.centers = t.centers;
  a.desc = t.desc;
  a.n_probes = (int)t.probes.size();
  a.done = t.done;
  a.loss_part = t.loss_part;
  a.wtab = ctx->wtab;
  a.htab = ctx->htab;
  a.sigma = ctx->cfg.sigma;
  a.sigma_pi = (float)((double)ctx->cfg.sigma / M_PI);
  a.alpha = ctx->cfg.alpha;
  a.thr = (float)(ctx->cfg.tau * ctx->probe_norm / ctx->cfg.n);
  // >= 2 tile chains share the GPU: the forward-pass build with room for more CTAs (same-box A/B,
  // LT-small: 1 chain 374 vs 329 probe-loc/s for the 2-CTA build; 2 chains 446 vs 430 and 8 tiles
  // 452 vs 425 for the 3-CTA build)
  a.high_occupancy = ctx->local.size() >= 2 ? 1 : 0;
  if (const char* e = getenv("PTYCHO_HIGH_OCC")) a.high_occupancy = atoi(e) != 0;  // A/B override
  a.batch = 1;  // the batched graph overrides (set_schedule)
  a.stash_slot = (long long)stash_slices(ctx->cfg) * ctx->cfg.n * ctx->cfg.n;
  a.stash_store = 1;
  a.wf_slot = (long long)ctx->cfg.n * ctx->cfg.n;
  a.no_acc = ctx->hve ? 1 : 0;
  a.dbg = (unsigned*)(ctx->iscratch + 32);  // error bits of PTYCHO_DEBUG_CHECKS builds
  return a;
}

struct ChainProfile {  // optional per-kind event timing (ptycho_profile_chain)
  std::vector<cudaEvent_t> ev;
  std::vector<int> kind;
};

static ptycho_status enqueue_chain(ptycho_ctx ctx, Tile& t, ChainMode mode, cudaStream_t st,
                                   ChainProfile* prof = nullptr, std::vector<cudaEvent_t>* slab_ev = nullptr,
                                   int slab = 0) {
  const int S = ctx->cfg.slices, n = ctx->cfg.n;
  PassArgs a = base_args(ctx, t);
  const bool ring = stash_free(ctx->cfg) && (mode == CHAIN_GRAD || mode == CHAIN_DEBUG_GRAD || mode == CHAIN_BATCH);
  int pass = 0, rpass = 0;  // chi chain / phi chain (stash-free) ping-pong positions
  auto go = [&](PassKind kind, int s, bool last) -> ptycho_status {
    PassArgs b = a;
    b.s = s;
    b.tmV = t.tm_dev + (s & 1);
    b.tmA = t.tm_dev + 2 + (s & 1);
    const bool recon = kind == K_RECON_FIRST || kind == K_RECON_MID || kind == K_RECON_END;
    b.stash_s = ring ? (s & 1) : s;
    // stash-free: the forward keeps only phi_{S-1}; the phi chain recomputes the others
    if (ring && (kind == K_FWD_FIRST_PROP || kind == K_FWD_MID)) b.stash_store = 0;
    if (recon) {
      b.in = t.wfr[rpass & 1];
      b.out = t.wfr[(rpass + 1) & 1];
    } else {
      b.in = t.wf[pass & 1];
      b.out = t.wf[(pass + 1) & 1];
    }
    b.advance = (last && (mode == CHAIN_GRAD || mode == CHAIN_SIMULATE)) ? 1 : 0;
    if (mode == CHAIN_BATCH) b.batch = ctx->batch;  // descriptors set per batch by the host
    if (mode == CHAIN_DEBUG_GRAD) b.gexport = ctx->debug;
    if (mode == CHAIN_DEBUG_EXIT) {
      b.natural_out = (float2*)ctx->debug;
      b.natural_transposed = S & 1;
    }
    if (prof) {
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      CK(cudaEventRecord(e0, st));
      CK(launch_pass(n, kind, b, st, false));
      CK(cudaEventRecord(e1, st));
      prof->ev.push_back(e0);
      prof->ev.push_back(e1);
      prof->kind.push_back((int)kind);
    } else {
      CK(launch_pass(n, kind, b, st, ctx->use_pdl));
      if (ctx->debug_sync) {  // PTYCHO_DEBUG_SYNC=1: name the pass that faults (not during capture)
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(ctx, PTYCHO_ECUDA, "pass kind %d slice %d: %s", (int)kind, s, cudaGetErrorString(e));
      }
    }
    ++ctx->launches;
    const bool bwd = kind == K_BWD_LAST_PROP || kind == K_BWD_LAST_END || kind == K_BWD_MID || kind == K_BWD_END;
    if (slab_ev && bwd && s % slab == 0) CK(cudaEventRecord((*slab_ev)[s / slab], st));
    if (recon) ++rpass;
    else ++pass;
    return PTYCHO_OK;
  };
  // forward: pass s finishes psi_s's propagation along its axis, transmits, starts the next
  const bool exit_mode = (mode == CHAIN_DEBUG_EXIT);
  if (S == 1) {
    PASS(go(exit_mode ? K_FWD_FIRST_PROP : K_FWD_FIRST_FFT, 0, false));
  } else {
    PASS(go(K_FWD_FIRST_PROP, 0, false));
    for (int s = 1; s < S - 1; ++s) PASS(go(K_FWD_MID, s, false));
    PASS(go(exit_mode ? K_FWD_MID : K_FWD_LAST, S - 1, false));
  }
  if (exit_mode) return go(K_EXIT_COMPLETE, S, true);
  if (mode == CHAIN_SIMULATE) return go(K_SIMULATE, S, true);
  PASS(go(K_TURN, S, false));
  if (S == 1) return go(K_BWD_LAST_END, 0, true);
  if (!ring) {
    PASS(go(K_BWD_LAST_PROP, S - 1, false));
    for (int s = S - 2; s >= 1; --s) PASS(go(K_BWD_MID, s, false));
    return go(K_BWD_END, 0, true);
  }
  // Stash-free adjoint: phi_{s-1} = P^H(conj(t_s) phi_s), from the stashed
  // phi_{S-1}.  The phi chain runs one slice ahead of the gradient chain, so every stash-ring
  // slot a gradient pass prefetches (before griddepcontrol.wait) was written >= 2 kernels earlier,
  // and RECON(s) reads V_s before the gradient pass of slice s updates it.
  auto recon = [&](int s) { return go(s == 0 ? K_RECON_END : K_RECON_MID, s, false); };
  PASS(go(K_RECON_FIRST, S - 1, false));
  PASS(recon(S - 2));
  PASS(go(K_BWD_LAST_PROP, S - 1, false));
  for (int s = S - 2; s >= 1; --s) {
    PASS(recon(s - 1));
    PASS(go(K_BWD_MID, s, false));
  }
  return go(K_BWD_END, 0, true);
}

static int chain_len(int S, bool ring = false) { return 2 * S + 1 + (ring && S > 1 ? S : 0); }

static ptycho_status ensure_graph(ptycho_ctx ctx, Tile& t, ChainMode mode = CHAIN_GRAD) {
  cudaGraphExec_t* slot = mode == CHAIN_BATCH ? &t.graph_b : &t.graph;
  if (*slot || !ctx->use_graph) return PTYCHO_OK;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(t.stream, cudaStreamCaptureModeThreadLocal));
  const long long before = ctx->launches;
  ptycho_status st = enqueue_chain(ctx, t, mode, t.stream);
  cudaError_t e = cudaStreamEndCapture(t.stream, &g);
  ctx->launches = before;  // captured, not launched
  if (st != PTYCHO_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  CK(e);
  e = cudaGraphInstantiateWithFlags(slot, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  return PTYCHO_OK;
}

// Batched schedule (north_star item 3): local probes [first, first+m) of tile t
// in batches of pairwise non-overlapping windows.  Round of probe i = 1 + the largest round of an
// earlier probe whose window (clipped to R_k) meets it; a round's probes, ascending, are split
// into batches of at most `batch`.  Every voxel then sees the updates of the probes covering it in
// ascending index order, and every probe reads V after all earlier overlapping probes -> results
// bit-identical to the sequential schedule (V, AccBuf).
static void make_batches(ptycho_ctx ctx, Tile& t, int64_t first, int64_t m) {
  if (t.bfirst == first && t.bcount == m) return;
  const int n = ctx->cfg.n;
  std::vector<int> y0(m), y1(m), x0(m), x1(m), round(m, 0);
  int nround = 0;
  for (int64_t i = 0; i < m; ++i) {
    const int64_t g = t.probes[first + i];
    const int cy = ctx->centers[2 * g], cx = ctx->centers[2 * g + 1];
    y0[i] = std::max(cy - n / 2, t.ey0);
    y1[i] = std::min(cy - n / 2 + n, t.ey1);
    x0[i] = std::max(cx - n / 2, t.ex0);
    x1[i] = std::min(cx - n / 2 + n, t.ex1);
    int r = 0;
    for (int64_t j = 0; j < i; ++j)
      if (round[j] >= r && y0[j] < y1[i] && y0[i] < y1[j] && x0[j] < x1[i] && x0[i] < x1[j]) r = round[j] + 1;
    round[i] = r;
    nround = std::max(nround, r + 1);
  }
  t.batches.clear();
  std::vector<std::vector<int>> byr(nround);
  for (int64_t i = 0; i < m; ++i) byr[round[i]].push_back((int)(first + i));
  for (auto& r : byr)
    for (size_t o = 0; o < r.size(); o += ctx->batch)
      t.batches.emplace_back(r.begin() + o, r.begin() + std::min(r.size(), o + (size_t)ctx->batch));
  t.bfirst = first;
  t.bcount = m;
}

static ptycho_status run_batched(ptycho_ctx ctx, int64_t first, int64_t count);

static ptycho_status set_cursor(ptycho_ctx ctx, Tile& t, int v, cudaStream_t st) {
  CK(launch_set_desc(t.desc, t.centers, v, (int)t.probes.size(), ctx->cfg.n, st));
  ++ctx->launches;
  return PTYCHO_OK;
}

static ptycho_status fork_tiles(ptycho_ctx ctx) {
  CK(cudaEventRecord(ctx->ev_fork, ctx->stream));
  for (int k : ctx->local) CK(cudaStreamWaitEvent(ctx->tiles[k].stream, ctx->ev_fork, 0));
  return PTYCHO_OK;
}

static ptycho_status join_tiles(ptycho_ctx ctx) {
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    CK(cudaEventRecord(t.ev, t.stream));
    CK(cudaStreamWaitEvent(ctx->stream, t.ev, 0));
  }
  return PTYCHO_OK;
}

static ptycho_status need_run(ptycho_ctx ctx) {
  PASS(need_ws(ctx));
  if (!ctx->probe_set) return fail(ctx, PTYCHO_ESTATE, "set_probe first");
  return PTYCHO_OK;
}

static ptycho_status sum_loss(ptycho_ctx ctx, double* out_host) {
  // fixed-order sum: per tile (deterministic kernel), then tiles in increasing index on the host
  const int parts = ctx->batch * (ctx->cfg.n / LINES_PER_CTA);
  int j = 0;
  for (int k : ctx->local) {
    CK(launch_sum_double(ctx->tiles[k].loss_part, parts, ctx->dscratch + j, ctx->stream));
    ++ctx->launches;
    ++j;
  }
  std::vector<double> h(std::max(j, 1), 0.0);
  if (j) CK(cudaMemcpyAsync(h.data(), ctx->dscratch, j * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  PASS(check_p2p(ctx));
  double tot = 0.0;
  for (int i = 0; i < j; ++i) tot += h[i];
  *out_host = tot;
  return PTYCHO_OK;
}

static ptycho_status zero_loss(ptycho_ctx ctx) {
  for (int k : ctx->local)
    CK(cudaMemsetAsync(ctx->tiles[k].loss_part, 0, ctx->batch * (ctx->cfg.n / LINES_PER_CTA) * sizeof(double),
                       ctx->stream));
  return PTYCHO_OK;
}

// Probes [first, first + cnt[k]) of every local tile k in one cooperative chain-kernel launch on
// ctx->stream (tiles in lockstep; a tile with fewer probes idles in the later steps).
static ptycho_status run_chain_kernel(ptycho_ctx ctx, int64_t first, const std::vector<int64_t>& cnt) {
  ChainArgs c{};
  int64_t maxn = 0;
  int nt = 0;
  for (int k : ctx->local) {
    if (nt == MAX_CHAIN_TILES) return fail(ctx, PTYCHO_EARG, "persistent chain: more than %d local tiles", MAX_CHAIN_TILES);
    Tile& t = ctx->tiles[k];
    c.t[nt] = base_args(ctx, t);
    c.t[nt].high_occupancy = 0;
    c.wf[nt][0] = t.wf[0];
    c.wf[nt][1] = t.wf[1];
    c.count[nt] = (int)cnt[k];
    maxn = std::max(maxn, cnt[k]);
    ++nt;
  }
  if (maxn == 0) return PTYCHO_OK;
  c.ntiles = nt;
  c.first = (int)first;
  c.maxn = (int)maxn;
  c.S = ctx->cfg.slices;
  c.bar = (unsigned*)ctx->iscratch;
  PASS(amp_settle(ctx, ctx->stream));
  CK(cudaMemsetAsync(ctx->iscratch, 0, sizeof(unsigned), ctx->stream));
  CK(launch_chain(ctx->cfg.n, c, ctx->stream));
  ctx->launches += 1;
  return PTYCHO_OK;
}

// Probes [first, first + cnt[k]) of every local tile k in cluster-resident chains (one 16-CTA
// cluster per tile, up to MAX_CHAIN_TILES tiles per launch) on ctx->stream.
static ptycho_status run_cluster_chain(ptycho_ctx ctx, int64_t first, int64_t count) {
  PASS(amp_settle(ctx, ctx->stream));
  ChainArgs c{};
  int nt = 0;
  auto flush = [&]() -> ptycho_status {
    if (nt == 0) return PTYCHO_OK;
    c.ntiles = nt;
    c.first = (int)first;
    c.S = ctx->cfg.slices;
    CK(launch_cluster(ctx->cfg.n, c, ctx->stream));
    ctx->launches += 1;
    nt = 0;
    return PTYCHO_OK;
  };
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t m = std::max<int64_t>(0, std::min<int64_t>(first + count, (int64_t)t.probes.size()) - first);
    if (m == 0) continue;
    c.t[nt] = base_args(ctx, t);
    c.count[nt] = (int)m;
    if (++nt == MAX_CHAIN_TILES) PASS(flush());
  }
  return flush();
}

static ptycho_status run_probes(ptycho_ctx ctx, int64_t first, int64_t count, ChainMode mode) {
  if (mode == CHAIN_GRAD && ctx->batched) return run_batched(ctx, first, count);
  if (mode == CHAIN_GRAD && ctx->cluster) return run_cluster_chain(ctx, first, count);
  if (mode == CHAIN_GRAD && ctx->persist) {
    std::vector<int64_t> cnt(ctx->tiles.size(), 0);
    for (int k : ctx->local)
      cnt[k] = std::max<int64_t>(0, std::min<int64_t>(first + count, (int64_t)ctx->tiles[k].probes.size()) - first);
    return run_chain_kernel(ctx, first, cnt);
  }
  PASS(fork_tiles(ctx));
  int64_t maxn = 0;
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t nk = (int64_t)t.probes.size();
    const int64_t m = std::max<int64_t>(0, std::min(first + count, nk) - first);
    maxn = std::max(maxn, m);
    if (m > 0) PASS(set_cursor(ctx, t, (int)first, t.stream));
    if (mode == CHAIN_GRAD) PASS(ensure_graph(ctx, t));
  }
  // interleave the tiles' probe chains so every tile stream is fed
  for (int64_t j = 0; j < maxn; ++j)
    for (int k : ctx->local) {
      Tile& t = ctx->tiles[k];
      const int64_t nk = (int64_t)t.probes.size();
      if (first + j >= nk) continue;
      PASS(amp_wait(ctx, t, first + j, t.stream));
      if (mode == CHAIN_GRAD && t.graph) {
        CK(cudaGraphLaunch(t.graph, t.stream));
        ctx->launches += chain_len(ctx->cfg.slices, stash_free(ctx->cfg));
      } else {
        PASS(enqueue_chain(ctx, t, mode, t.stream));
      }
    }
  return join_tiles(ctx);
}

static ptycho_status run_batched(ptycho_ctx ctx, int64_t first, int64_t count) {
  PASS(fork_tiles(ctx));
  for (int k : ctx->local) PASS(amp_wait(ctx, ctx->tiles[k], INT64_MAX, ctx->tiles[k].stream));
  size_t maxb = 0;
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const int64_t m = std::max<int64_t>(0, std::min<int64_t>(first + count, (int64_t)t.probes.size()) - first);
    make_batches(ctx, t, first, m);
    std::vector<int> flat;
    for (auto& b : t.batches) flat.insert(flat.end(), b.begin(), b.end());
    if (!flat.empty())
      CK(cudaMemcpyAsync(t.order, flat.data(), flat.size() * sizeof(int), cudaMemcpyHostToDevice, t.stream));
    PASS(ensure_graph(ctx, t, CHAIN_BATCH));
    maxb = std::max(maxb, t.batches.size());
  }
  std::vector<size_t> off(ctx->tiles.size(), 0);
  for (size_t j = 0; j < maxb; ++j)
    for (int k : ctx->local) {
      Tile& t = ctx->tiles[k];
      if (j >= t.batches.size()) continue;
      const int cnt = (int)t.batches[j].size();
      CK(launch_set_batch(t.desc, t.centers, t.order + off[k], cnt, ctx->batch, ctx->cfg.n, t.stream));
      ++ctx->launches;
      off[k] += cnt;
      if (t.graph_b) {
        CK(cudaGraphLaunch(t.graph_b, t.stream));
        ctx->launches += chain_len(ctx->cfg.slices, stash_free(ctx->cfg));
      } else {
        PASS(enqueue_chain(ctx, t, CHAIN_BATCH, t.stream));
      }
    }
  return join_tiles(ctx);
}

extern "C" ptycho_status ptycho_set_schedule(ptycho_ctx ctx, int32_t batched, int32_t max_batch) {
  if (!ctx) return PTYCHO_EARG;
  if (!ctx->tiles_set || !ctx->scan_set) return fail(ctx, PTYCHO_ESTATE, "set_tiles and set_scan first");
  if (ctx->ws_set) return fail(ctx, PTYCHO_ESTATE, "set_schedule must precede set_workspace");
  if (batched && (max_batch < 1 || max_batch > 64)) return fail(ctx, PTYCHO_EARG, "max_batch %d not in [1, 64]", max_batch);
  ctx->batched = batched != 0;
  ctx->batch = batched ? max_batch : 1;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_forward_grad(ptycho_ctx ctx, int64_t first, int64_t count, double* loss_out) {
  PASS(need_run(ctx));
  if (first < 0 || count < 0) return fail(ctx, PTYCHO_EARG, "bad probe range");
  CK(cudaSetDevice(ctx->device));
  if (loss_out) PASS(zero_loss(ctx));
  PASS(run_probes(ctx, first, count, CHAIN_GRAD));
  if (loss_out) PASS(sum_loss(ctx, loss_out));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_simulate_measurements(ptycho_ctx ctx) {
  PASS(need_run(ctx));
  CK(cudaSetDevice(ctx->device));
  int64_t maxn = 0;
  for (int k : ctx->local) maxn = std::max<int64_t>(maxn, (int64_t)ctx->tiles[k].probes.size());
  return run_probes(ctx, 0, maxn, CHAIN_SIMULATE);
}

// ------------------------------------------------------------------------------------------
// APPP passes (Alg. 1 steps 10-13) and the accumulated step (steps 14-16)
// ------------------------------------------------------------------------------------------
static ptycho_status hop_local(ptycho_ctx ctx, const Hop& h, int z0, int z1) {
  const Tile& a = ctx->tiles[h.src];
  const Tile& b = ctx->tiles[h.dst];
  for (int par = 0; par < 2; ++par) {
    SliceView vs = region_view(a, h.vol ? a.V : a.acc, par, z0, z1, h.y0, h.y1, h.x0, h.x1);
    SliceView vd = region_view(b, h.vol ? b.V : b.acc, par, z0, z1, h.y0, h.y1, h.x0, h.x1);
    if (vs.nslices == 0) continue;
    CK(launch_copy2d(vd.base, vd.ld, vd.ss, vs.base, vs.ld, vs.ss, vs.rows, vs.cols, vs.nslices, h.add, ctx->stream));
    ++ctx->launches;
  }
  return PTYCHO_OK;
}

// Remote hop: the region is moved in slabs of whole slices, packed [slice][rows][cols] per
// parity (even slices [y][x], odd [x][y]); sender packs + ncclSend, receiver ncclRecv + (add|copy).
static ptycho_status hop_remote(ptycho_ctx ctx, const Hop& h, bool sender, int z0, int z1) {
  const Tile& me = ctx->tiles[sender ? h.src : h.dst];
  const int peer = ctx->tiles[sender ? h.dst : h.src].owner;
  const size_t area = (size_t)(h.y1 - h.y0) * (h.x1 - h.x0);
  const int slab = (int)std::max<size_t>(1, ctx->msg_floats / area);
  for (int par = 0; par < 2; ++par) {
    SliceView v = region_view(me, h.vol ? me.V : me.acc, par, z0, z1, h.y0, h.y1, h.x0, h.x1);
    for (int q0 = 0; q0 < v.nslices; q0 += slab) {
      const int nz = std::min(slab, v.nslices - q0);
      const size_t cnt = area * nz;
      float* base = v.base + (long long)q0 * v.ss;
      const long long per = (long long)v.rows * v.cols;
      if (sender) {
        CK(launch_copy2d(ctx->sendbuf, v.cols, per, base, v.ld, v.ss, v.rows, v.cols, nz, 0, ctx->stream));
        ++ctx->launches;
        NK(ncclSend(ctx->sendbuf, cnt, ncclFloat, peer, ctx->comm, ctx->stream));
      } else {
        NK(ncclRecv(ctx->recvbuf, cnt, ncclFloat, peer, ctx->comm, ctx->stream));
        CK(launch_copy2d(base, v.ld, v.ss, ctx->recvbuf, v.cols, per, v.rows, v.cols, nz, h.add, ctx->stream));
        ++ctx->launches;
      }
    }
  }
  return PTYCHO_OK;
}

// P2P transport (SURVEY §8(e) "fused"): the receiver's copy2d reads the sender's AccBuf region
// in place through the CUDA IPC mapping of the sender's workspace (NVLink) and adds / copies it
// into its own AccBuf -- no pack, no staging, no NCCL.  READY / DONE flags (kernels.cu) order the
// two ranks exactly as a blocking send/recv pair would.
static ptycho_status hop_p2p(ptycho_ctx ctx, const Hop& h, size_t hid, bool sender, int z0, int z1,
                             unsigned ep) {
  const size_t nh = ctx->hops.size();
  const Tile& a = ctx->tiles[h.src];
  const Tile& b = ctx->tiles[h.dst];
  auto peer_flag = [&](int r, int which) {
    return (unsigned*)(ctx->peer_ws[r] + ctx->peer_flags[r]) + which * nh + hid;
  };
  if (sender) {
    cudaEvent_t s0 = nullptr, s1 = nullptr;
    if (ctx->signal_ev) {
      CK(cudaEventCreate(&s0));
      CK(cudaEventCreate(&s1));
      ctx->signal_ev->push_back(s0);
      ctx->signal_ev->push_back(s1);
      CK(cudaEventRecord(s0, ctx->stream));
    }
    CK(launch_p2p_signal(peer_flag(b.owner, 0), ep, ctx->flags + nh + hid, ctx->p2p_timeout_ns, ctx->p2p_err_dev,
                         ctx->stream));
    if (s1) CK(cudaEventRecord(s1, ctx->stream));
    ++ctx->launches;
    return PTYCHO_OK;
  }
  cudaEvent_t w0 = nullptr, w1 = nullptr;
  if (ctx->wait_ev) {
    CK(cudaEventCreate(&w0));
    CK(cudaEventCreate(&w1));
    ctx->wait_ev->push_back(w0);
    ctx->wait_ev->push_back(w1);
    CK(cudaEventRecord(w0, ctx->stream));
  }
  CK(launch_p2p_wait(ctx->flags + hid, ep, ctx->p2p_timeout_ns, ctx->p2p_err_dev, ctx->stream));
  if (w1) CK(cudaEventRecord(w1, ctx->stream));
  ++ctx->launches;
  float* src_acc = (float*)(ctx->peer_ws[a.owner] + ctx->peer_acc[a.owner][a.k]);
  cudaEvent_t c0 = nullptr, c1 = nullptr;
  if (ctx->copy_ev) {  // ptycho_profile_iteration: the NVLink pull itself
    CK(cudaEventCreate(&c0));
    CK(cudaEventCreate(&c1));
    ctx->copy_ev->push_back(c0);
    ctx->copy_ev->push_back(c1);
    CK(cudaEventRecord(c0, ctx->stream));
  }
  for (int par = 0; par < 2; ++par) {
    SliceView vs = region_view(a, src_acc, par, z0, z1, h.y0, h.y1, h.x0, h.x1);
    SliceView vd = region_view(b, b.acc, par, z0, z1, h.y0, h.y1, h.x0, h.x1);
    if (vs.nslices == 0) continue;
    CK(launch_copy2d(vd.base, vd.ld, vd.ss, vs.base, vs.ld, vs.ss, vs.rows, vs.cols, vs.nslices, h.add, ctx->stream));
    ++ctx->launches;
    ctx->copy_bytes += 4.0 * vs.rows * vs.cols * vs.nslices;
  }
  if (c1) CK(cudaEventRecord(c1, ctx->stream));
  CK(launch_p2p_post(peer_flag(a.owner, 1), ep, ctx->stream));
  ++ctx->launches;
  return PTYCHO_OK;
}

// Decide the APPP transport once, collectively: P2P needs every rank to map every other rank's
// workspace (CUDA IPC on the allocation that holds it) with peer access; otherwise (or on request)
// NCCL send/recv.  All ranks take the same decision (second all-gather of the verdicts).
static ptycho_status appp_transport_setup(ptycho_ctx ctx) {
  if (ctx->transport_set) return PTYCHO_OK;
  ctx->transport_set = true;
  ctx->transport = PTYCHO_APPP_NCCL;
  if (ctx->nranks == 1 || ctx->transport_req == PTYCHO_APPP_NCCL) return PTYCHO_OK;
  const int nr = ctx->nranks, nt = (int)ctx->tiles.size();
  struct Rec {
    cudaIpcMemHandle_t h;
    long long ws_off, flags_off;
    int device, ok;
  };
  const size_t rec = align_up(sizeof(Rec) + nt * sizeof(long long), 8);
  std::vector<char> mine(rec, 0), all(rec * nr, 0);
  Rec* r = (Rec*)mine.data();
  r->ok = 1;
  r->device = ctx->device;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  GetRange get_range = nullptr;
  cudaDriverEntryPointQueryResult q;
  CUdeviceptr base = 0;
  size_t sz = 0;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", (void**)&get_range, cudaEnableDefault, &q) != cudaSuccess ||
      !get_range || get_range(&base, &sz, (CUdeviceptr)ctx->ws) != CUDA_SUCCESS ||
      cudaIpcGetMemHandle(&r->h, (void*)base) != cudaSuccess) {
    r->ok = 0;
    cudaGetLastError();
  }
  r->ws_off = (long long)(ctx->ws - (char*)base);
  r->flags_off = (long long)((char*)ctx->flags - ctx->ws);
  long long* acc = (long long*)(mine.data() + sizeof(Rec));
  for (const Tile& t : ctx->tiles) acc[t.k] = t.owner == ctx->rank ? (long long)((char*)t.acc - ctx->ws) : -1;
  char* dsend = (char*)ctx->staging;
  char* drecv = dsend + align_up(rec);
  CK(cudaMemcpyAsync(dsend, mine.data(), rec, cudaMemcpyHostToDevice, ctx->stream));
  NK(ncclAllGather(dsend, drecv, rec, ncclUint8, ctx->comm, ctx->stream));
  CK(cudaMemcpyAsync(all.data(), drecv, rec * nr, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  int ok = 1;
  ctx->peer_ws.assign(nr, nullptr);
  ctx->peer_flags.assign(nr, 0);
  ctx->peer_acc.assign(nr, std::vector<long long>(nt, -1));
  for (int j = 0; j < nr && ok; ++j) {
    const Rec* o = (const Rec*)(all.data() + rec * j);
    ok &= o->ok;
    ctx->peer_flags[j] = o->flags_off;
    const long long* oa = (const long long*)(all.data() + rec * j + sizeof(Rec));
    for (int k = 0; k < nt; ++k) ctx->peer_acc[j][k] = oa[k];
    if (j == ctx->rank) {
      ctx->peer_ws[j] = ctx->ws;
      continue;
    }
    int can = 0;
    if (o->device == ctx->device || cudaDeviceCanAccessPeer(&can, ctx->device, o->device) != cudaSuccess || !can) {
      ok = 0;
      break;
    }
    void* m = nullptr;
    if (cudaIpcOpenMemHandle(&m, o->h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      ok = 0;
      break;
    }
    ctx->peer_map.push_back(m);
    ctx->peer_ws[j] = (char*)m + o->ws_off;
  }
  cudaGetLastError();
  // every rank must agree
  int* dv = (int*)dsend;
  CK(cudaMemcpyAsync(dv, &ok, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  NK(ncclAllGather(dv, dv + 64, 1, ncclInt32, ctx->comm, ctx->stream));
  std::vector<int> votes(nr, 0);
  CK(cudaMemcpyAsync(votes.data(), dv + 64, nr * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  bool all_ok = true;
  for (int v : votes) all_ok &= v != 0;
  if (all_ok) {
    ctx->transport = PTYCHO_APPP_P2P;
    CK(cudaHostAlloc((void**)&ctx->p2p_err, sizeof(unsigned), cudaHostAllocMapped));
    *ctx->p2p_err = 0;
    CK(cudaHostGetDevicePointer((void**)&ctx->p2p_err_dev, ctx->p2p_err, 0));
    return PTYCHO_OK;
  }
  for (void* m : ctx->peer_map) cudaIpcCloseMemHandle(m);
  ctx->peer_map.clear();
  if (ctx->transport_req == PTYCHO_APPP_P2P)
    return fail(ctx, PTYCHO_ECUDA, "APPP P2P transport requested but some rank cannot map its peers");
  return PTYCHO_OK;
}

// The four passes on the slices [z0, z1) of every AccBuf (every rank walks the same hop list).
static ptycho_status appp_range(ptycho_ctx ctx, int z0, int z1) {
  PASS(appp_transport_setup(ctx));
  const bool p2p = ctx->transport == PTYCHO_APPP_P2P;
  const unsigned ep = ++ctx->epoch;
  for (size_t hid = 0; hid < ctx->hops.size(); ++hid) {
    const Hop& h = ctx->hops[hid];
    if (h.y1 <= h.y0 || h.x1 <= h.x0) continue;  // disjoint extended rects: empty message
    const int so = ctx->tiles[h.src].owner, d = ctx->tiles[h.dst].owner;
    if (so == ctx->rank && d == ctx->rank) PASS(hop_local(ctx, h, z0, z1));
    else if (so == ctx->rank) PASS(p2p ? hop_p2p(ctx, h, hid, true, z0, z1, ep) : hop_remote(ctx, h, true, z0, z1));
    else if (d == ctx->rank) PASS(p2p ? hop_p2p(ctx, h, hid, false, z0, z1, ep) : hop_remote(ctx, h, false, z0, z1));
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_set_appp_transport(ptycho_ctx ctx, int32_t mode) {
  if (!ctx) return PTYCHO_EARG;
  if (mode < PTYCHO_APPP_AUTO || mode > PTYCHO_APPP_P2P) return fail(ctx, PTYCHO_EARG, "transport %d", mode);
  if (ctx->transport_set) return fail(ctx, PTYCHO_ESTATE, "the APPP transport is fixed at the first APPP call");
  ctx->transport_req = mode;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_appp_transport(ptycho_ctx ctx, int32_t* mode) {
  if (!ctx || !mode) return PTYCHO_EARG;
  *mode = ctx->transport_set ? ctx->transport : PTYCHO_APPP_AUTO;
  return PTYCHO_OK;
}

static ptycho_status step_range(ptycho_ctx ctx, int z0, int z1) {
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    const long long off = (long long)z0 * t.slice_stride;
    CK(launch_acc_step(t.V + off, t.acc + off, (long long)(z1 - z0) * t.slice_stride, ctx->cfg.alpha_acc,
                       ctx->stream));
    ++ctx->launches;
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_appp_passes(ptycho_ctx ctx) {
  PASS(need_ws(ctx));
  CK(cudaSetDevice(ctx->device));
  return appp_range(ctx, 0, ctx->cfg.slices);
}

extern "C" ptycho_status ptycho_step(ptycho_ctx ctx) {
  PASS(need_ws(ctx));
  if (ctx->hve) return fail(ctx, PTYCHO_ESTATE, "HVE has no accumulated step (Alg. 1 steps 14-16 are GD's)");
  CK(cudaSetDevice(ctx->device));
  return step_range(ctx, 0, ctx->cfg.slices);
}

// One pass segment with the APPP chains pipelined by slabs of slices (§8(a) a11):
// every tile's last probe of the segment runs as direct launches that record an event when its
// backward pass has finished the lowest slice of each slab (AccBuf of that slab is then final);
// the passes and the accumulated step of a slab start as soon as every local tile reached it,
// overlapping the backward passes of the lower slices.
static ptycho_status segment_pipelined(ptycho_ctx ctx, int64_t first, int64_t count) {
  if (ctx->batched || ctx->cluster) {  // whole batches / one cluster launch: passes after the segment
    PASS(run_probes(ctx, first, count, CHAIN_GRAD));
    PASS(appp_range(ctx, 0, ctx->cfg.slices));
    return step_range(ctx, 0, ctx->cfg.slices);
  }
  const int S = ctx->cfg.slices, slab = ctx->slab, nslab = (S + slab - 1) / slab;
  int64_t maxn = 0;
  std::vector<int64_t> m(ctx->tiles.size(), 0);
  for (int k : ctx->local) {
    m[k] = std::max<int64_t>(0, std::min<int64_t>(first + count, (int64_t)ctx->tiles[k].probes.size()) - first);
    maxn = std::max(maxn, m[k]);
  }
  std::vector<int64_t> done(ctx->tiles.size(), 0);  // probes already run by the chain kernel
  if (ctx->persist) {
    for (int k : ctx->local) done[k] = m[k] > 0 ? m[k] - 1 : 0;
    PASS(run_chain_kernel(ctx, first, done));
  }
  PASS(fork_tiles(ctx));
  for (int k : ctx->local) {
    Tile& t = ctx->tiles[k];
    if (m[k] > 0) PASS(set_cursor(ctx, t, (int)(first + done[k]), t.stream));
    PASS(ensure_graph(ctx, t));
    if ((int)t.slab_ev.size() < nslab) {
      for (cudaEvent_t e : t.slab_ev) cudaEventDestroy(e);
      t.slab_ev.assign(nslab, nullptr);
      for (auto& e : t.slab_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  }
  for (int64_t j = 0; j < maxn; ++j)
    for (int k : ctx->local) {
      Tile& t = ctx->tiles[k];
      if (j >= m[k] || j < done[k]) continue;
      PASS(amp_wait(ctx, t, first + j, t.stream));
      if (j < m[k] - 1 && t.graph) {
        CK(cudaGraphLaunch(t.graph, t.stream));
        ctx->launches += chain_len(S, stash_free(ctx->cfg));
      } else if (j < m[k] - 1) {
        PASS(enqueue_chain(ctx, t, CHAIN_GRAD, t.stream));
      } else {
        PASS(enqueue_chain(ctx, t, CHAIN_GRAD, t.stream, nullptr, &t.slab_ev, slab));
      }
    }
  for (int b = nslab - 1; b >= 0; --b) {
    for (int k : ctx->local)
      if (m[k] > 0) CK(cudaStreamWaitEvent(ctx->stream, ctx->tiles[k].slab_ev[b], 0));
    const int z0 = b * slab, z1 = std::min(S, z0 + slab);
    PASS(appp_range(ctx, z0, z1));
    PASS(step_range(ctx, z0, z1));
  }
  return join_tiles(ctx);
}

extern "C" ptycho_status ptycho_profile_iteration(ptycho_ctx ctx, double* ms_out) {
  PASS(need_run(ctx));
  if (!ms_out) return fail(ctx, PTYCHO_EARG, "ms_out is NULL");
  if (ctx->hve) return fail(ctx, PTYCHO_ESTATE, "profile_iteration: GD contexts only");
  CK(cudaSetDevice(ctx->device));
  for (int i = 0; i < 8; ++i) ms_out[i] = 0.0;
  size_t nmax = 0;
  for (const Tile& t : ctx->tiles) nmax = std::max(nmax, t.probes.size());
  if (nmax == 0) return PTYCHO_OK;
  const int64_t T = ctx->cfg.pass_period > 0 ? ctx->cfg.pass_period : (int64_t)nmax;
  const int64_t nseg = ((int64_t)nmax + T - 1) / T;
  std::vector<cudaEvent_t> ev(4 * nseg + 1, nullptr), wait_ev, signal_ev, copy_ev;
  ctx->copy_bytes = 0.0;
  for (auto& e : ev) CK(cudaEventCreate(&e));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaEventRecord(ev[0], ctx->stream));
  ptycho_status st = PTYCHO_OK;
  ctx->wait_ev = &wait_ev;
  ctx->signal_ev = &signal_ev;
  ctx->copy_ev = &copy_ev;
  for (int64_t j = 0; j < nseg && st == PTYCHO_OK; ++j) {
    if (j) CK(cudaEventRecord(ev[4 * j], ctx->stream));
    st = run_probes(ctx, j * T, T, CHAIN_GRAD);
    if (st == PTYCHO_OK) st = cudaEventRecord(ev[4 * j + 1], ctx->stream) == cudaSuccess ? PTYCHO_OK : PTYCHO_ECUDA;
    if (st == PTYCHO_OK) st = appp_range(ctx, 0, ctx->cfg.slices);
    if (st == PTYCHO_OK) st = cudaEventRecord(ev[4 * j + 2], ctx->stream) == cudaSuccess ? PTYCHO_OK : PTYCHO_ECUDA;
    if (st == PTYCHO_OK) st = step_range(ctx, 0, ctx->cfg.slices);
    if (st == PTYCHO_OK) st = cudaEventRecord(ev[4 * j + 3], ctx->stream) == cudaSuccess ? PTYCHO_OK : PTYCHO_ECUDA;
  }
  ctx->wait_ev = nullptr;
  ctx->signal_ev = nullptr;
  ctx->copy_ev = nullptr;
  if (st == PTYCHO_OK) {
    CK(cudaEventRecord(ev[4 * nseg], ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    PASS(check_p2p(ctx));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, ev[0], ev[4 * nseg]));
    ms_out[0] = ms;
    double appp = 0.0;
    for (int64_t j = 0; j < nseg; ++j) {
      CK(cudaEventElapsedTime(&ms, ev[4 * j], ev[4 * j + 1]));
      ms_out[1] += ms;
      CK(cudaEventElapsedTime(&ms, ev[4 * j + 1], ev[4 * j + 2]));
      appp += ms;
      CK(cudaEventElapsedTime(&ms, ev[4 * j + 2], ev[4 * j + 3]));
      ms_out[4] += ms;
    }
    for (size_t i = 0; i + 1 < wait_ev.size(); i += 2) {
      CK(cudaEventElapsedTime(&ms, wait_ev[i], wait_ev[i + 1]));
      ms_out[2] += ms;
    }
    for (size_t i = 0; i + 1 < signal_ev.size(); i += 2) {
      CK(cudaEventElapsedTime(&ms, signal_ev[i], signal_ev[i + 1]));
      ms_out[5] += ms;
    }
    ms_out[3] = std::max(0.0, appp - ms_out[2] - ms_out[5]);
    for (size_t i = 0; i + 1 < copy_ev.size(); i += 2) {
      CK(cudaEventElapsedTime(&ms, copy_ev[i], copy_ev[i + 1]));
      ms_out[6] += ms;
    }
    ms_out[7] = ctx->copy_bytes;
  }
  for (auto e : ev) cudaEventDestroy(e);
  for (auto e : wait_ev) cudaEventDestroy(e);
  for (auto e : signal_ev) cudaEventDestroy(e);
  for (auto e : copy_ev) cudaEventDestroy(e);
  return st == PTYCHO_OK ? PTYCHO_OK : (ctx->err.empty() ? fail(ctx, st, "profile_iteration failed") : st);
}

extern "C" ptycho_status ptycho_iterate(ptycho_ctx ctx, double* loss_out) {
  PASS(need_run(ctx));
  CK(cudaSetDevice(ctx->device));
  size_t nmax = 0;
  for (const Tile& t : ctx->tiles) nmax = std::max(nmax, t.probes.size());
  if (nmax == 0) return PTYCHO_OK;
  const int64_t T = ctx->cfg.pass_period > 0 ? ctx->cfg.pass_period : (int64_t)nmax;
  const int64_t nseg = ((int64_t)nmax + T - 1) / T;
  if (loss_out) PASS(zero_loss(ctx));
  if (ctx->hve) {  // HVE: one independent SGD sweep per tile, then the copy-paste exchange
    PASS(run_probes(ctx, 0, (int64_t)nmax, CHAIN_GRAD));
    PASS(appp_range(ctx, 0, ctx->cfg.slices));
  }
  for (int64_t j = 0; j < nseg && !ctx->hve; ++j) {
    if (ctx->slab > 0) {
      PASS(segment_pipelined(ctx, j * T, T));
    } else {
      PASS(run_probes(ctx, j * T, T, CHAIN_GRAD));
      PASS(ptycho_appp_passes(ctx));
      PASS(ptycho_step(ctx));
    }
  }
  if (loss_out) {
    double local = 0.0;
    PASS(sum_loss(ctx, &local));
    if (ctx->nranks > 1) {
      CK(cudaMemcpyAsync(ctx->dscratch, &local, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      NK(ncclAllReduce(ctx->dscratch, ctx->dscratch, 1, ncclDouble, ncclSum, ctx->comm, ctx->stream));
      CK(cudaMemcpyAsync(&local, ctx->dscratch, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
    *loss_out = local;
  }
  return PTYCHO_OK;
}

// ------------------------------------------------------------------------------------------
// stitch (Alg. 1 step 20)
// ------------------------------------------------------------------------------------------
extern "C" ptycho_status ptycho_stitch(ptycho_ctx ctx, float* V_out, int out_on_device, int32_t root) {
  PASS(need_ws(ctx));
  if (root < 0 || root >= ctx->nranks) return fail(ctx, PTYCHO_EARG, "bad root %d", root);
  const bool am_root = ctx->rank == root;
  if (am_root && !V_out) return fail(ctx, PTYCHO_EARG, "V_out is NULL on the root");
  CK(cudaSetDevice(ctx->device));
  const auto& cfg = ctx->cfg;
  const size_t hw = (size_t)cfg.height * cfg.width;
  // A pinned host V_out (cudaHostAlloc / registered, e.g. torch pin_memory) is written in place by
  // the gather kernels through its device alias (zero-copy): no staging, no per-slice sync.
  float* host_dev = nullptr;
  if (am_root && !out_on_device) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, V_out) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
      host_dev = (float*)at.devicePointer;
    cudaGetLastError();
  }
  float* gout = out_on_device ? V_out : host_dev;
  if (ctx->nranks == 1 && gout) {
    // every tile local: one gather per tile and slice parity (even slices copy, odd transpose)
    for (const Tile& t : ctx->tiles)
      for (int par = 0; par < 2; ++par) {
        SliceView v = region_view(t, t.V, par, 0, cfg.slices, t.iy0, t.iy1, t.ix0, t.ix1);
        if (v.nslices == 0) continue;
        float* dst = gout + (size_t)par * hw + (size_t)t.iy0 * cfg.width + t.ix0;
        if (par == 0)
          CK(launch_copy2d(dst, cfg.width, 2 * (long long)hw, v.base, v.ld, v.ss, v.rows, v.cols, v.nslices, 0,
                           ctx->stream));
        else
          CK(launch_transpose2d(dst, cfg.width, 2 * (long long)hw, v.base, v.ld, v.ss, t.iy1 - t.iy0, t.ix1 - t.ix0,
                                v.nslices, 0, ctx->stream));
        ++ctx->launches;
      }
    CK(cudaStreamSynchronize(ctx->stream));
    return check_p2p(ctx);
  }
  for (int s = 0; s < cfg.slices; ++s) {
    float* g = am_root ? (gout ? gout + (size_t)s * hw : ctx->staging) : nullptr;
    for (const Tile& t : ctx->tiles) {
      const int ih = t.iy1 - t.iy0, iw = t.ix1 - t.ix0;
      if (t.owner == ctx->rank && am_root) {
        PASS(tile_to_global(ctx, t, t.V, s, g, t.iy0, t.iy1, t.ix0, t.ix1));
      } else if (t.owner == ctx->rank) {  // pack my interior [ih][iw] and send it to the root
        float* tmp = ctx->sendbuf;
        const float* sl = t.V + (long long)s * t.slice_stride;
        if ((s & 1) == 0)
          CK(launch_copy2d(tmp, iw, 0, sl + (long long)(t.iy0 - t.ey0) * t.pitch0 + (t.ix0 - t.ex0), t.pitch0, 0, ih, iw,
                           1, 0, ctx->stream));
        else
          CK(launch_transpose2d(tmp, iw, 0, sl + (long long)(t.ix0 - t.ex0) * t.pitch1 + (t.iy0 - t.ey0), t.pitch1, 0,
                                ih, iw, 1, 0, ctx->stream));
        ++ctx->launches;
        NK(ncclSend(tmp, (size_t)ih * iw, ncclFloat, root, ctx->comm, ctx->stream));
      } else if (am_root) {
        NK(ncclRecv(ctx->recvbuf, (size_t)ih * iw, ncclFloat, t.owner, ctx->comm, ctx->stream));
        CK(launch_copy2d(g + (size_t)t.iy0 * cfg.width + t.ix0, cfg.width, 0, ctx->recvbuf, iw, 0, ih, iw, 1, 0,
                         ctx->stream));
        ++ctx->launches;
      }
    }
    if (am_root && !gout) {
      CK(cudaMemcpyAsync(V_out + (size_t)s * hw, ctx->staging, hw * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
    }
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return check_p2p(ctx);
}

// A P2P flag wait that timed out (the peer stalled longer than PTYCHO_P2P_TIMEOUT_S) is reported
// at the next synchronisation point; the AccBuf contents of that APPP call are then undefined.
static ptycho_status check_p2p(ptycho_ctx ctx) {
  if (ctx->p2p_err && *(volatile unsigned*)ctx->p2p_err)
    return fail(ctx, PTYCHO_ECUDA, "APPP P2P: a peer did not reach its hop within %.0f s (PTYCHO_P2P_TIMEOUT_S)",
                ctx->p2p_timeout_ns * 1e-9);
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_synchronize(ptycho_ctx ctx) {
  if (!ctx) return PTYCHO_EARG;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k : ctx->local)
    if (ctx->tiles[k].stream) CK(cudaStreamSynchronize(ctx->tiles[k].stream));
  if (ctx->copy_stream) CK(cudaStreamSynchronize(ctx->copy_stream));
  return check_p2p(ctx);
}

extern "C" ptycho_status ptycho_debug_errors(ptycho_ctx ctx, uint32_t* bits, int32_t* checks_built) {
  PASS(need_ws(ctx));
  if (!bits || !checks_built) return fail(ctx, PTYCHO_EARG, "outputs are NULL");
#ifdef PTYCHO_DEBUG_CHECKS
  *checks_built = 1;
#else
  *checks_built = 0;
#endif
  PASS(ptycho_synchronize(ctx));
  CK(cudaMemcpy(bits, ctx->iscratch + 32, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  CK(cudaMemset(ctx->iscratch + 32, 0, sizeof(uint32_t)));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_kernel_launches(ptycho_ctx ctx, int64_t* count) {
  if (!ctx || !count) return PTYCHO_EARG;
  *count = ctx->launches;
  return PTYCHO_OK;
}

// ------------------------------------------------------------------------------------------
// debug exports
// ------------------------------------------------------------------------------------------
static ptycho_status local_tile(ptycho_ctx ctx, int tile, Tile** out) {
  if (tile < 0 || tile >= (int)ctx->tiles.size() || ctx->tiles[tile].owner != ctx->rank)
    return fail(ctx, PTYCHO_EARG, "tile %d is not local", tile);
  *out = &ctx->tiles[tile];
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_debug_read_tile(ptycho_ctx ctx, int32_t tile, int32_t which, float* out) {
  PASS(need_ws(ctx));
  Tile* t = nullptr;
  PASS(local_tile(ctx, tile, &t));
  if (!out) return fail(ctx, PTYCHO_EARG, "out is NULL");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k : ctx->local) CK(cudaStreamSynchronize(ctx->tiles[k].stream));
  const float* buf = which ? t->acc : t->V;
  if (!buf) return fail(ctx, PTYCHO_EARG, "tile %d has no AccBuf (HVE context)", tile);
  const size_t area = (size_t)t->eh * t->ew;
  for (int s = 0; s < ctx->cfg.slices; ++s) {
    // staging viewed as [eh][ew]: use a private pitch = ew by calling the kernels directly
    const float* sl = buf + (long long)s * t->slice_stride;
    if ((s & 1) == 0) CK(launch_copy2d(ctx->staging, t->ew, 0, sl, t->pitch0, 0, t->eh, t->ew, 1, 0, ctx->stream));
    else CK(launch_transpose2d(ctx->staging, t->ew, 0, sl, t->pitch1, 0, t->eh, t->ew, 1, 0, ctx->stream));
    ++ctx->launches;
    CK(cudaMemcpyAsync(out + s * area, ctx->staging, area * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_debug_write_tile(ptycho_ctx ctx, int32_t tile, int32_t which, const float* in) {
  PASS(need_ws(ctx));
  Tile* t = nullptr;
  PASS(local_tile(ctx, tile, &t));
  if (!in) return fail(ctx, PTYCHO_EARG, "in is NULL");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  float* buf = which ? t->acc : t->V;
  if (!buf) return fail(ctx, PTYCHO_EARG, "tile %d has no AccBuf (HVE context)", tile);
  const size_t area = (size_t)t->eh * t->ew;
  for (int s = 0; s < ctx->cfg.slices; ++s) {
    float* sl = buf + (long long)s * t->slice_stride;
    CK(cudaMemcpyAsync(ctx->staging, in + s * area, area * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    if ((s & 1) == 0) CK(launch_copy2d(sl, t->pitch0, 0, ctx->staging, t->ew, 0, t->eh, t->ew, 1, 0, ctx->stream));
    else CK(launch_transpose2d(sl, t->pitch1, 0, ctx->staging, t->ew, 0, t->ew, t->eh, 1, 0, ctx->stream));
    ++ctx->launches;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  return PTYCHO_OK;
}

static ptycho_status debug_chain(ptycho_ctx ctx, int tile, int64_t probe, ChainMode mode, Tile** tout) {
  PASS(need_run(ctx));
  Tile* t = nullptr;
  PASS(local_tile(ctx, tile, &t));
  if (probe < 0 || probe >= (int64_t)t->probes.size()) return fail(ctx, PTYCHO_EARG, "bad probe %lld", (long long)probe);
  CK(cudaSetDevice(ctx->device));
  PASS(zero_loss(ctx));
  PASS(amp_settle(ctx, ctx->stream));
  PASS(set_cursor(ctx, *t, (int)probe, ctx->stream));
  PASS(enqueue_chain(ctx, *t, mode, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  *tout = t;
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_debug_probe_grad(ptycho_ctx ctx, int32_t tile, int64_t probe, float* grad_out,
                                                 double* loss_out) {
  Tile* t = nullptr;
  PASS(debug_chain(ctx, tile, probe, CHAIN_DEBUG_GRAD, &t));
  const size_t cnt = (size_t)ctx->cfg.slices * ctx->cfg.n * ctx->cfg.n;
  if (grad_out) CK(cudaMemcpy(grad_out, ctx->debug, cnt * sizeof(float), cudaMemcpyDeviceToHost));
  if (loss_out) PASS(sum_loss(ctx, loss_out));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_debug_exit_wave(ptycho_ctx ctx, int32_t tile, int64_t probe, void* psi_out) {
  Tile* t = nullptr;
  PASS(debug_chain(ctx, tile, probe, CHAIN_DEBUG_EXIT, &t));
  const size_t cnt = (size_t)ctx->cfg.n * ctx->cfg.n;
  if (psi_out) CK(cudaMemcpy(psi_out, ctx->debug, cnt * sizeof(float2), cudaMemcpyDeviceToHost));
  return PTYCHO_OK;
}

// Global probe id -> (local tile holding it, index in that tile's list); EARG if not local.
static ptycho_status find_probe(ptycho_ctx ctx, int64_t probe, int* tile, int64_t* local) {
  for (int k : ctx->local) {
    const auto& pr = ctx->tiles[k].probes;
    const auto it = std::lower_bound(pr.begin(), pr.end(), probe);
    if (it != pr.end() && *it == probe) {
      *tile = k;
      *local = it - pr.begin();
      return PTYCHO_OK;
    }
  }
  return fail(ctx, PTYCHO_EARG, "probe %lld is not assigned to a tile of this rank", (long long)probe);
}

extern "C" ptycho_status ptycho_probe_grad(ptycho_ctx ctx, int64_t probe, float* g_out, double* loss_out) {
  PASS(need_run(ctx));
  int tile = 0;
  int64_t j = 0;
  PASS(find_probe(ctx, probe, &tile, &j));
  Tile* t = nullptr;
  PASS(debug_chain(ctx, tile, j, CHAIN_DEBUG_GRAD, &t));
  const size_t cnt = (size_t)ctx->cfg.slices * ctx->cfg.n * ctx->cfg.n;
  if (g_out) CK(cudaMemcpy(g_out, ctx->debug, cnt * sizeof(float), cudaMemcpyDefault));
  if (loss_out) PASS(sum_loss(ctx, loss_out));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_probe_exitwave(ptycho_ctx ctx, int64_t probe, void* psi_out) {
  PASS(need_run(ctx));
  int tile = 0;
  int64_t j = 0;
  PASS(find_probe(ctx, probe, &tile, &j));
  Tile* t = nullptr;
  PASS(debug_chain(ctx, tile, j, CHAIN_DEBUG_EXIT, &t));
  if (psi_out) CK(cudaMemcpy(psi_out, ctx->debug, (size_t)ctx->cfg.n * ctx->cfg.n * sizeof(float2), cudaMemcpyDefault));
  return PTYCHO_OK;
}

extern "C" ptycho_status ptycho_profile_chain(ptycho_ctx ctx, int32_t tile, int64_t first, int64_t count,
                                              double* ms_out, int64_t* launches_out) {
  PASS(need_run(ctx));
  Tile* t = nullptr;
  PASS(local_tile(ctx, tile, &t));
  if (!ms_out || !launches_out) return fail(ctx, PTYCHO_EARG, "outputs are NULL");
  CK(cudaSetDevice(ctx->device));
  for (int k = 0; k < K_COUNT; ++k) {
    ms_out[k] = 0.0;
    launches_out[k] = 0;
  }
  const int64_t nk = (int64_t)t->probes.size();
  const int64_t m = std::max<int64_t>(0, std::min(first + count, nk) - first);
  if (m == 0) return PTYCHO_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  PASS(set_cursor(ctx, *t, (int)first, t->stream));
  ChainProfile prof;
  PASS(amp_settle(ctx, t->stream));
  for (int64_t j = 0; j < m; ++j) PASS(enqueue_chain(ctx, *t, CHAIN_GRAD, t->stream, &prof));
  CK(cudaStreamSynchronize(t->stream));
  for (size_t i = 0; i < prof.kind.size(); ++i) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, prof.ev[2 * i], prof.ev[2 * i + 1]));
    ms_out[prof.kind[i]] += ms;
    launches_out[prof.kind[i]] += 1;
  }
  for (cudaEvent_t e : prof.ev) cudaEventDestroy(e);
  return PTYCHO_OK;
}
