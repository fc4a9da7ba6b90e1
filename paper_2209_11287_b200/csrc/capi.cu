// extern "C" entry points of libtedjoin.so (declared in include/tedjoin.h).
// Every entry point converts internal failures into a status code and keeps
// the message for tj_last_error(); no C++ exception crosses the ABI.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "internal.cuh"
#include "scan.cuh"

namespace tj {

[[noreturn]] void fail(int status, const std::string& msg) { throw Error{status, msg}; }

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::mutex g_err_mu;
static std::string g_err;  // failures without a ctx (tj_ctx_create)

template <class F>
static int guarded(tj_ctx* ctx, F&& f) {
  try {
    if (ctx) {
      int cur = -1;
      cudaGetDevice(&cur);
      if (cur != ctx->device) TJ_CUDA(cudaSetDevice(ctx->device));
    }
    f();
    return TJ_OK;
  } catch (const Error& e) {
    if (ctx) ctx->err = e.msg;
    else {
      std::lock_guard<std::mutex> lk(g_err_mu);
      g_err = e.msg;
    }
    return e.status;
  } catch (const std::exception& e) {
    if (ctx) ctx->err = e.what();
    return TJ_ECUDA;
  }
}

static DevCounters* counters(tj_ctx* ctx) { return ctx->counters.as<DevCounters>(); }

static void require_grid(tj_ctx* ctx) {
  if (!ctx->g.built) fail(TJ_EINVAL, "no grid has been built on this context");
}

static void zero_results(tj_ctx* ctx, cudaStream_t s) {
  ctx->ctr_valid = false;
  ctx->rows_range_done = false;
  ctx->counters.ensure(2 * sizeof(DevCounters), s);  // live counters + a checkpoint
  TJ_CUDA(cudaMemsetAsync(ctx->counters.ptr, 0, 2 * sizeof(DevCounters), s));
  if (ctx->g.n > 0) {
    ctx->qcount.ensure(sizeof(uint32_t) * ctx->g.n, s);
    TJ_CUDA(cudaMemsetAsync(ctx->qcount.ptr, 0, sizeof(uint32_t) * ctx->g.n, s));
  }
}

// Dense hit-mask layout over all cells (low-d path); depends only on the grid.
static void ensure_masks(tj_ctx* ctx, cudaStream_t s) {
  if (ctx->masks_ready) return;
  if (ctx->symmetric) build_symmetric_tables(ctx, s);
  build_mask_bases(ctx, 0, ctx->g.n_cells, s);
  if (ctx->symmetric) build_bt_desc(ctx, s);
  ctx->masks.ensure(sizeof(unsigned long long) * std::max<int64_t>(ctx->g.tiles, 1), s);
  build_window_cells(ctx, s);
  ctx->masks_ready = true;
}


// Grow the pair append buffer to `pairs` entries, keeping the first `keep`.
static void reserve_pairs(tj_ctx* ctx, unsigned long long pairs, unsigned long long keep,
                          cudaStream_t s) {
  pairs = std::max<unsigned long long>(pairs, 1024);
  if (pairs <= ctx->pair_cap) return;
  keep = std::min(keep, ctx->pair_cap);
  DevBuf grown;
  grown.ensure(sizeof(uint2) * pairs, s);
  if (keep) TJ_CUDA(cudaMemcpyAsync(grown.ptr, ctx->pairs.ptr, sizeof(uint2) * keep,
                                    cudaMemcpyDeviceToDevice, s));
  ctx->pairs.release(s);
  ctx->pairs = grown;
  grown.ptr = nullptr;
  ctx->pair_cap = pairs;
}

__global__ void zero_query_counts_kernel(const int64_t* __restrict__ cell_start, int64_t cb,
                                         int64_t ce, uint32_t* __restrict__ qcount) {
  const int64_t a = cell_start[cb], b = cell_start[ce];
  for (int64_t p = a + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < b;
       p += int64_t(gridDim.x) * blockDim.x)
    qcount[p] = 0;
}

// Guard-band half-width relative to |q|^2 + max|c|^2 (+eps^2); see refine_dmma.cu.
static double guard_rel(int d, int d_pad) { return (4.0 * d_pad + 4.0 * d + 64.0) * std::ldexp(1.0, -53); }

}  // namespace tj

using namespace tj;

extern "C" {

int tj_version(void) { return 100; }

int64_t tj_launch_count(void) { return g_launches.load(); }

int tj_ctx_create(int device, tj_ctx** out) {
  if (!out) return TJ_EINVAL;
  *out = nullptr;
  return guarded(nullptr, [&] {
    int count = 0;
    TJ_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      fail(TJ_EINVAL, "device " + std::to_string(device) + " out of range (" +
                          std::to_string(count) + " visible)");
    TJ_CUDA(cudaSetDevice(device));
    cudaMemPool_t pool;
    TJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;  // keep freed blocks cached: repeated joins allocate nothing
    TJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    tj_ctx* c = new tj_ctx();
    c->device = device;
    const char* sym = std::getenv("TJ_SYMMETRIC");  // low-d symmetric join (default off)
    c->symmetric = sym && sym[0] == '1';
    cudaEventCreate(&c->ev0);
    cudaEventCreate(&c->ev1);
    cudaEventCreate(&c->ev2);
    cudaEventCreate(&c->ev3);
    *out = c;
  });
}

void tj_ctx_destroy(tj_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&ctx->P,        &ctx->NRM,       &ctx->CN,       &ctx->perm,      &ctx->keys,
                    &ctx->cell_key, &ctx->cell_key_hi, &ctx->keys_hi, &ctx->cell_start, &ctx->cell_runs, &ctx->runs,      &ctx->run_off,
                    &ctx->cell_cand, &ctx->cell_cost, &ctx->keys_alt,  &ctx->vals_alt,  &ctx->sort_hist,
                    &ctx->scan_partial, &ctx->scan_total, &ctx->minmax, &ctx->tmp64,   &ctx->items,
                    &ctx->pairs,    &ctx->qcount,    &ctx->counters, &ctx->fill,
                    &ctx->masks,    &ctx->win_cell, &ctx->cell_mbase, &ctx->dense,
                    &ctx->pos_off,  &ctx->rows_tmp,  &ctx->SFX,      &ctx->ipos,      &ctx->pcell,
                    &ctx->fwd,      &ctx->bt_start,  &ctx->bt,       &ctx->chunk_key,
                    &ctx->bt_desc,  &ctx->nid,       &ctx->route_dest,
                    &ctx->route_tiles};
  for (DevBuf* b : bufs) b->release(0);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  cudaEventDestroy(ctx->ev2);
  cudaEventDestroy(ctx->ev3);
  cudaDeviceSynchronize();
  delete ctx;
}

const char* tj_last_error(const tj_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_err.c_str();
}

int tj_build_grid(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                  int32_t k_idx, double eps, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n < 1 || d < 1) fail(TJ_EINVAL, "need n >= 1 and d >= 1");
    if (n >= (int64_t(1) << 32) - 1) fail(TJ_EINVAL, "n must be < 2^32 - 1 (32-bit point ids)");
    if (d > TJ_MAX_DIM) fail(TJ_EINVAL, "d must be <= " + std::to_string(TJ_MAX_DIM));
    if (!(std::isfinite(eps) && eps > 0))
      fail(TJ_EINVAL, "epsilon must be positive and finite");
    if (k_idx < 1 || k_idx > d)
      fail(TJ_EINVAL, "k_idx must be in [1, " + std::to_string(d) + "], got " +
                          std::to_string(k_idx));
    if (k_idx > TJ_MAX_K_IDX)
      fail(TJ_EINVAL, "k_idx must be <= " + std::to_string(TJ_MAX_K_IDX) +
                          " on the device grid, got " + std::to_string(k_idx));
    if (!coords) fail(TJ_EINVAL, "coords is null");
    if (ld < d) fail(TJ_EINVAL, "ld must be >= d");
    ctx->masks_ready = false;
    ctx->id_maps_ready = false;
    ctx->out_ids = nullptr;
    ctx->nid_ready = false;
    build_grid(ctx, coords, n, d, ld, k_idx, eps, s);
    zero_results(ctx, s);
    ctx->last_stream = s;
  });
}

int tj_get_grid_info(tj_ctx* ctx, tj_grid_info* out) {
  if (!ctx || !out) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    const GridState& g = ctx->g;
    out->n = g.n;
    out->d = g.d;
    out->d_pad = g.d_pad;
    out->k_idx = g.k;
    out->key_bits = g.key_bits;
    out->eps = g.eps;
    out->eps_sq = g.eps_sq;
    out->n_cells = g.n_cells;
    out->n_runs = g.n_runs;
    out->candidates = g.candidates;
    out->tiles = g.tiles;
    out->max_cell = g.max_cell;
  });
}

// Decode packed cell keys (one or two words) back into cell coordinates.
struct KeyLayout {
  int k;
  int shift[TJ_MAX_K_IDX], bits[TJ_MAX_K_IDX], word[TJ_MAX_K_IDX];
  long long cmin[TJ_MAX_K_IDX];
};
__global__ void decode_keys_kernel(const uint64_t* keys, const uint64_t* keys_hi, int64_t n_cells,
                                   KeyLayout L, int64_t* out) {
  for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < n_cells;
       c += int64_t(gridDim.x) * blockDim.x) {
    for (int j = 0; j < L.k; ++j) {
      const uint64_t w = L.word[j] ? keys_hi[c] : keys[c];
      const int bits = L.bits[j];
      const uint64_t f = (w >> L.shift[j]) & (bits >= 64 ? ~0ull : ((1ull << bits) - 1));
      out[c * L.k + j] = int64_t(f) - 1 + L.cmin[j];
    }
  }
}

int tj_grid_export(tj_ctx* ctx, uint32_t* point_order, int64_t* cell_start, int64_t* cell_coords,
                   int64_t* cell_cands, int64_t* cell_runs, uint32_t* runs) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    const GridState& g = ctx->g;
    cudaStream_t s = ctx->last_stream;
    TJ_CUDA(cudaStreamSynchronize(s));
    if (point_order)
      TJ_CUDA(cudaMemcpy(point_order, ctx->perm.ptr, sizeof(uint32_t) * g.n, cudaMemcpyDeviceToHost));
    if (cell_start)
      TJ_CUDA(cudaMemcpy(cell_start, ctx->cell_start.ptr, sizeof(int64_t) * (g.n_cells + 1),
                         cudaMemcpyDeviceToHost));
    if (cell_cands)
      TJ_CUDA(cudaMemcpy(cell_cands, ctx->cell_cand.ptr, sizeof(int64_t) * g.n_cells,
                         cudaMemcpyDeviceToHost));
    if (cell_runs)
      TJ_CUDA(cudaMemcpy(cell_runs, ctx->cell_runs.ptr, sizeof(int64_t) * (g.n_cells + 1),
                         cudaMemcpyDeviceToHost));
    if (runs)
      TJ_CUDA(cudaMemcpy(runs, ctx->runs.ptr, sizeof(uint2) * g.n_runs, cudaMemcpyDeviceToHost));
    if (cell_coords) {
      DevBuf tmp;
      tmp.ensure(sizeof(int64_t) * g.n_cells * g.k, s);
      KeyLayout L{};
      L.k = g.k;
      for (int j = 0; j < g.k; ++j) {
        L.shift[j] = g.shift[j];
        L.bits[j] = g.bits[j];
        L.word[j] = g.word[j];
        L.cmin[j] = g.cmin[j];
      }
      decode_keys_kernel<<<256, 256, 0, s>>>(ctx->cell_key.as<uint64_t>(),
                                             g.wide ? ctx->cell_key_hi.as<uint64_t>() : nullptr,
                                             g.n_cells, L, tmp.as<int64_t>());
      TJ_CHECK_LAUNCH();
      TJ_CUDA(cudaMemcpyAsync(cell_coords, tmp.ptr, sizeof(int64_t) * g.n_cells * g.k,
                              cudaMemcpyDeviceToHost, s));
      TJ_CUDA(cudaStreamSynchronize(s));
      tmp.release(s);
    }
  });
}

int tj_reserve_results(tj_ctx* ctx, int64_t pairs) {
  if (!ctx || pairs < 0) return TJ_EINVAL;
  return guarded(ctx, [&] {
    // keep what was appended so far (the batches before an overflowing one)
    DevCounters c{};
    if (ctx->counters.ptr) {
      TJ_CUDA(cudaMemcpyAsync(&c, counters(ctx), sizeof(c), cudaMemcpyDeviceToHost, ctx->last_stream));
      TJ_CUDA(cudaStreamSynchronize(ctx->last_stream));
    }
    reserve_pairs(ctx, (unsigned long long)pairs, c.pairs, ctx->last_stream);
  });
}

int tj_checkpoint_results(tj_ctx* ctx, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    TJ_CUDA(cudaMemcpyAsync(counters(ctx) + 1, counters(ctx), sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
  });
}

int tj_rollback_results(tj_ctx* ctx, int64_t cell_begin, int64_t cell_end, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    if (cell_begin < 0 || cell_end > ctx->g.n_cells || cell_begin > cell_end)
      fail(TJ_EINVAL, "cell range out of bounds");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->ctr_valid = false;
    ctx->rows_range_done = false;
    TJ_CUDA(cudaMemcpyAsync(counters(ctx), counters(ctx) + 1, sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
    if (cell_end > cell_begin) {
      zero_query_counts_kernel<<<kNumSMs * 4, 256, 0, s>>>(ctx->cell_start.as<int64_t>(),
                                                           cell_begin, cell_end,
                                                           ctx->qcount.as<uint32_t>());
      TJ_CHECK_LAUNCH();
    }
  });
}

// Which refine kernel a tj_refine call runs and how it cuts work items.
struct RefinePlan {
  bool lowd, dmma, gram, core_gram;
  int variant;     // CUDA-core variant (refine_core.cu)
  int qpi;         // queries per work item
  int64_t target;  // candidate-slice target of build_work_items
};

static RefinePlan plan_refine(const tj_ctx* ctx, int32_t kernel) {
  const GridState& g = ctx->g;
  RefinePlan r{};
  // The expanded form needs finite norms; beyond that the exact kernel decides.
  const bool norms_ok = std::isfinite(g.max_norm) && g.max_norm < 1e290;
  r.dmma = kernel == TJ_KERNEL_DMMA && norms_ok && g.d <= 64;
  r.lowd = r.dmma && g.d_pad == 4;
  // big cells at d_pad >= 12: the CTA-blocked Gram kernel (refine_gram.cu)
  r.gram = r.dmma && !r.lowd && gram_applies(g.d_pad, g.n, g.n_cells);
  // the expanded form in DFMA on big cells: the same CTA blocking on CUDA cores
  r.core_gram = kernel == TJ_KERNEL_CORE_EXPANDED && norms_ok && g.d <= 64 &&
                gram_applies(g.d_pad, g.n, g.n_cells);
  r.variant = kernel == TJ_KERNEL_CORE_FMA                   ? 1
              : kernel == TJ_KERNEL_CORE_EXPANDED && norms_ok ? 2
                                                              : 0;
  r.qpi = r.lowd                  ? lowd_queries_per_item(g.n, g.n_cells)
          : (r.gram || r.core_gram) ? kGramQueries
          : r.dmma ? tc_queries_per_item(g.d_pad, g.n, g.n_cells)
                   : core_queries_per_item(g.d, g.d_pad);
  // lowd: items never split a candidate list (each query row comes from one item);
  // gram: 64-query items x 32k-candidate slices
  r.target = r.lowd                  ? (int64_t(1) << 60)
             : (r.gram || r.core_gram) ? int64_t(kGramQueries) * kGramSlice
                      : std::max<int64_t>(g.candidates / (int64_t(kNumSMs) * 8), 1 << 16);
  return r;
}

static RefineArgs refine_args(tj_ctx* ctx, const RefinePlan& rp, int32_t short_circuit) {
  const GridState& g = ctx->g;
  RefineArgs a{};
  a.P = ctx->P.as<double>();
  a.NRM = ctx->NRM.as<double>();
  a.CN = ctx->CN.as<double>();
  a.SFX = ctx->SFX.as<double>();
  a.runs = ctx->runs.as<uint2>();
  a.run_off = ctx->run_off.as<uint32_t>();
  a.cell_runs = ctx->cell_runs.as<int64_t>();
  a.cell_start = ctx->cell_start.as<int64_t>();
  a.items = ctx->items.as<WorkItem>();
  a.n_items = ctx->n_items;
  a.n_items_dev = rp.lowd ? &counters(ctx)->n_items : nullptr;
  a.ctr = counters(ctx);
  a.pairs = ctx->pairs.as<uint2>();
  a.pair_cap = ctx->pair_cap;
  a.qcount = ctx->qcount.as<uint32_t>();
  a.masks = ctx->masks.as<unsigned long long>();
  a.cell_mbase = ctx->cell_mbase.as<int64_t>();
  a.cell_base = 0;
  a.fwd = rp.lowd && ctx->symmetric ? ctx->fwd.as<uint32_t>() : nullptr;
  a.d = g.d;
  a.d_pad = g.d_pad;
  a.nchunks = g.nchunks;
  a.eps_sq = g.eps_sq;
  a.guard_rel = guard_rel(g.d, g.d_pad);
  a.max_norm = g.max_norm + g.eps_sq;
  a.short_circuit = short_circuit ? 1 : 0;
  return a;
}

static void launch_refine(const tj_ctx* ctx, const RefinePlan& rp, const RefineArgs& a,
                          cudaStream_t s) {
  const GridState& g = ctx->g;
  if (rp.lowd) launch_refine_lowd(a, g.n, g.n_cells, s);
  else if (rp.gram) launch_refine_gram(a, false, s);
  else if (rp.core_gram) launch_refine_gram(a, true, s);
  else if (rp.dmma) launch_refine_tc(a, g.n, g.n_cells, s);
  else launch_refine_core(a, rp.variant, s);
}

static void refine_range(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
                         int64_t cell_end, cudaStream_t s, bool count_rows);

int tj_refine_masks(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
                    int64_t cell_end, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const RefinePlan rp = plan_refine(ctx, kernel);
    if (!rp.lowd || !ctx->symmetric) return;  // only the symmetric low-d join reads them
    // the counters (stats, totals) stay as they were: these cells are not this
    // result set's rows, only the masks its rows read back
    TJ_CUDA(cudaMemcpyAsync(counters(ctx) + 1, counters(ctx), sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
    refine_range(ctx, kernel, short_circuit, cell_begin, cell_end, s, false);
    TJ_CUDA(cudaMemcpyAsync(counters(ctx), counters(ctx) + 1, sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
  });
}

int tj_refine(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
              int64_t cell_end, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    refine_range(ctx, kernel, short_circuit, cell_begin, cell_end,
                 static_cast<cudaStream_t>(stream), true);
  });
}

static void refine_range(tj_ctx* ctx, int32_t kernel, int32_t short_circuit, int64_t cell_begin,
                         int64_t cell_end, cudaStream_t s, bool count_rows) {
  {
    require_grid(ctx);
    ctx->last_stream = s;
    const GridState& g = ctx->g;
    if (kernel < TJ_KERNEL_CORE || kernel > TJ_KERNEL_CORE_EXPANDED)
      fail(TJ_EINVAL, "kernel must be one of TJ_KERNEL_CORE, _DMMA, _CORE_FMA, _CORE_EXPANDED");
    if (cell_begin < 0 || cell_end > g.n_cells || cell_begin > cell_end)
      fail(TJ_EINVAL, "cell range out of bounds");
    ctx->have_refine_timing = false;
    ctx->ctr_valid = false;
    ctx->rows_range_done = false;
    if (cell_begin == cell_end) return;
    const RefinePlan rp = plan_refine(ctx, kernel);
    if (!rp.lowd && ctx->pair_cap == 0)  // callers size it (tj_reserve_results); a floor otherwise
      reserve_pairs(ctx, std::min<unsigned long long>((unsigned long long)g.candidates, 1ull << 20),
                    0, s);
    if (rp.lowd) ensure_masks(ctx, s);
    ctx->n_items = build_work_items(ctx, cell_begin, cell_end, rp.qpi, rp.target, s,
                                    rp.lowd ? &counters(ctx)->n_items : nullptr);
    TJ_CUDA(cudaMemsetAsync(&counters(ctx)->item_next, 0, sizeof(unsigned long long), s));
    const RefineArgs a = refine_args(ctx, rp, short_circuit);
    TJ_CUDA(cudaEventRecord(ctx->ev0, s));
    launch_refine(ctx, rp, a, s);
    TJ_CUDA(cudaEventRecord(ctx->ev1, s));
    ctx->have_refine_timing = true;
    // low-d rows are counted from the hit masks (pairs per query + total hits)
    if (rp.lowd && count_rows)
      launch_count_rows(ctx, cell_begin, cell_end, &counters(ctx)->hits, &counters(ctx)->max_row, s);
  }
}

__global__ void zero_sample_counts_kernel(const WorkItem* __restrict__ items, int64_t n_items,
                                          uint32_t* __restrict__ qcount) {
  for (int64_t i = blockIdx.x; i < n_items; i += gridDim.x)
    for (uint32_t q = threadIdx.x; q < items[i].nq; q += blockDim.x) qcount[items[i].q0 + q] = 0;
}

int tj_estimate_pairs(tj_ctx* ctx, int32_t kernel, int64_t cell_begin, int64_t cell_end,
                      int32_t samples, uint64_t seed, double* pairs_per_candidate, void* stream) {
  if (!ctx || !pairs_per_candidate) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    const GridState& g = ctx->g;
    if (kernel < TJ_KERNEL_CORE || kernel > TJ_KERNEL_CORE_EXPANDED)
      fail(TJ_EINVAL, "kernel must be one of TJ_KERNEL_CORE, _DMMA, _CORE_FMA, _CORE_EXPANDED");
    if (cell_begin < 0 || cell_end > g.n_cells || cell_begin > cell_end || samples < 1)
      fail(TJ_EINVAL, "need a valid cell range and samples >= 1");
    *pairs_per_candidate = 0.0;
    if (cell_begin == cell_end) return;
    const RefinePlan rp = plan_refine(ctx, kernel);
    if (rp.lowd) fail(TJ_EINVAL, "the low-d DMMA kernel records hit masks: nothing to size");
    // sample items: cells drawn with probability |cell|*|cand| (the estimator),
    // one query block at a random offset of the cell against its whole list
    const int64_t nc = cell_end - cell_begin;
    std::vector<int64_t> cost(nc), start(nc + 1), cand(nc);
    TJ_CUDA(cudaStreamSynchronize(s));
    TJ_CUDA(cudaMemcpy(cost.data(), ctx->cell_cost.as<int64_t>() + cell_begin, sizeof(int64_t) * nc,
                       cudaMemcpyDeviceToHost));
    TJ_CUDA(cudaMemcpy(start.data(), ctx->cell_start.as<int64_t>() + cell_begin,
                       sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost));
    TJ_CUDA(cudaMemcpy(cand.data(), ctx->cell_cand.as<int64_t>() + cell_begin, sizeof(int64_t) * nc,
                       cudaMemcpyDeviceToHost));
    std::vector<double> cum(nc + 1, 0.0);
    for (int64_t c = 0; c < nc; ++c) cum[c + 1] = cum[c] + double(cost[c]);
    if (cum[nc] <= 0) return;
    uint64_t st = seed * 0x9e3779b97f4a7c15ull + 0x632be59bd9b4e019ull;
    auto next = [&]() {  // splitmix64
      uint64_t z = (st += 0x9e3779b97f4a7c15ull);
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      return z ^ (z >> 31);
    };
    std::vector<WorkItem> items;
    for (int i = 0; i < samples; ++i) {
      const double u = double(next() >> 11) * 0x1.0p-53 * cum[nc];
      const int64_t c = std::min<int64_t>(
          nc - 1, std::upper_bound(cum.begin(), cum.end(), u) - cum.begin() - 1);
      const int64_t sz = start[c + 1] - start[c];
      if (sz <= 0 || cand[c] <= 0) continue;
      const int64_t nq = std::min<int64_t>(rp.qpi, sz);
      const int64_t q0 = start[c] + int64_t(next() % uint64_t(sz - nq + 1));
      WorkItem w{};
      w.cell = uint32_t(cell_begin + c);
      w.q0 = uint32_t(q0);
      w.nq = uint32_t(nq);
      w.s0 = 0;
      w.s1 = uint32_t(cand[c]);
      items.push_back(w);
    }
    if (items.empty()) return;
    // run them on the refine kernel, appends counted (not stored) past the buffer;
    // the counters and the sampled queries' counts are restored afterwards
    ctx->items.ensure(sizeof(WorkItem) * items.size(), s);
    TJ_CUDA(cudaMemcpyAsync(ctx->items.ptr, items.data(), sizeof(WorkItem) * items.size(),
                            cudaMemcpyHostToDevice, s));
    ctx->n_items = int64_t(items.size());
    TJ_CUDA(cudaMemcpyAsync(counters(ctx) + 1, counters(ctx), sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
    DevCounters before{};
    TJ_CUDA(cudaMemcpyAsync(&before, counters(ctx), sizeof(before), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaMemsetAsync(&counters(ctx)->item_next, 0, sizeof(unsigned long long), s));
    RefineArgs a = refine_args(ctx, rp, 1);
    a.pair_cap = std::min<unsigned long long>(ctx->pair_cap, before.pairs);  // store nothing new
    launch_refine(ctx, rp, a, s);
    DevCounters after{};
    TJ_CUDA(cudaMemcpyAsync(&after, counters(ctx), sizeof(after), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaMemcpyAsync(counters(ctx), counters(ctx) + 1, sizeof(DevCounters),
                            cudaMemcpyDeviceToDevice, s));
    zero_sample_counts_kernel<<<unsigned(std::min<size_t>(items.size(), 4096)), 64, 0, s>>>(
        ctx->items.as<WorkItem>(), int64_t(items.size()), ctx->qcount.as<uint32_t>());
    TJ_CHECK_LAUNCH();
    TJ_CUDA(cudaStreamSynchronize(s));
    ctx->ctr_valid = false;
    const double refined = double(after.refined - before.refined);
    *pairs_per_candidate = refined > 0 ? double(after.pairs - before.pairs) / refined : 0.0;
  });
}

int tj_set_output_ids(tj_ctx* ctx, const uint32_t* id_map) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    ctx->out_ids = id_map;
    ctx->nid_ready = false;
  });
}

int tj_set_symmetric(tj_ctx* ctx, int32_t on) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    const bool want = on != 0;
    if (want != ctx->symmetric) {
      ctx->symmetric = want;
      ctx->masks_ready = false;  // the mask layout depends on the mode
    }
  });
}

int tj_last_refine_ms(tj_ctx* ctx, double* ms) {
  if (!ctx || !ms) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (!ctx->have_refine_timing) fail(TJ_EINVAL, "no refine launch recorded");
    TJ_CUDA(cudaEventSynchronize(ctx->ev1));
    float t = 0;
    TJ_CUDA(cudaEventElapsedTime(&t, ctx->ev0, ctx->ev1));
    *ms = t;
  });
}

int tj_last_emit_ms(tj_ctx* ctx, double* ms) {
  if (!ctx || !ms) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (!ctx->have_emit_timing) fail(TJ_EINVAL, "no row-emission launch recorded");
    TJ_CUDA(cudaEventSynchronize(ctx->ev3));
    float t = 0;
    TJ_CUDA(cudaEventElapsedTime(&t, ctx->ev2, ctx->ev3));
    *ms = t;
  });
}

int tj_result_count(tj_ctx* ctx, int64_t* total, int32_t* overflowed) {
  if (!ctx || !total) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    cudaStream_t s = ctx->last_stream;
    DevCounters c{};
    TJ_CUDA(cudaMemcpyAsync(&c, counters(ctx), sizeof(c), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaStreamSynchronize(s));
    ctx->ctr = c;
    ctx->ctr_valid = true;
    *total = int64_t(c.pairs + c.hits);  // exact: appends are counted past the capacity
    if (overflowed) *overflowed = c.pairs > ctx->pair_cap ? 1 : 0;
  });
}

int tj_reset_results(tj_ctx* ctx, void* stream) {
  if (!ctx) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    zero_results(ctx, s);
  });
}

static void finalize_phase(tj_ctx* ctx, int64_t* offsets, uint32_t* neighbors, void* stream,
                           int phase) {
  require_grid(ctx);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ctx->last_stream = s;
  DevCounters c = ctx->ctr;  // read by tj_result_count since the last refine
  if (!ctx->ctr_valid) {
    TJ_CUDA(cudaMemcpyAsync(&c, counters(ctx), sizeof(c), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaStreamSynchronize(s));
    ctx->ctr = c;
    ctx->ctr_valid = true;
  }
  if (c.pairs > ctx->pair_cap)
    fail(TJ_ECAPACITY, "result buffer overflowed; call tj_result_count and re-run the batch");
  if (c.pairs > 0 && c.hits > 0)
    fail(TJ_EINVAL, "one result set mixes the low-d DMMA kernel with another kernel");
  if ((phase & 2) && c.pairs + c.hits > 0 && !neighbors) fail(TJ_EINVAL, "neighbors is null");
  finalize_csr(ctx, offsets, neighbors, int64_t(c.pairs), int64_t(c.hits), int64_t(c.max_row), s,
               phase);
}

int tj_finalize(tj_ctx* ctx, int64_t* offsets, uint32_t* neighbors, void* stream) {
  if (!ctx || !offsets) return TJ_EINVAL;
  return guarded(ctx, [&] { finalize_phase(ctx, offsets, neighbors, stream, 3); });
}

int tj_finalize_offsets(tj_ctx* ctx, int64_t* offsets, void* stream) {
  if (!ctx || !offsets) return TJ_EINVAL;
  return guarded(ctx, [&] { finalize_phase(ctx, offsets, nullptr, stream, 1); });
}

int tj_finalize_rows(tj_ctx* ctx, const int64_t* offsets, uint32_t* neighbors, void* stream) {
  if (!ctx || !offsets) return TJ_EINVAL;
  return guarded(ctx, [&] {
    finalize_phase(ctx, const_cast<int64_t*>(offsets), neighbors, stream, 2);
  });
}

int tj_finalize_rows_chunk(tj_ctx* ctx, const int64_t* offsets, uint32_t* neighbors,
                           int32_t chunk, int32_t chunks, void* stream) {
  if (!ctx || !offsets) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    if (chunks < 1 || chunks > 256 || chunk < 0 || chunk >= chunks)
      fail(TJ_EINVAL, "need 0 <= chunk < chunks <= 256");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->last_stream = s;
    DevCounters c = ctx->ctr;
    if (!ctx->ctr_valid) {
      TJ_CUDA(cudaMemcpyAsync(&c, counters(ctx), sizeof(c), cudaMemcpyDeviceToHost, s));
      TJ_CUDA(cudaStreamSynchronize(s));
      ctx->ctr = c;
      ctx->ctr_valid = true;
    }
    if (c.pairs > ctx->pair_cap)
      fail(TJ_ECAPACITY, "result buffer overflowed; call tj_result_count and re-run the batch");
    if (c.pairs + c.hits > 0 && !neighbors) fail(TJ_EINVAL, "neighbors is null");
    if (c.pairs + c.hits == 0) return;
    finalize_rows_range(ctx, offsets, neighbors, int64_t(c.pairs), int64_t(c.hits),
                        int64_t(c.max_row), chunk, chunks, s);
  });
}

int tj_get_stats(tj_ctx* ctx, tj_stats* out) {
  if (!ctx || !out) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    DevCounters c{};
    cudaStream_t s = ctx->last_stream;
    TJ_CUDA(cudaMemcpyAsync(&c, counters(ctx), sizeof(c), cudaMemcpyDeviceToHost, s));
    TJ_CUDA(cudaStreamSynchronize(s));
    out->tiles_processed = int64_t(c.tiles);
    out->chunks_executed = int64_t(c.chunks_exec);
    out->chunks_skipped = int64_t(c.chunks_skip);
    out->candidates_refined = int64_t(c.refined);
    out->pairs_emitted = int64_t(c.pairs + c.hits);
    out->guard_rechecks = int64_t(c.rechecks);
  });
}

int tj_cell_costs(tj_ctx* ctx, int64_t* costs) {
  if (!ctx || !costs) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    TJ_CUDA(cudaStreamSynchronize(ctx->last_stream));
    TJ_CUDA(cudaMemcpy(costs, ctx->cell_cost.ptr, sizeof(int64_t) * ctx->g.n_cells,
                       cudaMemcpyDeviceToHost));
  });
}

int tj_pair_sq_dists(tj_ctx* ctx, const double* coords, int64_t ld, int32_t d,
                     const int64_t* offsets, int64_t n, const uint32_t* neighbors, int64_t m,
                     double* out, void* stream) {
  if (!ctx || !coords || !offsets || (m > 0 && (!neighbors || !out))) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (d < 1 || ld < d || n < 0 || m < 0) fail(TJ_EINVAL, "need d >= 1, ld >= d, n, m >= 0");
    launch_pair_sq_dists(coords, ld, d, offsets, n, neighbors, m, out,
                         static_cast<cudaStream_t>(stream));
  });
}

int tj_write_pairs(const char* path, const int64_t* offsets, int64_t n,
                   const uint32_t* neighbors, const double* sq, int32_t threads) {
  if (!path || !offsets || n < 0) return TJ_EINVAL;
  return guarded(nullptr, [&] {
    if (offsets[n] > 0 && (!neighbors || !sq)) fail(TJ_EINVAL, "neighbors / sq is null");
    write_pairs_file(path, offsets, n, neighbors, sq, threads);
  });
}

int tj_expand_pairs(const int64_t* offsets, int64_t n, const uint32_t* neighbors, int64_t* out,
                    int32_t threads) {
  if (!offsets || n < 0 || !out) return TJ_EINVAL;
  return guarded(nullptr, [&] {
    if (offsets[n] > 0 && !neighbors) fail(TJ_EINVAL, "neighbors is null");
    expand_pairs(offsets, n, neighbors, out, threads);
  });
}

int tj_column_moments(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                      double* mean, double* var, void* stream) {
  if (!ctx || !coords || !mean || !var) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (n < 1 || d < 1 || ld < d) fail(TJ_EINVAL, "need n >= 1, d >= 1, ld >= d");
    column_moments(ctx, coords, n, d, ld, mean, var, static_cast<cudaStream_t>(stream));
  });
}

int tj_permute_columns(tj_ctx* ctx, const double* src, int64_t n, int32_t d, int64_t ld,
                       const int32_t* perm, double* dst, int64_t ld_out, void* stream) {
  if (!ctx || !src || !perm || !dst) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (n < 1 || d < 1 || ld < d || ld_out < d) fail(TJ_EINVAL, "need n, d >= 1, ld, ld_out >= d");
    for (int j = 0; j < d; ++j)
      if (perm[j] < 0 || perm[j] >= d) fail(TJ_EINVAL, "perm entries must be in [0, d)");
    permute_columns(src, n, d, ld, perm, dst, ld_out, static_cast<cudaStream_t>(stream));
  });
}

int tj_brute_force(tj_ctx* ctx, const double* coords, int64_t n, int32_t d, int64_t ld,
                   double eps, int64_t* offsets, uint32_t* neighbors, int64_t* total,
                   void* stream) {
  if (!ctx || !coords || !offsets || (!neighbors && !total)) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (n < 1 || d < 1 || ld < d) fail(TJ_EINVAL, "need n >= 1, d >= 1, ld >= d");
    if (!(std::isfinite(eps) && eps > 0)) fail(TJ_EINVAL, "epsilon must be positive and finite");
    if (n >= (int64_t(1) << 32) - 1) fail(TJ_EINVAL, "n must be < 2^32 - 1 (32-bit point ids)");
    brute_force_join(ctx, coords, n, d, ld, eps, offsets, neighbors, total,
                     static_cast<cudaStream_t>(stream));
  });
}

// ---- page-locked host memory -------------------------------------------------------
int tj_host_register(void* ptr, int64_t bytes, int32_t mapped, void** device_ptr) {
  if (!ptr || bytes <= 0) return TJ_EINVAL;
  return guarded(nullptr, [&] {
    unsigned flags = cudaHostRegisterPortable | (mapped ? cudaHostRegisterMapped : 0u);
    cudaError_t e = cudaHostRegister(ptr, size_t(bytes), flags);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
      (void)cudaGetLastError();  // already page-locked: usable as is, no stale error left behind
    } else if (e != cudaSuccess) {
      (void)cudaGetLastError();
      fail(TJ_ECUDA, std::string("cudaHostRegister failed: ") + cudaGetErrorString(e));
    }
    if (device_ptr) {
      *device_ptr = nullptr;
      e = cudaHostGetDevicePointer(device_ptr, ptr, 0);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(TJ_ECUDA, std::string("cudaHostGetDevicePointer failed: ") + cudaGetErrorString(e));
      }
    }
  });
}

int tj_host_unregister(void* ptr) {
  if (!ptr) return TJ_EINVAL;
  return guarded(nullptr, [&] {
    cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      fail(TJ_ECUDA, std::string("cudaHostUnregister failed: ") + cudaGetErrorString(e));
    }
  });
}

// ---- multi-GPU strong layout (shard.cu) ----------------------------------------
static void check_bins(int32_t pdims, const int64_t* origin, const int64_t* span) {
  if (pdims < 1 || pdims > 2) fail(TJ_EINVAL, "pdims must be 1 or 2");
  if (!origin || !span) fail(TJ_EINVAL, "origin / span is null");
  for (int j = 0; j < pdims; ++j)
    if (span[j] < 1) fail(TJ_EINVAL, "span entries must be >= 1");
}

int tj_shard_bounds(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t pdims,
                    double eps, int64_t* lo, int64_t* hi, void* stream) {
  if (!ctx || !lo || !hi) return TJ_EINVAL;
  return guarded(ctx, [&] {
    if (pdims < 1 || pdims > 2) fail(TJ_EINVAL, "pdims must be 1 or 2");
    if (n > 0 && (!coords || ld < pdims)) fail(TJ_EINVAL, "need coords and ld >= pdims");
    if (!(std::isfinite(eps) && eps > 0)) fail(TJ_EINVAL, "epsilon must be positive and finite");
    shard_bounds(ctx, coords, n, ld, pdims, eps, lo, hi, static_cast<cudaStream_t>(stream));
  });
}

int tj_shard_histogram(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t pdims,
                       double eps, const int64_t* origin, const int64_t* span, int64_t* hist,
                       void* stream) {
  if (!ctx || !hist) return TJ_EINVAL;
  return guarded(ctx, [&] {
    check_bins(pdims, origin, span);
    if (n > 0 && (!coords || ld < pdims)) fail(TJ_EINVAL, "need coords and ld >= pdims");
    shard_histogram(coords, n, ld, pdims, eps, origin, span, hist,
                    static_cast<cudaStream_t>(stream));
  });
}

int tj_shard_select(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t d,
                    int32_t pdims, double eps, const int64_t* origin, const int64_t* span,
                    int64_t own_lo, int64_t own_hi, double* out, int64_t ld_out, uint32_t* gid,
                    int64_t gid_base, int64_t capacity, int64_t* selected, void* stream) {
  if (!ctx || !selected) return TJ_EINVAL;
  return guarded(ctx, [&] {
    check_bins(pdims, origin, span);
    if (n > 0 && (!coords || ld < d || d < pdims)) fail(TJ_EINVAL, "need coords, ld >= d >= pdims");
    if (out && (!gid || ld_out < d)) fail(TJ_EINVAL, "need gid and ld_out >= d with out");
    *selected = shard_select(ctx, coords, n, ld, d, pdims, eps, origin, span, own_lo, own_hi, out,
                             ld_out, gid, gid_base, capacity, static_cast<cudaStream_t>(stream));
  });
}

int tj_shard_route(tj_ctx* ctx, const double* coords, int64_t n, int64_t ld, int32_t d,
                   int32_t pdims, double eps, const int64_t* origin, const int64_t* span,
                   const int64_t* own_lo, const int64_t* own_hi, int32_t ranks, int64_t* counts,
                   double* out, int64_t ld_out, uint32_t* gid, int64_t gid_base, int64_t capacity,
                   void* stream) {
  if (!ctx || !counts || !own_lo || !own_hi || ranks < 1 || ranks > 1024) return TJ_EINVAL;
  return guarded(ctx, [&] {
    check_bins(pdims, origin, span);
    if (n > 0 && (!coords || ld < d || d < pdims)) fail(TJ_EINVAL, "need coords, ld >= d >= pdims");
    if (out && (!gid || ld_out < d)) fail(TJ_EINVAL, "need gid and ld_out >= d with out");
    shard_route(ctx, coords, n, ld, d, pdims, eps, origin, span, own_lo, own_hi, ranks, counts, out,
                ld_out, gid, gid_base, capacity, static_cast<cudaStream_t>(stream));
  });
}

int tj_shard_cell_range(tj_ctx* ctx, int32_t pdims, const int64_t* origin, const int64_t* span,
                        int64_t own_lo, int64_t own_hi, int64_t* cell_begin, int64_t* cell_end) {
  if (!ctx || !cell_begin || !cell_end) return TJ_EINVAL;
  return guarded(ctx, [&] {
    require_grid(ctx);
    check_bins(pdims, origin, span);
    if (pdims > ctx->g.k) fail(TJ_EINVAL, "pdims exceeds the grid's k_idx");
    shard_cell_range(ctx, pdims, origin, span, own_lo, own_hi, cell_begin, cell_end,
                     ctx->last_stream);
  });
}

int tj_remap_ids(tj_ctx* ctx, uint32_t* ids, int64_t m, const uint32_t* gid, void* stream) {
  if (!ctx || (m > 0 && (!ids || !gid))) return TJ_EINVAL;
  return guarded(ctx, [&] { shard_remap_ids(ids, m, gid, static_cast<cudaStream_t>(stream)); });
}

int tj_scatter_counts(tj_ctx* ctx, const int64_t* offsets, int64_t n_rows, const uint32_t* gid,
                      int32_t* counts, void* stream) {
  if (!ctx || (n_rows > 0 && (!offsets || !gid || !counts))) return TJ_EINVAL;
  return guarded(ctx, [&] {
    shard_scatter_counts(offsets, n_rows, gid, counts, static_cast<cudaStream_t>(stream));
  });
}

int tj_scatter_counts_u8(tj_ctx* ctx, const int64_t* offsets, int64_t n_rows, const uint32_t* gid,
                         uint8_t* counts, int32_t* overflow, void* stream) {
  if (!ctx || !overflow || (n_rows > 0 && (!offsets || !gid || !counts))) return TJ_EINVAL;
  return guarded(ctx, [&] {
    shard_scatter_counts_u8(offsets, n_rows, gid, counts, overflow, static_cast<cudaStream_t>(stream));
  });
}

int tj_counts_u8_to_offsets(tj_ctx* ctx, const uint8_t* counts, int64_t n, int64_t* offsets,
                            void* stream) {
  if (!ctx || !offsets || (n > 0 && !counts) || n < 0) return TJ_EINVAL;
  return guarded(ctx, [&] {
    counts_to_offsets_u8(ctx, counts, n, offsets, static_cast<cudaStream_t>(stream));
  });
}

int tj_counts_to_offsets(tj_ctx* ctx, const int32_t* counts, int64_t n, int64_t* offsets,
                         void* stream) {
  if (!ctx || !offsets || (n > 0 && !counts) || n < 0) return TJ_EINVAL;
  return guarded(ctx, [&] {
    counts_to_offsets(ctx, counts, n, offsets, static_cast<cudaStream_t>(stream));
  });
}

int tj_place_rows(tj_ctx* ctx, const int64_t* offsets, const uint32_t* neighbors, int64_t n_rows,
                  const uint32_t* gid, const int64_t* global_offsets, uint32_t* dst, void* stream) {
  if (!ctx || (n_rows > 0 && (!offsets || !gid || !global_offsets || !dst))) return TJ_EINVAL;
  return guarded(ctx, [&] {
    shard_place_rows(offsets, neighbors, n_rows, gid, global_offsets, dst,
                     static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
