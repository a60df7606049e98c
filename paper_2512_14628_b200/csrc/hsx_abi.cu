// Host side of libhsx: plan construction (layer table, work lists, scratch)
// and the extern "C" entry points declared in include/hsx.h.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/hsx.h"
#include "hsx_kernels.cuh"

using hsx::DevLayer;
using hsx::Item;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int check_cuda(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HSX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return HSX_OK;
}

#define HSX_CUDA(call)                                                              \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) return fail(HSX_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr long long kAlign = 32;        // arena layer alignment in elements (128 B)
constexpr int kSubElems = 4096;         // target elements per shared-memory sub-tile
constexpr int hsx_tile_quads = 64;      // quad tiles: rows x 64 column quads (hsx_kernels.cu)
#ifndef HSX_CAND_QUADS
#define HSX_CAND_QUADS 64
#endif
constexpr int hsx_cand_quads = HSX_CAND_QUADS;  // K1's own quad tiles (hsx_kernels.cu kCandQuads)
// rows per quad tile (K1; K6/K7; K3); HSX_CAND_TILE_ROWS / HSX_STREAM_TILE_ROWS / HSX_PROJ_TILE_ROWS
// override them for tuning runs (multiples of 4, <= kMaxTileRows = 128)
int tile_rows_env(const char* name, int dflt) {
  const char* v = std::getenv(name);
  int r = v ? std::atoi(v) : dflt;
  if (r < 4 || r > 128 || (r & 3)) r = dflt;
  return r;
}
int env_flag(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
// select_layer's shared memory: G u64 keys + G flag bytes, then the structured
// keep-set derivation of the layer (one node)
size_t select_need(const DevLayer& ly, int q) {
  return hsx::select_smem_bytes(ly.G[q]) + hsx::structured_smem_bytes(ly.rows, ly.L, ly.cin);
}
constexpr long long kItemElems = 8192;  // elements per streaming work item
constexpr long long kProjElems = 1024;  // K3 items of layers without row-quad tiles (32 words)
constexpr long long kWordItem = 512;    // mask words per keep-mark item
constexpr int kMaxSelectGroups = 8192;  // radix top-k capacity of one selection CTA (keys + flags in smem)
constexpr size_t kMaxSmem = 200 * 1024;

template <typename T>
int upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return HSX_OK;
  HSX_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), src.size() * sizeof(T)));
  HSX_CUDA(cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
  return HSX_OK;
}

template <typename T>
int alloc0(T** dst, long long n) {
  *dst = nullptr;
  if (n <= 0) return HSX_OK;
  HSX_CUDA(cudaMalloc(reinterpret_cast<void**>(dst), (size_t)n * sizeof(T)));
  HSX_CUDA(cudaMemset(*dst, 0, (size_t)n * sizeof(T)));
  return HSX_OK;
}

}  // namespace

struct hsx_plan {
  int n_layers = 0;
  int max_passes = 0;
  int identity = 0;
  long long arena = 0;
  long long mask_words = 0;
  long long gtotal[hsx::kMaxPasses] = {0, 0, 0};
  long long ptotal[hsx::kMaxPasses] = {0, 0, 0};
  long long ktotal[2] = {0, 0};
  long long ctotal = 0;  // column-map entries (sum of L over prunable layers, padded to 4)
  std::vector<DevLayer> layers;
  std::vector<Item> cand_dyn, elem_items, stream_items, proj_items, word_items;
  std::vector<int> pass_list[hsx::kMaxPasses];
  std::vector<int> sel_list[hsx::kMaxPasses];  // layers whose pass-q selection needs the K2 launch
  std::vector<int> prunable;
  size_t cand_smem = 0, select_smem[hsx::kMaxPasses] = {0, 0, 0}, mark_smem = 0, fixup_smem = 0;
  int single_node = 0;  // structured keep sets in the selection tail (M == 1)
  int sqcap = 0;
  // device
  DevLayer* d_layers = nullptr;
  Item *d_cand = nullptr, *d_elem = nullptr, *d_stream = nullptr, *d_proj = nullptr, *d_word = nullptr;
  unsigned int* d_layer_done = nullptr;
  unsigned int* d_cand_done = nullptr;
  unsigned int* d_sched = nullptr;
  int *d_sfirst = nullptr, *d_scount = nullptr;  // per layer: first stream item, item count
  double* d_rpart = nullptr;                       // residual partials [stream item][9]
  unsigned int *d_ready = nullptr, *d_pdone = nullptr;  // merged K2 + K3: per layer / prunable layer
  cudaEvent_t fetch_ev = nullptr;                  // recorded after the summary D2H (external in graphs)
  unsigned long long* d_acc = nullptr;
  uint8_t *d_rk_prev = nullptr, *d_ck_prev = nullptr, *d_ch_prev = nullptr;
  int *d_irr = nullptr, *d_irr_any = nullptr;
  unsigned int* d_k1done = nullptr;  // chained K2: K1 tiles finished per prunable layer (0 between steps)
  float* d_stage = nullptr;          // staged peer operand (two ranks): local copy of the peer's send
  unsigned int *d_sready = nullptr, *d_sepoch = nullptr, *d_scounter = nullptr;
  int k2_armed = 0;                  // the last launch was such a K1: hsx_select(0) chains behind it
  int k2_pending = 0;                // a counting K1 ran whose counts no chained K2 consumed yet
  // split two-rank K1 (hsx_plan_set_split): this rank's work list (dense items and
  // every other prunable tile), the peer's partials / tile counts; partials[0] and
  // the counts then live in caller-owned peer-mapped memory (not freed here)
  Item* d_cand_split = nullptr;
  int n_cand_split = 0;
  int split_me = -1;
  double* partials_peer = nullptr;
  unsigned int* k1done_peer = nullptr;
  int ext_partials = 0, ext_k1done = 0;
  int k3_armed = 0;                  // the last launch was a chained single-pass K2: K3 chains behind it
  int k67_armed = 0;                 // the last launch was a chained one-node K3 with fixups: K67 chains
  int k67_chain = 0;                 // hsx_plan_set_k67_chain: the caller follows every one-node projection with K67
  unsigned int *d_ready3 = nullptr, *d_cnt67 = nullptr, *d_up = nullptr;  // K3 -> K67 chain flags
  long long* h_pub = nullptr;        // mapped host summary the chained K3 publishes into (+ seq word after)
  unsigned int* d_seq_ctr = nullptr;
  unsigned int last_seq = 0;
  int pub_mapped = 0;                // dynamic one-node steps publish the summary from the device
  int big_first = 0;                 // work-list order (set_order)
  int* d_sel[hsx::kMaxPasses] = {nullptr, nullptr, nullptr};
  int* d_prunable = nullptr;
  double* d_partials[hsx::kMaxPasses] = {nullptr, nullptr, nullptr};
  double* d_norms[hsx::kMaxPasses] = {nullptr, nullptr, nullptr};
  uint8_t* d_flags[hsx::kMaxPasses] = {nullptr, nullptr, nullptr};
  uint8_t *d_oflag = nullptr, *d_iflag = nullptr;
  int *d_pos_out = nullptr, *d_pos_in = nullptr;
  long long* d_summary = nullptr;
  unsigned int* d_done = nullptr;
  std::vector<long long> summary;  // host mirror (dense rows, installed keep sets)

  ~hsx_plan() {
    if (ext_k1done) d_k1done = nullptr;
    if (ext_partials) d_partials[0] = nullptr;
    if (d_cand_split) cudaFree(d_cand_split);
    void* ptrs[] = {d_stage, d_sready, d_sepoch, d_scounter, d_ready3, d_cnt67, d_up, d_k1done, d_layers, d_cand, d_layer_done, d_cand_done, d_sched, d_sfirst, d_scount, d_rpart, d_ready, d_pdone, d_acc, d_rk_prev, d_ck_prev, d_irr, d_irr_any, d_elem, d_stream, d_proj, d_word, d_prunable, d_oflag, d_iflag,
                    d_pos_out, d_pos_in, d_summary, d_done,
                    d_ch_prev};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (fetch_ev) cudaEventDestroy(fetch_ev);
    if (h_pub) cudaFreeHost(h_pub);
    if (d_seq_ctr) cudaFree(d_seq_ctr);
    for (int i = 0; i < hsx::kMaxPasses; ++i) {
      if (d_sel[i]) cudaFree(d_sel[i]);
      if (d_partials[i]) cudaFree(d_partials[i]);
      if (d_norms[i]) cudaFree(d_norms[i]);
      if (d_flags[i]) cudaFree(d_flags[i]);
    }
  }
};

namespace {

// lay out flat-buffer offsets from the host summary mirror (layer order)
void host_layout(hsx_plan* p) {
  long long off = 0;
  for (int l = 0; l < p->n_layers; ++l) {
    long long* row = &p->summary[(size_t)l * HSX_SUM_COLS];
    row[HSX_SUM_OFFSET] = off;
    off += row[HSX_SUM_ELEMS];
  }
  p->summary[(size_t)p->n_layers * HSX_SUM_COLS] = off;
}

// Work-list order of K1 / K2 / K3. big_first: the layers with the costliest
// selection tails first, so their chained K2 CTAs select while K1 streams the rest
// (B200 r2m, one GPU: RN18 0.130 -> 0.122 ms with the chain). Otherwise layer order
// (group-norm tiles first, dense items last): measured faster when K1 reads the
// node's sums over NVLink (r2n, RN50 2x2: 0.649 vs 0.663 ms).
void set_order(hsx_plan* p, bool big_first) {
  auto cost = [&](int l) {
    const DevLayer& ly = p->layers[l];
    if (ly.ncons == 0) return -1LL;
    long long c = (long long)ly.rows + ly.cin;
    for (int q = 0; q < ly.ncons; ++q) c += ly.G[q];
    return c;
  };
  auto before = [&](int x, int y) {  // strict order of layers x, y
    if (big_first) return cost(x) > cost(y);
    const bool dx = cost(x) < 0, dy = cost(y) < 0;
    return dx != dy ? dy : x < y;
  };
  std::stable_sort(p->cand_dyn.begin(), p->cand_dyn.end(),
                   [&](const Item& x, const Item& y) { return x.layer != y.layer && before(x.layer, y.layer); });
  for (int q = 0; q < hsx::kMaxPasses; ++q)
    std::stable_sort(p->sel_list[q].begin(), p->sel_list[q].end(), before);
  std::stable_sort(p->proj_items.begin(), p->proj_items.end(),
                   [&](const Item& x, const Item& y) { return x.layer != y.layer && before(x.layer, y.layer); });
  p->big_first = big_first ? 1 : 0;
}

int build(hsx_plan* p, const hsx_layer_desc* in, int n) {
  p->n_layers = n;
  long long off = 0, mword = 0, okeep = 0, ikeep = 0, cpoff = 0;
  long long goff[hsx::kMaxPasses] = {0, 0, 0}, poff[hsx::kMaxPasses] = {0, 0, 0};
  int sqcap = 0, quadcap = 0;
  std::vector<Item> dense_items;
  size_t mark_smem = 0;
  p->summary.assign((size_t)n * HSX_SUM_COLS + 1, 0);
  for (int l = 0; l < n; ++l) {
    const hsx_layer_desc& d = in[l];
    DevLayer ly;
    std::memset(&ly, 0, sizeof(ly));
    if (d.rank != 2 && d.rank != 4) return fail(HSX_ESHAPE, "layer %d: rank must be 2 or 4, got %d", l, d.rank);
    for (int i = 0; i < d.rank; ++i)
      if (d.shape[i] <= 0) return fail(HSX_ESHAPE, "layer %d: non-positive dimension", l);
    ly.rank = d.rank;
    ly.rows = d.shape[0];
    ly.cin = d.shape[1];
    ly.k = d.rank == 4 ? d.shape[2] * d.shape[3] : 1;
    ly.L = ly.cin * ly.k;
    ly.n = (long long)ly.rows * ly.L;
    if (ly.n >= (1LL << 31)) return fail(HSX_ESHAPE, "layer %d: more than 2^31 elements", l);
    ly.off = off;
    off += (ly.n + kAlign - 1) / kAlign * kAlign;
    ly.divL = hsx::make_fastdiv((unsigned)ly.L);
    ly.divk = hsx::make_fastdiv((unsigned)ly.k);
    ly.rho1 = d.rho1;
    ly.rho2 = d.rho2;
    ly.gamma = 1.0;
    ly.rgamma = 1.0;
    ly.mword = -1;
    ly.okeep = ly.ikeep = ly.cpoff = -1;
    for (int q = 0; q < hsx::kMaxPasses; ++q) ly.goff[q] = ly.poff[q] = -1;
    if (d.n_constraints < 0 || d.n_constraints > HSX_MAX_CONSTRAINTS)
      return fail(HSX_ESHAPE, "layer %d: %d constraints (max %d)", l, d.n_constraints, HSX_MAX_CONSTRAINTS);
    ly.ncons = d.n_constraints;
    long long* srow = &p->summary[(size_t)l * HSX_SUM_COLS];
    if (ly.ncons > 0) {
      if (d.rank != 4) return fail(HSX_ESHAPE, "layer %d: only conv layers are prunable", l);
      if (ly.L > 16384) return fail(HSX_ESHAPE, "layer %d: row of %d elements exceeds 16384", l, ly.L);
      for (int q = 0; q < ly.ncons; ++q) {
        int g = d.group[q];
        if (g < 0 || g > 2) return fail(HSX_ESHAPE, "layer %d: bad group kind %d", l, g);
        for (int r = 0; r < q; ++r)
          if (d.group[r] == g) return fail(HSX_ESHAPE, "layer %d: duplicate constraint kinds", l);
        int G = g == HSX_GROUP_FILTER ? ly.rows : (g == HSX_GROUP_CHANNEL ? ly.cin : ly.L);
        if (d.keep[q] < 1) return fail(HSX_ESHAPE, "layer %d: keep_count must be positive", l);
        if (d.keep[q] > G) return fail(HSX_ESHAPE, "layer %d: keep_count %d exceeds group count %d", l, d.keep[q], G);
        if (G > kMaxSelectGroups) return fail(HSX_ESHAPE, "layer %d: %d groups exceed %d", l, G, kMaxSelectGroups);
        ly.group[q] = g;
        ly.keep[q] = d.keep[q];
        ly.G[q] = G;
      }
      ly.rsub = std::max(1, kSubElems / ly.L);
      // quad tiling when every pass groups columns (CHANNEL / SHAPE) and rows are
      // a multiple of 4 elements; otherwise row tiling (FILTER, stems)
      // quad tiles of 64 column quads (1 KB-aligned row segments, per-column
      // partials folded into channels by the selection); HSX_K1_PERCOL=0 makes a
      // tile hold whole channels instead (cq quads, 4*cq a multiple of kh*kw,
      // per-channel partials)
      const int kmul = ly.k / std::gcd(ly.k, 4);
      const bool percol = env_flag("HSX_K1_PERCOL", 1) != 0;
      const int cq = percol ? hsx_cand_quads : hsx_cand_quads / kmul * kmul;
      ly.percol = percol ? 1 : 0;
      bool quads = (ly.L & 3) == 0 && cq > 0;
      for (int q = 0; q < ly.ncons; ++q) quads = quads && ly.group[q] != HSX_GROUP_FILTER;
      ly.tiling = quads ? 1 : 0;
      ly.pidx = (int)p->prunable.size();
      if (quads) {
        const int tr = tile_rows_env("HSX_CAND_TILE_ROWS", 128);
        const int nchunks = (ly.L / 4 + cq - 1) / cq;
        ly.cq = cq;
        // lanes per row: the tile's quads rounded up to a power of two (HSX_K1_NARROW=0:
        // always hsx_cand_quads); a narrow layer's spare lanes take more row phases
        ly.cw = hsx_cand_quads;
        if (env_flag("HSX_K1_NARROW", 1)) {
          const int q = std::min(cq, ly.L / 4);
          ly.cw = 1;
          while (ly.cw < q) ly.cw <<= 1;
          ly.cw = std::min(ly.cw, hsx_cand_quads);
        }
        ly.nparts = (ly.rows + tr - 1) / tr;
        for (int pt = 0; pt < ly.nparts; ++pt)
          for (int cc = 0; cc < nchunks; ++cc) {
            Item it{l, pt, cc, 1, (long long)pt * tr, std::min<long long>((long long)(pt + 1) * tr, ly.rows)};
            p->cand_dyn.push_back(it);
          }
        ly.ncitems = ly.nparts * nchunks;
        quadcap = std::max(quadcap, 4 * hsx_cand_quads * (256 / hsx_cand_quads));
      } else {
        sqcap = std::max(sqcap, ly.rsub * ly.L);
        // one shared-memory sub-tile of rows per item
        const long long rows_item = std::min<long long>(ly.rsub, ly.rows);
        ly.nparts = (int)((ly.rows + rows_item - 1) / rows_item);
        for (int pt = 0; pt < ly.nparts; ++pt) {
          Item it{l, pt, 0, 0, pt * rows_item * ly.L, std::min<long long>((pt + 1) * rows_item, ly.rows) * ly.L};
          p->cand_dyn.push_back(it);
        }
        ly.ncitems = ly.nparts;
      }
      for (int q = 0; q < ly.ncons; ++q) {
        ly.goff[q] = goff[q];
        goff[q] += ly.G[q];
        ly.poff[q] = poff[q];
        poff[q] += ly.group[q] == HSX_GROUP_FILTER ? ly.rows : (long long)ly.nparts * (ly.percol ? ly.L : ly.G[q]);
        p->pass_list[q].push_back(l);
        p->max_passes = std::max(p->max_passes, q + 1);
      }
      ly.mword = mword;
      mword += (ly.n + 31) / 32;
      ly.okeep = okeep;
      okeep += (ly.rows + 15) / 16 * 16;  // 16-B aligned per layer (cp.async of the byte flags)
      ly.ikeep = ikeep;
      ikeep += (ly.cin + 15) / 16 * 16;
      ly.cpoff = cpoff;
      cpoff += (ly.L + 15) / 16 * 16;
      p->prunable.push_back(l);
      ly.qtile = (ly.L % 32) == 0 ? 1 : 0;
      if (ly.qtile) {
        // row-quad tiles for K3 / K6 / K7 (same shape as the K1 quad tiles)
        const int tq = hsx_tile_quads, tr = tile_rows_env("HSX_STREAM_TILE_ROWS", 32);
        const int trp = tile_rows_env("HSX_PROJ_TILE_ROWS", 64);
        const int nchunks = (ly.L / 4 + tq - 1) / tq;
        for (int r0 = 0; r0 < ly.rows; r0 += tr)
          for (int cc = 0; cc < nchunks; ++cc) {
            Item it{l, r0 / tr, cc, 1, (long long)r0, std::min<long long>(r0 + tr, ly.rows)};
            p->stream_items.push_back(it);
          }
        for (int r0 = 0; r0 < ly.rows; r0 += trp)
          for (int cc = 0; cc < nchunks; ++cc) {
            Item it{l, r0 / trp, cc, 1, (long long)r0, std::min<long long>(r0 + trp, ly.rows)};
            p->proj_items.push_back(it);
            ++ly.npitems;
          }
      } else {
        // K3's warp-per-word path is latency-bound: small items, many CTAs
        for (long long b = 0; b < ly.n; b += kProjElems) {
          Item it{l, 0, 0, 0, b, std::min(ly.n, b + kProjElems)};
          p->proj_items.push_back(it);
          ++ly.npitems;
        }
        for (long long b = 0; b < ly.n; b += kItemElems) {
          Item it{l, 0, 0, 0, b, std::min(ly.n, b + kItemElems)};
          p->stream_items.push_back(it);
        }
      }
      // fused K3 + K5: the keep-set tail reuses the ring's shared memory for positions
      p->fixup_smem = std::max<size_t>(p->fixup_smem, (size_t)ly.cin + ly.rows);
      const int nwi = (int)((ly.n + kWordItem * 32 - 1) / (kWordItem * 32));
      for (long long b = 0; b < ly.n; b += kWordItem * 32) {
        Item it{l, ly.pidx, nwi, 0, b, std::min(ly.n, b + kWordItem * 32)};
        p->word_items.push_back(it);
        long long r_lo = b / ly.L, r_hi = (it.end - 1) / ly.L;
        // flags (c_in + rows of the item), 16-B aligned, then the column words of a row
        mark_smem = std::max<size_t>(mark_smem, (((size_t)ly.cin + (size_t)(r_hi - r_lo + 1) + 15) & ~(size_t)15) +
                                                    (ly.L % 32 == 0 ? (size_t)(ly.L / 32) * 4 : 0));
      }
    } else {
      for (long long b = 0; b < ly.n; b += kItemElems) {
        Item it{l, 0, 0, 0, b, std::min(ly.n, b + kItemElems)};
        dense_items.push_back(it);
      }
    }
    for (long long b = 0; b < ly.n; b += kItemElems) {
      Item it{l, 0, 0, 0, b, std::min(ly.n, b + kItemElems)};
      p->elem_items.push_back(it);
      if (ly.ncons == 0) p->stream_items.push_back(it);
    }
    // initial keep sets: everything kept (all-ones initial masks, consensus.py:418)
    srow[HSX_SUM_KOUT] = ly.rows;
    srow[HSX_SUM_KIN] = ly.cin;
    srow[HSX_SUM_ELEMS] = ly.n;
    p->layers.push_back(ly);
  }
  // dynamic candidate launch: group-norm tiles first, short dense items fill the
  // tail; persistent CTAs take the largest items first
  p->cand_dyn.insert(p->cand_dyn.end(), dense_items.begin(), dense_items.end());
  // launch order: set_order() below, once the selection lists exist
  // the last layer needs no trailing pad: arenas may be exactly-sized tensors
  if (n > 0) off = p->layers.back().off + p->layers.back().n;
  p->arena = off;
  p->mask_words = mword;
  p->ktotal[0] = okeep;
  p->ktotal[1] = ikeep;
  p->ctotal = cpoff;
  for (int q = 0; q < hsx::kMaxPasses; ++q) {
    p->gtotal[q] = goff[q];
    p->ptotal[q] = poff[q];
    p->select_smem[q] = 0;
    for (int l : p->pass_list[q]) p->select_smem[q] = std::max(p->select_smem[q], select_need(p->layers[l], q));
  }
  p->sqcap = sqcap;
  // k_candidate: cp.async ring (kDepth x 4 x 256 float4 = 64 KB; the 8 KB quad fold
  // aliases it once drained: three CTAs per SM), or the row-tile path's sub-tile
  // squares + group accumulators
  p->cand_smem = std::max((size_t)sqcap * sizeof(double),
                          std::max((size_t)4 * 4 * 256 * 16, (size_t)quadcap * sizeof(double)));
  p->mark_smem = mark_smem;
  // selection as its own launch (K2, one CTA per layer on otherwise idle SMs) by
  // default: in K1's tail (HSX_FUSE_SELECT=1) a layer's selection shares its SM
  // with streaming tiles and every dependent L2 round trip of the tail stalls
  // behind their traffic (measured: K1 + fused tails 77-85 us vs K1 56 + K2 25)
  const bool fuse = env_flag("HSX_FUSE_SELECT", 0) != 0;
  for (int q = 0; q < hsx::kMaxPasses; ++q) {
    for (int l : p->pass_list[q]) {
      DevLayer& ly = p->layers[l];
      if (fuse && select_need(ly, q) <= p->cand_smem)
        ly.fsel |= 1 << q;
      else
        p->sel_list[q].push_back(l);
    }
  }
  set_order(p, env_flag("HSX_K1_ORDER", 1) != 0);
  if (p->cand_smem > kMaxSmem) return fail(HSX_ESHAPE, "candidate tile needs %zu B of shared memory", p->cand_smem);
  host_layout(p);
  return HSX_OK;
}

int upload_plan(hsx_plan* p) {
  int rc;
  if ((rc = upload(&p->d_layers, p->layers))) return rc;
  if ((rc = upload(&p->d_cand, p->cand_dyn))) return rc;
  if ((rc = alloc0(&p->d_layer_done, (long long)p->prunable.size()))) return rc;
  if ((rc = alloc0(&p->d_cand_done, (long long)p->prunable.size()))) return rc;
  if ((rc = alloc0(&p->d_sched, 2))) return rc;
  if ((rc = alloc0(&p->d_ready, std::max(1, p->n_layers)))) return rc;
  if ((rc = alloc0(&p->d_pdone, (long long)p->prunable.size() + 1))) return rc;  // + layers-done counter
  if ((rc = alloc0(&p->d_acc, 2 * (long long)p->prunable.size()))) return rc;
  if ((rc = alloc0(&p->d_irr, (long long)p->prunable.size()))) return rc;
  if ((rc = alloc0(&p->d_irr_any, 1))) return rc;
  // previous rectangle: the all-ones initial mask (consensus.py:418)
  const std::vector<uint8_t> ones_r(p->ktotal[0], 1), ones_c(p->ctotal, 1), ones_i(p->ktotal[1], 1);
  rc = upload(&p->d_rk_prev, ones_r);
  if (rc) return rc;
  rc = upload(&p->d_ck_prev, ones_c);
  if (rc) return rc;
  rc = upload(&p->d_ch_prev, ones_i);
  if (rc) return rc;
  if ((rc = upload(&p->d_elem, p->elem_items))) return rc;
  if ((rc = upload(&p->d_stream, p->stream_items))) return rc;
  {  // stream items are laid out layer by layer: per-layer ranges for the residual fold
    std::vector<int> first(p->n_layers, 0), count(p->n_layers, 0);
    for (size_t i = p->stream_items.size(); i-- > 0;) {
      first[p->stream_items[i].layer] = (int)i;
      ++count[p->stream_items[i].layer];
    }
    if ((rc = upload(&p->d_sfirst, first))) return rc;
    if ((rc = upload(&p->d_scount, count))) return rc;
    if ((rc = alloc0(&p->d_rpart, (long long)std::max<size_t>(1, p->stream_items.size()) * hsx::kResidSlots)))
      return rc;
  }
  if ((rc = upload(&p->d_proj, p->proj_items))) return rc;
  if ((rc = upload(&p->d_word, p->word_items))) return rc;
  if ((rc = upload(&p->d_prunable, p->prunable))) return rc;
  for (int q = 0; q < hsx::kMaxPasses; ++q) {
    if ((rc = upload(&p->d_sel[q], p->sel_list[q]))) return rc;
    if ((rc = alloc0(&p->d_partials[q], p->ptotal[q]))) return rc;
    if ((rc = alloc0(&p->d_norms[q], p->gtotal[q]))) return rc;
    if ((rc = alloc0(&p->d_flags[q], p->gtotal[q]))) return rc;
  }
  if ((rc = alloc0(&p->d_oflag, p->ktotal[0]))) return rc;
  if ((rc = alloc0(&p->d_iflag, p->ktotal[1]))) return rc;
  // identity positions (all kept) until the first keep-set derivation
  std::vector<int> po(p->ktotal[0], -1), pi(p->ktotal[1], -1);  // per-layer padding: -1
  for (int l : p->prunable) {
    const DevLayer& ly = p->layers[l];
    for (int i = 0; i < ly.rows; ++i) po[ly.okeep + i] = i;
    for (int i = 0; i < ly.cin; ++i) pi[ly.ikeep + i] = i;
  }
  if ((rc = upload(&p->d_pos_out, po))) return rc;
  if ((rc = upload(&p->d_pos_in, pi))) return rc;
  if ((rc = upload(&p->d_summary, p->summary))) return rc;
  if ((rc = alloc0(&p->d_done, 1))) return rc;
  if ((rc = alloc0(&p->d_k1done, (long long)p->prunable.size() + 1))) return rc;
  if ((rc = alloc0(&p->d_ready3, std::max(1, p->n_layers)))) return rc;
  if ((rc = alloc0(&p->d_cnt67, std::max(1, p->n_layers)))) return rc;
  if ((rc = alloc0(&p->d_up, 2))) return rc;   // [0] upstream complete, [1] K67 items done
  return HSX_OK;
}

}  // namespace

// ===========================================================================
// extern "C" entry points
// ===========================================================================

#define HSX_TRY(body)                                                      \
  try {                                                                    \
    body                                                                   \
  } catch (const std::bad_alloc&) {                                        \
    return fail(HSX_EINVAL, "host allocation failed");                     \
  } catch (...) {                                                          \
    return fail(HSX_EINVAL, "unexpected C++ exception");                   \
  }

#define HSX_LAUNCHED(what)        \
  do {                            \
    g_launches.fetch_add(1);      \
    int rc_ = check_cuda(what);   \
    if (rc_) return rc_;          \
  } while (0)

extern "C" {

int hsx_abi_version(void) { return HSX_ABI_VERSION; }
const char* hsx_last_error(void) { return g_err.c_str(); }
int64_t hsx_launch_count(void) { return g_launches.load(); }
void hsx_note_graph_replay(int64_t kernels) { if (kernels > 0) g_launches.fetch_add(kernels); }

int hsx_plan_create(const hsx_layer_desc* layers, int32_t n_layers, hsx_plan** out) {
  if (!out || (!layers && n_layers > 0) || n_layers < 0) return fail(HSX_EINVAL, "null argument");
  *out = nullptr;
  HSX_TRY({
    hsx_plan* p = new hsx_plan();
    int rc = build(p, layers, n_layers);
    if (!rc) rc = upload_plan(p);
    if (rc) {
      delete p;
      return rc;
    }
    *out = p;
    return HSX_OK;
  })
}

void hsx_plan_destroy(hsx_plan* plan) { delete plan; }

int64_t hsx_plan_arena_elements(const hsx_plan* p) { return p ? p->arena : -1; }
int64_t hsx_plan_layer_offset(const hsx_plan* p, int32_t l) {
  return (p && l >= 0 && l < p->n_layers) ? p->layers[l].off : -1;
}
int64_t hsx_plan_mask_words(const hsx_plan* p) { return p ? p->mask_words : -1; }
int64_t hsx_plan_mask_word_offset(const hsx_plan* p, int32_t l) {
  return (p && l >= 0 && l < p->n_layers) ? p->layers[l].mword : -1;
}
int64_t hsx_plan_group_offset(const hsx_plan* p, int32_t l, int32_t pass) {
  if (!p || l < 0 || l >= p->n_layers || pass < 0 || pass >= hsx::kMaxPasses) return -1;
  return p->layers[l].goff[pass];
}
int64_t hsx_plan_group_total(const hsx_plan* p, int32_t pass) {
  return (p && pass >= 0 && pass < hsx::kMaxPasses) ? p->gtotal[pass] : -1;
}
int64_t hsx_plan_keep_offset(const hsx_plan* p, int32_t l, int32_t which) {
  if (!p || l < 0 || l >= p->n_layers) return -1;
  return which == 0 ? p->layers[l].okeep : p->layers[l].ikeep;
}
int64_t hsx_plan_keep_total(const hsx_plan* p, int32_t which) {
  return p ? p->ktotal[which ? 1 : 0] : -1;
}
int32_t hsx_plan_max_passes(const hsx_plan* p) { return p ? p->max_passes : -1; }

int hsx_plan_set_penalties(hsx_plan* p, const double* rho1, const double* rho2, double wd,
                           int32_t num_nodes, int32_t per_node, int32_t identity) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (num_nodes < 1 || per_node < 1) return fail(HSX_ECONFIG, "topology dimensions must be positive");
  for (int l = 0; l < p->n_layers; ++l) {
    DevLayer& ly = p->layers[l];
    if (rho1) ly.rho1 = rho1[l];
    if (rho2) ly.rho2 = rho2[l];
    // consensus.py:157-159, same fp64 expression order
    double gamma = wd / (double)num_nodes + (double)per_node * ly.rho1 + ly.rho2;
    if (!identity && !(gamma > 0.0))
      return fail(HSX_ECONFIG, "non-positive candidate normalizer gamma=%g (layer %d)", gamma, l);
    ly.gamma = gamma;
    ly.rgamma = 1.0 / gamma;
  }
  p->identity = identity ? 1 : 0;
  if (p->n_layers)
    HSX_CUDA(cudaMemcpy(p->d_layers, p->layers.data(), p->layers.size() * sizeof(DevLayer),
                        cudaMemcpyHostToDevice));
  return HSX_OK;
}

int hsx_pack_theta_u(const hsx_plan* p, const float* theta, const float* u, float* send,
                     void* stream) {
  if (!p || !theta || !u || !send) return fail(HSX_EINVAL, "null argument");
  hsx::launch_add(theta, u, send, p->arena, S(stream));
  HSX_LAUNCHED("pack_theta_u");
  return HSX_OK;
}

static hsx::KeepArgs keep_args(hsx_plan* p, const Item* items, const uint32_t* uni, const uint32_t* prev) {
  hsx::KeepArgs ka;
  ka.layers = p->d_layers;
  ka.items = items;
  ka.uni = uni;
  ka.usrc.n = 0;
  ka.uni_out = nullptr;
  ka.prev = prev;
  ka.oflag = p->d_oflag;
  ka.iflag = p->d_iflag;
  ka.pos_out = p->d_pos_out;
  ka.pos_in = p->d_pos_in;
  for (int q = 0; q < hsx::kMaxPasses; ++q) ka.flags.f[q] = p->d_flags[q];
  ka.summary = p->d_summary;
  ka.layer_done = p->d_layer_done;
  ka.done = p->d_done;
  ka.acc = p->d_acc;
  ka.rk_prev = p->d_rk_prev;
  ka.ch_prev = p->d_ch_prev;
  ka.ck_prev = p->d_ck_prev;
  ka.irr = p->d_irr;
  ka.irr_any = p->d_irr_any;
  ka.n_layers = p->n_layers;
  ka.n_prunable = (int)p->prunable.size();
  return ka;
}

static hsx::CandArgs cand_args(hsx_plan* p, const float* sum, const float* theta, const float* u,
                               const float* z, const float* v) {
  hsx::CandArgs a;
  std::memset(&a, 0, sizeof(a));
  p->k2_armed = 0;   // only a counting dynamic K1 (arm_chain) is chained to
  p->k3_armed = 0;
  p->k67_armed = 0;
  a.s = sum;
  a.theta = theta;
  a.u = u;
  a.z = z;
  a.v = v;
  a.layers = p->d_layers;
  a.items = p->d_cand;
  a.identity = p->identity;
  a.sqcap = p->sqcap;
  for (int q = 0; q < hsx::kMaxPasses; ++q) a.fw.f[q] = p->d_flags[q];
  a.cand_done = p->d_cand_done;
  a.sched = p->d_sched;
  a.ka = keep_args(p, nullptr, nullptr, nullptr);
  a.structured = p->single_node;
  return a;
}

// K2 chained behind this dynamic K1 (HSX_K2_CHAIN=0: off): K1 counts the tiles of
// the layers K2 selects; the selections start as K1's first CTAs (short dense items)
// exit. HSX_K1_RESERVE CTA slots are left free for them from the start (default 0:
// every SM then holds the same number of K1 CTAs; one slot per K2 CTA measured
// 0.5% slower on RN18 / RN50 / RN152, profiles/r2zo_*). K1 never waits for K2, so the
// selection always gets its slots.
static void arm_chain(hsx_plan* p, hsx::CandArgs& a, cudaStream_t st) {
  static const int on = env_flag("HSX_K2_CHAIN", 1);
  static const int reserve = env_flag("HSX_K1_RESERVE", 0);
  p->k2_armed = 0;
  if (!on || p->sel_list[0].empty()) return;
  // counts of an earlier K1 that no chained selection consumed: start from zero
  if (p->k2_pending) cudaMemsetAsync(p->d_k1done, 0, sizeof(unsigned) * p->prunable.size(), st);
  p->k2_pending = 1;
  a.k1done = p->d_k1done;
  // cross-tile prologue: parity green, measured neutral (r2zt), so opt-in
  static const int xtile = env_flag("HSX_K1_XTILE", 0);
  a.xtile = xtile;
  a.reserve = reserve >= 0 ? reserve : (int)p->sel_list[0].size();  // < 0: one per selection CTA
  p->k2_armed = 1;
}

static int check_cand_inputs(const hsx_plan* p, const float* sum, const float* theta,
                             const float* u, const float* z, const float* v) {
  if (!sum && (!theta || !u)) return fail(HSX_EINVAL, "candidate needs sum or theta and u");
  if (!p->identity && (!z || !v)) return fail(HSX_EINVAL, "candidate needs z and v");
  return HSX_OK;
}

int hsx_candidate(hsx_plan* p, const float* sum, const float* theta, const float* u,
                  const float* z, const float* v, float* z_node, const uint32_t* frozen_mask,
                  void* stream) {
  if (!p || !z_node) return fail(HSX_EINVAL, "null argument");
  if (int rc = check_cand_inputs(p, sum, theta, u, z, v)) return rc;
  hsx::CandArgs a = cand_args(p, sum, theta, u, z, v);
  a.zn = z_node;
  a.fmask = frozen_mask;
  a.pass = 0;
  a.partials = p->d_partials[0];
  a.norms = p->d_norms[0];
  if (frozen_mask) {
    a.items = p->d_elem;  // frozen: plain elementwise over every layer
    hsx::launch_candidate(a, (int)p->elem_items.size(), 1, p->cand_smem, S(stream));
  } else {
    a.items = p->d_cand;
    arm_chain(p, a, S(stream));
    hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  }
  HSX_LAUNCHED("candidate");
  return HSX_OK;
}

int hsx_candidate_peers(hsx_plan* p, const float* const* sends, int32_t n, const float* z,
                        const float* v, float* z_node, const uint32_t* frozen_mask, void* stream) {
  if (!p || !z_node || !sends || !z || !v) return fail(HSX_EINVAL, "null argument");
  if (n < 1 || n > hsx::kMaxPeers) return fail(HSX_EINVAL, "peer count %d outside [1, %d]", n, hsx::kMaxPeers);
  if (p->identity) return fail(HSX_EINVAL, "peer candidate needs a penalty plan");
  hsx::CandArgs a = cand_args(p, nullptr, nullptr, nullptr, z, v);
  a.peers.n = n;
  for (int j = 0; j < n; ++j) {
    if (!sends[j]) return fail(HSX_EINVAL, "null peer pointer %d", j);
    a.peers.p[j] = sends[j];
  }
  a.zn = z_node;
  a.fmask = frozen_mask;
  a.pass = 0;
  a.partials = p->d_partials[0];
  a.norms = p->d_norms[0];
  if (frozen_mask) {
    a.items = p->d_elem;
    hsx::launch_candidate(a, (int)p->elem_items.size(), 1, p->cand_smem, S(stream));
  } else {
    a.items = p->d_cand;
    arm_chain(p, a, S(stream));
    hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  }
  HSX_LAUNCHED("candidate_peers");
  return HSX_OK;
}

int hsx_candidate_dist(hsx_plan* p, const float* const* slices, int32_t n, const float* z, const float* v,
                       float* z_node, const uint32_t* frozen_mask, void* stream) {
  if (!p || !z_node || !slices || !z || !v) return fail(HSX_EINVAL, "null argument");
  if (n < 2 || n > hsx::kMaxPeers) return fail(HSX_EINVAL, "slice count %d outside [2, %d]", n, hsx::kMaxPeers);
  if (p->identity) return fail(HSX_EINVAL, "distributed candidate needs a penalty plan");
  hsx::CandArgs a = cand_args(p, nullptr, nullptr, nullptr, z, v);
  // the slices of hsx_slices_peers(part = j) over the whole arena
  const long long total = p->arena;
  const long long slice = ((total + n - 1) / n + 31) / 32 * 32;
  a.peers.n = n;
  for (int j = 0; j < n; ++j) {
    if (!slices[j]) return fail(HSX_EINVAL, "null slice pointer %d", j);
    a.peers.p[j] = slices[j];
    a.sbound[j] = std::min<long long>((long long)j * slice, total);
  }
  a.sdist = 1;
  a.zn = z_node;
  a.fmask = frozen_mask;
  a.pass = 0;
  a.partials = p->d_partials[0];
  a.norms = p->d_norms[0];
  if (frozen_mask) {
    a.items = p->d_elem;
    hsx::launch_candidate(a, (int)p->elem_items.size(), 1, p->cand_smem, S(stream));
  } else {
    a.items = p->d_cand;
    arm_chain(p, a, S(stream));
    hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  }
  HSX_LAUNCHED("candidate_dist");
  return HSX_OK;
}

int hsx_plan_set_peer_staging(hsx_plan* p, int32_t on) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (!on || p->d_stage) return HSX_OK;
  HSX_CUDA(cudaMalloc(&p->d_stage, (size_t)std::max<long long>(p->arena, 1) * sizeof(float)));
  const size_t ni = std::max<size_t>(p->cand_dyn.size(), 1);
  HSX_CUDA(cudaMalloc(&p->d_sready, ni * sizeof(unsigned int)));
  HSX_CUDA(cudaMemset(p->d_sready, 0, ni * sizeof(unsigned int)));
  HSX_CUDA(cudaMalloc(&p->d_sepoch, 2 * sizeof(unsigned int)));
  HSX_CUDA(cudaMemset(p->d_sepoch, 0, 2 * sizeof(unsigned int)));
  HSX_CUDA(cudaMalloc(&p->d_scounter, 2 * sizeof(unsigned int)));
  HSX_CUDA(cudaMemset(p->d_scounter, 0, 2 * sizeof(unsigned int)));
  return HSX_OK;
}

int hsx_candidate_peers_staged(hsx_plan* p, const float* const* sends, int32_t n, int32_t me, const float* z,
                               const float* v, float* z_node, void* stream, void* side_stream) {
  if (!p || !z_node || !sends || !z || !v || !side_stream) return fail(HSX_EINVAL, "null argument");
  if (n != 2 || me < 0 || me > 1 || !sends[0] || !sends[1]) return fail(HSX_EINVAL, "staging takes two ranks");
  if (p->identity) return fail(HSX_EINVAL, "peer candidate needs a penalty plan");
  if (!p->d_stage) return fail(HSX_EPROTOCOL, "hsx_plan_set_peer_staging(plan, 1) first");
  static const int grid = std::max(8, env_flag("HSX_STAGE_CTAS", 64));
  // the staging copy of the peer's send on the side stream (the caller forked it from
  // `stream` and joins it back later); K1 reads own send + stage: two fp64 operands,
  // the theta + u kernel (their sum is commutative: the rank order is immaterial)
  hsx::launch_stage(sends[1 - me], p->d_stage, p->d_layers, p->d_cand, (int)p->cand_dyn.size(), p->d_sready,
                    p->d_sepoch, p->d_scounter, grid, S(side_stream));
  HSX_LAUNCHED("stage_peer");
  hsx::CandArgs a = cand_args(p, nullptr, sends[me], p->d_stage, z, v);
  a.u_alt = sends[1 - me];
  a.sready = p->d_sready;
  a.sepoch = p->d_sepoch;
  a.zn = z_node;
  a.pass = 0;
  a.partials = p->d_partials[0];
  a.norms = p->d_norms[0];
  a.items = p->d_cand;
  arm_chain(p, a, S(stream));
  a.reserve += grid;   // slots for the staging CTAs
  hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  HSX_LAUNCHED("candidate_staged");
  return HSX_OK;
}

int hsx_candidate_renorm_peers(hsx_plan* p, int32_t pass, const float* const* sends, int32_t n,
                               const float* z, const float* v, void* stream) {
  if (!p || !sends || !z || !v) return fail(HSX_EINVAL, "null argument");
  if (pass < 1 || pass >= p->max_passes) return fail(HSX_EINVAL, "renorm pass %d out of range", pass);
  if (n < 1 || n > hsx::kMaxPeers) return fail(HSX_EINVAL, "peer count %d outside [1, %d]", n, hsx::kMaxPeers);
  hsx::CandArgs a = cand_args(p, nullptr, nullptr, nullptr, z, v);
  a.peers.n = n;
  for (int j = 0; j < n; ++j) a.peers.p[j] = sends[j];
  a.pass = pass;
  a.partials = p->d_partials[pass];
  a.norms = p->d_norms[pass];
  for (int q = 0; q < pass; ++q) a.flags[q] = p->d_flags[q];
  a.items = p->d_cand;
  hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  HSX_LAUNCHED("candidate_renorm_peers");
  return HSX_OK;
}

int hsx_candidate_renorm(hsx_plan* p, int32_t pass, const float* sum, const float* theta,
                         const float* u, const float* z, const float* v, void* stream) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (pass < 1 || pass >= p->max_passes) return fail(HSX_EINVAL, "renorm pass %d out of range", pass);
  if (int rc = check_cand_inputs(p, sum, theta, u, z, v)) return rc;
  hsx::CandArgs a = cand_args(p, sum, theta, u, z, v);
  a.pass = pass;
  a.partials = p->d_partials[pass];
  a.norms = p->d_norms[pass];
  for (int q = 0; q < pass; ++q) a.flags[q] = p->d_flags[q];
  a.items = p->d_cand;
  hsx::launch_candidate(a, (int)p->cand_dyn.size(), 0, p->cand_smem, S(stream));
  HSX_LAUNCHED("candidate_renorm");
  return HSX_OK;
}

int hsx_select(hsx_plan* p, int32_t pass, void* stream) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (pass < 0 || pass >= hsx::kMaxPasses) return fail(HSX_EINVAL, "pass %d out of range", pass);
  // layers selected in the candidate kernel's tail need nothing here
  int n = (int)p->sel_list[pass].size();
  if (n == 0) return HSX_OK;
  hsx::FlagPtrs fl = {{p->d_flags[0], p->d_flags[1], p->d_flags[2]}};
  // pass 0 right behind a counting K1 (same stream, next launch): chained
  const bool chained = pass == 0 && p->k2_armed;
  p->k2_armed = 0;
  if (chained) p->k2_pending = 0;
  // a single-pass plan's chained selection also publishes per-layer ready flags, so
  // the K3 launched next (hsx_project / hsx_project_keep_sets) chains behind it
  // (alone measured RN18 +1%, RN50 -1%, r2n: on by default only for one-node plans,
  // where K67 chains behind it as well)
  const bool k3 = chained && p->max_passes == 1 && p->sel_list[0].size() == p->prunable.size() &&
                  env_flag("HSX_K3_CHAIN", p->single_node && p->k67_chain ? 1 : 0);
  p->k3_armed = k3 ? 1 : 0;
  hsx::launch_select(p->d_layers, p->d_sel[pass], n, pass, p->d_partials[pass], p->d_norms[pass],
                     fl, keep_args(p, nullptr, nullptr, nullptr), p->single_node, p->select_smem[pass], S(stream),
                     chained ? p->d_k1done : nullptr, k3 ? p->d_ready : nullptr);
  HSX_LAUNCHED("select");
  return HSX_OK;
}

int hsx_read_groups(const hsx_plan* p, int32_t pass, double* norms, uint8_t* flags, void* stream) {
  if (!p || pass < 0 || pass >= hsx::kMaxPasses) return fail(HSX_EINVAL, "bad argument");
  long long n = p->gtotal[pass];
  if (n == 0) return HSX_OK;
  if (norms)
    HSX_CUDA(cudaMemcpyAsync(norms, p->d_norms[pass], n * sizeof(double), cudaMemcpyDeviceToDevice, S(stream)));
  if (flags)
    HSX_CUDA(cudaMemcpyAsync(flags, p->d_flags[pass], n, cudaMemcpyDeviceToDevice, S(stream)));
  return HSX_OK;
}

int hsx_mask_or(const uint32_t* gathered, int32_t n_ranks, int64_t words, uint32_t* out,
                void* stream) {
  if (!gathered || !out || n_ranks < 1 || n_ranks > 8 || words < 0) return fail(HSX_EINVAL, "bad argument");
  hsx::MaskPtrs g;
  g.n = n_ranks;
  for (int r = 0; r < n_ranks; ++r) g.p[r] = gathered + (size_t)r * words;
  hsx::launch_mask_or(g, words, out, S(stream));
  HSX_LAUNCHED("mask_or");
  return HSX_OK;
}

int hsx_mask_or_ptrs(const uint32_t* const* srcs, int32_t n, int64_t words, uint32_t* out,
                     void* stream) {
  if (!srcs || !out || n < 1 || n > 8 || words < 0) return fail(HSX_EINVAL, "bad argument");
  hsx::MaskPtrs g;
  g.n = n;
  for (int r = 0; r < n; ++r) {
    if (!srcs[r]) return fail(HSX_EINVAL, "null mask pointer %d", r);
    g.p[r] = srcs[r];
  }
  hsx::launch_mask_or(g, words, out, S(stream));
  HSX_LAUNCHED("mask_or_ptrs");
  return HSX_OK;
}

int hsx_project(hsx_plan* p, float* z_node, uint32_t* local_mask, void* stream) {
  if (!p || !z_node || (!local_mask && p->mask_words)) return fail(HSX_EINVAL, "null argument");
  hsx::KeepArgs ka = keep_args(p, p->d_proj, nullptr, nullptr);
  const bool chained = p->k3_armed;
  p->k3_armed = 0;
  hsx::launch_project(ka, (int)p->proj_items.size(), z_node, local_mask, 0, S(stream),
                      chained ? p->d_ready : nullptr, p->d_pdone);
  HSX_LAUNCHED("project");
  return HSX_OK;
}

int hsx_project_keep_sets(hsx_plan* p, float* z_node, uint32_t* mask, const uint32_t* prev_mask,
                          void* stream) {
  if (!p || !z_node || (!mask && p->mask_words)) return fail(HSX_EINVAL, "null argument");
  if (p->prunable.empty()) return HSX_OK;
  if (!p->single_node) {  // keep sets from the mask bits (K3, then K5)
    if (int rc = hsx_project(p, z_node, mask, stream)) return rc;
    return hsx_keep_sets(p, mask, prev_mask, stream);
  }
  // the selection's last pass derived the keep sets of the rectangles R x C; K3
  // flags layers whose mask has a kept zero and the fixup re-derives those
  hsx::KeepArgs ka = keep_args(p, p->d_proj, mask, prev_mask);
  const bool chained = p->k3_armed;
  p->k3_armed = 0;
  if (chained && p->k67_chain) {
    // K3 behind the chained K2 runs each layer's fixup in its last item and publishes
    // the layer to a chained K67 (hsx_local_sync next on this stream)
    hsx::ChainK67 c{p->d_ready3, p->d_up, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
    if (p->pub_mapped) {
      long long* dsum = nullptr;
      HSX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dsum), p->h_pub, 0));
      c.pub_sum = dsum;
      c.pub_seq = reinterpret_cast<unsigned int*>(dsum + p->summary.size());
      c.seq_ctr = p->d_seq_ctr;
      c.n_sum = (int)p->summary.size();
    }
    hsx::launch_project(ka, (int)p->proj_items.size(), z_node, mask, 1, S(stream), p->d_ready, p->d_pdone, c,
                        p->fixup_smem);
    HSX_LAUNCHED("project_check_fixup");
    p->k67_armed = 1;
    return HSX_OK;
  }
  hsx::launch_project(ka, (int)p->proj_items.size(), z_node, mask, 1, S(stream), chained ? p->d_ready : nullptr,
                      p->d_pdone);
  HSX_LAUNCHED("project_check");
  hsx::launch_keep_fixup(ka, p->d_prunable, (int)p->prunable.size(), p->fixup_smem, S(stream));
  HSX_LAUNCHED("keep_fixup");
  return HSX_OK;
}

int hsx_select_project_keep_sets(hsx_plan* p, float* z_node, uint32_t* mask, const uint32_t* prev_mask,
                                 void* stream) {
  if (!p || !z_node || (!mask && p->mask_words)) return fail(HSX_EINVAL, "null argument");
  if (p->prunable.empty()) return HSX_OK;
  const bool merge = p->single_node && p->max_passes == 1 && !p->sel_list[0].empty() &&
                     p->sel_list[0].size() == p->prunable.size() && env_flag("HSX_MERGE_SELECT_PROJECT", 0);
  if (!merge) {
    for (int q = 0; q < p->max_passes; ++q)
      if (int rc = hsx_select(p, q, stream)) return rc;
    return hsx_project_keep_sets(p, z_node, mask, prev_mask, stream);
  }
  hsx::KeepArgs ka = keep_args(p, p->d_proj, mask, prev_mask);
  hsx::SelProjArgs sp;
  sp.list = p->d_sel[0];
  sp.nsel = (int)p->sel_list[0].size();
  sp.partials = p->d_partials[0];
  sp.norms = p->d_norms[0];
  sp.ready = p->d_ready;
  sp.pdone = p->d_pdone;
  sp.structured = 1;
  // selection, projection and the keep-set fixup (in the layers' last K3 items) in one launch
  hsx::launch_select_project(sp, ka, (int)p->proj_items.size(), z_node, mask,
                             std::max(p->select_smem[0], p->fixup_smem), S(stream));
  HSX_LAUNCHED("select_project");
  return HSX_OK;
}

int hsx_plan_set_k67_chain(hsx_plan* p, int32_t on) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  p->k67_chain = on && env_flag("HSX_K67_CHAIN", 1) ? 1 : 0;
  // every dynamic one-node step then runs the chained projection, which publishes
  // the summary from the device into the mapped host buffer (hsx_plan_summary_host)
  const bool always = p->k67_chain && p->single_node && env_flag("HSX_K2_CHAIN", 1) && p->max_passes == 1 &&
                      !p->prunable.empty() && p->sel_list[0].size() == p->prunable.size();
  p->pub_mapped = 0;
  if (always && hsx_plan_summary_host(p)) {
    if (!p->d_seq_ctr) HSX_CUDA(cudaMalloc(&p->d_seq_ctr, sizeof(unsigned int)));
    HSX_CUDA(cudaMemset(p->d_seq_ctr, 0, sizeof(unsigned int)));
    p->h_pub[p->summary.size()] = 0;
    p->last_seq = 0;
    p->pub_mapped = 1;
  }
  return HSX_OK;
}

// split two-rank K1: rank `split_me` takes every dense item (both ranks compute the
// dense layers, which no tile count orders) and the prunable tiles at its parity
// in K1's work-list order
static int upload_split_items(hsx_plan* p) {
  std::vector<Item> mine;
  int k = 0;
  for (const Item& it : p->cand_dyn) {
    if (p->layers[it.layer].ncons == 0)
      mine.push_back(it);
    else if ((k++ & 1) == p->split_me)
      mine.push_back(it);
  }
  if (!p->d_cand_split) HSX_CUDA(cudaMalloc(&p->d_cand_split, std::max<size_t>(p->cand_dyn.size(), 1) * sizeof(Item)));
  if (!mine.empty())
    HSX_CUDA(cudaMemcpy(p->d_cand_split, mine.data(), mine.size() * sizeof(Item), cudaMemcpyHostToDevice));
  p->n_cand_split = (int)mine.size();
  return HSX_OK;
}

int hsx_plan_split_sizes(const hsx_plan* p, int64_t* partials_elems, int32_t* counters) {
  if (!p || !partials_elems || !counters) return fail(HSX_EINVAL, "null argument");
  *partials_elems = p->ptotal[0];
  *counters = (int32_t)p->prunable.size() + 1;
  return HSX_OK;
}

int hsx_plan_set_split(hsx_plan* p, int32_t me, double* partials, double* partials_peer, uint32_t* k1done,
                       uint32_t* k1done_peer) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (me < 0 || me > 1 || !partials || !partials_peer || !k1done || !k1done_peer)
    return fail(HSX_EINVAL, "split K1 takes two ranks and peer-mapped partials / counts");
  if (p->identity || p->max_passes != 1) return fail(HSX_EINVAL, "split K1 needs a single-pass penalty plan");
  if (!env_flag("HSX_K2_CHAIN", 1) || p->sel_list[0].size() != p->prunable.size())
    return fail(HSX_EINVAL, "split K1 needs the chained selection of every prunable layer");
  if (p->split_me >= 0) return fail(HSX_EINVAL, "split already set");
  if (p->d_partials[0] && !p->ext_partials) cudaFree(p->d_partials[0]);
  if (p->d_k1done && !p->ext_k1done) cudaFree(p->d_k1done);
  p->d_partials[0] = partials;
  p->d_k1done = k1done;
  p->ext_partials = p->ext_k1done = 1;
  p->partials_peer = partials_peer;
  p->k1done_peer = k1done_peer;
  p->split_me = me;
  return upload_split_items(p);
}

int hsx_candidate_peers_split(hsx_plan* p, const float* const* sends, int32_t n, const float* z, const float* v,
                              float* z_node, float* z_node_peer, void* stream) {
  if (!p || !z_node || !z_node_peer || !sends || !z || !v) return fail(HSX_EINVAL, "null argument");
  if (p->split_me < 0) return fail(HSX_EINVAL, "split K1 not set up (hsx_plan_set_split)");
  if (n != 2 || !sends[0] || !sends[1]) return fail(HSX_EINVAL, "split K1 takes two ranks");
  // the peer counts into this rank's counters concurrently: they cannot be reset here
  if (p->k2_pending) return fail(HSX_EINVAL, "split K1 behind a counting K1 no selection consumed");
  hsx::CandArgs a = cand_args(p, nullptr, nullptr, nullptr, z, v);
  a.peers.n = 2;
  a.peers.p[0] = sends[0];
  a.peers.p[1] = sends[1];
  a.zn = z_node;
  a.zn_peer = z_node_peer;
  a.pass = 0;
  a.partials = p->d_partials[0];
  a.partials_peer = p->partials_peer;
  a.norms = p->d_norms[0];
  a.items = p->d_cand_split;
  arm_chain(p, a, S(stream));
  if (!a.k1done) return fail(HSX_EINVAL, "split K1 needs the chained selection");
  a.k1done_peer = p->k1done_peer;
  hsx::launch_candidate(a, p->n_cand_split, 0, p->cand_smem, S(stream));
  HSX_LAUNCHED("candidate_peers_split");
  return HSX_OK;
}

int hsx_plan_set_order(hsx_plan* p, int32_t big_first) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if ((big_first != 0) == (p->big_first != 0)) return HSX_OK;
  set_order(p, big_first != 0);
  HSX_CUDA(cudaMemcpy(p->d_cand, p->cand_dyn.data(), p->cand_dyn.size() * sizeof(Item), cudaMemcpyHostToDevice));
  HSX_CUDA(cudaMemcpy(p->d_proj, p->proj_items.data(), p->proj_items.size() * sizeof(Item), cudaMemcpyHostToDevice));
  if (p->split_me >= 0)
    if (int rc = upload_split_items(p)) return rc;
  for (int q = 0; q < hsx::kMaxPasses; ++q)
    if (!p->sel_list[q].empty())
      HSX_CUDA(cudaMemcpy(p->d_sel[q], p->sel_list[q].data(), p->sel_list[q].size() * sizeof(int),
                          cudaMemcpyHostToDevice));
  return HSX_OK;
}

int hsx_plan_set_single_node(hsx_plan* p, int32_t on) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  p->single_node = on ? 1 : 0;
  return HSX_OK;
}

int hsx_keep_sets(hsx_plan* p, const uint32_t* union_mask, const uint32_t* prev_mask,
                  void* stream) {
  if (!p || (!union_mask && p->mask_words)) return fail(HSX_EINVAL, "null argument");
  if (p->prunable.empty()) return HSX_OK;
  // K_out / K_in flags and the popcount accumulators are zero here (zero at
  // allocation, re-zeroed by every keep-set tail)
  hsx::KeepArgs ka = keep_args(p, p->d_word, union_mask, prev_mask);
  hsx::launch_keep_sets(ka, (int)p->word_items.size(), p->mark_smem, S(stream));
  HSX_LAUNCHED("keep_sets");
  return HSX_OK;
}

int hsx_keep_sets_ptrs(hsx_plan* p, const uint32_t* const* srcs, int32_t n, uint32_t* union_out,
                       const uint32_t* prev_mask, void* stream) {
  if (!p || !srcs || (!union_out && p->mask_words)) return fail(HSX_EINVAL, "null argument");
  if (n < 1 || n > 8) return fail(HSX_EINVAL, "source count %d outside [1, 8]", n);
  if (p->prunable.empty()) return HSX_OK;
  if (p->single_node) return fail(HSX_EINVAL, "one-node plans derive keep sets in K3 (structured)");
  hsx::KeepArgs ka = keep_args(p, p->d_word, nullptr, prev_mask);
  ka.usrc.n = n;
  for (int r = 0; r < n; ++r) {
    if (!srcs[r]) return fail(HSX_EINVAL, "null mask pointer %d", r);
    ka.usrc.p[r] = srcs[r];
  }
  ka.uni_out = union_out;
  hsx::launch_keep_sets(ka, (int)p->word_items.size(), p->mark_smem, S(stream));
  HSX_LAUNCHED("keep_sets_ptrs");
  return HSX_OK;
}

int hsx_keep_sets_fetch(hsx_plan* p, int64_t* host_summary, void* stream) {
  if (!p || !host_summary) return fail(HSX_EINVAL, "null argument");
  size_t bytes = p->summary.size() * sizeof(long long);
  HSX_CUDA(cudaMemcpyAsync(host_summary, p->d_summary, bytes, cudaMemcpyDeviceToHost, S(stream)));
  HSX_CUDA(cudaStreamSynchronize(S(stream)));
  std::memcpy(p->summary.data(), host_summary, bytes);
  return HSX_OK;
}

int hsx_keep_sets_fetch_async(hsx_plan* p, int64_t* host_summary, void* stream) {
  if (!p || !host_summary) return fail(HSX_EINVAL, "null argument");
  if (p->pub_mapped && host_summary == reinterpret_cast<int64_t*>(p->h_pub))
    return HSX_OK;   // the chained projection publishes it from the device (hsx_keep_sets_fetch_wait)
  HSX_CUDA(cudaMemcpyAsync(host_summary, p->d_summary, p->summary.size() * sizeof(long long),
                           cudaMemcpyDeviceToHost, S(stream)));
  // completion marker the host can wait on mid-step; under stream capture an
  // external event-record node, so a replayed graph signals it at this point
  if (!p->fetch_ev) HSX_CUDA(cudaEventCreateWithFlags(&p->fetch_ev, cudaEventDisableTiming));
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HSX_CUDA(cudaStreamIsCapturing(S(stream), &cs));
  HSX_CUDA(cudaEventRecordWithFlags(p->fetch_ev, S(stream),
                                    cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0));
  return HSX_OK;
}

int hsx_keep_sets_fetch_wait(hsx_plan* p) {
  if (!p) return fail(HSX_EINVAL, "null plan");
  if (p->pub_mapped) {
    // the device bumps the mapped sequence word once per published summary, and the
    // host waits once per dynamic step (before the next one is launched)
    volatile unsigned int* seq = reinterpret_cast<volatile unsigned int*>(p->h_pub + p->summary.size());
    unsigned v;
    while ((v = *seq) == p->last_seq) {
      cudaError_t e = cudaGetLastError();   // a failed context would never publish
      if (e != cudaSuccess) return fail(HSX_ECUDA, "waiting for the keep-set summary: %s", cudaGetErrorString(e));
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    p->last_seq = v;
    return HSX_OK;
  }
  if (p->fetch_ev) HSX_CUDA(cudaEventSynchronize(p->fetch_ev));
  return HSX_OK;
}

int64_t* hsx_plan_summary_host(hsx_plan* p) {
  if (!p) return nullptr;
  if (!p->h_pub) {
    if (cudaHostAlloc(reinterpret_cast<void**>(&p->h_pub), (p->summary.size() + 1) * sizeof(long long),
                      cudaHostAllocMapped) != cudaSuccess) {
      p->h_pub = nullptr;
      return nullptr;
    }
    std::memcpy(p->h_pub, p->summary.data(), p->summary.size() * sizeof(long long));
    p->h_pub[p->summary.size()] = 0;
  }
  return reinterpret_cast<int64_t*>(p->h_pub);
}

int hsx_set_keep_sets(hsx_plan* p, int32_t l, const int32_t* k_out, int32_t n_out,
                      const int32_t* k_in, int32_t n_in) {
  if (!p || l < 0 || l >= p->n_layers) return fail(HSX_EINVAL, "bad layer");
  const DevLayer& ly = p->layers[l];
  if (ly.ncons == 0) return fail(HSX_ESHAPE, "layer %d: only conv layers are shrunk", l);
  if (n_out < 0 || n_in < 0 || n_out > ly.rows || n_in > ly.cin || (n_out && !k_out) || (n_in && !k_in))
    return fail(HSX_ESHAPE, "layer %d: keep sets inconsistent with shape", l);
  std::vector<int> po(ly.rows, -1), pi(ly.cin, -1);
  for (int i = 0; i < n_out; ++i) {
    if (k_out[i] < 0 || k_out[i] >= ly.rows || (i && k_out[i] <= k_out[i - 1]))
      return fail(HSX_ESHAPE, "layer %d: K_out must be sorted, unique and in range", l);
    po[k_out[i]] = i;
  }
  for (int i = 0; i < n_in; ++i) {
    if (k_in[i] < 0 || k_in[i] >= ly.cin || (i && k_in[i] <= k_in[i - 1]))
      return fail(HSX_ESHAPE, "layer %d: K_in must be sorted, unique and in range", l);
    pi[k_in[i]] = i;
  }
  HSX_CUDA(cudaMemcpy(p->d_pos_out + ly.okeep, po.data(), po.size() * sizeof(int), cudaMemcpyHostToDevice));
  HSX_CUDA(cudaMemcpy(p->d_pos_in + ly.ikeep, pi.data(), pi.size() * sizeof(int), cudaMemcpyHostToDevice));
  long long* row = &p->summary[(size_t)l * HSX_SUM_COLS];
  row[HSX_SUM_KOUT] = n_out;
  row[HSX_SUM_KIN] = n_in;
  row[HSX_SUM_ELEMS] = (long long)n_out * n_in * ly.k;
  host_layout(p);
  HSX_CUDA(cudaMemcpy(p->d_summary, p->summary.data(), p->summary.size() * sizeof(long long),
                      cudaMemcpyHostToDevice));
  return HSX_OK;
}

int hsx_read_keep_positions(const hsx_plan* p, int32_t which, int32_t* dst, void* stream) {
  if (!p || !dst) return fail(HSX_EINVAL, "null argument");
  long long n = p->ktotal[which ? 1 : 0];
  if (n)
    HSX_CUDA(cudaMemcpyAsync(dst, which ? p->d_pos_in : p->d_pos_out, n * sizeof(int),
                             cudaMemcpyDeviceToDevice, S(stream)));
  return HSX_OK;
}

static hsx::ElemArgs elem_args(const hsx_plan* p) {
  hsx::ElemArgs a;
  std::memset(&a, 0, sizeof(a));
  a.layers = p->d_layers;
  a.items = p->d_stream;
  a.pos_out = p->d_pos_out;
  a.pos_in = p->d_pos_in;
  a.summary = p->d_summary;
  a.divisor = 1.0f;
  return a;
}

int hsx_compact_dual(const hsx_plan* p, const float* theta, float* u, const float* z_node,
                     const float* v, float* flat, void* stream) {
  if (!p || !z_node || !flat) return fail(HSX_EINVAL, "null argument");
  if ((theta == nullptr) != (u == nullptr)) return fail(HSX_EINVAL, "theta and u go together");
  hsx::ElemArgs a = elem_args(p);
  a.theta = theta;
  a.u = u;
  a.zn = z_node;
  a.vin = v;
  a.flat_out = flat;
  hsx::launch_compact(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("compact_dual");
  return HSX_OK;
}

int hsx_dual_intra(const hsx_plan* p, const float* theta, float* u, const float* z_node,
                   void* stream) {
  if (!p || !theta || !u || !z_node) return fail(HSX_EINVAL, "null argument");
  hsx::launch_dual(theta, u, z_node, p->arena, S(stream));
  HSX_LAUNCHED("dual_intra");
  return HSX_OK;
}

int hsx_decompact_dual(const hsx_plan* p, const float* flat, float divisor, const float* z_node,
                       float* v, float* z, void* stream) {
  if (!p || !flat || !z) return fail(HSX_EINVAL, "null argument");
  if (v && !z_node) return fail(HSX_EINVAL, "v update needs z_node");
  if (!(divisor > 0.0f)) return fail(HSX_EINVAL, "divisor must be positive");
  hsx::ElemArgs a = elem_args(p);
  a.flat_in = flat;
  a.divisor = divisor;
  a.zn = z_node;
  a.v = v;
  a.z = z;
  hsx::launch_decompact(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("decompact_dual");
  return HSX_OK;
}

int hsx_decompact_average(const hsx_plan* p, const float* const* srcs, int32_t n, double divisor, float* zhat_out,
                          const float* z_node, const float* z_node_prev, float* v, float* z, int32_t residuals,
                          void* stream) {
  if (!p || !srcs || !z_node || !v || !z) return fail(HSX_EINVAL, "null argument");
  if (n != 2 || !srcs[0] || !srcs[1]) return fail(HSX_EINVAL, "the fused average takes exactly two leaders");
  if (!(divisor > 0.0)) return fail(HSX_EINVAL, "divisor must be positive");
  if (residuals && !z_node_prev) return fail(HSX_EINVAL, "residuals need z_node_prev");
  hsx::ElemArgs a = elem_args(p);
  a.flat_in = srcs[0];
  a.flat_in2 = srcs[1];
  a.avg_div = divisor;
  a.zhat_out = zhat_out;
  a.zn = z_node;
  a.zn_prev = z_node_prev;
  a.v = v;
  a.z = z;
  a.rpart = residuals ? p->d_rpart : nullptr;
  hsx::launch_decompact(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("decompact_average");
  return HSX_OK;
}

int hsx_compact_dual_resid(const hsx_plan* p, const float* theta, float* u, const float* z_node,
                           const float* v, float* flat, void* stream) {
  if (!p || !theta || !u || !z_node) return fail(HSX_EINVAL, "null argument");
  if (flat && !v) return fail(HSX_EINVAL, "compaction needs v");
  hsx::ElemArgs a = elem_args(p);
  a.theta = theta;
  a.u = u;
  a.zn = z_node;
  a.vin = v;
  a.flat_out = flat;
  a.rpart = p->d_rpart;
  hsx::launch_compact(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("compact_dual_resid");
  return HSX_OK;
}

int hsx_decompact_dual_resid(const hsx_plan* p, const float* flat, float divisor, const float* z_node,
                             const float* z_node_prev, float* v, float* z, void* stream) {
  if (!p || !z_node || !z_node_prev || !v || !z) return fail(HSX_EINVAL, "null argument");
  if (!(divisor > 0.0f)) return fail(HSX_EINVAL, "divisor must be positive");
  hsx::ElemArgs a = elem_args(p);
  a.flat_in = flat;
  a.divisor = divisor;
  a.zn = z_node;
  a.zn_prev = z_node_prev;
  a.v = v;
  a.z = z;
  a.rpart = p->d_rpart;
  hsx::launch_decompact(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("decompact_dual_resid");
  return HSX_OK;
}

int hsx_local_sync(hsx_plan* p, const float* theta, float* u, const float* z_node, float* v, float* z,
                   const float* z_node_prev, int32_t residuals, void* stream) {
  if (!p || !theta || !u || !z_node || !v || !z) return fail(HSX_EINVAL, "null argument");
  if (residuals && !z_node_prev) return fail(HSX_EINVAL, "residuals need z_node_prev");
  hsx::ElemArgs a = elem_args(p);
  if (p->k67_armed)  // right behind the chained one-node K3: per-layer waits instead of the grid's
    a.c67 = hsx::ChainK67{p->d_ready3, p->d_up, p->d_cnt67, p->d_scount, p->d_up + 1};
  p->k67_armed = 0;
  a.theta = theta;
  a.u = u;
  a.zn = z_node;
  a.v = v;
  a.z = z;
  a.zn_prev = z_node_prev;
  a.rpart = residuals ? p->d_rpart : nullptr;
  hsx::launch_local_sync(a, (int)p->stream_items.size(), S(stream));
  HSX_LAUNCHED("local_sync");
  return HSX_OK;
}

static hsx::ResidArgs resid_args(hsx_plan* p) {
  hsx::ResidArgs a;
  std::memset(&a, 0, sizeof(a));
  a.layers = p->d_layers;
  a.n_layers = p->n_layers;
  a.first = p->d_sfirst;
  a.count = p->d_scount;
  a.rpart = p->d_rpart;
  return a;
}

int hsx_residual_fold(hsx_plan* p, int32_t leader, double* vec, void* stream) {
  if (!p || !vec) return fail(HSX_EINVAL, "null argument");
  hsx::ResidArgs a = resid_args(p);
  a.vec = vec;
  a.leader = leader ? 1 : 0;
  hsx::launch_resid_fold(a, S(stream));
  HSX_LAUNCHED("residual_fold");
  return HSX_OK;
}

int hsx_residual_report(hsx_plan* p, const double* global, double* report, double* scales,
                        const hsx_resid_params* prm, void* stream) {
  if (!p || !report || !scales || !prm) return fail(HSX_EINVAL, "null argument");
  if (prm->num_nodes < 1 || prm->accels_per_node < 1) return fail(HSX_ECONFIG, "topology dimensions must be positive");
  hsx::ResidArgs a = resid_args(p);
  a.global = global;
  a.report = report;
  a.scales = scales;
  a.wd = prm->weight_decay;
  a.eps_abs = prm->eps_abs;
  a.eps_rel = prm->eps_rel;
  a.mu = prm->mu;
  a.tau_inc = prm->tau_inc;
  a.tau_dec = prm->tau_dec;
  a.rho1_max = prm->rho1_max;
  a.rho2_max = prm->rho2_max;
  a.num_nodes = prm->num_nodes;
  a.per_node = prm->accels_per_node;
  a.adapt = prm->adapt ? 1 : 0;
  a.flat = prm->flat ? 1 : 0;
  hsx::launch_report(a, S(stream));
  HSX_LAUNCHED("residual_report");
  return HSX_OK;
}

int hsx_scale_duals(const hsx_plan* p, const double* scales, float* u, float* v, void* stream) {
  if (!p || !scales || !u || !v) return fail(HSX_EINVAL, "null argument");
  // contiguous 8192-element items of every layer (balanced; unscaled layers exit at once)
  hsx::launch_scale_duals(p->d_layers, p->d_elem, (int)p->elem_items.size(), scales, p->n_layers, u, v,
                          S(stream));
  HSX_LAUNCHED("scale_duals");
  return HSX_OK;
}

int hsx_prox_sgd_step(const hsx_plan* p, const float* grad, float* theta, const float* z_node, const float* u,
                      float* velocity, double lr, double momentum, int32_t first, float* send, void* stream) {
  if (!p || !grad || !theta || !z_node || !u || !velocity) return fail(HSX_EINVAL, "null argument");
  if (!(lr > 0.0)) return fail(HSX_ECONFIG, "learning rate must be positive, got %g", lr);
  hsx::launch_prox_sgd(p->d_layers, p->d_elem, (int)p->elem_items.size(), grad, theta, z_node, u, velocity, send, lr,
                       momentum, first ? 1 : 0, S(stream));
  HSX_LAUNCHED("prox_sgd_step");
  return HSX_OK;
}

int hsx_dense_grad_pack(const float* grad, const float* params, double weight_decay, float* send, int64_t n,
                        void* stream) {
  if (n < 0) return fail(HSX_EINVAL, "negative element count");
  if (n && (!grad || !params || !send)) return fail(HSX_EINVAL, "null argument");
  if ((reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(params) | reinterpret_cast<uintptr_t>(send)) & 15)
    return fail(HSX_EINVAL, "buffers must be 16-byte aligned");
  hsx::launch_dense_pack(grad, params, weight_decay, send, n, S(stream));
  HSX_LAUNCHED("dense_grad_pack");
  return HSX_OK;
}

int hsx_dense_apply(const float* const* sends, int32_t n_sends, double divisor, float* params, float* velocity,
                    double lr, double momentum, int32_t first, int64_t n, void* stream) {
  if (n < 0) return fail(HSX_EINVAL, "negative element count");
  if (!sends || !params || !velocity) return fail(HSX_EINVAL, "null argument");
  if (n_sends < 1 || n_sends > hsx::kMaxPeers)
    return fail(HSX_EINVAL, "peer count %d outside [1, %d]", n_sends, hsx::kMaxPeers);
  if (!(divisor > 0.0)) return fail(HSX_EINVAL, "divisor must be positive");
  if (!(lr > 0.0)) return fail(HSX_ECONFIG, "learning rate must be positive, got %g", lr);
  hsx::PeerPtrs src;
  src.n = n_sends;
  for (int j = 0; j < n_sends; ++j) {
    if (!sends[j] || (reinterpret_cast<uintptr_t>(sends[j]) & 15)) return fail(HSX_EINVAL, "send pointer %d null or unaligned", j);
    src.p[j] = sends[j];
  }
  if ((reinterpret_cast<uintptr_t>(params) | reinterpret_cast<uintptr_t>(velocity)) & 15)
    return fail(HSX_EINVAL, "buffers must be 16-byte aligned");
  hsx::launch_dense_apply(src, divisor, params, velocity, lr, momentum, first ? 1 : 0, n, S(stream));
  HSX_LAUNCHED("dense_apply");
  return HSX_OK;
}

struct hsx_topk {
  int n_layers = 0;
  long long ktotal = 0, span = 0;
  std::vector<hsx::TkLayer> layers;
  std::vector<hsx::TkTile> tiles;
  hsx::TkLayer* d_layers = nullptr;
  hsx::TkTile* d_tiles = nullptr;
  hsx::TkState* d_state = nullptr;
  unsigned* d_hist = nullptr;
  int2 *d_cnt = nullptr, *d_base = nullptr;
  ~hsx_topk() {
    void* ptrs[] = {d_layers, d_tiles, d_state, d_hist, d_cnt, d_base};
    for (void* q : ptrs)
      if (q) cudaFree(q);
  }
};

int hsx_topk_create(const int64_t* offsets, const int64_t* elements, double rate, int32_t n_layers, hsx_topk** out) {
  if (!out || (n_layers > 0 && (!offsets || !elements))) return fail(HSX_EINVAL, "null argument");
  if (n_layers < 0) return fail(HSX_EINVAL, "negative layer count");
  if (!(rate > 0.0) || rate > 1.0) return fail(HSX_ECONFIG, "top-k rate must be in (0, 1], got %g", rate);
  *out = nullptr;
  HSX_TRY({
    std::unique_ptr<hsx_topk> t(new hsx_topk());
    t->n_layers = n_layers;
    constexpr long long kTile = 8192;
    for (int l = 0; l < n_layers; ++l) {
      if (elements[l] <= 0 || offsets[l] < 0) return fail(HSX_ESHAPE, "layer %d: bad extent", l);
      if (elements[l] > INT32_MAX) return fail(HSX_ESHAPE, "layer %d: more than 2^31 elements", l);
      hsx::TkLayer ly;
      ly.off = offsets[l];
      ly.n = elements[l];
      // k = max(1, ceil(rate * n)) with the reference's float expression (:132)
      ly.k = std::max<long long>(1, (long long)std::ceil(rate * (double)elements[l]));
      if (ly.k > ly.n) ly.k = ly.n;
      ly.koff = t->ktotal;
      ly.tile0 = (int)t->tiles.size();
      for (long long b = 0; b < ly.n; b += kTile) {
        hsx::TkTile tt;
        tt.layer = l;
        tt.pad = 0;
        tt.begin = b;
        tt.end = std::min(ly.n, b + kTile);
        t->tiles.push_back(tt);
      }
      ly.ntiles = (int)t->tiles.size() - ly.tile0;
      t->ktotal += ly.k;
      t->span = std::max(t->span, ly.off + ly.n);
      t->layers.push_back(ly);
    }
    if (n_layers) {
      int rc;
      if ((rc = upload(&t->d_layers, t->layers))) return rc;
      if ((rc = upload(&t->d_tiles, t->tiles))) return rc;
      HSX_CUDA(cudaMalloc(&t->d_state, sizeof(hsx::TkState) * n_layers));
      HSX_CUDA(cudaMalloc(&t->d_hist, sizeof(unsigned) * 256 * n_layers));
      HSX_CUDA(cudaMalloc(&t->d_cnt, sizeof(int2) * t->tiles.size()));
      HSX_CUDA(cudaMalloc(&t->d_base, sizeof(int2) * t->tiles.size()));
    }
    *out = t.release();
  })
  return HSX_OK;
}

void hsx_topk_destroy(hsx_topk* t) { delete t; }

int64_t hsx_topk_total(const hsx_topk* t) { return t ? t->ktotal : -1; }

int hsx_topk_layer_keep(const hsx_topk* t, int32_t layer, int64_t* k, int64_t* offset) {
  if (!t || !k || !offset) return fail(HSX_EINVAL, "null argument");
  if (layer < 0 || layer >= t->n_layers) return fail(HSX_EINVAL, "layer %d out of range", layer);
  *k = t->layers[layer].k;
  *offset = t->layers[layer].koff;
  return HSX_OK;
}

int hsx_topk_select(const hsx_topk* t, const float* grad, const float* params, double weight_decay, double* residual,
                    float* values, int32_t* indices, void* stream) {
  if (!t || !grad || !params || !residual || !values || !indices) return fail(HSX_EINVAL, "null argument");
  const int n = hsx::launch_topk_select(t->d_tiles, (int)t->tiles.size(), t->d_layers, t->n_layers, t->d_state,
                                        t->d_hist, t->d_cnt, t->d_base, residual, grad, params, weight_decay, values,
                                        indices, S(stream));
  if (n > 1) g_launches.fetch_add(n - 1);
  HSX_LAUNCHED("topk_select");
  return HSX_OK;
}

int hsx_topk_scatter(const hsx_topk* t, const float* values, const int32_t* indices, double* dense, void* stream) {
  if (!t || !values || !indices || !dense) return fail(HSX_EINVAL, "null argument");
  hsx::launch_topk_scatter(t->d_layers, t->n_layers, values, indices, t->ktotal, dense, S(stream));
  HSX_LAUNCHED("topk_scatter");
  return HSX_OK;
}

int hsx_topk_apply(const hsx_topk* t, double* dense, double divisor, float* params, float* velocity, double lr,
                   double momentum, int32_t first, void* stream) {
  if (!t || !dense || !params || !velocity) return fail(HSX_EINVAL, "null argument");
  if (!(divisor > 0.0)) return fail(HSX_EINVAL, "divisor must be positive");
  if (!(lr > 0.0)) return fail(HSX_ECONFIG, "learning rate must be positive, got %g", lr);
  hsx::launch_topk_apply(dense, divisor, params, velocity, lr, momentum, first ? 1 : 0, t->span, S(stream));
  HSX_LAUNCHED("topk_apply");
  return HSX_OK;
}

int hsx_plan_read_penalties(hsx_plan* p, double* rho1, double* rho2) {
  if (!p || !rho1 || !rho2) return fail(HSX_EINVAL, "null argument");
  if (p->n_layers)
    HSX_CUDA(cudaMemcpy(p->layers.data(), p->d_layers, p->layers.size() * sizeof(DevLayer),
                        cudaMemcpyDeviceToHost));
  for (int l = 0; l < p->n_layers; ++l) {
    rho1[l] = p->layers[l].rho1;
    rho2[l] = p->layers[l].rho2;
  }
  return HSX_OK;
}

int hsx_average_peers(const hsx_plan* p, const float* const* srcs, int32_t n, double divisor, float* out,
                      void* stream) {
  if (!p || !srcs || !out) return fail(HSX_EINVAL, "null argument");
  if (n < 1 || n > hsx::kMaxPeers) return fail(HSX_EINVAL, "peer count %d outside [1, %d]", n, hsx::kMaxPeers);
  if (!(divisor > 0.0)) return fail(HSX_EINVAL, "divisor must be positive");
  hsx::PeerPtrs src;
  src.n = n;
  for (int j = 0; j < n; ++j) {
    if (!srcs[j] || (reinterpret_cast<uintptr_t>(srcs[j]) & 15)) return fail(HSX_EINVAL, "peer pointer %d null or unaligned", j);
    src.p[j] = srcs[j];
  }
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(HSX_EINVAL, "output not 16-byte aligned");
  // payload size of the last keep-set derivation, read on the device
  hsx::launch_average(src, p->d_summary + (size_t)p->n_layers * HSX_SUM_COLS, p->arena, divisor, out, S(stream));
  HSX_LAUNCHED("average_peers");
  return HSX_OK;
}

int hsx_slices_peers(const hsx_plan* p, const float* const* srcs, int32_t n, int32_t part, double divisor,
                     int32_t payload, float* out, void* stream) {
  if (!p || !srcs || !out) return fail(HSX_EINVAL, "null argument");
  if (n < 1 || n > hsx::kMaxPeers) return fail(HSX_EINVAL, "peer count %d outside [1, %d]", n, hsx::kMaxPeers);
  if (part >= n) return fail(HSX_EINVAL, "slice %d of %d", part, n);
  if (!(divisor > 0.0)) return fail(HSX_EINVAL, "divisor must be positive");
  hsx::PeerPtrs src;
  src.n = n;
  for (int j = 0; j < n; ++j) {
    if (!srcs[j] || (reinterpret_cast<uintptr_t>(srcs[j]) & 15)) return fail(HSX_EINVAL, "peer pointer %d null or unaligned", j);
    src.p[j] = srcs[j];
  }
  if (reinterpret_cast<uintptr_t>(out) & 15) return fail(HSX_EINVAL, "output not 16-byte aligned");
  const long long* total_p = payload ? p->d_summary + (size_t)p->n_layers * HSX_SUM_COLS : nullptr;
  hsx::launch_slices(src, total_p, p->arena, p->arena, part, divisor, out, S(stream));
  HSX_LAUNCHED("slices_peers");
  return HSX_OK;
}

int hsx_group_barrier(int32_t* const* flags, const int32_t* slots, int32_t n, int32_t me, int32_t epoch,
                      void* stream) {
  return hsx_group_barrier_mode(flags, slots, n, me, epoch, 0, 0, stream);
}

int hsx_group_barrier_mode(int32_t* const* flags, const int32_t* slots, int32_t n, int32_t me, int32_t epoch,
                           int32_t mode, int32_t root, void* stream) {
  if (!flags || !slots || n < 1 || n > 32 || me < 0 || me >= n) return fail(HSX_EINVAL, "bad barrier arguments");
  if (mode < 0 || mode > 2 || root < 0 || root >= n) return fail(HSX_EINVAL, "bad barrier mode / root");
  hsx::BarrierArgs b;
  b.n = n;
  b.me = me;
  b.epoch = epoch;
  b.mode = mode;
  b.root = root;
  for (int i = 0; i < n; ++i) {
    if (!flags[i]) return fail(HSX_EINVAL, "null flag pointer %d", i);
    b.flags[i] = flags[i];
    b.slots[i] = slots[i];
  }
  hsx::launch_barrier(b, S(stream));
  HSX_LAUNCHED("group_barrier");
  return HSX_OK;
}

int hsx_barrier_timeouts(uint32_t* count, int32_t reset) {
  if (!count) return fail(HSX_EINVAL, "null argument");
  if (hsx::barrier_timeouts(count, reset) != 0) return check_cuda("barrier_timeouts");
  return HSX_OK;
}

int hsx_nonzero_u8(const float* t, int64_t n, uint8_t* out, void* stream) {
  if ((!t || !out) && n > 0) return fail(HSX_EINVAL, "null argument");
  hsx::launch_nonzero(t, n, out, S(stream));
  HSX_LAUNCHED("nonzero_u8");
  return HSX_OK;
}
int hsx_pack_bits(const uint8_t* m, int64_t n, uint32_t* bits, void* stream) {
  if ((!m || !bits) && n > 0) return fail(HSX_EINVAL, "null argument");
  hsx::launch_pack(m, n, bits, S(stream));
  HSX_LAUNCHED("pack_bits");
  return HSX_OK;
}
int hsx_unpack_bits(const uint32_t* bits, int64_t n, uint8_t* m, void* stream) {
  if ((!m || !bits) && n > 0) return fail(HSX_EINVAL, "null argument");
  hsx::launch_unpack(bits, n, m, S(stream));
  HSX_LAUNCHED("unpack_bits");
  return HSX_OK;
}
int hsx_selftest_division(const double* num, int64_t n, double den, double* out, void* stream) {
  if ((!num || !out) && n > 0) return fail(HSX_EINVAL, "null argument");
  if (!(den != 0.0)) return fail(HSX_EINVAL, "zero denominator");
  hsx::launch_div_selftest(num, n, den, out, S(stream));
  HSX_LAUNCHED("selftest_division");
  return HSX_OK;
}

int hsx_count_diff_u8(const uint8_t* a, const uint8_t* b, int64_t n, uint64_t* count_dev,
                      void* stream) {
  if ((!a || !b || !count_dev) && n > 0) return fail(HSX_EINVAL, "null argument");
  hsx::launch_count_diff(a, b, n, reinterpret_cast<unsigned long long*>(count_dev), S(stream));
  HSX_LAUNCHED("count_diff_u8");
  return HSX_OK;
}

}  // extern "C"
