// Device side of libhsx: the sm_100a kernels of the H-SADMM sync step.
// All kernels are HBM-bound streaming / gather-scatter work (no tensor cores:
// arithmetic intensity <= 0.3 flop/B). Conventions:
//  * fp32 state, fp64 arithmetic for every compound expression so each output
//    is the fp32 rounding of the reference's fp64 value on the same inputs;
//  * 128-bit loads/stores on the contiguous streams, scalar (warp-coalesced)
//    stores for the compact payload whose offsets are not 16-B aligned;
//  * deterministic reductions: fixed per-thread ownership and fixed shuffle
//    trees, no floating-point atomics (leaders must agree bit-for-bit).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hsx {

constexpr int kMaxPasses = 3;
constexpr int kSumCols = 6;  // HSX_SUM_COLS
enum { kFilter = 0, kChannel = 1, kShape = 2 };

// n / d for n < 2^32, d < 2^32 via one 64-bit mul-hi: m = ceil(2^64 / d).
struct FastDiv {
  unsigned long long m;
  unsigned int d;
  unsigned int pad;
};

__host__ inline FastDiv make_fastdiv(unsigned int d) {
  FastDiv f;
  f.d = d;
  f.pad = 0;
  f.m = d > 1 ? (~0ULL / d + 1ULL) : 0ULL;
  return f;
}

__device__ __forceinline__ unsigned int fdiv(unsigned int n, const FastDiv& f) {
  return f.d == 1 ? n : (unsigned int)__umul64hi((unsigned long long)n, f.m);
}

// Per-layer table entry (one per weight tensor, layer order = reference order).
struct DevLayer {
  long long off;    // element offset in every fp32 arena
  long long n;      // elements
  long long mword;  // mask word offset, -1 for dense layers
  long long okeep;  // offset of this layer's K_out flags / positions
  long long ikeep;  // offset of this layer's K_in flags / positions
  long long cpoff;  // offset of this layer's column maps (colpos / colkeep), multiple of 4
  long long goff[kMaxPasses];  // offset into norms / keep flags per pass
  long long poff[kMaxPasses];  // offset into group-norm partials per pass ([nparts][G]; FILTER [G])
  int rows, cin, k, L;         // rank-4: c_out, c_in, kh*kw, c_in*kh*kw; rank-2: d0, d1, 1, d1
  int ncons;                   // number of constraints (0 = dense path)
  int nparts;                  // row tiles of the candidate kernel (partials rows)
  int rsub;                    // rows per shared-memory sub-tile
  int rank;
  int tiling;                  // 0: row tiles (partials per group / row), 1: quad tiles (per column)
  int qtile;                   // K3/K6/K7 use row-quad tiles (prunable, c_in*kh*kw % 32 == 0)
  int fsel;                    // bit q: pass q's selection runs in K1's tail (no K2 launch)
  int pidx;                    // index among prunable layers
  int group[kMaxPasses];
  int keep[kMaxPasses];
  int G[kMaxPasses];
  int ncitems;                 // K1 items of the layer (dynamic launch)
  int npitems;                 // K3 items of the layer
  int cq;                      // K1 quad tiles: column quads per tile (whole channels unless percol)
  int percol;                  // K1 writes per-column partials [nparts][L]; the selection folds channels
  int cw;                      // K1 quad tiles: lanes per row (power of two >= the tile's quads, <= 64);
                               // the CTA's other lanes take more rows (narrow layers keep every lane busy)
  FastDiv divL, divk;
  double rho1, rho2, gamma;
  double rgamma;               // RN(1 / gamma), for the FMA-corrected division
};

// A contiguous slice [begin, end) of one layer's elements.
struct Item {
  int layer;
  int part;   // candidate: row-tile index; keep-mark: prunable-layer index
  int chunk;  // quad tiles: column chunk of 64 quads; keep-mark: items of the layer
  int tile;   // 1: row-quad tile, [begin, end) are rows; 0: element range
  long long begin, end;  // element range (quad tiling: rows [begin, end))
};

constexpr int kMaxPeers = 4;  // ranks whose buffers a fused peer kernel reads

// device pointers of the same buffer on every rank of a group (member order)
struct PeerPtrs {
  const float* p[kMaxPeers];
  int n;
};

struct MaskPtrs {
  const uint32_t* p[8];
  int n;
};

struct FlagPtrs {
  uint8_t* f[kMaxPasses];
};

struct KeepArgs {
  const DevLayer* layers;
  const Item* items;
  const uint32_t* uni;
  // usrc.n > 0: the union is the OR of these mask-bit arrays (the leaders' local
  // masks, peer-mapped), formed while marking and stored to uni_out (K4 fused into K5)
  MaskPtrs usrc;
  uint32_t* uni_out;
  const uint32_t* prev;
  uint8_t* oflag;
  uint8_t* iflag;
  int* pos_out;
  int* pos_in;
  FlagPtrs flags;            // group keep flags of every pass (K3: kept = AND of the passes)
  long long* summary;
  unsigned int* layer_done;  // per prunable layer
  unsigned int* done;        // prunable layers finished
  unsigned long long* acc;   // per prunable layer: drift, popcount accumulators (zero between launches)
  // structured keep sets (one node)
  uint8_t* rk_prev;          // [sum rows] rows of the previous rectangle R x C
  uint8_t* ch_prev;          // [sum c_in] its channels (layers without SHAPE groups)
  uint8_t* ck_prev;          // [sum L]    its columns (layers with SHAPE groups)
  int* irr;                  // per prunable layer: bit 0 a kept zero now, bit 1 previously
  int* irr_any;              // some layer has a kept zero now
  int n_layers;
  int n_prunable;
};

struct CandArgs {
  const float* __restrict__ s;
  const float* __restrict__ theta;
  const float* __restrict__ u;
  const float* __restrict__ z;
  const float* __restrict__ v;
  float* __restrict__ zn;
  const uint32_t* __restrict__ fmask;  // frozen global mask bits or nullptr
  const DevLayer* __restrict__ layers;
  const Item* __restrict__ items;
  double* __restrict__ partials;       // this pass
  const uint8_t* flags[kMaxPasses];    // keep flags of earlier passes (renorm)
  PeerPtrs peers;                      // n > 0: S = sum of the peers' theta + u (rank order)
  unsigned int* k1done;                // chained K2: +1 per finished tile of a prunable layer (or nullptr)
  // split two-rank K1 (hsx_candidate_peers_split): this rank computes half of the
  // prunable layers' tiles and writes z_node, the partials and the tile counts into
  // its own and the peer's buffers (peer-mapped; nullptr: not split)
  float* zn_peer;
  double* partials_peer;
  unsigned int* k1done_peer;
  // distributed sum (P > 2, hsx_candidate_dist): S lives in the P ranks' reduce-scatter
  // slices, peers.p[j] = rank j's slice buffer (valid on [sbound[j], sbound[j + 1]))
  long long sbound[kMaxPeers];
  int sdist;
  // cross-tile pipelining (hsx: HSX_K1_XTILE): a persistent CTA claims its next item
  // when a quad tile's loads are consumed and puts the next quad tile's first ring
  // stages in flight before the tile's fold; the fold then uses the ring's last stage
  int xtile;
  // staged peer operand (two ranks): u is a local copy of the peer's send that a
  // staging kernel fills item by item on a side stream; sready[item] == epoch + 1
  // once the item's region landed, else K1 reads u_alt (the peer's send) directly
  const float* u_alt;
  const unsigned int* sready;          // nullptr = not staged
  unsigned int* sepoch;                // [0] epoch (K1's last CTA bumps it), [1] K1 exit counter
  int reserve;                         // persistent grid: CTA slots left free for the chained K2
  // fused selection (K2 in the tail of each layer's last K1 tile)
  double* norms;                       // this pass
  FlagPtrs fw;                         // keep flags, all passes (this pass written)
  unsigned int* cand_done;             // per prunable layer: K1 tiles finished
  unsigned int* sched;                 // [2] persistent-CTA item counter + exit counter (left zeroed)
  int n_items;
  KeepArgs ka;                         // structured keep sets at the last pass (one node)
  int structured;
  int pass;
  int identity;                        // candidate = input (per-tensor API)
  int sqcap;                           // doubles of the sq sub-tile region
};

// K3 -> K67 chain of one node: per-layer "projected + fixed" flags published by the
// chained K3, the upstream-complete flag (K1 and K2 done), per-layer item counters
// of K67 (stream items per layer: count[]), and a launch-wide counter
struct ChainK67 {
  unsigned int* ready3;    // [layers]; nullptr = not chained
  unsigned int* upstream;
  unsigned int* cnt;       // [layers]
  const int* count;        // [layers] stream items per layer
  unsigned int* all;
  // the chained K3 publishes the finished keep-set summary straight into mapped host
  // memory (pub_sum, n_sum int64), then bumps the mapped sequence word pub_seq
  long long* pub_sum;
  unsigned int* pub_seq;
  unsigned int* seq_ctr;   // device-side publish counter
  int n_sum;
};

struct ElemArgs {
  const float* __restrict__ theta;
  float* __restrict__ u;
  const float* __restrict__ zn;
  float* __restrict__ v;
  const float* __restrict__ vin;
  const float* __restrict__ flat_in;
  float* __restrict__ flat_out;
  float* __restrict__ z;
  const DevLayer* __restrict__ layers;
  const Item* __restrict__ items;
  const int* __restrict__ pos_out;     // K_out position of each row, -1: dropped
  const int* __restrict__ pos_in;      // K_in position of each channel, -1: dropped
  const long long* __restrict__ summary;
  float divisor;
  // phase-5 residuals (consensus.py:537-563): per-item fp64 partial sums of squares,
  // [item][kResidSlots] (K6 / K6f: slots 0-2, K7: slots 3-8); nullptr = off
  double* __restrict__ rpart;
  const float* __restrict__ zn_prev;   // K7: the previous iteration's z_node
  // K7 with the two-leader average fused (F1): flat_in, flat_in2 in rank order,
  // z = fp32((a + b) / avg_div) in fp64; zhat_out (optional) receives the average
  const float* flat_in2;
  float* zhat_out;
  double avg_div;
  ChainK67 c67;                        // K67 chained behind the chained K3 (ready3 == nullptr: off)
};
constexpr int kResidSlots = 9;         // consensus.py:235 (_INTER_SLOTS)

void launch_candidate(const CandArgs& a, int n_items, int frozen, size_t smem, cudaStream_t st);
// the staging copy of the peer's send for a staged K1 (side stream): K1's dynamic
// items in order, each region copied from peer to stage, then sready[item] = epoch + 1
void launch_stage(const float* peer, float* stage, const DevLayer* layers, const Item* items, int n_items,
                  unsigned int* sready, const unsigned int* sepoch, unsigned int* counter, int grid, cudaStream_t st);
// K2; k1done != nullptr: chained behind the K1 launch that counted its tiles into
// k1done (a layer's selection starts once k1done[pidx] reaches its tile count and
// subtracts it again; the grid-completion wait moves to the end)
void launch_select(const DevLayer* layers, const int* list, int n, int pass, const double* partials,
                   double* norms, FlagPtrs flags, const KeepArgs& ka, int structured, size_t smem, cudaStream_t st,
                   unsigned int* k1done = nullptr, unsigned int* ready = nullptr);
void launch_mask_or(const MaskPtrs& g, long long words, uint32_t* out, cudaStream_t st);
void launch_keep_sets(const KeepArgs& a, int n_items, size_t smem, cudaStream_t st);
void launch_keep_fixup(const KeepArgs& a, const int* prunable, int n, size_t smem, cudaStream_t st);
// K3; check != 0: flag layers with a kept zero (structured keep sets)
// ready != nullptr: chained behind a chained K2 that publishes ready[layer] (pdone:
// per prunable layer item counters, left zeroed)
// c67.ready3 != nullptr (with ready): the layer's last item also runs the keep-set
// fixup (fix_smem bytes) and publishes ready3[layer] for a chained K67
void launch_project(const KeepArgs& a, int n_items, float* zn, uint32_t* mask, int check, cudaStream_t st,
                    unsigned int* ready = nullptr, unsigned int* pdone = nullptr, ChainK67 c67 = ChainK67{},
                    size_t fix_smem = 0);
struct SelProjArgs {
  const int* list;          // layers to select (pass 0)
  int nsel;
  const double* partials;   // pass 0
  double* norms;
  unsigned int* ready;      // per layer: selection published (left zeroed)
  unsigned int* pdone;      // per prunable layer: K3 items finished (left zeroed)
  int structured;
};
void launch_select_project(const SelProjArgs& sp, const KeepArgs& a, int n_items, float* zn, uint32_t* mask,
                           size_t smem, cudaStream_t st);
// shared memory of the structured keep-set derivation (K1 / K2 tail)
size_t structured_smem_bytes(int rows, int L, int cin);
size_t select_smem_bytes(int G);
void launch_compact(const ElemArgs& a, int n_items, cudaStream_t st);
void launch_decompact(const ElemArgs& a, int n_items, cudaStream_t st);
void launch_local_sync(const ElemArgs& a, int n_items, cudaStream_t st);
// phase 5: per-layer fold of the residual partials, report + adaptation, dual rescale
struct ResidArgs {
  DevLayer* layers;                     // penalties updated in place when adapting
  int n_layers;
  const int* first;                     // per layer: first stream item, item count
  const int* count;
  const double* rpart;                  // [item][kResidSlots]
  double* vec;                          // [layer][kResidSlots]
  int leader;                           // 0: slots 3-8 zeroed (the leader contributes them)
  const double* global;                 // globally summed [layer][kResidSlots], or nullptr: adapt from report
  double* report;                       // [layer][8] + 5 (consensus.py:291-300 layout)
  double* scales;                       // [2][layer]: u scale, v scale
  double wd, eps_abs, eps_rel, mu, tau_inc, tau_dec, rho1_max, rho2_max;
  int num_nodes, per_node, adapt, flat;
};
void launch_resid_fold(const ResidArgs& a, cudaStream_t st);
void launch_report(const ResidArgs& a, cudaStream_t st);
// Top-K baseline (baselines.py:101-148)
struct TkLayer {
  long long off;    // arena offset of the layer
  long long n;      // elements
  long long k;      // keep count, max(1, ceil(rate * n)) (:132)
  long long koff;   // offset of the layer's pairs in the payload
  int tile0, ntiles;
};
struct TkTile {
  int layer;
  int pad;
  long long begin, end;  // layer-local element range
};
struct TkState {
  unsigned long long prefix, mask;  // radix-select prefix of bits(|acc|) so far
  long long k_rem;                  // keys still to take inside the prefix bin
  int done, pad;
};
int launch_topk_select(const TkTile* tiles, int n_tiles, const TkLayer* tl, int L, TkState* st, unsigned* hist,
                       int2* cnt, int2* base, double* res, const float* g, const float* p, double wd, float* vals,
                       int* idx, cudaStream_t stq);
void launch_topk_scatter(const TkLayer* tl, int L, const float* vals, const int* idx, long long ktotal, double* dense,
                         cudaStream_t st);
void launch_topk_apply(double* dense, double div, float* p, float* v, double lr, double mom, int first, long long n,
                       cudaStream_t st);
void launch_dense_pack(const float* g, const float* p, double wd, float* send, long long n, cudaStream_t st);
void launch_dense_apply(const PeerPtrs& src, double div, float* p, float* v, double lr, double mom, int first,
                        long long n, cudaStream_t st);
void launch_prox_sgd(const DevLayer* layers, const Item* items, int n_items, const float* g, float* th,
                     const float* zn, const float* u, float* vel, float* send, double lr, double mom, int first,
                     cudaStream_t st);
void launch_scale_duals(const DevLayer* layers, const Item* items, int n_items, const double* scales,
                        int n_layers, float* u, float* v, cudaStream_t st);
void launch_slices(const PeerPtrs& src, const long long* total_p, long long total_h, long long max_elems,
                   int part, double div, float* out, cudaStream_t st);
struct BarrierArgs {
  int* flags[32];  // members' flag arrays (peer-mapped), member order
  int slots[32];   // members' slot indices (their world ranks)
  int n, me, epoch;
  int mode;    // 0: everyone publishes and waits; 1: publish only (root); 2: wait for member `root` only
  int root;
  unsigned long long timeout_ns;  // 0: wait forever (set by launch_barrier)
};
void launch_barrier(const BarrierArgs& b, cudaStream_t st);
// barriers that timed out on the current device (synchronous read; reset != 0 zeroes it)
int barrier_timeouts(unsigned int* count, int reset);
void launch_average(const PeerPtrs& src, const long long* total, long long max_elems, double div, float* out,
                    cudaStream_t st);
void launch_add(const float* a, const float* b, float* out, long long n, cudaStream_t st);
void launch_dual(const float* theta, float* u, const float* zn, long long n, cudaStream_t st);
void launch_nonzero(const float* t, long long n, uint8_t* out, cudaStream_t st);
void launch_pack(const uint8_t* m, long long n, uint32_t* bits, cudaStream_t st);
void launch_unpack(const uint32_t* bits, long long n, uint8_t* m, cudaStream_t st);
void launch_div_selftest(const double* num, long long n, double den, double* out, cudaStream_t st);
void launch_count_diff(const uint8_t* a, const uint8_t* b, long long n, unsigned long long* c,
                       cudaStream_t st);

}  // namespace hsx
