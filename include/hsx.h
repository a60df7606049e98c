/*
 * libhsx — B200-native (sm_100a) kernels for the PruneX H-SADMM
 * synchronization step. Plain C ABI: device pointers, sizes, a cudaStream_t
 * passed as void*. No torch types. Every entry point returns 0 (HSX_OK) or an
 * HSX_E* code; hsx_last_error() returns the thread-local message. Nothing is
 * thrown across the ABI and no call synchronizes the device except
 * hsx_keep_sets_fetch() (one D2H of per-layer counts per dynamic sync,
 * SURVEY.md §7.3 H5).
 *
 * The reference (admmprune 0.1.0, pure numpy) has no FFI; the entry points
 * below replace the numpy bodies its Python API calls. Each comment cites the
 * reference function it replaces (paths relative to
 * /root/reference/pkg/src/admmprune/). INTEGRATION.md shows the ctypes
 * binding a maintainer adds on the reference side.
 *
 * Memory: the caller owns every large buffer (the fp32 state arenas theta,
 * u, z_node, v, z, the intra-sum buffer, the flat compact buffer, mask-bit
 * arenas). A plan owns only its layer tables, work lists and small scratch
 * (group-norm partials, norms, keep flags, keep-set positions, counts).
 * A plan may be used by one stream at a time.
 *
 * Layout: all fp32 arenas share one layout: layer l occupies elements
 * [hsx_plan_layer_offset(l), +elements(l)), offsets are multiples of 32
 * (128 B), gaps are zero. Mask arenas hold one bit per element of each
 * prunable layer: bit b of 32-bit word (hsx_plan_mask_word_offset(l) + w) is
 * element 32*w + b of layer l in row-major order.
 */
#ifndef HSX_H_
#define HSX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HSX_ABI_VERSION 1

/* return codes; map 1:1 onto admmprune.errors (errors.py:4-13) */
enum {
  HSX_OK = 0,
  HSX_ESHAPE = 1,     /* ShapeError    */
  HSX_EPROTOCOL = 2,  /* ProtocolError */
  HSX_ECONFIG = 3,    /* ConfigError   */
  HSX_ECUDA = 4,      /* CUDA runtime error */
  HSX_EINVAL = 5      /* bad argument (null pointer, out-of-range index) */
};

/* structured groups (tensors.py:25-30 GroupBy; sparsity.py:20-30 ConstraintKind) */
enum { HSX_GROUP_FILTER = 0, HSX_GROUP_CHANNEL = 1, HSX_GROUP_SHAPE = 2 };
#define HSX_MAX_CONSTRAINTS 3

/* per-layer summary row returned by hsx_keep_sets_fetch */
enum {
  HSX_SUM_KOUT = 0,     /* |K_out| */
  HSX_SUM_KIN = 1,      /* |K_in|  */
  HSX_SUM_ELEMS = 2,    /* payload elements of the layer in the flat buffer */
  HSX_SUM_OFFSET = 3,   /* element offset of the layer's payload in the flat buffer */
  HSX_SUM_DRIFT = 4,    /* popcount(union ^ prev) — mask_drift numerator (sparsity.py:118-122) */
  HSX_SUM_POP = 5,      /* popcount(union) */
  HSX_SUM_COLS = 6
};

typedef struct hsx_plan hsx_plan;

/* One weight tensor (tensors.py:33-56 LayerSpec + its constraint list). */
typedef struct hsx_layer_desc {
  int32_t rank;                          /* 2 (fc / BN / bias as (1,d)) or 4 (conv) */
  int32_t shape[4];                      /* rank-2 uses shape[0..1] */
  int32_t n_constraints;                 /* 0 = travels dense */
  int32_t group[HSX_MAX_CONSTRAINTS];    /* HSX_GROUP_* in application order */
  int32_t keep[HSX_MAX_CONSTRAINTS];     /* keep counts, resolved by the caller with the
                                            reference expression (sparsity.py:53-62) */
  double rho1, rho2;                     /* PenaltySchedule entries (consensus.py:43-69) */
} hsx_layer_desc;

int hsx_abi_version(void);
const char* hsx_last_error(void);
/* number of kernels libhsx has launched in this process */
int64_t hsx_launch_count(void);
/* a CUDA graph holding `kernels` libhsx launches (captured through this ABI) was
   replayed: counted like eager launches */
void hsx_note_graph_replay(int64_t kernels);
/* L2 eviction-priority hints in the streaming kernels (z_node and the compact
 * buffer kept resident between K1 / K3 / K6 / K7, single-use streams evict
 * first) are a build choice (-DHSX_NO_L2_HINTS turns them off); returns 0 when
 * the library was built with the requested setting, 1 otherwise. */
int hsx_set_l2_hints(int32_t on);

/* ---- plans ----------------------------------------------------------------- */
int hsx_plan_create(const hsx_layer_desc* layers, int32_t n_layers, hsx_plan** out);
void hsx_plan_destroy(hsx_plan* plan);
int64_t hsx_plan_arena_elements(const hsx_plan* plan);
int64_t hsx_plan_layer_offset(const hsx_plan* plan, int32_t layer);
int64_t hsx_plan_mask_words(const hsx_plan* plan);
int64_t hsx_plan_mask_word_offset(const hsx_plan* plan, int32_t layer);   /* -1 if dense */
/* Offset of (layer, pass) in the concatenated norms / keep-flag vectors, -1 if none. */
int64_t hsx_plan_group_offset(const hsx_plan* plan, int32_t layer, int32_t pass);
int64_t hsx_plan_group_total(const hsx_plan* plan, int32_t pass);
/* Offset of a layer's K_out (which=0) / K_in (which=1) positions, -1 if dense. */
int64_t hsx_plan_keep_offset(const hsx_plan* plan, int32_t layer, int32_t which);
int64_t hsx_plan_keep_total(const hsx_plan* plan, int32_t which);
int32_t hsx_plan_max_passes(const hsx_plan* plan);
/* gamma = weight_decay/num_nodes + accels_per_node*rho1 + rho2 per layer
 * (consensus.py:157); HSX_ECONFIG if any gamma <= 0 (consensus.py:158-159).
 * rho1/rho2 may be NULL to keep the plan's values. identity != 0 makes the
 * candidate the raw input (used by the per-tensor project/group_norms API). */
int hsx_plan_set_penalties(hsx_plan* plan, const double* rho1, const double* rho2,
                           double weight_decay, int32_t num_nodes, int32_t accels_per_node,
                           int32_t identity);

/* ---- K0: intra-sum send buffer  send = theta + u  (consensus.py:439) -------- */
int hsx_pack_theta_u(const hsx_plan* plan, const float* theta, const float* u, float* send,
                     void* stream);

/* ---- K1: node candidate + first-pass group-norm partials -------------------
 * z_node <- (rho1*S + rho2*(z - v)) / gamma   in fp64, rounded once to fp32
 * (node_candidate, consensus.py:142-160). S is `sum` or, when sum == NULL,
 * theta + u (P == 1: the intra all-reduce is the identity).
 * frozen_mask == NULL: dynamic — prunable layers also accumulate fp64
 *   sum-of-squares partials of the unrounded candidate for their first
 *   constraint (group_norms, tensors.py:75-93), deterministic two-stage order.
 * frozen_mask != NULL: frozen — prunable layers get cand * mask
 *   (update_node_consensus frozen branch, consensus.py:177-180). */
int hsx_candidate(hsx_plan* plan, const float* sum, const float* theta, const float* u,
                  const float* z, const float* v, float* z_node, const uint32_t* frozen_mask,
                  void* stream);
/* Composite constraints, pass >= 1: recompute the candidate, apply the keep
 * flags of passes < pass, accumulate partials for this pass
 * (project_composite re-norms the projected tensor, sparsity.py:97-110). */
int hsx_candidate_renorm(hsx_plan* plan, int32_t pass, const float* sum, const float* theta,
                         const float* u, const float* z, const float* v, void* stream);

/* ---- K2: group norms -> top-k keep flags -----------------------------------
 * norms = sqrt(sum of partials); keep the `keep` largest, lower index on ties
 * (SparsityConstraint.resolve + _kept_group_indices, sparsity.py:53-68).
 * With HSX_FUSE_SELECT=1 layers are selected inside the candidate launch (tail
 * of the layer's last tile); this call completes the others. Always call it after
 * hsx_candidate / hsx_candidate_renorm of the same pass. Pass 0 issued as the
 * next launch on the same stream as a dynamic hsx_candidate /
 * hsx_candidate_peers is chained behind it when HSX_K2_CHAIN=1 (off by default:
 * measured slower on B200, the selection's dependent L2 round trips stall behind
 * K1's streaming traffic): that K1 counts
 * each prunable layer's finished tiles, the selection launch starts while K1
 * still streams and each layer's selection begins once its tiles are done;
 * completion still implies K1's completion. */
int hsx_select(hsx_plan* plan, int32_t pass, void* stream);
/* copy pass `pass` norms (fp64) / keep flags (uint8) to caller device buffers
 * of hsx_plan_group_total(pass) entries; either may be NULL. */
int hsx_read_groups(const hsx_plan* plan, int32_t pass, double* norms, uint8_t* flags,
                    void* stream);

/* ---- K3: projection + local support mask ------------------------------------
 * zero every element of z_node whose group is dropped by any pass; write the
 * packed mask bit  kept && z != 0  (project, sparsity.py:71-94; extract_mask
 * :113-115; update_node_consensus dynamic branch, consensus.py:181-182). */
int hsx_project(hsx_plan* plan, float* z_node, uint32_t* local_mask, void* stream);
/* K3 + keep sets for one node (M == 1: the union is the local mask): writes
 * the mask bits into `mask` and leaves the keep sets, payload sizes,
 * flat-buffer offsets and drift / popcount columns exactly as hsx_project
 * followed by hsx_keep_sets(mask, prev_mask) would (derive_keep_sets,
 * shrinkage.py:45-58; mask_drift numerator, sparsity.py:118-122).
 * With hsx_plan_set_single_node(plan, 1) the last selection pass has already
 * derived them from the group flags (the mask is the rectangle of kept rows x
 * kept columns unless a kept element is exactly zero); this call then only
 * checks for kept zeros and re-derives such layers from their bits. In that
 * mode prev_mask must be the `mask` of the previous call (drift is counted
 * against the previous rectangle). */
int hsx_project_keep_sets(hsx_plan* plan, float* z_node, uint32_t* mask, const uint32_t* prev_mask,
                          void* stream);
/* K2 + K3 (+ fixup) of a one-node plan in one launch when every prunable layer
 * has a single constraint: the selection CTAs publish per-layer ready flags and
 * the projection items of a layer start as soon as its selection is done (falls
 * back to hsx_select + hsx_project_keep_sets otherwise). Replaces the last
 * hsx_select + hsx_project_keep_sets of a dynamic step. */
int hsx_select_project_keep_sets(hsx_plan* plan, float* z_node, uint32_t* mask,
                                 const uint32_t* prev_mask, void* stream);
/* Single-node mode on / off (default off): see hsx_project_keep_sets. */
int hsx_plan_set_single_node(hsx_plan* plan, int32_t on);
/* Work-list order of the candidate / selection / projection launches (results do
 * not depend on it): big_first != 0 (default, HSX_K1_ORDER) takes the layers with
 * the costliest selection first so the chained selection overlaps K1 (one GPU);
 * 0 keeps layer order (measured faster when K1 reads the intra sum over NVLink).
 * Synchronous (re-uploads the work lists); call between steps. */
int hsx_plan_set_order(hsx_plan* plan, int32_t big_first);
/* One-node chain K1 -> K2 -> K3 -> K67 (default off; HSX_K67_CHAIN=0 forces it
 * off): the caller promises that every hsx_project_keep_sets of this single-node
 * plan is followed, as the next launch on the same stream, by hsx_local_sync.
 * The projection then runs behind the chained selection with the keep-set fixups
 * in its items, and K67 starts per layer as soon as the layer is projected. */
int hsx_plan_set_k67_chain(hsx_plan* plan, int32_t on);
/* Host buffer (page-locked, mapped) of the plan's keep-set summary rows, the same
 * layout hsx_keep_sets_fetch writes. With the K67 chain on (and the plan's
 * selection fully chained) the projection publishes the summary into it from the
 * device as soon as it is final; hsx_keep_sets_fetch_async with this buffer is
 * then a no-op and hsx_keep_sets_fetch_wait waits for the publication. */
int64_t* hsx_plan_summary_host(hsx_plan* plan);

/* ---- K4: leader mask union  out = OR_m gathered[m]  (transport.py:455-457) -- */
int hsx_mask_or(const uint32_t* gathered, int32_t n_ranks, int64_t words, uint32_t* out,
                void* stream);

/* ---- K5: keep sets from the union mask -------------------------------------
 * K_out = filters with any bit, K_in = channels with any bit, their prefix
 * positions, per-layer payload sizes and flat-buffer offsets in layer order
 * (derive_keep_sets shrinkage.py:45-58; bucketize concatenation
 * transport.py:239-280), plus popcount(union ^ prev) for mask_drift when
 * prev != NULL. */
int hsx_keep_sets(hsx_plan* plan, const uint32_t* union_mask, const uint32_t* prev_mask,
                  void* stream);
/* K4 fused into K5 (peer transport, M > 1): the union is the OR of the n leaders'
 * local mask bits `srcs` (peer-mapped), formed while K5 marks the keep sets and
 * stored to union_out; replaces hsx_mask_or_ptrs + hsx_keep_sets (and the
 * followers' copy of their leader's union). Multi-node plans only. */
int hsx_keep_sets_ptrs(hsx_plan* p, const uint32_t* const* srcs, int32_t n, uint32_t* union_out,
                       const uint32_t* prev_mask, void* stream);
/* D2H of the per-layer summary (n_layers x HSX_SUM_COLS int64, then 1 int64
 * total payload elements) into host memory; synchronizes `stream`. */
int hsx_keep_sets_fetch(hsx_plan* plan, int64_t* host_summary, void* stream);
/* Same copy without the synchronization: the caller records an event on
 * `stream` and waits on it before reading host_summary (lets the compaction
 * kernel run while the host sizes the leader all-reduce). Does not refresh
 * the plan's host mirror used by hsx_set_keep_sets. */
int hsx_keep_sets_fetch_async(hsx_plan* plan, int64_t* host_summary, void* stream);
/* Host wait for the last hsx_keep_sets_fetch_async copy (also when it was
 * captured into a CUDA graph and replayed: the copy is followed by an external
 * event-record node, so the host resumes mid-graph, before the step ends). */
int hsx_keep_sets_fetch_wait(hsx_plan* plan);
/* Install keep sets from host index lists (KeepSetCache hit path / per-tensor
 * compress): k_out/k_in sorted ascending, lengths n_out/n_in. Recomputes the
 * flat-buffer offsets of every layer. */
int hsx_set_keep_sets(hsx_plan* plan, int32_t layer, const int32_t* k_out, int32_t n_out,
                      const int32_t* k_in, int32_t n_in);
/* Copy positions (int32, -1 = dropped) of all layers: which=0 K_out, 1 K_in. */
int hsx_read_keep_positions(const hsx_plan* plan, int32_t which, int32_t* dst, void* stream);

/* ---- K6: leader compaction fused with the intra dual update -----------------
 * flat[payload] <- z_node + v gathered onto K_out x K_in (prunable) or raveled
 * (dense)  (consensus.py:476-483; compress shrinkage.py:61-68), and, when
 * theta/u != NULL, u <- u + (theta - z_node) (dual_update_intra,
 * consensus.py:185-186, 535). v == NULL compresses z_node alone. */
int hsx_compact_dual(const hsx_plan* plan, const float* theta, float* u, const float* z_node,
                     const float* v, float* flat, void* stream);
/* K6f: follower / non-sync intra dual update u <- u + (theta - z_node). */
int hsx_dual_intra(const hsx_plan* plan, const float* theta, float* u, const float* z_node,
                   void* stream);

/* ---- K7: decompaction fused with the inter dual update ----------------------
 * z <- zero-filled scatter of flat/divisor onto K_out x K_in (prunable) or
 * reshape (dense) (decompress shrinkage.py:71-82; consensus.py:491-504; the
 * leader average's "/ g", transport.py:461-462), and, when v != NULL,
 * v <- v + (z_node - z) (consensus.py:505). */
int hsx_decompact_dual(const hsx_plan* plan, const float* flat, float divisor,
                       const float* z_node, float* v, float* z, void* stream);

/* ---- phase 5: residuals, report, adaptive penalties --------------------------
 * (hierarchical_program phase 5, consensus.py:537-598; build_residual_report
 * :239-288; adapt_penalties :189-219). Per-layer fp64 squared norms are
 * accumulated inside K6 / K7 (no extra pass over the arenas), folded per layer
 * in a fixed order, summed over the node (intra) and the leaders (inter) by
 * the caller's collectives, turned into the report on the device, and the
 * adapted penalties are written into the plan's device layer table (the next
 * K1 uses them; no host round trip). */
typedef struct hsx_resid_params {
  double weight_decay, eps_abs, eps_rel;          /* ConsensusSettings (consensus.py:94-110) */
  double mu, tau_inc, tau_dec, rho1_max, rho2_max; /* PenaltySchedule (consensus.py:42-69) */
  int32_t num_nodes, accels_per_node, adapt;
  /* flat != 0: flat_consensus_program's report (baselines.py:229-254) on a one-node
   * (1 x W) plan with rho2 = 0 and v = 0: the per-layer intra entries as for one node
   * (z == z_node, so (z_node - z_node_prev)^2 is (z - z_prev)^2 and z_node^2 is z^2),
   * the inter entries 0; adaptation then moves rho1 only. */
  int32_t flat;
} hsx_resid_params;
/* K6 + residual slots 0-2 per layer: (theta - z_node)^2, theta^2, u'^2
 * (consensus.py:541-545). flat == NULL: the intra dual alone (followers). */
int hsx_compact_dual_resid(const hsx_plan* plan, const float* theta, float* u, const float* z_node,
                           const float* v, float* flat, void* stream);
/* K7 + residual slots 3-8: (z_node - z)^2, (z_node - z_node_prev)^2, z_node^2, v'^2,
 * (z - z_prev)^2, z^2 (consensus.py:552-563; z_prev is z as it was before this
 * call). flat == NULL: a non-sync iteration (z, v unchanged, dz = 0, no stores). */
int hsx_decompact_dual_resid(const hsx_plan* plan, const float* flat, float divisor,
                             const float* z_node, const float* z_node_prev, float* v, float* z,
                             void* stream);
/* F1: the leader average of two leaders fused into K7 (transport.py:453-462 AVG +
 * decompress, consensus.py:486-505): srcs[0], srcs[1] are the two leaders' flat
 * compact buffers in rank order (one is read over NVLink); every kept coordinate
 * gets z = fp32((srcs[0][i] + srcs[1][i]) / divisor) in fp64 — bitwise what
 * hsx_average_peers then hsx_decompact_dual(divisor 1) produce — written to
 * zhat_out[i] (the node's payload for the intra broadcast; may be NULL) and
 * decompacted with the inter dual v += z_node - z in the same pass.
 * residuals != 0: slots 3-8 as hsx_decompact_dual_resid. */
int hsx_decompact_average(const hsx_plan* plan, const float* const* srcs, int32_t n, double divisor,
                          float* zhat_out, const float* z_node, const float* z_node_prev, float* v, float* z,
                          int32_t residuals, void* stream);
/* K6 + K7 of a one-node cluster (M == 1) in one pass: the leader average is the
 * identity, so z = z_node + v on the kept rectangle (0 elsewhere), u += theta -
 * z_node, v += z_node - z, in place and bitwise equal to hsx_compact_dual then
 * hsx_decompact_dual(divisor 1) — without the compact buffer. residuals != 0
 * also accumulates all nine residual slots (z_node_prev required).
 * Issued as the next launch on the same stream after a one-node
 * hsx_project_keep_sets that ran chained (hsx_plan_set_k67_chain), it is
 * chained too: that projection runs each layer's keep-set
 * fixup in its last item and publishes the layer, and this kernel's items start
 * per layer as soon as their layer is published (dense layers once the candidate
 * and selection launches are complete); completion still implies the projection's. */
int hsx_local_sync(hsx_plan* plan, const float* theta, float* u, const float* z_node, float* v,
                   float* z, const float* z_node_prev, int32_t residuals, void* stream);
/* vec[layer][9] = the layer's slot sums (leader == 0 zeroes slots 3-8: the
 * node's leader contributes them to the intra SUM, consensus.py:550-563). */
int hsx_residual_fold(hsx_plan* plan, int32_t leader, double* vec, void* stream);
/* global != NULL: report[layer][8] + (r_pri, r_dual, eps_pri, eps_dual, converged)
 * from the globally summed vec (pack_report layout, consensus.py:291-300), then
 * adaptation; global == NULL: adaptation from a received report. scales[0][l] /
 * scales[1][l] receive the u / v rescale factors (1 when unchanged). */
int hsx_residual_report(hsx_plan* plan, const double* global, double* report, double* scales,
                        const hsx_resid_params* params, void* stream);
/* u *= scales[0][l], v *= scales[1][l] for the layers whose factor != 1. */
int hsx_scale_duals(const hsx_plan* plan, const double* scales, float* u, float* v, void* stream);
/* Phase-1 boundary: one proximal-SGD step (proximal_sgd, workloads.py:316-320) over
 * every layer: combined = grad + rho1*(theta - z_node + u); velocity = momentum *
 * velocity + combined (first != 0: velocity starts at 0, :312); theta -= lr *
 * velocity. fp64 math in the reference's order, fp32 state; rho1 from the plan's
 * device layer table. send != NULL also writes theta + u (the intra-sum send
 * buffer, K0 fused into the last step). HSX_ECONFIG if lr <= 0 (workloads.py:46-47). */
int hsx_prox_sgd_step(const hsx_plan* plan, const float* grad, float* theta, const float* z_node,
                      const float* u, float* velocity, double lr, double momentum, int32_t first,
                      float* send, void* stream);
/* Dense synchronous SGD baseline (dense_sync_program, baselines.py:77-98), flat fp32
 * arenas of n elements, fp64 math:
 *   send = grad + weight_decay * params                          (:88)
 * then, after the all-rank exchange, with avg = (sum_j sends[j], in order) / divisor:
 *   velocity = momentum * velocity + avg (first != 0: velocity starts at 0, :82);
 *   params -= lr * velocity                                       (:90-92)
 * n_sends == 1, divisor 1: sends[0] is the NCCL-averaged buffer; n_sends == W,
 * divisor W: sends are the W ranks' peer-mapped send buffers (NVLink), the AVG fused
 * into the update. HSX_ECONFIG if lr <= 0 (workloads.py:46-47). */
int hsx_dense_grad_pack(const float* grad, const float* params, double weight_decay, float* send, int64_t n,
                        void* stream);
int hsx_dense_apply(const float* const* sends, int32_t n_sends, double divisor, float* params, float* velocity,
                    double lr, double momentum, int32_t first, int64_t n, void* stream);
/* Top-K gradient compression with error feedback (topk_program, baselines.py:101-148).
 * A selector over layers at arena offsets[l] with elements[l] elements keeps
 * k_l = max(1, ceil(rate * elements[l])) entries per layer (:132); pairs of layer l
 * sit at [koff_l, koff_l + k_l) of the (values, indices) payload, K = sum k_l.
 *   select:  acc = residual + grad + wd * params (fp64, in place in residual, :128-129);
 *            the k_l largest |acc| per layer, ties to the lower index (stable argsort of
 *            -|x|, :71-74), written in ascending index order as fp32 values and
 *            layer-local int32 indices; selected residual entries become 0 (:142-144).
 *   scatter: dense[offset + index] += value for one rank's pairs (call in rank order, :137-139).
 *   apply:   avg = dense / divisor; velocity = momentum * velocity + avg (first: from 0);
 *            params -= lr * velocity (:145-146); dense is cleared for the next step. */
typedef struct hsx_topk hsx_topk;
int hsx_topk_create(const int64_t* offsets, const int64_t* elements, double rate, int32_t n_layers, hsx_topk** out);
void hsx_topk_destroy(hsx_topk* topk);
int64_t hsx_topk_total(const hsx_topk* topk);
int hsx_topk_layer_keep(const hsx_topk* topk, int32_t layer, int64_t* k, int64_t* offset);
int hsx_topk_select(const hsx_topk* topk, const float* grad, const float* params, double weight_decay,
                    double* residual, float* values, int32_t* indices, void* stream);
int hsx_topk_scatter(const hsx_topk* topk, const float* values, const int32_t* indices, double* dense, void* stream);
int hsx_topk_apply(const hsx_topk* topk, double* dense, double divisor, float* params, float* velocity, double lr,
                   double momentum, int32_t first, void* stream);
/* Current per-layer penalties (after device-side adaptation); synchronous. */
int hsx_plan_read_penalties(hsx_plan* plan, double* rho1, double* rho2);

/* ---- fused peer-memory collectives (one process per GPU, NVLink) ---------------
 * Pointer arrays are HOST arrays of DEVICE pointers to the same buffer on every
 * rank of a group, in member (rank) order, mapped into this process (e.g. torch
 * symmetric memory); n <= 4. The caller orders them after the peers' producers
 * with a group barrier. */
/* K1 with the intra all-reduce fused: S = sum_j sends[j] (fp64, rank order, the
 * reference's serial fold transport.py:453-462) read over NVLink. */
int hsx_candidate_peers(hsx_plan* plan, const float* const* sends, int32_t n, const float* z,
                        const float* v, float* z_node, const uint32_t* frozen_mask, void* stream);
/* Composite pass >= 1 of the peer candidate (same sources as hsx_candidate_peers). */
int hsx_candidate_renorm_peers(hsx_plan* plan, int32_t pass, const float* const* sends, int32_t n,
                               const float* z, const float* v, void* stream);
/* Staged peer operand for two ranks (allocate once): hsx_candidate_peers_staged
 * copies the peer's send into a plan-owned local buffer on a side stream, item by
 * item in K1's order, and K1 (the theta + u kernel with own send + that copy)
 * waits per item for its copy to land, reading the peer directly for an item whose
 * copy is late. Same values as hsx_candidate_peers with n = 2. */
int hsx_plan_set_peer_staging(hsx_plan* plan, int32_t on);
/* sends[0..1] in rank order, me = this rank's index among them; side_stream must be
 * forked from `stream` after the sends are valid (the caller joins it back before
 * the next staged call). Dynamic (non-frozen) steps only. */
int hsx_candidate_peers_staged(hsx_plan* plan, const float* const* sends, int32_t n, int32_t me, const float* z,
                               const float* v, float* z_node, void* stream, void* side_stream);
/* K4 over mapped pointers: out = OR_j srcs[j] (leaders' local masks, transport.py:455-457). */
int hsx_mask_or_ptrs(const uint32_t* const* srcs, int32_t n, int64_t words, uint32_t* out,
                     void* stream);
/* Leader average as a contiguous NVLink stream: out[i] = fp32((sum_j srcs[j][i],
 * rank order, fp64) / divisor) for i below the payload size of the plan's last
 * keep-set derivation (read on the device: no host sync). srcs are the leaders'
 * flat buffers (transport.py:453-462 AVG); with n = 1, divisor = 1 it is a
 * follower's read of its leader's averaged payload (the intra broadcast). */
int hsx_average_peers(const hsx_plan* plan, const float* const* srcs, int32_t n, double divisor,
                      float* out, void* stream);

/* Reduce-scatter / all-gather halves over mapped pointers for groups of >= 3
 * ranks: part >= 0 writes slice `part` of the rank-order average (divisor) of
 * srcs into out; part < 0 gathers every slice from its owner srcs[owner] into
 * out. The range is the plan's arena (payload == 0) or the payload size of the
 * last keep-set derivation read on the device (payload != 0). */
int hsx_slices_peers(const hsx_plan* plan, const float* const* srcs, int32_t n, int32_t part,
                     double divisor, int32_t payload, float* out, void* stream);
/* Device-side barrier of a group over NVLink: flags[i] is member i's int32 flag
 * array (peer-mapped, indexed by world rank), slots[i] member i's world rank,
 * me this rank's member index, epoch a per-group counter identical on all
 * members (incremented by the caller for every barrier). Enqueued on `stream`.
 * A member that has not arrived within HSX_BARRIER_TIMEOUT_S seconds (default
 * 600; 0 = wait forever, like an NCCL collective) does not trap the context: the
 * waiter counts a timeout and the stream continues; hsx_barrier_timeouts reports
 * it so the host can raise ProtocolError. */
int hsx_group_barrier(int32_t* const* flags, const int32_t* slots, int32_t n, int32_t me, int32_t epoch,
                      void* stream);
/* K1 on a distributed intra sum (P > 2, peer transport): after the reduce-scatter
 * (hsx_slices_peers with part = j on rank j), slices[j] = rank j's slice buffer;
 * each quad's S is read from its slice owner over NVLink (no all-gather of S,
 * no local copy). Same results as hsx_candidate on the all-gathered sum. */
int hsx_candidate_dist(hsx_plan* p, const float* const* slices, int32_t n, const float* z, const float* v,
                       float* z_node, const uint32_t* frozen_mask, void* stream);
/* Split two-rank K1 (P = 2, peer transport): each rank computes the candidate and
 * the group-norm partials of every dense item and of half of the prunable tiles,
 * reading both ranks' theta + u sends, and writes z_node, the partials and the
 * chained selection's tile counts into its own AND the peer's buffers (peer-mapped
 * memory), so each rank reads only half of the peer's send over NVLink. The
 * chained K2 (each layer's selection waits for both ranks' tiles) orders the peer's
 * writes before the selection, K3 and the rest of the step. Sizes of the
 * peer-mapped partials (doubles) and tile counters (uint32) the caller allocates: */
int hsx_plan_split_sizes(const hsx_plan* p, int64_t* partials_elems, int32_t* counters);
/* Install them (me = this rank's index in the pair); needs a single-pass plan with
 * the chained selection. */
int hsx_plan_set_split(hsx_plan* p, int32_t me, double* partials, double* partials_peer, uint32_t* k1done,
                       uint32_t* k1done_peer);
/* The split K1 (dynamic steps; z_node_peer = the peer's z_node arena). */
int hsx_candidate_peers_split(hsx_plan* p, const float* const* sends, int32_t n, const float* z, const float* v,
                              float* z_node, float* z_node_peer, void* stream);
/* One-sided variant: mode 0 = hsx_group_barrier; mode 1 = this member (the root)
 * only publishes the epoch and does not wait; mode 2 = this member waits for member
 * `root`'s epoch only (a producer -> readers hand-off; all members still count the
 * epoch). */
int hsx_group_barrier_mode(int32_t* const* flags, const int32_t* slots, int32_t n, int32_t me, int32_t epoch,
                           int32_t mode, int32_t root, void* stream);
/* Number of group barriers on the current device that timed out (synchronous
 * device read); reset != 0 zeroes the counter. */
int hsx_barrier_timeouts(uint32_t* count, int32_t reset);

/* ---- mask helpers for the per-tensor API -------------------------------------- */
/* out[i] = |t[i]| > 0  (extract_mask, sparsity.py:113-115) */
int hsx_nonzero_u8(const float* t, int64_t n, uint8_t* out, void* stream);
/* pack / unpack bool bytes <-> bits (n elements, bits zero-padded to a word) */
int hsx_pack_bits(const uint8_t* m, int64_t n, uint32_t* bits, void* stream);
int hsx_unpack_bits(const uint32_t* bits, int64_t n, uint8_t* m, void* stream);
/* *count_dev (uint64, device) += number of i with a[i] != b[i]  (mask_drift numerator) */
int hsx_count_diff_u8(const uint8_t* a, const uint8_t* b, int64_t n, uint64_t* count_dev,
                      void* stream);

/* Self-test of the candidate kernel's division: out[i] = num[i] / den computed
 * exactly as K1 does (q = RN(num*y), r = fma(-q, den, num), q' = fma(r, y, q)
 * with y = RN(1/den), Markstein's FMA correction). Tests compare it bit for
 * bit with IEEE division (numpy) to back the claim that K1's fp64 candidate is
 * the reference's (rho1*S + rho2*(z-v)) / gamma. */
int hsx_selftest_division(const double* num, int64_t n, double den, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HSX_H_ */
