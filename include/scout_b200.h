/*
 * scout_b200.h — C ABI of the B200-native ScoutAttention decode hot path.
 *
 * Drop-in boundary for the reference's hot-path functions
 * (/root/reference/proj/include/scout/{digest,attention,kv_store}.hpp).  Every entry point here replaces
 * one reference function, batched over "units" = (request, KV head) pairs of
 * one layer; the header-only C++ wrapper include/scout_b200.hpp restates the
 * reference signatures on top of these calls.
 *
 * Conventions:
 *   - every call returns an int status (SCOUT_OK == 0); the message of the
 *     last failure on the calling thread is scout_last_error();
 *   - all buffers are caller-owned device pointers unless a parameter says
 *     "host" (pinned, device-mapped host memory for K4);
 *   - each launching call takes a cudaStream_t (as void*; NULL = legacy default
 *     stream) and neither allocates nor synchronises the host;
 *   - argument errors -> SCOUT_ERR_INVALID_ARGUMENT (the reference throws
 *     std::invalid_argument), sequencing errors -> SCOUT_ERR_LOGIC
 *     (std::logic_error), launch failures -> SCOUT_ERR_CUDA.
 *
 * Fixed geometry (the reference's configs): head_dim d = 128,
 * block size B = 64 tokens, GQA group G = Hq/Hkv in {1,2,4,8}.
 *
 * Data layouts in HBM:
 *   KV pool    : slot-major array of blocks. Slot s holds K then V of one block
 *                (64 tokens x 128 channels). bf16 slots are 32 KiB, stored in the
 *                "half/slab/row" 128B-swizzled order (scout_kv_write_tokens
 *                writes it); f32 slots are 64 KiB, plain row-major. Slot
                indices are < 2^26.
 *   digests    : per unit [2][128][nb_stride] (lo then hi, channel-major, block
 *                id fastest) in the KV dtype for minmax; [128][nb_stride] f64
 *                for the mean method.
 *   queries    : [req][Hq][128] f32 (f64 for the generic f64 scoring path), or
 *                bf16 where a q_dtype field says SCOUT_BF16 (the model's own
 *                query dtype: half the bytes, products still exact in K1).
 *   partials   : o [req][Hq][128] f32 (normalised) + ml [req][Hq][2] f32
 *                = (max logit, denominator); empty partial = (0, -inf, 0).
 */
#ifndef SCOUT_B200_H
#define SCOUT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCOUT_HEAD_DIM 128
#define SCOUT_BLOCK_SIZE 64
#define SCOUT_MAX_BLOCKS 4096 /* per unit (256K tokens) */
#define SCOUT_MAX_K 512

enum scout_status {
    SCOUT_OK = 0,
    SCOUT_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
    SCOUT_ERR_LOGIC = 2,            /* reference: std::logic_error */
    SCOUT_ERR_CUDA = 3,
    SCOUT_ERR_UNSUPPORTED = 4
};

enum scout_dtype { SCOUT_F32 = 0, SCOUT_BF16 = 1, SCOUT_F64 = 2 };
#define SCOUT_TIER_ERR_SPLIT 3 /* scout_tier_layer.err: check_split failed (std::logic_error) */

/* Launch flags. SCOUT_LAUNCH_PDL launches with programmatic stream
 * serialization: K1 scores before waiting on the preceding kernel (it only
 * waits to publish its lists), K2 waits before reading K1's lists, so
 * consecutive K1/K2 launches overlap their prologues and tails. Every kernel
 * still observes all prior stream work before it reads dependent data. */
#define SCOUT_LAUNCH_PDL 1

/* DigestMethod, digest.hpp:23 */
enum scout_digest_method { SCOUT_DIGEST_MINMAX = 0, SCOUT_DIGEST_MEAN = 1 };

/* Message of the last failed call on this thread ("" if none). */
const char* scout_last_error(void);
int scout_version(void);
/* Bytes of one KV slot (K + V) for a dtype (SCOUT_F32 / SCOUT_BF16); 0 if unsupported. */
size_t scout_slot_bytes(int kv_dtype);

/* ------------------------------------------------------------------ K0 --
 * Write token rows into KV slots (kv_store.hpp:90-117 append_token's data
 * movement). Row i of k_rows/v_rows (f32, [n][128]) goes to slot slots[i],
 * row rows[i] (0..63), converted to kv_dtype.                              */
int scout_kv_write_tokens(void* kv_pool, int kv_dtype, const int32_t* slots, const int32_t* rows,
                          const float* k_rows, const float* v_rows, int n, void* stream);
/* Inverse of the above (tests / host tier spill): rows back to f32. */
int scout_kv_read_tokens(const void* kv_pool, int kv_dtype, const int32_t* slots,
                         const int32_t* rows, float* k_rows, float* v_rows, int n, void* stream);

/* Digest build for n blocks (build_digest, digest.hpp:34-60; the open-block
 * refresh of kv_store.hpp:108). Block i = slot slots[i] with block_rows[i]
 * valid rows (>= 1) is summarised into unit units[i], column block_ids[i] of
 * the digest array. minmax: digests in kv_dtype, exact. mean: f64 digests,
 * sequential double sum / rows (bit-exact with the reference).             */
int scout_digest_build(const void* kv_pool, int kv_dtype, int method, int n, const int32_t* slots,
                       const int32_t* block_rows, const int32_t* units, const int32_t* block_ids,
                       void* digests, int nb_stride, void* stream);

/* Decode-time append (append_token kv_store.hpp:90-117, one layer, data
 * side): for every unit u, the f32 rows k_rows[u] / v_rows[u] ([n_units][128])
 * go to row n_tokens[u] % 64 of pool slot open_slot[u] (the caller hands a
 * fresh slot when that row is 0, i.e. a new block opens), and the digest column
 * of block n_tokens[u] / 64 is updated in place: minmax continues the
 * reference's min/max fold by one row (bit-identical to rebuilding the open
 * block, kv_store.hpp:108); mean recomputes the sequential double column sum
 * of the stored rows / rows (f64 digests). advance != 0 also increments
 * n_tokens[u] (set it on the last layer appended: n_tokens is shared by the
 * layers). A block is sealed when n_tokens becomes a multiple of 64.        */
int scout_kv_append(void* kv_pool, int kv_dtype, int method, int n_units, const int32_t* open_slot,
                    int32_t* n_tokens, const float* k_rows, const float* v_rows, void* digests, int nb_stride,
                    int advance, void* stream);

/* ------------------------------------------------------------------ K1 --
 * Score + top-k + resident/CPU split for n_units units of one layer
 * (digest_score digest.hpp:62-72, select_topk :101-118, set_intersection /
 * set_difference :77-87 as called at engine.hpp:238-242).
 *
 * q: [n_units/Hkv... ] laid out as [unit][G][128] — i.e. [req][Hq][128] with
 *    unit = req*Hkv + kvh and head = kvh*G + g. f32 for bf16/f32 digests,
 *    f64 for f64 digests.
 * Score of block b = sum over c (outer) and g (inner) of
 *    max(q_g[c]*lo[c], q_g[c]*hi[c])   (minmax)   or   q_g[c]*mean[c]   (mean),
 *    accumulated sequentially in double from +0.0: the reference's
 *    digest_score on the stacked G*128-vector q_s[c*G+g].
 * n_tokens[u]: tokens cached for unit u; blocks = ceil(n_tokens/64); the last
 *    block is the open block with n_tokens - 64*(blocks-1) rows.
 * Selection: the min(k, blocks) best scores, ties to the lower block id; ids
 *    written ascending to sel_ids[u*k_stride ...], count to n_sel[u].
 * block_table (optional, [unit][nb_stride] int32): slot of a block that is
 *    (or will be, for planned recalls) GPU-resident, -1 otherwise. If given,
 *    res_slots/res_ids/n_res receive the resident share (ascending ids) and
 *    cpu_ids/n_cpu the rest; res_tokens/cpu_tokens (optional) the row counts.
 * last_selected (optional, [unit][nb_stride] int32): set to `step` for every
 *    selected block (mark_selected, kv_store.hpp:222-228).
 * scores_out (optional, [unit][nb_stride] f64): the raw scores.
 * k == 0 -> SCOUT_ERR_INVALID_ARGUMENT (digest.hpp:103).                    */
typedef struct scout_topk_args {
    int n_units;
    int group;      /* G */
    int digest_dtype;
    int method;
    int k;
    int k_stride;   /* row stride of the id/slot outputs (>= k) */
    int nb_stride;  /* digest / table row stride in blocks (multiple of 8) */
    int step;
    const void* q;
    const void* digests;
    const int32_t* n_tokens;
    const int32_t* block_table;
    int32_t* sel_ids;
    int32_t* n_sel;
    int32_t* res_slots;
    int32_t* res_ids;
    int32_t* n_res;
    int32_t* cpu_ids;
    int32_t* n_cpu;
    int32_t* res_tokens;
    int32_t* cpu_tokens;
    int32_t* last_selected;
    double* scores_out;
    int flags;      /* SCOUT_LAUNCH_PDL: programmatic dependent launch */
    /* optional completion flag: when every CTA has written its lists, the
     * last one stores done_token to *done_flag (release, gpu scope);
     * done_ctr is a zero-initialised counter it leaves zeroed */
    unsigned* done_flag;
    unsigned* done_ctr;
    unsigned done_token;
    int q_dtype;    /* minmax bf16/f32 digests: SCOUT_F32 (0, default) or SCOUT_BF16 queries */
} scout_topk_args;

int scout_score_topk_split(const scout_topk_args* args, void* stream);
/* The same for n layers in ONE launch (grid = units x layers): every
 * args[i] must share n_units, group, nb_stride, digest dtype and method. */
int scout_score_topk_split_batch(const scout_topk_args* args, int n, void* stream);

/* ------------------------------------------------------------------ K2 --
 * Block-sparse flash-decode over the GPU-resident selected blocks of every
 * unit (partial_attention attention.hpp:73-95 with accumulate_token :38-50,
 * GPU side of engine.hpp:257-258), optionally LSE-merged with a CPU partial
 * (merge :100-114, finalize :117-122, empty -> zeros engine.hpp:273).
 *
 * q [req][Hq][128] f32 (the true query), res_slots/res_ids/n_res as written
 * by K1 (row stride k_stride), n_tokens per unit (for the open block's rows).
 * Outputs o [req][Hq][128] f32 normalised and ml [req][Hq][2] = (m, l) with m
 * the max scaled logit and l the softmax denominator relative to m.
 * cpu_o / cpu_ml (optional, same layout): the co-attention partial to merge.
 * workspace: scout_sparse_decode_workspace_bytes(); zero it ONCE after
 * allocation (the kernel leaves its counters zeroed).                      */
typedef struct scout_decode_args {
    int n_units;
    int group;
    int kv_dtype;
    int k_stride;
    float scale;
    const void* q;  /* f32 (or bf16, see q_dtype) */
    const void* kv_pool;
    const int32_t* res_slots;
    const int32_t* res_ids;
    const int32_t* n_res;
    const int32_t* n_tokens;
    const float* cpu_o;
    const float* cpu_ml;
    float* o;
    float* ml;
    void* workspace;
    size_t workspace_bytes;
    int max_ctas; /* 0 = one persistent CTA per SM */
    int flags;    /* SCOUT_LAUNCH_PDL: programmatic dependent launch */
    int q_dtype;  /* bf16 KV: SCOUT_F32 (0, default) or SCOUT_BF16 queries (q then points to bf16) */
} scout_decode_args;

size_t scout_sparse_decode_workspace_bytes(int n_units, int group, int max_ctas);
/* CTAs the bf16 launch uses: max_ctas, or one persistent CTA per SM when 0
 * (capped at 1024), whatever the unit count or list length: a CTA plans a
 * range of any size in chunks. */
int scout_sparse_decode_grid(int n_units, int k_stride, int max_ctas);
int scout_sparse_decode(const scout_decode_args* args, void* stream);

/* ------------------------------------------------------------------ K3 --
 * Standalone LSE merge of two partial sets (merge attention.hpp:100-114):
 * out = merge(a, b) row-wise over n_rows heads. Empty operands are exact
 * identities; both empty -> o = 0, ml = (-inf, 0).  out may alias a.       */
int scout_merge_partials(const float* a_o, const float* a_ml, const float* b_o, const float* b_ml,
                         float* out_o, float* out_ml, int n_rows, void* stream);

/* ------------------------------------------------------------------ K4 --
 * Periodic-recall gather (the slow->fast move that kv_store.hpp:201-218
 * applies as a tier flip): copy n whole block images from device-mapped
 * pinned host memory (host_blocks + src_index[i]*slot_bytes) into pool slots
 * dst_slots[i]. Launch it on a side stream and gate the consumer with an
 * event; the kernel streams over PCIe / C2C with 16-byte loads.            */
int scout_recall_gather(void* kv_pool, int kv_dtype, const void* host_blocks,
                        const int64_t* src_index, const int32_t* dst_slots, int n, void* stream);
/* Same move on the copy engines (no SM time): one cudaMemcpyAsync per run of
 * consecutive (src_index, dst_slot) pairs, so it suits contiguous runs; a
 * scattered list is per-call bound (~6.7 GB/s, profiles/r02a_pcie_recall.txt)
 * and belongs on scout_recall_gather. src_index / dst_slots are HOST arrays
 * here; `stream` must not be the legacy default stream.                    */
int scout_recall_copy(void* kv_pool, int kv_dtype, const void* host_blocks, const int64_t* src_index,
                      const int32_t* dst_slots, int n, void* stream);

/* ------------------------------------------------------------------ K5 --
 * Device-resident tier bookkeeping: the GPU mirror of TieredKvCache's
 * per-layer state (kv_store.hpp:296-305) for n_units units of ONE layer, so
 * residency planning, LRU eviction and recall tickets never leave the device.
 * Clock ticks encode the reference's (step, layer) pairs as
 * step * n_layers + layer (pair order == integer order).
 * All arrays are device memory, row stride nb_stride blocks ([U][nb_stride])
 * or slots_per_unit (free ring); zero-initialise tier, fill table / ready /
 * warm / free_owner with -1, zero free_head, and put the (layer, unit)'s
 * pool slots in free_slots[u][0 .. n_free).                                */
typedef struct scout_tier_layer {
    int32_t* table;       /* [U][nbs] pool slot of a fast or in-flight block, -1 otherwise */
    uint8_t* tier;        /* [U][nbs] 1 = fast, 0 = slow (Tier, kv_store.hpp:19) */
    int32_t* last_sel;    /* [U][nbs] last_selected step (K1 writes it: mark_selected) */
    int32_t* ready;       /* [U][nbs] ready tick of an in-flight recall, -1 none */
    int32_t* ticket;      /* [U][nbs] issue number of that recall (apply order) */
    int32_t* free_slots;  /* [U][slots_per_unit] ring of free pool slots */
    int32_t* n_free;      /* [U] */
    int32_t* err;         /* [U] sticky first error of the unit (0 none): 1 invalid
                             argument (reference throws std::invalid_argument), 2 out of slots,
                             3 (engine) K1's split broke check_split (engine.hpp:317-329) */
    int capacity;         /* sealed fast blocks per unit; <= 0: pinned layer (pin_layer) */
    int slots_per_unit;   /* row stride of the free ring (>= the slots a (layer, unit) owns) */
    /* The free slots form a FIFO ring per unit: entries (head + i) % slots_per_unit,
     * i < n_free; allocation takes the oldest entry, a freed slot goes to the back.
     * Device victim cache (optional: free_owner and warm both set, or both NULL):
     * a slot freed by an eviction keeps the evicted block's image, so while the
     * slot waits in the ring the block has a WARM copy in HBM. A recall of a warm
     * block takes that slot back and moves no bytes (the reference moves none
     * either: the tier flip is the recall, kv_store.hpp:201-218); the tier state
     * is exactly the reference's either way. An allocation that reuses a slot
     * forgets its image. Sealed blocks are immutable, so a warm
     * image stays equal to the host-tier image.                             */
    int32_t* free_head;   /* [U] ring head */
    int32_t* free_owner;  /* [U][slots_per_unit] block whose image the entry's slot holds, -1 */
    int32_t* warm;        /* [U][nbs] ring position of a slow block's warm image, -1 */
} scout_tier_layer;

/* append_token's bookkeeping (kv_store.hpp:95-115), n_tokens = count BEFORE
 * the append: a new block takes a free slot, is fast and marked clock_step;
 * the append that fills a block seals it (mark = clock_step) and enforces
 * capacity (LRU victim, ties -> lower id, kv_store.hpp:333-345). open_slot[u]
 * receives the slot to hand scout_kv_append; sealed_id[u] the block sealed by
 * this append or -1 (its image goes to the host tier: write-through).     */
int scout_tier_append(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                      int clock_step, int32_t* open_slot, int32_t* sealed_id, void* stream);
/* begin_layer's application for this layer (kv_store.hpp:201-218): blocks
 * whose recall is ready at or before due_tick become fast, ticket by ticket,
 * each followed by enforce_capacity. n_applied[u] (optional) counts them.  */
int scout_tier_apply(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                     int due_tick, int32_t* n_applied, void* stream);
/* schedule_recall (kv_store.hpp:175-197) per unit: ids[u][0..n_ids[u]) an
 * ascending set of sealed, slow, not-in-flight blocks (else the unit's ticket
 * is rejected: err = 1, dst_slots = -1); n_ids[u] == 0 skips the unit.
 * Accepted blocks get a pool slot and ready_tick / ticket. dst_slots[u][i]:
 * the slot (>= 0) the block's image must be copied into, or -2 - slot when
 * the block's warm image already sits in that slot (no copy).             */
int scout_tier_schedule_recall(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                               const int32_t* ids, const int32_t* n_ids, int k_stride, int ready_tick, int ticket,
                               int32_t* dst_slots, void* stream);
/* residency_set (kv_store.hpp:156-170) as K1's block table [U][nb_stride]:
 * the slot of every fast block and of every in-flight block ready by
 * next_tick (= next_run_of(layer), kv_store.hpp:328-331), -1 elsewhere.    */
int scout_tier_plan(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                    int next_tick, int32_t* block_table, void* stream);
/* Bulk prefill of a FRESH layer (the caller side of the decode path): the
 * state n_tokens[u] append_token calls at clock_step leave
 * (kv_store.hpp:90-117; the last `capacity` sealed blocks and the open block
 * fast, the others slow, every mark clock_step), in one pass: the rows
 * k_rows / v_rows [U][max_tokens][128] f32 go into the pool slots of the
 * fast blocks (and of warm images of the highest-id slow blocks while free
 * slots remain), min/max digests [U][2][128][nb_stride] of every block in
 * the KV dtype, and every sealed block's image to the host tier at
 * (host_base + u * nb_stride + id) % host_blocks (write-through; host_tier
 * NULL: none). blk_slot: device scratch [U][nb_stride] int32. Follow with
 * scout_tier_place for place_after_prefill (kv_store.hpp:271-283).         */
int scout_tier_prefill(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                       int clock_step, const float* k_rows, const float* v_rows, int max_tokens, void* kv_pool,
                       int kv_dtype, void* digests, void* host_tier, long long host_base, long long host_blocks,
                       int32_t* blk_slot, void* stream);
/* mark_selected (kv_store.hpp:222-228) for explicit ascending id lists
 * (K1 marks its own selections through scout_topk_args.last_selected).     */
int scout_tier_mark(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* ids,
                    const int32_t* n_ids, int k_stride, int step, void* stream);
/* place_after_prefill (kv_store.hpp:271-283): keep[u] = ascending ids of the
 * top-capacity sealed blocks (K1 over the sealed blocks, k = capacity); the
 * other sealed blocks go slow and free their slots; a kept block that was
 * slow takes a free slot, returned in fill_slots[u][i] (optional, else -1)
 * so the caller copies its image in. No-op for pinned layers.              */
int scout_tier_place(const scout_tier_layer* layer, int n_units, int nb_stride, const int32_t* n_tokens,
                     const int32_t* keep, const int32_t* n_keep, int k_stride, int32_t* fill_slots, void* stream);

/* ------------------------------------------------------------------ K6 --
 * Layer-ahead query prediction on the tcgen05 tensor
 * cores: q_pred[b] = predict_next_query(rms_normalize(x[b]), W_Q^{i+1})
 * (model.hpp:215-217, numerics.hpp:99-123, called at engine.hpp:237).
 * W [hidden][n_out] bf16 (the reference's hidden x out layout) is packed once
 * into UMMA core-matrix tiles (w_packed: hidden*n_out bf16). x [batch][hidden]
 * f32, batch <= 256, hidden % 128 == 0, n_out % 128 == 0. Outputs q_pred
 * [batch][n_out] as f32 and/or bf16 (either may be NULL): fp32 accumulation of
 * bf16 products. Stream-K over (128-feature tile, 64-wide K chunk) units on
 * max_ctas CTAs (0 = one per SM); a tile shared by several CTAs is summed in
 * CTA order (deterministic). workspace: scout_qpred_workspace_bytes() for the
 * same max_ctas, zeroed once (the kernel leaves its counters zeroed).      */
size_t scout_qpred_workspace_bytes(int hidden, int n_out, int batch, int max_ctas);
int scout_qpred_pack_weights(const void* w, int hidden, int n_out, void* w_packed, void* stream);
int scout_predict_query(const float* x, int batch, int hidden, const void* w_packed, int n_out, float* out_f32,
                        void* out_bf16, void* workspace, size_t workspace_bytes, int max_ctas, void* stream);

/* Device-driven tier data movement. Host tier layout: the image of block
 * (layer, unit, id) at index host_base + unit * nb_stride + id, with
 * host_base = layer * n_units * nb_stride, modulo host_blocks when > 0 (a
 * bounded synthetic tier whose images alias) (pinned, device-mapped memory).
 * scout_recall_gather_ids: unit u's blocks ids[u][0..n_ids[u]) (e.g. K1's
 * CPU-side ids) into the slots K5 assigned (dst_slots, -1 = skipped), SM
 * loads over PCIe / C2C on `ctas` CTAs (0 = 32: a narrow footprint next to
 * a persistent K2).
 * scout_kv_writeback: write-through of the blocks scout_tier_append sealed
 * (sealed_id[u] >= 0 at slot open_slot[u]) into their host images.        */
int scout_recall_gather_ids(void* kv_pool, int kv_dtype, const void* host_tier, long long host_base, int nb_stride,
                            long long host_blocks, int n_units, const int32_t* ids, const int32_t* n_ids, const int32_t* dst_slots,
                            int k_stride, int ctas, void* stream);
int scout_kv_writeback(const void* kv_pool, int kv_dtype, void* host_tier, long long host_base, int nb_stride,
                       long long host_blocks, int n_units, const int32_t* open_slot, const int32_t* sealed_id, void* stream);

/* ------------------------------------------------------------- host CPU --
 * CPU co-attention worker (the reference's PrecomputeWorker
 * engine.hpp:88-150 running partial_attention attention.hpp:73-95 on the
 * CPU-side blocks): HOST memory throughout. Unit u's G heads
 * q[(u*G+g)*128] (f32) attend over n_blocks[u] block images
 * host_tier + host_index[u*k_stride+i] * slot_bytes (the pool's layout: bf16
 * swizzled tiles or f32 rows), block_rows[u*k_stride+i] valid rows (NULL: 64).
 * Writes o [(u*G+g)][128] normalised and ml [(u*G+g)][2] = (max logit, denom),
 * empty = (0, -inf, 0): K2's CPU-partial input. bf16 images on an AMX-BF16
 * CPU: tile products (q split bf16 hi + lo, P rounded to bf16 as in K2);
 * otherwise fp32 AVX-512 (SCOUT_CPU_AMX=0 forces this). `threads` workers of
 * a persistent pool (0 = all hardware threads).                           */
int scout_cpu_partial_attention(const void* host_tier, int kv_dtype, const int64_t* host_index,
                                const int32_t* block_rows, const int32_t* n_blocks, int k_stride, const float* q,
                                int group, float scale, int n_units, float* o, float* ml, int threads);
/* The same with the model's dtypes: q in q_dtype and o in o_dtype (SCOUT_F32
 * or SCOUT_BF16; ml stays f32). A bf16 query is widened exactly; a bf16 o is
 * the f32 result rounded to nearest even, bit for bit what the f32 entry point
 * followed by that rounding gives. This is what the decode calls' CPU-partial
 * input takes with cfg.cpu_dtype = SCOUT_BF16 (no host-side conversion).   */
int scout_cpu_partial_attention_ex(const void* host_tier, int kv_dtype, const int64_t* host_index,
                                   const int32_t* block_rows, const int32_t* n_blocks, int k_stride, const void* q,
                                   int q_dtype, int group, float scale, int n_units, void* o, int o_dtype, float* ml,
                                   int threads);
/* Which kernel scout_cpu_partial_attention runs for kv_dtype on this CPU now:
 * 2 = AMX-BF16 tiles, 1 = AVX-512 fp32, 0 = scalar.                        */
int scout_cpu_coattn_kernel(int kv_dtype);

/* ------------------------------------------------------ recall policy --
 * calibrate_intervals (recall.hpp:66-95), host only: per layer, the longest
 * run of leading steps of a recall-free profiling trace whose CPU ratio
 * cpu_tokens / budget_tokens stays <= beta (a ratio equal to beta counts),
 * floor 1. cpu_tokens / budget_tokens: [layers][steps] in step order (the
 * reference records cpu_partial.token_count / k * block_size per (layer,
 * step), engine.hpp:283; a batched engine's aggregate is
 * scout_engine_cpu_tokens). beta in (0, 1), every budget > 0.            */
int scout_calibrate_intervals(const int64_t* cpu_tokens, const int64_t* budget_tokens, int layers, int steps,
                              double beta, int32_t* intervals);

/* ------------------------------------------------------------- engine --
 * Host-side layer-ahead decode orchestration (ScoutEngine::decode_step,
 * engine.hpp:205-314, GPU side): per layer i, K1 for layer i+1 with the
 * predicted query (layer 0: K1 with the true query, pinned resident,
 * engine.hpp:227-233), K2+K3 for layer i with the true query over the
 * resident share chosen during layer i-1, merged with layer i's CPU partial;
 * then, when layer i is due for a recall (the cadence below), K4 moves that
 * layer's recall host->device on a side stream; layer i's next attention
 * waits for it (issue (m, i) -> visible (m+1, i), kv_store.hpp:175-218).
 * Static mode: the caller owns the tables and the recall plans. Device tier
 * mode (cfg.tier): the engine runs the reference's policy on the device. */
typedef struct scout_layer_desc {
    const void* digests;         /* [U][2][128][nb_stride] in kv dtype */
    const int32_t* block_table;  /* [U][nb_stride] slot or -1 (planning view) */
    const int64_t* recall_src;   /* optional recall plan (HOST arrays, copied at create):
                                    host block indices ... */
    const int32_t* recall_dst;   /* ... and destination pool slots */
    int recall_n;
} scout_layer_desc;

typedef struct scout_engine_config {
    int layers, batch, hq, hkv, k, nb_stride, kv_dtype;
    float scale;
    int recall_interval;       /* 0 disables K4 */
    void* kv_pool;
    const int32_t* n_tokens;   /* [U] device */
    const void* host_tier;     /* pinned host block images (K4 source) */
    int max_ctas;              /* K2 grid (0 = one CTA per SM) */
    int host_staging;          /* 1: allocate device staging for decode_step_host */
    int chunk_layers;          /* layers per H2D/D2H chunk of the host path (0 = 8) */
    int recall_mode;           /* 1: SM gather kernel over the mapped host tier (K4, the default
                                  of the Python engine); 0: copy engines, one cudaMemcpyAsync per
                                  contiguous run (scout_recall_copy) */
    int q_dtype;               /* q_true / q_pred element type: SCOUT_F32 (0) or SCOUT_BF16 */
    /* device tier mode (optional): per-layer K5 state (host array of `layers`
     * descs over device arrays). Residency is then planned on the device
     * (layers[].block_table and recall plans are ignored), decode steps take
     * the new token's K/V (scout_engine_decode_step_kv) and append it, seal
     * blocks with write-through to host_tier, evict LRU, and recall each
     * layer's CPU-side selected blocks every recall_interval steps straight
     * from K1's lists (no host round trip). host_tier holds block images at
     * ((layer * U + unit) * nb_stride + id) % host_blocks (host_blocks <= 0:
     * no wrap; the bench bounds it and lets images alias; see host_units).  */
    const scout_tier_layer* tier;
    long long host_blocks;
    int cpu_dtype;             /* CPU-partial o element type: SCOUT_F32 (0) or SCOUT_BF16 (half the
                                * host-path bytes; its (max, denominator) pairs stay f32)        */
    /* Recall cadence (engine.hpp:35, recall.hpp:97-126). recall_intervals
     * (optional host array [layers], each >= 1; copied at create) gives each
     * layer its calibrated interval; NULL: recall_interval for every layer.
     * Layer i is due at step s when s - last_recall(i) >= interval(i), with
     * last_recall = 0 at prefill (so at steps n, 2n, ...), and a due trigger
     * resets the cadence even when it moves nothing. recall_stagger = 1 keeps
     * round 1's staggered cadence instead ((s + i) % interval == 0, one
     * interval for all layers): it spreads the PCIe traffic over the steps. */
    const int32_t* recall_intervals;
    int recall_stagger;
    /* In-engine CPU co-attention (the reference's PrecomputeWorker,
     * engine.hpp:88-150, 243-271), device tier mode host path only: 1 = the
     * engine itself computes every step's CPU partials on cpu_threads host
     * threads (0 = all) over the host tier, from the CPU-side ids K1 selects
     * in THIS step and the step's predicted queries (layer i's partial with
     * q_pred[i]), and publishes them layer chunk by layer chunk to the running
     * K2, which merges each layer as soon as its chunk landed. The decode
     * calls' cpu_o / cpu_ml inputs must then be NULL. 0 = the caller supplies
     * the partials. */
    int cpu_worker;
    int cpu_threads;
    /* GpuSidePolicy (engine.hpp:25-29): SCOUT_GPU_SIDE_PREDICTED (0, the
     * default) attends to K1's predicted-and-resident share of each layer;
     * SCOUT_GPU_SIDE_ALL_RESIDENT (1) to the layer's whole fast tier at
     * attention time (residency_set after begin_layer, engine.hpp:253-256;
     * the CPU share is unchanged and check_split is not applied, as in the
     * reference). */
    int gpu_side_policy;
    /* layer-by-layer mode (scout_engine_decode_layer): K2 CTAs of a
     * single-layer launch; the SMs it leaves free run K1 of the next layer
     * beside it. 0: automatic (the grid less 68), < 0: the whole grid. */
    int layer_ctas;
    /* Device tier mode: the host tier's unit index space when it is shared by
     * several engines (request-sharded ranks): block (layer, unit u, id) of
     * this engine is image ((layer * host_units + host_unit0 + u) * nb_stride
     * + id) % host_blocks. host_units = 0: this engine's U, host_unit0 = 0. */
    int host_units;
    int host_unit0;
    /* K6 inside the layer-by-layer mode (scout_engine_decode_layer_x): the
     * model's hidden size (0: off). The engine then keeps the predictor's
     * workspace and a q_pred buffer of one layer. */
    int hidden;
} scout_engine_config;

#define SCOUT_GPU_SIDE_PREDICTED 0
#define SCOUT_GPU_SIDE_ALL_RESIDENT 1

typedef struct scout_engine scout_engine;

int scout_engine_create(const scout_engine_config* cfg, const scout_layer_desc* layers, scout_engine** out);
int scout_engine_destroy(scout_engine* eng);
/* One decode step, device-resident inputs: q_true / q_pred [L][U*G][128] in
 * cfg.q_dtype, cpu_o [L][U*G][128] in cfg.cpu_dtype, cpu_ml [L][U*G][2] f32; outputs out_o
 * [L][U*G][128], out_ml [L][U*G][2] f32. */
int scout_engine_decode_step(scout_engine* eng, int step, const void* q_true, const void* q_pred,
                             const void* cpu_o, const float* cpu_ml, float* out_o, float* out_ml, void* stream);
/* Same step from pinned HOST buffers (same layouts): H2D of the inputs and
 * D2H of the outputs plus each layer's CPU-side block ids (h_cpu_ids
 * [L][U][k], h_n_cpu [L][U], the host co-attention worker's input) are
 * pipelined by layer chunks on copy streams. Completion is ordered on
 * `stream`: synchronise it before reading the host outputs. As with
 * cudaMemcpyAsync, the input copies start as soon as the call is made (they
 * overlap the previous step's attention), so the host inputs must be final
 * at the call and stay unchanged until `stream` completes the step. */
int scout_engine_decode_step_host(scout_engine* eng, int step, const void* h_q_true, const void* h_q_pred,
                                  const void* h_cpu_o, const float* h_cpu_ml, float* h_out_o, float* h_out_ml,
                                  int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream);
/* Device tier mode: one decode step with the token's new K/V rows k_new /
 * v_new [L][U][128] f32 appended after each layer's attention (the order of
 * engine.hpp:220-307: plan, select + mark, begin_layer's ticket application,
 * attention + merge, append, recall). The other arguments as
 * scout_engine_decode_step. n_tokens (cfg) advances by one per step.      */
int scout_engine_decode_step_kv(scout_engine* eng, int step, const void* q_true, const void* q_pred,
                                const void* cpu_o, const float* cpu_ml, const float* k_new, const float* v_new,
                                float* out_o, float* out_ml, void* stream);
/* Device tier mode from pinned HOST buffers (the pipeline of
 * scout_engine_decode_step_host plus h_k_new / h_v_new [L][U][128] f32).
 * The step's selection follows the previous step's engine work, not other
 * work the caller queued on `stream` after it: the engine owns every device
 * buffer it reads, and the previous step's output copies need not finish
 * before the next step's selection starts. */
int scout_engine_decode_step_kv_host(scout_engine* eng, int step, const void* h_q_true, const void* h_q_pred,
                                     const void* h_cpu_o, const float* h_cpu_ml, const float* h_k_new,
                                     const float* h_v_new, float* h_out_o, float* h_out_ml, int32_t* h_cpu_ids,
                                     int32_t* h_n_cpu, void* stream);
/* Device tier mode: the tier state's sticky per-unit errors (a rejected
 * recall ticket, out of pool slots, a split that broke check_split,
 * engine.hpp:317-329, checked after every step). Synchronises; returns
 * SCOUT_OK, or SCOUT_ERR_INVALID_ARGUMENT / SCOUT_ERR_LOGIC naming the first
 * (layer, unit) with an error. */
int scout_engine_check_state(scout_engine* eng);
/* Device tier mode, layer by layer: the calls a decoder makes inside its
 * layer loop (engine.hpp:219-307 per layer), for layers 0, 1, ..., L-1 of a
 * step in order. Layer i's call applies layer i's due recall tickets, selects
 * layer i+1 with its predicted query q_pred_next [U*G][128] (q dtype; NULL for
 * the last layer; layer 0 also selects itself with q_true), runs layer i's
 * attention + merge with q_true [U*G][128] over the share selected one call
 * earlier (cpu_o / cpu_ml: layer i's CPU partial, optional), writes out_o
 * [U*G][128] / out_ml [U*G][2], and appends k_new / v_new [U][128] f32 after
 * the attention. A layer's inputs need only exist at its call (they come from
 * the previous layer's output in a decoder); the selection of layer i+1 runs
 * on the engine's own stream beside layer i's attention. */
int scout_engine_decode_layer(scout_engine* eng, int step, int layer, const void* q_true, const void* q_pred_next,
                              const void* cpu_o, const float* cpu_ml, const float* k_new, const float* v_new,
                              float* out_o, float* out_ml, void* stream);
/* The same call with the layer-ahead prediction inside (engine.hpp:237,
 * cfg.hidden > 0): q_pred of layer + 1 = predict_next_query(rms_normalize(
 * x_next), W_Q^{layer+1}) on K6 (the tcgen05 GEMM, scout_predict_query) into
 * an engine buffer, then K1 of layer + 1 on it. x_next [batch][hidden] f32 is
 * the hidden state the model feeds layer + 1's prediction; wq_next_packed is
 * W_Q^{layer+1} packed by scout_qpred_pack_weights (hidden x hq*128). Both
 * NULL for the last layer.                                                 */
int scout_engine_decode_layer_x(scout_engine* eng, int step, int layer, const void* q_true, const float* x_next,
                                const void* wq_next_packed, const void* cpu_o, const float* cpu_ml, const float* k_new,
                                const float* v_new, float* out_o, float* out_ml, void* stream);
/* Order all outstanding side-stream work (recalls) before `stream`. */
int scout_engine_sync(scout_engine* eng, void* stream);
/* Device tier mode: the caller changed the K5 state outside the engine
 * between steps (e.g. scout_tier_place for a newly admitted request). Each
 * step's post-attention launch writes the next step's planning view; this
 * makes the next step plan again from the current state instead. */
int scout_engine_tier_changed(scout_engine* eng);
/* Instrumentation: when enabled, CUDA events bracket every K2 launch (on the
 * launching stream). scout_engine_stats synchronises, reports the summed K2
 * event time, K2 count and the number of kernels launched since the last
 * call, then resets. */
int scout_engine_set_timing(scout_engine* eng, int enable);
int scout_engine_stats(scout_engine* eng, double* k2_ms_total, int* k2_count, long long* launches);
/* The same window's K2 launch durations one by one (ms[0..min(n, max_n))),
 * without resetting it (call before scout_engine_stats); synchronises. */
int scout_engine_k2_times(scout_engine* eng, float* ms, int max_n, int* n);
/* Device tier mode: recalled blocks since the last reset that were served by
 * a warm image in HBM (no bytes moved) and that were copied from the host
 * tier; reset != 0 zeroes the counts. Synchronises the device.            */
int scout_engine_recall_stats(scout_engine* eng, long long* warm_blocks, long long* copied_blocks, int reset);
/* The overlapped step (whole-step calls: device tier mode, and the static
 * view when it has no recall plans): K1 of the step runs beside K2 on a share
 * of the SMs (K2 polls K1's per-layer flags) instead of before it, from the
 * second step on, when no begin_layer ticket is due, the policy is the
 * predicted top-k, the KV is bf16 and a unit has <= 1024 blocks; the
 * environment variable SCOUT_K1K2_OVERLAP=<SMs> sets the share (0: off),
 * scout_engine_set_overlap per engine (-1: the environment / default 35% of
 * the grid, 0: off, > 0: K1's SMs). Never under a kernel-serialising tool
 * (CUDA_INJECTION64_PATH, CUDA_LAUNCH_BLOCKING). The stats: steps run that
 * way since the last reset, and the last share.                            */
int scout_engine_set_overlap(scout_engine* eng, int k1_sms);
int scout_engine_overlap_stats(scout_engine* eng, long long* steps, int* k1_sms, int reset);
/* ScoutEngine::prefill + place_after_prefill (engine.hpp:192-201), device
 * tier mode, on FRESH tier state: every layer filled from the model's rows
 * k_rows / v_rows [L][U][max_tokens][128] f32 with n_tokens[u] tokens per
 * unit (device) by scout_tier_prefill (slots, digests into the layers'
 * digest arrays, write-through to the host tier), the engine's token counts
 * set to n_tokens; then, with q_place [L][U*G][128] (q dtype, the layers'
 * last prefill queries; NULL: skip), every unpinned layer keeps its
 * top-capacity sealed blocks fast, the promoted blocks' images taken from
 * warm slots or gathered from the host tier (required then). Allocates
 * scratch and synchronises. Once per engine (a second call: LOGIC).       */
int scout_engine_prefill(scout_engine* eng, const float* k_rows, const float* v_rows, const int32_t* n_tokens,
                         int max_tokens, const void* q_place, void* stream);
/* The last step's CPU-side tokens per layer summed over the units (K1's
 * split: the tokens the host co-attention attends) and the matching budget,
 * U * k * 64 (engine.hpp:189, 283): one RatioTrace sample per layer for
 * scout_calibrate_intervals. Synchronises.                                 */
int scout_engine_cpu_tokens(scout_engine* eng, int64_t* cpu_tokens, int64_t* budget_tokens);
/* In-engine CPU worker (cfg.cpu_worker): the wall time its partials took
 * on the host pool, summed over the steps since the last call, then reset. */
int scout_engine_worker_stats(scout_engine* eng, double* cpu_ms_total, int* steps);
/* Device views of the engine's per-layer K1 outputs ([L][U][k] / [L][U]). */
int scout_engine_k1_outputs(scout_engine* eng, int32_t** res_slots, int32_t** res_ids, int32_t** n_res,
                            int32_t** cpu_ids, int32_t** n_cpu, int32_t** res_tokens, int32_t** cpu_tokens);

#ifdef __cplusplus
}
#endif

#endif /* SCOUT_B200_H */
