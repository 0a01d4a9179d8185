/*
 * hgca_b200.h -- C ABI of the B200-native hybrid decode-attention library
 * (libhgca_b200.so). Plain device pointers, sizes and a CUDA stream; no torch
 * types. Every entry point returns 0 on success, HGCA_EINVAL for a contract
 * violation (the reference raises ContractError, errors.py:1-2) or
 * HGCA_ECUDA for a CUDA failure; hgca_last_error() describes the last failure
 * of the calling thread.
 *
 * Reference interfaces each entry replaces (paths under
 * /root/reference/pkg/src/tierkv/):
 *   hgca_attend_dense          backends.active.attend_dense   backends.py:8-20, _core.pyx:22-84
 *   hgca_attend_indexed        backends.active.attend_indexed backends.py:8-20, _core.pyx:87-150
 *   hgca_attend_indexed_heads  per-head attend_indexed loop   engine.py:139-148
 *   hgca_attend_gqa            append-mode attend over window / archive  engine.py:127-132, 161-164
 *   hgca_attend_gqa_indexed    decode a_cpu: per-head attend_indexed over the engine's KV  engine.py:139-148
 *   hgca_append_bf16           the same append step for BF16 storage on the tensor cores (+ row-mean weights)
 *   hgca_merge_states          merge_states                   attention.py:153-188
 *   hgca_select_threshold      select_salient                 sparsifier.py:32-42
 *   hgca_mask_to_indices       np.nonzero / context index lists sparsifier.py:42, 77-87
 *   hgca_popcount_rows         ContextCache.sizes             sparsifier.py:74-75
 *   hgca_group_need            pack_head_groups targets       sparsifier.py:209-217
 *   hgca_select_topk           pack_head_groups padding order sparsifier.py:219-226
 *   hgca_write_rows            WindowCache.append_kv          kv_cache.py:122-169
 *   hgca_maw_update            WindowCache.update_maw / StoreTier.reevaluate kv_cache.py:171-187, sparsifier.py:158-177
 *   hgca_maw_ema               WindowCache.update_maw on fp64 weights   kv_cache.py:171-187
 *   hgca_union_build(_items)   (device layout of the context cache for the decode kernel)
 *   hgca_decode_step           HybridEngine._run_step, decode mode engine.py:151-195
 *   hgca_decode_step_host      the same step with host q|k|v in / out|lse back (one call)
 *   hgca_decode_step_host_async  ... without the final stream synchronization
 *   hgca_merge_partials        P-way merge of sharded (out, lse) partials
 *   hgca_merge_packed          P-way merge of the allgathered packed partials
 *   hgca_merge_packed_wait     the same merge behind the one-shot NVLink push (flags), hgca_peer_*
 */
#ifndef HGCA_B200_H
#define HGCA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGCA_OK 0
#define HGCA_EINVAL 1
#define HGCA_ECUDA 2

#define HGCA_DTYPE_F32 0
#define HGCA_DTYPE_F64 1
#define HGCA_DTYPE_BF16 2

typedef void* hgca_stream_t; /* a cudaStream_t */

int hgca_version(void);
const char* hgca_last_error(void);

/* ---- plugin boundary (tierkv backend contract) ---------------------------
 * Dense: q [H,nq,d], k/v [H,nkv,d] of one dtype (F32 or F64), C-contiguous.
 * out [H,nq,d] (input dtype), lse [H,nq] fp64, weights [H,nq,nkv] or NULL.
 * ws: caller scratch of hgca_attend_ws_bytes(H*nq, nkv) bytes.
 * nkv == 0 gives zero output and lse = -inf (_core.pyx:41-45). */
int64_t hgca_attend_ws_bytes(int64_t rows, int64_t nkeys);
int hgca_attend_dense(int dtype, const void* q, const void* k, const void* v, int64_t H,
                      int64_t nq, int64_t nkv, int64_t d, double scale, int keep_weights,
                      void* out, double* lse, void* weights, void* ws, hgca_stream_t stream);

/* Indexed (single head): q [nq,d], k/v [M,d], idx int64 [n] (rows of k/v). */
int hgca_attend_indexed(int dtype, const void* q, const void* k, const void* v,
                        const int64_t* idx, int64_t n, int64_t M, int64_t nq, int64_t d,
                        double scale, int keep_weights, void* out, double* lse, void* weights,
                        void* ws, hgca_stream_t stream);

/* Many heads at once: q [H,nq,d], k/v [H,M,d]; head h attends
 * idx[idx_off[h] .. idx_off[h]+idx_cnt[h]) (device arrays); weights for head h
 * are written at weights + h*nq*max_n with row stride max_n. */
int hgca_attend_indexed_heads(int dtype, const void* q, const void* k, const void* v,
                              int64_t H, int64_t M, const int64_t* idx, const int64_t* idx_off,
                              const int64_t* idx_cnt, int64_t max_n, int64_t nq, int64_t d,
                              double scale, void* out, double* lse, void* weights, void* ws,
                              hgca_stream_t stream);

/* Grouped-query attention over rows [row0, row0+n) of the interleaved
 * position buffer KV [B*Hkv, T, 2, d] (F32 or BF16 storage; BF16 rows in the
 * position-rotated layout hgca_write_rows produces): q [B*Hq, nq, d];
 * q-head h of batch b reads kv-head b*Hkv + h/(Hq/Hkv). out float32,
 * weights [B*Hq, nq, wts_ld] float32 or NULL. */
int hgca_attend_gqa(int dtype, const void* q, const void* KV, int64_t B, int64_t Hq, int64_t Hkv,
                    int64_t T, int64_t row0, int64_t n, int64_t nq, int64_t d, double scale, void* out,
                    double* lse, void* weights, int64_t wts_ld, void* ws, hgca_stream_t stream);
/* attend_indexed per query head over the engine's HBM layout (KV [B*Hkv, T, 2, d],
 * bf16 rows position-rotated): head bh = b*Hq + h attends rows idx[idx_off[bh] ..
 * + idx_cnt[bh]) of kv head b*Hkv + h/(Hq/Hkv); weights [B*Hq, nq, max_n] in the
 * output dtype (float32). The decode step's store-tier weight rows a_cpu
 * (engine.py:139-148) when the engine keeps weights. ws: [B*Hq*nq*max_n] fp64. */
int hgca_attend_gqa_indexed(int dtype, const void* q, const void* KV, int64_t B, int64_t Hq, int64_t Hkv,
                            int64_t T, const int64_t* idx, const int64_t* idx_off, const int64_t* idx_cnt,
                            int64_t max_n, int64_t nq, int64_t d, double scale, void* out, double* lse,
                            void* weights, void* ws, hgca_stream_t stream);

/* merge_states over `rows` rows of d: outputs in dtype, lse fp64. Optional
 * weight rows (w_a [rows,na], w_b [rows,nb] -> w_out [rows,na+nb]). */
int hgca_merge_states(int dtype, const void* out_a, const double* lse_a, const void* out_b,
                      const double* lse_b, int64_t rows, int64_t d, void* out, double* lse,
                      const void* w_a, const void* w_b, int64_t na, int64_t nb, void* w_out,
                      hgca_stream_t stream);

/* P-way merge of fp32 partials: outs [P, rows, d], lses [P, rows] -> out, lse
 * (left fold of merge_states in p order). */
int hgca_merge_partials(const float* outs, const double* lses, int64_t P, int64_t rows, int64_t d,
                        float* out, double* lse, hgca_stream_t stream);

/* P-way merge of packed partials: partial p = out [rows, d] f32 at
 * parts + p*stride_bytes followed by lse [rows] f64 (the receive buffer of the
 * sequence-sharded (out, lse) allgather; rank order fold). */
/* Peer buffers for the one-shot exchange: device memory that other processes
 * map (CUDA IPC). hgca_peer_alloc returns the pointer and a 64-byte handle for
 * the peers; hgca_peer_open maps a peer's handle (hgca_peer_close unmaps it). */
int hgca_peer_alloc(int64_t bytes, void** ptr, void* handle64);
int hgca_peer_open(const void* handle64, void** ptr);
int hgca_peer_close(void* ptr);
int hgca_peer_free(void* ptr);
/* In stream order: wait on the device until flags[i] >= epoch for all i < P
 * (acquire loads at system scope; the peers' merge kernels publish them), then
 * hgca_merge_packed over parts. A wait longer than timeout_ms stores 1 to *err
 * (device int32, optional) instead of hanging, and the merge then writes NaN
 * to out / lse rather than folding stale slots (check *err at a sync point). */
int hgca_merge_packed_wait(const void* parts, int64_t P, int64_t rows, int64_t d, int64_t stride_bytes,
                           const uint64_t* flags, uint64_t epoch, int64_t timeout_ms, int32_t* err, float* out,
                           double* lse, hgca_stream_t stream);
int hgca_merge_packed(const void* parts, int64_t P, int64_t rows, int64_t d, int64_t stride_bytes,
                      float* out, double* lse, hgca_stream_t stream);

/* ---- selection ----------------------------------------------------------
 * Bit masks are [rows, words] uint32, bit p of row r = position p. */
/* keep: optional [words] position mask (NULL = every position); under
 * sequence sharding it holds the archive blocks this rank owns. */
int hgca_select_threshold(const double* maw, int64_t rows, int64_t ld, int64_t p0, int64_t p1,
                          double beta, int64_t divisor, uint32_t* mask, int64_t words,
                          int assign, const uint32_t* keep, hgca_stream_t stream);
int hgca_mask_to_indices(const uint32_t* mask_a, const uint32_t* mask_b, int64_t rows,
                         int64_t words, int64_t n, int64_t* idx, int64_t ld, uint8_t* flags,
                         int64_t* counts, hgca_stream_t stream);
int hgca_popcount_rows(const uint32_t* mask, int64_t rows, int64_t words, int64_t n,
                       int64_t* counts, hgca_stream_t stream);
int hgca_group_need(const int64_t* counts, int64_t B, int64_t H, int64_t g, int64_t* need,
                    hgca_stream_t stream);
/* Per row, OR into out the top k[row] candidates of [0,n) not in exclude
 * (NULL = none) by (maw descending, position ascending). */
int hgca_select_topk(const double* maw, int64_t rows, int64_t ld, int64_t n, const int64_t* k,
                     const uint32_t* exclude, uint32_t* out, int64_t words, hgca_stream_t stream);

/* ---- device-resident decode engine --------------------------------------- */
/* KV[bh, pos+i] = (k_new[bh, i], v_new[bh, i]) for the interleaved position
 * buffer KV [BH, T, 2, d] (WindowCache.append_kv, kv_cache.py:122-169).
 * BF16 rows are stored position-rotated: 16-byte chunk c of the 2d-element
 * row pair of position p lands at chunk (c & ~7) | ((c ^ p) & 7). */
int hgca_write_rows(int dtype, void* KV, int64_t BH, int64_t T, int64_t d, int64_t pos,
                    const void* k_new, const void* v_new, int64_t n, hgca_stream_t stream);
int hgca_decode_chunk_rows(int dtype, int64_t d);
/* Launch configuration of the decode kernel for (dtype, head_dim, Hq/Hkv):
 * out5 = {warps per CTA, smem bytes per warp, cp.async stages, rows per
 * sub-chunk, smem bytes per CTA}. */
int hgca_decode_config(int dtype, int64_t d, int64_t group, int64_t* out5);
/* Work-item granularity of hgca_decode_step for a storage dtype: out2 =
 * {shortest item (32 rows, one pipeline stage: size the partial buffers for
 * dense items this short), longest item (the sparse_rows to pass to
 * hgca_union_build and the descriptor)}: float32 {32, 64}, bfloat16
 * {32, 256}. hgca_union_build_items with item_target > 0 picks the item size
 * per union between the two (long items for big steps: per-item q load,
 * partial write and merge fold; short ones so small steps reach every warp);
 * the decode kernel cuts the window into dense items of the same size. */
int hgca_item_rows(int dtype, int64_t* out2);
/* MAW maintenance from float32 weight rows w [BH, nq, w_ld] (row mean in fp64):
 * mode 0 = window EMA for j < w_old and init for j >= w_old (kv_cache.py:171-187,
 * engine.py:177-191); mode 1 = replace (StoreTier.reevaluate, sparsifier.py:158-177). */
int hgca_maw_update(const float* w, int64_t BH, int64_t nq, int64_t W, int64_t w_ld, double* maw,
                    int64_t T, int64_t p0, int64_t w_old, double alpha, int mode, hgca_stream_t stream);
/* WindowCache.update_maw (kv_cache.py:171-187): maw[r, j] = (1 - alpha) * maw[r, j]
 * + alpha * a[r, j] for j < n, three separately rounded fp64 ops (kv_cache.py:186). */
int hgca_maw_ema(double* maw, int64_t rows, int64_t ld, int64_t n, const double* a, int64_t lda, double alpha,
                 hgca_stream_t stream);
/* Union of the Hq/Hkv query heads' selection masks per (batch, kv-head) as
 * entries u_ent [B*Hkv, T] = position | (query-head mask << 24), grouped by
 * mask value (grouped = 1), in position order (0), or position-class
 * interleaved (2: position order, each aligned window of 32 entries permuted
 * to (rank within class p & 7, class) order so groups of 8 have distinct p & 7
 * where the window's classes allow; the bfloat16 decode layout), or grouped by
 * mask value and then class-interleaved per window (3: the float32 decode
 * layout); u_cnt [B*Hkv]; and
 * the sparse work items: each list is cut into items of sparse_rows entries
 * followed by tail items of sparse_rows/4 entries covering its last twelfth or
 * more (all full items first, then all tail items, so the step ends on small
 * items). item_off
 * [2, B*Hkv+1] holds the full-item and tail-item prefixes, item_tab
 * [items][4] = (bk, lo, hi, 0). */
int hgca_union_build(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                     int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                     int32_t* item_tab, int64_t sparse_rows, int grouped, hgca_stream_t stream);
/* The same with step-adaptive items: item rows = the largest power-of-two
 * fraction of max_rows, not below min_rows, that still cuts the whole union
 * into >= item_target items (chosen on the device from u_cnt and stored at
 * item_off[2*(B*Hkv+1)]; item_off needs 2*(B*Hkv+1)+1 entries). Big steps keep
 * long items (few partials), small steps give every decode warp work. Pass
 * the same item_target in the step descriptor (it sizes the partials check). */
int hgca_union_build_items(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                           int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                           int32_t* item_tab, int64_t max_rows, int64_t min_rows, int64_t item_target, int grouped,
                           hgca_stream_t stream);
/* The same counting the step's dense window (window_rows per (batch, kv
 * head), e.g. the window capacity) into the work the item size is chosen for:
 * the window parts share the item granularity, so a big window beside a small
 * union keeps long items. */
int hgca_union_build_items_w(const uint32_t* sel_mask, int64_t B, int64_t Hq, int64_t Hkv, int64_t words,
                             int64_t n_arch, int64_t T, int32_t* u_ent, int32_t* u_cnt, int32_t* item_off,
                             int32_t* item_tab, int64_t max_rows, int64_t min_rows, int64_t item_target,
                             int64_t window_rows, int grouped, hgca_stream_t stream);

typedef struct hgca_decode_desc {
  int32_t dtype;            /* HGCA_DTYPE_F32 or HGCA_DTYPE_BF16 (storage) */
  int32_t pad0;
  int64_t B, Hq, Hkv, D, T; /* batch, query heads, kv heads, head_dim, positions (T < 2^24) */
  const void* KV;           /* [B*Hkv, T, 2, D]: K row then V row per position */
  const void* q;            /* [B*Hq, D] this step's queries (storage dtype) */
  const void* k_new;        /* optional [B*Hkv, D] kv_in keys: written into KV at position dhi-1
                               by the kernel itself (else the caller stored them, hgca_write_rows) */
  const void* v_new;        /* optional [B*Hkv, D] kv_in values (with k_new) */
  double scale;
  int64_t dlo, dhi;         /* dense positions [dlo, dhi): window + kv_in */
  int64_t w_old;            /* window entries before this step (EMA'd) */
  int64_t sparse_rows;      /* rows per sparse work item (as in hgca_union_build) */
  const int32_t* u_ent;     /* union entries from hgca_union_build */
  const int32_t* u_cnt;
  const int32_t* item_off;
  const int32_t* item_tab;  /* [items][4] from hgca_union_build */
  void* dsc;                /* [B*Hq, dsc_ld] dense-score scratch: fp64 (F32) or fp32 (BF16), dsc_ld >= dhi-dlo */
  int64_t dsc_ld;
  double* part_m;           /* [G*max_items] head-major item partials */
  double* part_z;           /* [G*max_items] */
  float* part_acc;          /* [G*max_items*D] */
  int64_t max_items;        /* >= B*Hkv*(ceil(dsc_ld/32) + 2 + ceil(4T / sparse_rows)) (+ 5/3 item_target + 5*B*Hkv when adaptive) */
  int32_t* counter;         /* int32 work counter (>= 1 element): zero it once before the first step;
                               every step leaves it 0 again */
  double* maw;              /* [B*Hq, T] or NULL */
  double alpha;
  float* out;               /* [B*Hq, D] */
  double* lse;              /* [B*Hq] */
  float* wts_out;           /* optional [B*Hq, dhi-dlo] dense weights (a_gpu) */
  float* out_sparse;        /* optional sparse-only partial [B*Hq, D] */
  double* lse_sparse;       /* optional [B*Hq] */
  /* Sequence-sharded one-shot exchange; push_n = 0 disables.
   * The merge kernel stores this rank's packed partial -- out / lse
   * (push_sparse 0: the rank whose partial includes the window) or the
   * sparse-only out / lse (push_sparse 1) -- straight into each push_dst[p]
   * (f32 [B*Hq, D] then f64 [B*Hq], the hgca_merge_packed slot layout; peer
   * memory from hgca_peer_open, so the stores go over NVLink while the merge
   * runs), fences at system scope, and its last CTA publishes `epoch` to each
   * *push_flag[p] with a release store. push_cnt: a uint32 counter, zero
   * before the first step (every step leaves it 0). */
  int32_t push_n;
  int32_t push_sparse;
  void* push_dst[8];
  uint64_t* push_flag[8];
  uint64_t epoch;
  uint32_t* push_cnt;
  int64_t item_target;      /* item_target of hgca_union_build_items (0: fixed sparse_rows items) */
  /* Graph mode (optional, NULL = off): a device int64[4] step state
   * {dlo, dhi, epoch, 0} (hgca_step_state_set). When set, both kernels read
   * the window range [dlo, dhi) (and the push epoch) from it at run time --
   * dlo / dhi / w_old / epoch above are only validated (dhi - dlo <= dsc_ld)
   * -- and the merge kernel advances dhi and epoch by one after the step, so
   * one captured launch sequence (CUDA graph) replays step after step. The
   * caller re-sets the state when the window moves otherwise (eviction). */
  int64_t* state;
  /* Split merge (optional; merge_split <= 1 = off): long per-head item lists
   * are folded by merge_split CTAs per query head (contiguous shares of the
   * sparse items, the last share with the dense window items), whose partials
   * the last CTA to arrive combines in share order -- deterministic, and the
   * merge of a 128K-context step is spread over the GPU instead of one CTA per
   * head walking ~300 partials. merge_scratch: hgca_merge_scratch_bytes(B, Hq,
   * D, merge_split) bytes, zeroed once before the first step (every step
   * leaves its counters zero). */
  int64_t merge_split;
  void* merge_scratch;
} hgca_decode_desc;

/* Device scratch of the split merge (hgca_decode_desc.merge_split / merge_scratch). */
int64_t hgca_merge_scratch_bytes(int64_t B, int64_t Hq, int64_t D, int64_t split);

/* Graph mode: state[0..3] = {dlo, dhi, epoch, 0}, in stream order (one tiny
 * kernel, so it can be captured too). */
int hgca_step_state_set(int64_t* state, int64_t dlo, int64_t dhi, uint64_t epoch, hgca_stream_t stream);

/* One decode step = two kernels on `stream`: the decode kernel (dense items =
 * window parts of hgca_item_rows(dtype)[0] rows, sparse items = union slices
 * -> per-item (m, z, acc) partials, head-major; it also writes k_new/v_new)
 * and the merge kernel (one CTA per query head, programmatic dependent launch;
 * folds the partials in item order, applies merge_states, the window weights
 * and the MAW EMA, and with push_n > 0 pushes the rank's packed partial). */
int hgca_decode_step(const hgca_decode_desc* desc, hgca_stream_t stream);

/* Append / re-evaluation attention for BF16 storage on the tensor cores
 * (engine.py:111-132, 161-169; sparsifier.py:158-177): q [B*Hq, nq, D]
 * (nq <= 128) attends the archive [0, lo) and the window + kv_in [lo, hi) of
 * the position buffer KV (kv_in already written); out [B*Hq, nq, D] f32 and
 * lse [B*Hq, nq] f64 are merge_states(archive, window); mean_archive
 * [B*Hq, lo] and mean_window [B*Hq, hi-lo] (optional) receive, per query head
 * and position, the mean attention weight over the nq rows (a_cpu / a_gpu
 * row means). ws: hgca_append_ws_bytes(...) bytes of device scratch.
 * Kernels: D = 128 runs both passes on tcgen05 for every row group (TMEM
 * accumulators; groups of < 64 rows loaded 2 or 4 times into the 128-row tile
 * with the keys split between the copies; two 128-row groups per CTA when a kv
 * head has two; the mean-weight pass key-major); D = 64 uses mma.sync. Same
 * results contract either way. */
int64_t hgca_append_ws_bytes(int64_t B, int64_t Hq, int64_t Hkv, int64_t D, int64_t nq, int64_t lo, int64_t hi);
int hgca_append_bf16(const void* KV, int64_t B, int64_t Hq, int64_t Hkv, int64_t T, int64_t D, const void* q,
                     int64_t nq, double scale, int64_t lo, int64_t hi, float* out, double* lse, float* mean_archive,
                     float* mean_window, void* ws, int64_t ws_bytes, hgca_stream_t stream);

/* End-to-end step from HOST buffers (pinned): copy in_bytes of in_host to
 * in_dev (the caller points desc->q / k_new / v_new into in_dev), run the
 * step, deliver out_bytes of out_dev (desc->out / lse point into it) to
 * out_host, and synchronize the stream. One call per decode step. When
 * out_host is pinned and mapped (cudaHostGetDevicePointer succeeds, as for
 * cudaHostAlloc memory under UVA) the merge kernel writes out / lse straight to
 * their mirror offsets in out_host and no D2H copy is issued; otherwise
 * out_dev is copied back. */
int hgca_decode_step_host(const hgca_decode_desc* desc, const void* in_host, void* in_dev, int64_t in_bytes,
                          void* out_host, const void* out_dev, int64_t out_bytes, hgca_stream_t stream);

/* The same step without the final synchronization: everything is enqueued on
 * `stream` and out_host holds the result once the stream reaches this point
 * (the caller synchronizes), so host work for the next step -- bookkeeping,
 * the next descriptor -- can overlap this one. */
int hgca_decode_step_host_async(const hgca_decode_desc* desc, const void* in_host, void* in_dev, int64_t in_bytes,
                                void* out_host, const void* out_dev, int64_t out_bytes, hgca_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
