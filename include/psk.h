/*
 * psk.h — C ABI of the PrefillShare B200 hot path (libpsk.so, sm_100a).
 *
 * Plain pointers and sizes only: no torch or C++ types cross this boundary.
 * Device pointers are caller-owned; `stream` is a cudaStream_t passed as
 * void*. Every function returns PSK_OK (0) or a negative PSK_E* code and
 * records a message retrievable with psk_last_error() (thread-local).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/pkg).
 */
#ifndef PSK_H_
#define PSK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define PSK_ABI_VERSION 1

#define PSK_OK 0
#define PSK_EINVAL (-1)        /* bad argument / stale block handle            */
#define PSK_ECUDA (-2)         /* CUDA runtime error                           */
#define PSK_ECAPACITY (-3)     /* kvstore.CapacityExhausted: all pinned        */
#define PSK_ECAPACITY_NEED (-4) /* kvstore.CapacityExhausted: need > capacity  */
#define PSK_EUNDERFLOW (-5)    /* kvstore.release underflow (RuntimeError)     */
#define PSK_ENOMEM (-6)        /* record table / staging too small; reserve()  */

int psk_abi_version(void);
const char* psk_last_error(void);
/* SM count of `device` (grid sizing is a multiple of it). */
int psk_sm_count(int device, int32_t* out);
/* SM budget for the persistent kernels' grids (0 = every SM). Lets a
 * serving loop run prefill kernels on a share of the SMs beside decode on
 * another stream; set before the launches (or graph capture) it applies to.
 * Process-wide, not per stream. No reference counterpart (a B200 serving knob). */
int psk_set_sm_budget(int32_t n);
int psk_get_sm_budget(int32_t* out);

/* ------------------------------------------------------------------------ *
 * Deterministic weight init (random-init models; no checkpoints).
 * dst[i] = bf16(std * N(0,1)) from a counter-based splitmix64 stream keyed
 * by (seed, i). Replaces frontend/src/model.ts:181-198 (TinyLM.init, seeded
 * Gaussian(0, 0.02)) for the Llama-shaped modules.
 * ------------------------------------------------------------------------ */
int psk_init_normal_bf16(void* dst, int64_t n, uint64_t seed, float std, void* stream);
int psk_fill_bf16(void* dst, int64_t n, float value, void* stream);

/* ------------------------------------------------------------------------ *
 * K7 — KV block pool: prefix-hash index + refcounted allocator on the GPU.
 * Replaces src/prefillsim/kvstore.py:59-250 (BlockPool) bit-exactly:
 * namespaced radix edges (ns, parent_id, token_span) (:69-70), walk (:109),
 * longest_prefix_match (:123), insert (:140), evict_until (:191),
 * LRU over unpinned leaves keyed (last_access, block_id) (:212-223),
 * pin / release (:237-250). Block ids are monotone and never reused; each
 * live block occupies one record slot, which doubles as its physical KV page
 * index when the pool backs KV memory.
 * ------------------------------------------------------------------------ */
typedef struct psk_pool psk_pool;

typedef struct psk_pool_result {
  int64_t status;          /* PSK_OK or error code of the op               */
  int64_t count;           /* matched blocks (lookup) / new blocks (insert) / evicted (evict) */
  int64_t first_block_id;  /* insert: id of the first new block            */
  int64_t evicted;         /* evictions performed by this op               */
  int64_t used_blocks;     /* live blocks after the op                     */
  int64_t matched_tokens;  /* cumulative (kvstore.py:74)                   */
  int64_t lookup_tokens;   /* cumulative (kvstore.py:75)                   */
  int64_t eviction_count;  /* cumulative (kvstore.py:76)                   */
  int64_t next_block_id;   /* kvstore.py:68                                */
  int64_t err_index;       /* release underflow: index into the list      */
  int64_t err_block_id;    /* release underflow: offending block id        */
  int64_t reserved[5];
} psk_pool_result;

/* capacity_blocks: logical capacity (kvstore.py:63); may be ~2^62 (unbounded).
 * records: record slots to allocate now (grow later with psk_pool_reserve).
 * max_query_tokens: size of the pinned token staging buffer. */
int psk_pool_create(psk_pool** out, int64_t capacity_blocks, int32_t block_size,
                    int64_t records, int64_t max_query_tokens, int device);
int psk_pool_destroy(psk_pool* pool);
/* Grow record slots (and the hash table) to at least `records`. */
int psk_pool_reserve(psk_pool* pool, int64_t records);
int64_t psk_pool_records(const psk_pool* pool);

/* Pinned host staging the caller fills before lookup/insert/pin/release:
 * tokens (int64[max_query_tokens]) and block handles (int32 slot + int64 id,
 * max_query_tokens entries each). Results of the last op land in *result,
 * the chain / new blocks in out_slots / out_ids (mapped host memory). */
int psk_pool_host_buffers(psk_pool* pool, int64_t** tokens, int32_t** in_slots,
                          int64_t** in_ids, int32_t** out_slots, int64_t** out_ids,
                          psk_pool_result** result);
/* Device mirrors of out_slots (the chain / new pages), for the engine. */
int psk_pool_device_out_slots(psk_pool* pool, int32_t** out_slots_dev);

/* kvstore.py:123-138. tokens: n_tokens ids in the staging buffer (or a
 * device pointer if tokens_dev != NULL). pin != 0: pin + last_access=now +
 * counters (longest_prefix_match); pin == 0: pure walk (kvstore.py:109). */
int psk_pool_lookup(psk_pool* pool, int32_t ns, const int64_t* tokens_dev,
                    int64_t n_tokens, int64_t now, int32_t pin, void* stream);
/* kvstore.py:140-189 (including evict_until :191-210 and the temporary
 * pin of the matched chain :153-164). */
int psk_pool_insert(psk_pool* pool, int32_t ns, const int64_t* tokens_dev,
                    int64_t n_tokens, int64_t now, void* stream);
/* kvstore.py:191-210 */
int psk_pool_evict_until(psk_pool* pool, int64_t need, void* stream);
/* kvstore.py:237-241 / 242-250, over n handles in the staging buffers. */
int psk_pool_pin(psk_pool* pool, int64_t n, int64_t now, void* stream);
int psk_pool_release(psk_pool* pool, int64_t n, void* stream);
/* Footprint / peak footprint tokens of namespace ns (kvstore.py:100-105). */
int psk_pool_footprint(psk_pool* pool, int32_t ns, int64_t* footprint, int64_t* peak);
/* Copy the record table to host arrays sized psk_pool_records() (block ids
 * -1 for free slots; tokens are records*block_size). Debug / parity only. */
int psk_pool_snapshot(psk_pool* pool, int64_t* block_id, int64_t* parent_id,
                      int32_t* ns, int32_t* ref_count, int32_t* child_count,
                      int64_t* last_access, int64_t* tokens);

/* One record: fields = {block_id, parent_id, ns, ref_count, child_count,
 * last_access, parent_slot}; tokens = its span (block_size ids). */
int psk_pool_read_record(psk_pool* pool, int32_t slot, int64_t* fields, int64_t* tokens);

/* ------------------------------------------------------------------------ *
 * Paged KV layout (shared by prefill, decode and transfer kernels).
 * One page holds `page_tokens` (=16 = kvstore block_size) consecutive
 * positions for ALL layers: page[layer][K|V][kv_head][token][head_dim] bf16,
 * so one page is one contiguous NVLink copy unit (2 MiB at the 8B shape) and
 * each (layer, K|V, head) tile is a contiguous 4 KiB run.
 * ------------------------------------------------------------------------ */
typedef struct psk_kv_layout {
  void* base;            /* bf16 [n_pages][page_elems]                      */
  int64_t page_elems;    /* n_layers * 2 * n_kv_heads * page_tokens * head_dim */
  int32_t n_layers;
  int32_t n_kv_heads;
  int32_t head_dim;      /* 128 */
  int32_t page_tokens;   /* 16  */
  int64_t n_pages;       /* pages in `base` (bounds TMA tensor maps)        */
} psk_kv_layout;

/* A batch of decode rows. Row r = (decode module row_mod[r], session
 * row_sess[r]); rows are grouped by module: module i owns rows
 * [mod_row_start[i], mod_row_start[i+1]). Session s shares its base-prefill
 * KV for positions [0, sess_len[s]) through sess_pages; row r's own KV
 * (positions sess_len + [0, priv_len[r])) lives in row_pages. All arrays are
 * device memory; the step kernels read lengths on the device so a whole
 * step can be captured in a CUDA graph. Mirrors the decode-module contract
 * of frontend/src/model.ts:363-399 (generate with an injected strict-prefix
 * cache; the module itself processes the last prompt token, :372-374 and
 * evaluate.ts:16-19). */
typedef struct psk_decode_batch {
  int32_t n_rows;
  int32_t n_sess;
  int32_t n_mod;
  int32_t max_rows_per_sess;   /* <= 16 (64 query heads per KV head tile)  */
  const int32_t* row_mod;      /* [n_rows] module index (0..n_mod)         */
  const int32_t* row_sess;     /* [n_rows]                                 */
  const int32_t* row_in_sess;  /* [n_rows] index of the row in its session */
  const int32_t* mod_row_start;/* [n_mod+1]                                */
  const int32_t* sess_rows;    /* [n_sess][max_rows_per_sess] row ids      */
  const int32_t* sess_nrows;   /* [n_sess]                                 */
  const int32_t* sess_len;     /* [n_sess] shared prefix tokens            */
  const int32_t* sess_pages;   /* [n_sess][max_sess_pages]                 */
  int32_t max_sess_pages;
  const int32_t* row_pages;    /* [n_rows][max_row_pages]                  */
  int32_t max_row_pages;
  int32_t* priv_len;           /* [n_rows] private tokens already written  */
  int32_t* tokens;             /* [n_rows] current input token             */
} psk_decode_batch;

/* h[r,:] = embed[row_mod[r]][tokens[r],:] (fp32 residual stream).
 * embed: device array of n_mod bf16 table pointers [vocab][d]. */
int psk_embed_rows(const psk_decode_batch* b, const void* const* embed, int32_t d,
                   float* h, void* stream);
/* out[r,:] = bf16(h[r,:] * rsqrt(mean(h^2)+eps) * gamma[mod(r)]) where
 * mod(r) = row_mod ? row_mod[r] : 0; gamma: device array of pointers. */
int psk_rmsnorm_rows(const float* h, int32_t n_rows, int32_t d, const void* const* gamma,
                     const int32_t* row_mod, float eps, void* out, void* stream);

/* Grouped weight-streaming GEMV (K5): for each module i and each of its
 * rows r, y[r, n] = sum_k x[r, k] * W_i[n, k]  (x bf16 [n_rows][K], W_i bf16
 * [N][K] row-major; K % 8 == 0, N % 16 == 0). Rows of module i are
 * [mod_row_start[i], mod_row_start[i+1]); max_rows_per_mod bounds any
 * module's row count (<= 32; 0 = use n_rows). Epilogues: */
#define PSK_EPI_STORE_BF16 0   /* out bf16 [n_rows][N]                          */
#define PSK_EPI_STORE_F32 1    /* out fp32 [n_rows][N]                          */
#define PSK_EPI_RESID_ADD 2    /* out fp32 [n_rows][N] += y (residual stream)   */
#define PSK_EPI_SILU_MUL 3     /* W rows interleaved [gate8|up8]...; out bf16 [n_rows][N/2] = silu(g)*u */
int psk_gemv(const void* x, int32_t n_rows, int32_t K, const void* const* W,
             const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod,
             int32_t N, int32_t epilogue, void* out, void* stream);

/* K5-TC: the same grouped GEMV on tcgen05 (M = 128 weight rows, N = rows of a
 * module padded to 16/32/64, accumulator in TMEM), for 9..64 rows per module.
 * W_host: HOST array of the n_mod (<= 16) weight pointers (TMA tensor maps
 * are encoded per call; capture the call in a CUDA graph). K % 64 == 0,
 * N % 128 == 0. The CTAs split the (128-row block, 64-column chunk) space
 * evenly (stream-K) and reduce split blocks in a fixed order through the
 * workspace. Replaces the same reference projections as psk_gemv. */
int psk_gemv_tc(const void* x, int32_t n_rows, int32_t K, const void* const* W_host,
                const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod,
                int32_t N, int32_t epilogue, void* out, void* workspace, void* stream);
/* K5-TC for the decode step's fused QKV projection of every row of `b`
 * (N = (n_q_heads + 2 n_kv_heads) * 128, unit = one head) with RoPE and the
 * KV append fused into the epilogue: q_rot bf16 [n_rows][nq][128] and the
 * rotated k / plain v of each row written into its private page at index
 * priv_len[r], exactly as psk_gemv_tc(PSK_EPI_STORE_F32) followed by
 * psk_rope_append (bit-identical). Same workspace as psk_gemv_tc. */
int psk_gemv_tc_qkv_rope(const void* x, int32_t K, const void* const* W_host, const psk_decode_batch* b,
                         int32_t max_rows_per_mod, int32_t n_q_heads, const float* rope, int32_t layer,
                         psk_kv_layout kv, void* q_rot, void* workspace, void* stream);
/* K5-TC residual projection with the next RMSNorm fused (o-proj -> MLP norm,
 * down-proj -> next layer's attention norm): h[r,:] += y, then
 * xn[r,:] = bf16(h[r,:] * rsqrt(mean(h[r,:]^2) + eps) * gamma[module]),
 * as psk_gemv_tc(PSK_EPI_RESID_ADD) followed by psk_rmsnorm_rows (sums of
 * squares in another order). When one CTA per 128-row unit fits the SMs
 * the units of a module meet at an in-kernel grid barrier; otherwise the
 * call runs those two kernels. Same workspace as psk_gemv_tc. */
int psk_gemv_tc_resid_norm(const void* x, int32_t n_rows, int32_t K, const void* const* W_host,
                           const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod, int32_t N,
                           float* h, const void* const* gamma, const int32_t* row_mod, float eps, void* xn,
                           void* workspace, void* stream);
/* Bytes of the psk_gemv_tc workspace (stream-K partials + flags); allocate
 * once ZEROED and reuse for every call on the stream (the kernel leaves the
 * flags zeroed). */
int psk_gemv_tc_workspace(int64_t* bytes);

/* RoPE (rotate-half, Llama) on q and k of the fused qkv rows (fp32
 * [n_rows][(nq+2*nkv)*hd]) at position sess_len[sess]+priv_len[r]; writes
 * q_rot bf16 [n_rows][nq][hd] and appends k,v (bf16) to the row's private
 * page at index priv_len[r]. rope: fp32 [max_pos][hd/2][2] (cos, sin). */
int psk_rope_append(const psk_decode_batch* b, const float* qkv, int32_t n_q_heads,
                    const float* rope, int32_t layer, psk_kv_layout kv, void* q_rot,
                    void* stream);

/* K6: shared-prefix paged decode attention for one layer. The page stream of
 * each (session, KV head) — the session's shared prompt pages followed by its
 * rows' private pages (incl. the token appended this step) — is cut into
 * `splits` slices; every page is streamed from HBM once per step (TMA) for
 * ALL of the session's decode rows (modules) and their GQA query heads; the
 * split partials merge by log-sum-exp in a second, PDL-overlapped kernel.
 * splits = 0 selects the stream-K schedule: all groups' pages laid end to
 * end and cut into one equal run per SM (segment partials merged through a
 * per-group CTA directory); it falls back to fixed splits that fit the same
 * workspace for > 32 query rows per KV head or > 64 sessions.
 * Above 32 query rows per KV head (fan-out) the tcgen05 kernel runs and, when
 * its CTAs fit one wave, merges the splits itself (no second kernel).
 * Launched with programmatic dependent launch: it may read the sessions'
 * shared prefix pages before waiting on the previous kernel of the stream
 * (only q and the private pages come from it), so those pages must be
 * complete when that kernel releases its dependents -- as in a decode step,
 * whose first kernel (psk_embed_rows) waits for all earlier work first.
 * PSK_ATTN_LATE=1 makes every read wait.
 * q_rot bf16 [n_rows][nq][hd] -> out bf16 [n_rows][nq][hd]. workspace: fp32,
 * psk_decode_attn_workspace() bytes (for the same `splits`); its first
 * 32 KiB are merge counters (generation << 16 | arrivals per (session, KV
 * head)) that must be zero before the first call (e.g. a zero-filled
 * allocation); every call leaves the arrival counts zero (generations
 * advance). */
int psk_decode_attn_workspace(const psk_decode_batch* b, int32_t n_kv_heads, int32_t splits,
                              int64_t* bytes);
/* How many kernels psk_decode_attn launches for this batch (1: the fan-out
 * kernel merging its own splits; 2: partial + merge; 0: no rows). */
int psk_decode_attn_kernels(const psk_decode_batch* b, int32_t n_q_heads, int32_t n_kv_heads, int32_t splits,
                            int32_t* n_kernels);
int psk_decode_attn(const psk_decode_batch* b, const void* q_rot, int32_t n_q_heads,
                    int32_t layer, psk_kv_layout kv, int32_t splits, void* workspace, void* out,
                    void* stream);
/* Diagnostics (no reference counterpart): with PSK_TRACE_RING=1 in the
 * environment every fan-out (tcgen05) launch stamps its CTAs' phases
 * (%globaltimer ns: entry, barriers, first TMA, last TMA, partial written,
 * group merged, exit) into the next slot of a 512-launch device ring of
 * ctas_stride x 8 stamps; this copies up to n_u64 values of the ring to host
 * (synchronizing the device; host may be NULL to query only) and reports
 * the launches recorded so far. */
int psk_decode_attn_trace_ring(uint64_t* host, int64_t n_u64, int32_t* launches, int32_t* ctas_stride);
/* Diagnostics: the same launch ring for the K5-TC GEMV (PSK_TRACE_RING=1;
 * 1024 launches of ctas_stride x 8 stamps: entry, setup done, first TMA,
 * PDL wait passed, last TMA, last MMA commit, epilogue done, exit); meta
 * (may be NULL) receives {N, grid} per slot (2 x 1024 ints). */
int psk_gemv_tc_trace_ring(uint64_t* host, int64_t n_u64, int32_t* meta, int32_t* launches,
                           int32_t* ctas_stride);

/* Greedy step end: tokens[r] = argmax(logits[r]) (first max, as tf.argMax /
 * torch.argmax), out_tokens[r*max_new + priv_len[r]] = it (if in range),
 * then priv_len[r] += 1 (the row's KV for this step was appended). */
int psk_argmax_advance(const psk_decode_batch* b, const float* logits, int32_t vocab,
                       int32_t* out_tokens, int32_t max_new, void* stream);
/* out[r] = argmax(logits[r, 0:vocab]) (first maximum) — greedy prediction of
 * evaluateSharing (frontend/src/evaluate.ts:36-42). */
int psk_argmax_rows(const float* logits, int32_t n_rows, int32_t vocab, int32_t* out, void* stream);

/* ------------------------------------------------------------------------ *
 * K1/K2 — prefill GEMMs on tcgen05 (TMA -> smem -> UMMA -> TMEM).
 * out = A[M,K] . B[N,K]^T with bf16 A/B (K-major), fp32 accumulation and a
 * fused epilogue (PSK_EPI_* above; ldo = output row stride in elements).
 * Replaces the q/k/v, o and MLP matmuls of frontend/src/model.ts:298-323.
 * N % 256 == 0, K % 64 == 0; any M (tail rows masked).
 * ------------------------------------------------------------------------ */
#define PSK_EPI_QKV_ROPE_KV 4  /* internal: see psk_gemm_qkv_rope_kv          */
/* Split-K workspace for the prefill GEMMs: when a GEMM's last wave of
 * 128x256 tiles would be at most half full, those tail tiles are split along
 * K and reduced in a fixed order through this buffer. Bind one ZEROED buffer
 * of psk_gemm_workspace() bytes per process (GEMMs on one stream at a time);
 * unbound (or NULL) = no split. */
int psk_gemm_workspace(int64_t* bytes);
int psk_gemm_bind_workspace(void* ws, int64_t bytes);
int psk_gemm(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epilogue,
             void* out, int64_t ldo, void* stream);
/* Fused QKV projection of T prompt tokens at positions pos0.. : RoPE on q
 * and k (rotate-half), q_rot bf16 [T][nq][128] out, k/v written straight into
 * the paged cache (page_table[pos/16]) — the base module's KV write
 * (buildBaseCache, model.ts:340-352; cache push model.ts:307-311). */
int psk_gemm_qkv_rope_kv(const void* A, const void* Wqkv, int32_t T, int32_t K, int32_t n_q_heads,
                         const float* rope, int32_t pos0, psk_kv_layout kv, int32_t layer,
                         const int32_t* page_table, void* q_out, void* stream);
/* Batched (varlen) form for several sequences' new tokens stacked in A
 * (partial prefills of many sessions in one forward):
 * row t sits at absolute position row_pos[t] and its k/v go to KV slot
 * row_slot[t] = page * 16 + token-in-page. */
int psk_gemm_qkv_rope_kv_rows(const void* A, const void* Wqkv, int32_t T, int32_t K, int32_t n_q_heads,
                              const float* rope, const int32_t* row_pos, const int32_t* row_slot,
                              psk_kv_layout kv, int32_t layer, void* q_out, void* stream);

/* K3 — causal prefill attention of T new positions [pos0, pos0+T) over the
 * paged cache (keys [0, pos0+T) through page_table; the new keys were
 * written by psk_gemm_qkv_rope_kv). q_rot bf16 [T][nq][128] -> out bf16
 * [T][nq*128]. frontend/src/model.ts:288-293, :312-315. */
int psk_prefill_attn(const void* q_rot, int32_t T, int32_t pos0, int32_t n_q_heads, psk_kv_layout kv,
                     int32_t layer, const int32_t* page_table, void* out, void* stream);
/* Batched K3 over stacked sequences: n_items work items, 8 int32 each
 * {token offset of the sequence in q_rot/out, its T, its pos0, offset of its
 * page table in `pages`, q-block (256 / GQA-group positions), 0, 0, 0}
 * (16-byte aligned), one CTA per (item, KV head); order items heaviest first. */
int psk_prefill_attn_batch(const void* q_rot, int32_t n_items, const int32_t* items, int32_t n_q_heads,
                           psk_kv_layout kv, int32_t layer, const int32_t* pages, void* out, void* stream);
/* h[t,:] = table[tokens[t],:] (fp32). model.ts:276-284 (token embedding). */
int psk_embed_tokens(const int64_t* tokens, int32_t T, const void* table, int32_t d, float* h,
                     void* stream);

/* K8 — copy whole KV pages src_base[src_pages[i]] -> dst_base[dst_pages[i]]
 * (page_bytes each; pools addressable from the launching device: same GPU
 * or a peer-mapped pool). Replaces the modelled handoff of
 * src/prefillsim/costs.py:66-83 for same-process moves; cross-process
 * handoffs use NCCL P2P of the same page units (paper_2602_12029_b200/
 * transfer.py). */
int psk_kv_copy_pages(const void* src_base, void* dst_base, const int32_t* src_pages,
                      const int32_t* dst_pages, int32_t n_pages, int64_t page_bytes, void* stream);

/* ------------------------------------------------------------------------ *
 * TinyLM — the reference's own model (frontend/src/model.ts:112-331) on the
 * GPU, fp32, over a paged prompt cache. Replaces TinyLM.forward(tokens,
 * past) (model.ts:246-331): `past_len` tokens already in the sequences'
 * pages (PromptCache, model.ts:41-88, as block tables: slice(n) is a shorter
 * table, so a decode module reads the base module's pages in place), n_new
 * tokens per sequence appended at positions past_len.. (their K/V written
 * into the pages the block table names; the caller gives a sequence a
 * private copy of a partially filled page before appending to it).
 * prev_first[b] = token before tokens[b][0] (the cache's last covered token;
 * -1 when the cache is empty), the prev-token channel of model.ts:262-270.
 * logits [batch][n_new][vocab] fp32. Pages: [page][layer][K|V][head][16][hd]
 * fp32. Errors as model.ts:249-258 (PSK_EINVAL: over-length, width not
 * divisible by heads). scratch: psk_tiny_scratch_floats floats.
 * ------------------------------------------------------------------------ */
typedef struct {
  int32_t layers, width, heads, context, vocab;
  const float* tok_emb;  /* [vocab][width] */
  const float* prev_emb; /* [vocab][width] */
  const float* pos_emb;  /* [context][width] */
  const float* lnf_g;
  const float* lnf_b;
  const float* head; /* [width][vocab] */
  /* device array of layers x 12 pointers (model.ts:147-169 order): ln1g ln1b
   * wq wk wv wo ([width][width], x @ W) ln2g ln2b wUp [width][4 width] bUp
   * wDown [4 width][width] bDown */
  const float* const* blocks;
} psk_tiny_model;
int psk_tiny_scratch_floats(const psk_tiny_model* m, int32_t batch, int32_t n_new, int64_t* out);
int psk_tiny_forward(const psk_tiny_model* m, int32_t batch, int32_t n_new, int32_t past_len,
                     const int32_t* tokens, const int32_t* prev_first, const int32_t* block_table,
                     int32_t max_pages, float* kv_pages, int64_t n_pages, float* scratch, float* logits,
                     void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* PSK_H_ */
