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

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* PSK_H_ */
