// K7 — GPU KV block pool: warp-parallel prefix-hash index + refcounted
// allocator with exact LRU-leaf eviction.
//
// Semantics are those of src/prefillsim/kvstore.py:59-250 (BlockPool),
// reproduced bit-exactly:
//   * the index is keyed by (namespace, parent block, token span)
//     (kvstore.py:69-70); only full blocks are indexed (:115, :148);
//   * longest_prefix_match pins the chain and stamps last_access=now, and
//     counts the whole query (tail included) into lookup_tokens (:123-138);
//   * insert protects the matched chain while evicting (:153-164), checks
//     need > capacity before touching anything (:197-200), keeps partial
//     evictions on failure (:194-196), gives new interior blocks a
//     provisional child_count of 1 and the new leaf 0 (:177, :184);
//   * eviction pops the unpinned leaf with the smallest (last_access,
//     block_id) one at a time; a parent whose last child goes becomes a
//     candidate immediately (:212-235). The lazy heap of the reference is
//     equivalent to "argmin over current unpinned leaves" because every
//     transition into candidacy pushes a fresh entry (:164, :185, :235,
//     :250) and stale entries are filtered on pop (:216-222).
//
// B200 design. State lives in HBM as structure-of-arrays record slots plus
// an open-addressing bucket array (linear probing, backward-shift deletion,
// so probes never see tombstones). Walks are parallel instead of
// pointer-chasing: the bucket key is a *path hash* H_k = mix(ns, sum_{i<=k}
// c_i) where c_i hashes block i's span and index, so all blocks of a query
// hash and probe independently after one CTA-wide prefix sum; the exact
// edge (ns, parent, span) is then verified in parallel (record span compare
// + parent == previous match). A 64-bit path-hash collision only reroutes to
// an exact sequential probe, never to a wrong answer. Each op is one CTA of
// 1024 threads and one launch; eviction keeps its candidate set (the
// current unpinned leaves) in shared memory and runs block-wide argmin pops.
#include "common.cuh"

#include <stdlib.h>
#include <string.h>

namespace psk {
namespace pool {

constexpr int kThreads = 1024;
constexpr int kMaxNs = 1024;
constexpr int32_t kEmpty = -1;
constexpr int kCandMax = 6144;  // candidates kept in smem (20 B each)
constexpr size_t kCandSmem = (size_t)kCandMax * (8 + 8 + 4);

struct State {
  int64_t free_top;  // free_stack[0:free_top) are free slots
  int64_t used;
  int64_t next_id;
  int64_t matched_tokens;
  int64_t lookup_tokens;
  int64_t eviction_count;
  int64_t footprint[kMaxNs];
  int64_t peak[kMaxNs];
};

struct Dev {
  int64_t* rec_id;
  int64_t* rec_parent_id;
  int32_t* rec_parent_slot;
  int32_t* rec_ns;
  int32_t* rec_ref;
  int32_t* rec_child;
  int64_t* rec_last;
  uint64_t* rec_hash;
  int64_t* rec_tokens;
  int32_t* buckets;
  int32_t* free_stack;
  State* st;
  int64_t records;
  uint64_t bucket_mask;
  int64_t capacity;
  int32_t bs;
};

struct OpIO {
  const int64_t* tokens;  // device
  int64_t n_tokens;
  int32_t ns;
  int64_t now;
  int32_t* found;    // scratch [max blocks]
  uint64_t* hashes;  // scratch [max blocks]
  int32_t* out_slots_host;  // mapped
  int64_t* out_ids_host;    // mapped
  int32_t* out_slots_dev;
  const int32_t* in_slots;  // device
  const int64_t* in_ids;    // device
  int64_t n_handles;
  psk_pool_result* res;     // mapped
};

// ---------------------------------------------------------------- hashing --

__device__ __forceinline__ uint64_t block_content_hash(const int64_t* toks, int bs, int64_t k) {
  uint64_t h = 0x8CB92BA72F3D8DD7ull ^ (uint64_t)(k + 1) * 0x9E3779B97F4A7C15ull;
  for (int j = 0; j < bs; ++j) h = mix64(h ^ ((uint64_t)toks[j] + (uint64_t)j * 0xD6E8FEB86659FD93ull));
  return h;
}

__device__ __forceinline__ uint64_t path_hash(uint64_t prefix_sum, int32_t ns) {
  return mix64(prefix_sum ^ ((uint64_t)(uint32_t)ns * 0xA0761D6478BD642Full + 0xE7037ED1A0B428DBull));
}

// CTA-wide inclusive scan of per-block contributions -> path hashes.
// Thread t owns the contiguous block range [t*per, (t+1)*per).
__device__ void compute_path_hashes(const Dev& d, const OpIO& io, int64_t nb, uint64_t* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t per = (nb + kThreads - 1) / kThreads;
  const int64_t b0 = (int64_t)tid * per;
  const int64_t b1 = min(b0 + per, nb);
  uint64_t local = 0;
  for (int64_t k = b0; k < b1; ++k) {
    uint64_t c = block_content_hash(io.tokens + k * d.bs, d.bs, k);
    io.hashes[k] = c;
    local += c;
  }
  // inclusive warp scan of thread totals
  uint64_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = s_warp[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    s_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint64_t run = (incl - local) + (warp > 0 ? s_warp[warp - 1] : 0ull);
  for (int64_t k = b0; k < b1; ++k) {
    run += io.hashes[k];
    io.hashes[k] = path_hash(run, io.ns);
  }
  __syncthreads();
}

__device__ __forceinline__ bool span_equal(const Dev& d, int32_t slot, const int64_t* q) {
  const int64_t* r = d.rec_tokens + (int64_t)slot * d.bs;
  for (int j = 0; j < d.bs; ++j)
    if (r[j] != q[j]) return false;
  return true;
}

// First record on block k's probe path whose (ns, path hash, span) match.
__device__ int32_t probe_block(const Dev& d, const OpIO& io, int64_t k) {
  const uint64_t h = io.hashes[k];
  const int64_t* q = io.tokens + k * d.bs;
  uint64_t b = h & d.bucket_mask;
  while (true) {
    int32_t s = d.buckets[b];
    if (s == kEmpty) return -1;
    if (d.rec_hash[s] == h && d.rec_ns[s] == io.ns && span_equal(d, s, q)) return s;
    b = (b + 1) & d.bucket_mask;
  }
}

// Exact edge probe (ns, parent, span) — the reference key itself.
__device__ int32_t probe_exact(const Dev& d, const OpIO& io, int64_t k, int32_t parent) {
  const uint64_t h = io.hashes[k];
  const int64_t* q = io.tokens + k * d.bs;
  uint64_t b = h & d.bucket_mask;
  while (true) {
    int32_t s = d.buckets[b];
    if (s == kEmpty) return -1;
    if (d.rec_hash[s] == h && d.rec_ns[s] == io.ns && d.rec_parent_slot[s] == parent &&
        span_equal(d, s, q))
      return s;
    b = (b + 1) & d.bucket_mask;
  }
}

// kvstore.py:109-121 (_walk). Returns the chain length; io.found[0:len) are
// the chain's record slots. No side effects on the pool.
__device__ int64_t walk(const Dev& d, const OpIO& io, uint64_t* s_warp, int64_t* s_chain) {
  const int64_t nb = io.n_tokens / d.bs;
  if (nb == 0) return 0;
  compute_path_hashes(d, io, nb, s_warp);
  for (int64_t k = threadIdx.x; k < nb; k += kThreads) io.found[k] = probe_block(d, io, k);
  if (threadIdx.x == 0) *s_chain = nb;
  __syncthreads();
  for (int64_t k = threadIdx.x; k < nb; k += kThreads) {
    int32_t f = io.found[k];
    int32_t want_parent = (k == 0) ? -1 : io.found[k - 1];
    bool ok = f >= 0 && d.rec_parent_slot[f] == want_parent;
    if (!ok) atomicMin((unsigned long long*)s_chain, (unsigned long long)k);
  }
  __syncthreads();
  int64_t chain = *s_chain;
  if (chain < nb && io.found[chain] >= 0) {
    // Path-hash collision with a foreign edge: finish the walk exactly.
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t k = chain;
      for (; k < nb; ++k) {
        int32_t parent = (k == 0) ? -1 : io.found[k - 1];
        int32_t s = probe_exact(d, io, k, parent);
        if (s < 0) break;
        io.found[k] = s;
      }
      *s_chain = k;
    }
    __syncthreads();
    chain = *s_chain;
  }
  __syncthreads();
  return chain;
}

// ------------------------------------------------------- bucket deletion --

__device__ void bucket_remove(const Dev& d, int32_t slot) {
  uint64_t i = d.rec_hash[slot] & d.bucket_mask;
  while (d.buckets[i] != slot) i = (i + 1) & d.bucket_mask;
  uint64_t j = i;
  while (true) {
    j = (j + 1) & d.bucket_mask;
    int32_t t = d.buckets[j];
    if (t == kEmpty) break;
    uint64_t home = d.rec_hash[t] & d.bucket_mask;
    bool stays = (i <= j) ? (i < home && home <= j) : (i < home || home <= j);
    if (stays) continue;
    d.buckets[i] = t;
    i = j;
  }
  d.buckets[i] = kEmpty;
}

__device__ void bucket_insert(const Dev& d, int32_t slot, uint64_t h) {
  uint64_t b = h & d.bucket_mask;
  while (atomicCAS(&d.buckets[b], kEmpty, slot) != kEmpty) b = (b + 1) & d.bucket_mask;
}

// ---------------------------------------------------------------- eviction --

struct Cand {
  int64_t* last;
  int64_t* id;
  int32_t* slot;
};

constexpr int64_t kRemoved = INT64_MAX;

// kvstore.py:191-235. Evicts unpinned leaves in (last_access, block_id) order
// until capacity - used >= need. Returns 0, or PSK_ECAPACITY if candidates ran
// out (evictions performed so far persist, as in the reference).
__device__ int evict_until_dev(const Dev& d, int64_t need, int64_t* s_used, int64_t* s_evicted,
                               unsigned char* smem_cand, Cand gcand) {
  __shared__ int s_ncand;
  __shared__ int64_t s_red_last[32];
  __shared__ int64_t s_red_id[32];
  __shared__ int s_red_idx[32];
  __shared__ int s_best;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (d.capacity - *s_used >= need) return PSK_OK;

  // Collect the current unpinned leaves.
  if (tid == 0) s_ncand = 0;
  __syncthreads();
  int64_t live_cands = 0;
  for (int64_t s = tid; s < d.records; s += kThreads)
    if (d.rec_id[s] >= 0 && d.rec_ref[s] == 0 && d.rec_child[s] == 0) ++live_cands;
  // count first to choose smem vs global storage
  __shared__ unsigned long long s_count;
  if (tid == 0) s_count = 0;
  __syncthreads();
  atomicAdd(&s_count, (unsigned long long)live_cands);
  __syncthreads();
  const bool use_smem = s_count <= (unsigned long long)kCandMax;
  Cand c;
  if (use_smem) {
    c.last = reinterpret_cast<int64_t*>(smem_cand);
    c.id = c.last + kCandMax;
    c.slot = reinterpret_cast<int32_t*>(c.id + kCandMax);
  } else {
    c = gcand;
  }
  for (int64_t s = tid; s < d.records; s += kThreads) {
    if (d.rec_id[s] >= 0 && d.rec_ref[s] == 0 && d.rec_child[s] == 0) {
      int i = atomicAdd(&s_ncand, 1);
      c.last[i] = d.rec_last[s];
      c.id[i] = d.rec_id[s];
      c.slot[i] = (int32_t)s;
    }
  }
  __syncthreads();
  const int ncand = s_ncand;

  while (d.capacity - *s_used < need) {
    // block-wide argmin over (last, id)
    int64_t bl = kRemoved, bi = kRemoved;
    int bidx = -1;
    for (int i = tid; i < ncand; i += kThreads) {
      int64_t l = c.last[i], id = c.id[i];
      if (id == kRemoved) continue;
      if (l < bl || (l == bl && id < bi)) { bl = l; bi = id; bidx = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      int64_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      int ox = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (ol < bl || (ol == bl && oi < bi)) { bl = ol; bi = oi; bidx = ox; }
    }
    if (lane == 0) { s_red_last[warp] = bl; s_red_id[warp] = bi; s_red_idx[warp] = bidx; }
    __syncthreads();
    if (warp == 0) {
      bl = s_red_last[lane]; bi = s_red_id[lane]; bidx = s_red_idx[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        int64_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        int ox = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ol < bl || (ol == bl && oi < bi)) { bl = ol; bi = oi; bidx = ox; }
      }
      if (lane == 0) {
        s_best = (bi == kRemoved) ? -1 : bidx;
        if (s_best >= 0) {
          // _evict (kvstore.py:225-235)
          int32_t s = c.slot[s_best];
          bucket_remove(d, s);
          int32_t ns = d.rec_ns[s];
          d.st->footprint[ns] -= d.bs;
          d.st->eviction_count += 1;
          *s_evicted += 1;
          *s_used -= 1;
          int32_t p = d.rec_parent_slot[s];
          d.rec_id[s] = -1;
          d.free_stack[d.st->free_top++] = s;
          c.id[s_best] = kRemoved;
          if (p >= 0) {
            int32_t ch = --d.rec_child[p];
            if (ch == 0 && d.rec_ref[p] == 0) {
              c.last[s_best] = d.rec_last[p];
              c.id[s_best] = d.rec_id[p];
              c.slot[s_best] = p;
            }
          }
        }
      }
    }
    __syncthreads();
    if (s_best < 0) return PSK_ECAPACITY;
  }
  return PSK_OK;
}

// ------------------------------------------------------------------ kernels --

__device__ void publish(const Dev& d, psk_pool_result* r, int64_t status, int64_t count,
                        int64_t first_id, int64_t evicted) {
  r->status = status;
  r->count = count;
  r->first_block_id = first_id;
  r->evicted = evicted;
  r->used_blocks = d.st->used;
  r->matched_tokens = d.st->matched_tokens;
  r->lookup_tokens = d.st->lookup_tokens;
  r->eviction_count = d.st->eviction_count;
  r->next_block_id = d.st->next_id;
  __threadfence_system();
}

__global__ void __launch_bounds__(kThreads, 1) lookup_kernel(Dev d, OpIO io, int pin) {
  __shared__ uint64_t s_warp[32];
  __shared__ int64_t s_chain;
  int64_t chain = walk(d, io, s_warp, &s_chain);
  for (int64_t k = threadIdx.x; k < chain; k += kThreads) {
    int32_t s = io.found[k];
    if (pin) {
      d.rec_ref[s] += 1;  // chain blocks are distinct: no atomics needed
      d.rec_last[s] = io.now;
    }
    io.out_slots_host[k] = s;
    io.out_ids_host[k] = d.rec_id[s];
    io.out_slots_dev[k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pin) {
      d.st->lookup_tokens += io.n_tokens;
      d.st->matched_tokens += chain * d.bs;
    }
    publish(d, io.res, PSK_OK, chain, -1, 0);
  }
}

__global__ void __launch_bounds__(kThreads, 1) insert_kernel(Dev d, OpIO io, Cand gcand) {
  extern __shared__ __align__(16) unsigned char smem_cand[];
  __shared__ uint64_t s_warp[32];
  __shared__ int64_t s_chain;
  __shared__ int64_t s_used, s_evicted;
  const int tid = threadIdx.x;
  const int64_t bs = d.bs;
  const int64_t n_full = io.n_tokens / bs;
  int64_t chain = walk(d, io, s_warp, &s_chain);
  const int64_t need = n_full - chain;
  if (need == 0) {
    if (tid == 0) publish(d, io.res, PSK_OK, 0, -1, 0);
    return;
  }
  if (tid == 0) { s_used = d.st->used; s_evicted = 0; }
  if (need > d.capacity) {  // kvstore.py:197-200, raised before any eviction
    if (tid == 0) publish(d, io.res, PSK_ECAPACITY_NEED, 0, -1, 0);
    return;
  }
  // Protect the matched chain (kvstore.py:153-156).
  for (int64_t k = tid; k < chain; k += kThreads) d.rec_ref[io.found[k]] += 1;
  __syncthreads();
  int st = evict_until_dev(d, need, &s_used, &s_evicted, smem_cand, gcand);
  __syncthreads();
  for (int64_t k = tid; k < chain; k += kThreads) d.rec_ref[io.found[k]] -= 1;
  if (st != PSK_OK) {
    __syncthreads();
    if (tid == 0) {
      d.st->used = s_used;
      publish(d, io.res, st, 0, -1, s_evicted);
    }
    return;
  }
  if (d.st->free_top < need) {  // physical record slots exhausted: host must reserve()
    __syncthreads();
    if (tid == 0) {
      d.st->used = s_used;
      publish(d, io.res, PSK_ENOMEM, 0, -1, s_evicted);
    }
    return;
  }
  // Allocate need blocks (kvstore.py:165-185).
  const int64_t top = d.st->free_top;
  const int64_t first_id = d.st->next_id;
  const int32_t root_parent = chain > 0 ? io.found[chain - 1] : -1;
  for (int64_t j = tid; j < need; j += kThreads) {
    int32_t s = d.free_stack[top - 1 - j];
    int32_t p = (j == 0) ? root_parent : d.free_stack[top - j];
    d.rec_id[s] = first_id + j;
    d.rec_parent_slot[s] = p;
    d.rec_parent_id[s] = (j == 0) ? (chain > 0 ? d.rec_id[root_parent] : -1) : first_id + j - 1;
    d.rec_ns[s] = io.ns;
    d.rec_ref[s] = 0;
    d.rec_child[s] = (j == need - 1) ? 0 : 1;
    d.rec_last[s] = io.now;
    uint64_t h = io.hashes[chain + j];
    d.rec_hash[s] = h;
    io.out_slots_host[j] = s;
    io.out_ids_host[j] = first_id + j;
    io.out_slots_dev[j] = s;
  }
  // span copy: thread per (block, token)
  for (int64_t e = tid; e < need * bs; e += kThreads) {
    int64_t j = e / bs, t = e % bs;
    int32_t s = d.free_stack[top - 1 - j];
    d.rec_tokens[(int64_t)s * bs + t] = io.tokens[(chain + j) * bs + t];
  }
  __syncthreads();
  for (int64_t j = tid; j < need; j += kThreads) {
    int32_t s = d.free_stack[top - 1 - j];
    bucket_insert(d, s, d.rec_hash[s]);
  }
  __syncthreads();
  if (tid == 0) {
    if (chain > 0) d.rec_child[root_parent] += 1;
    d.st->free_top = top - need;
    d.st->next_id = first_id + need;
    d.st->used = s_used + need;
    int64_t fp = d.st->footprint[io.ns] + need * bs;
    d.st->footprint[io.ns] = fp;
    if (fp > d.st->peak[io.ns]) d.st->peak[io.ns] = fp;
    publish(d, io.res, PSK_OK, need, first_id, s_evicted);
  }
}

__global__ void __launch_bounds__(kThreads, 1) evict_kernel(Dev d, int64_t need, psk_pool_result* res,
                                                            Cand gcand) {
  extern __shared__ __align__(16) unsigned char smem_cand[];
  __shared__ int64_t s_used, s_evicted;
  if (threadIdx.x == 0) { s_used = d.st->used; s_evicted = 0; }
  __syncthreads();
  int st = evict_until_dev(d, need, &s_used, &s_evicted, smem_cand, gcand);
  __syncthreads();
  if (threadIdx.x == 0) {
    d.st->used = s_used;
    publish(d, res, st, s_evicted, -1, s_evicted);
  }
}

// Handles must name live blocks (slot holds that block id).
__device__ bool handles_valid(const Dev& d, const OpIO& io, int* s_bad) {
  if (threadIdx.x == 0) *s_bad = -1;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < io.n_handles; i += kThreads) {
    int32_t s = io.in_slots[i];
    if (s < 0 || s >= d.records || d.rec_id[s] != io.in_ids[i]) atomicMax(s_bad, (int)i);
  }
  __syncthreads();
  return *s_bad < 0;
}

__global__ void __launch_bounds__(kThreads, 1) pin_kernel(Dev d, OpIO io) {
  __shared__ int s_bad;
  if (!handles_valid(d, io, &s_bad)) {
    if (threadIdx.x == 0) {
      io.res->err_index = s_bad;
      io.res->err_block_id = io.in_ids[s_bad];
      publish(d, io.res, PSK_EINVAL, 0, -1, 0);
    }
    return;
  }
  for (int64_t i = threadIdx.x; i < io.n_handles; i += kThreads) {
    int32_t s = io.in_slots[i];
    atomicAdd(&d.rec_ref[s], 1);
    d.rec_last[s] = io.now;
  }
  __syncthreads();
  if (threadIdx.x == 0) publish(d, io.res, PSK_OK, io.n_handles, -1, 0);
}

// kvstore.py:242-250. Underflow raises at the first offending element in list
// order, after the earlier elements were released; reproduced exactly by a
// sequential replay when the parallel pass detects any underflow.
__global__ void __launch_bounds__(kThreads, 1) release_kernel(Dev d, OpIO io) {
  __shared__ int s_bad;
  __shared__ int s_under;
  if (!handles_valid(d, io, &s_bad)) {
    if (threadIdx.x == 0) {
      io.res->err_index = s_bad;
      io.res->err_block_id = io.in_ids[s_bad];
      publish(d, io.res, PSK_EINVAL, 0, -1, 0);
    }
    return;
  }
  if (threadIdx.x == 0) s_under = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < io.n_handles; i += kThreads) {
    int old = atomicSub(&d.rec_ref[io.in_slots[i]], 1);
    if (old <= 0) s_under = 1;
  }
  __syncthreads();
  if (!s_under) {
    if (threadIdx.x == 0) publish(d, io.res, PSK_OK, io.n_handles, -1, 0);
    return;
  }
  for (int64_t i = threadIdx.x; i < io.n_handles; i += kThreads) atomicAdd(&d.rec_ref[io.in_slots[i]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t i = 0; i < io.n_handles; ++i) {
      int32_t s = io.in_slots[i];
      if (d.rec_ref[s] <= 0) {
        io.res->err_index = i;
        io.res->err_block_id = d.rec_id[s];
        publish(d, io.res, PSK_EUNDERFLOW, i, -1, 0);
        return;
      }
      d.rec_ref[s] -= 1;
    }
  }
}

__global__ void rebuild_kernel(Dev d) {
  // Clear buckets, then re-insert every live record (grid-stride).
  const int64_t nbuckets = (int64_t)d.bucket_mask + 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  (void)nbuckets;
  for (int64_t s = t0; s < d.records; s += stride)
    if (d.rec_id[s] >= 0) bucket_insert(d, (int32_t)s, d.rec_hash[s]);
}

__global__ void init_records_kernel(Dev d, int64_t from) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = from + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < d.records; s += stride) {
    d.rec_id[s] = -1;
    d.rec_ref[s] = 0;
    d.rec_child[s] = 0;
  }
}

}  // namespace pool
}  // namespace psk

using psk::pool::Dev;
using psk::pool::State;

struct psk_pool {
  int device;
  Dev d;
  int64_t max_q;
  // device scratch
  int64_t* d_tokens;
  int32_t* d_found;
  uint64_t* d_hashes;
  int32_t* d_out_slots;
  int32_t* d_in_slots;
  int64_t* d_in_ids;
  int64_t* d_cand_last;
  int64_t* d_cand_id;
  int32_t* d_cand_slot;
  // pinned host (mapped)
  int64_t* h_tokens;
  int32_t* h_in_slots;
  int64_t* h_in_ids;
  int32_t* h_out_slots;
  int64_t* h_out_ids;
  psk_pool_result* h_res;
  int32_t* m_out_slots;  // device aliases of the mapped buffers
  int64_t* m_out_ids;
  psk_pool_result* m_res;
};

namespace {

template <class T>
int dmalloc(T** p, int64_t n) {
  PSK_CUDA_TRY(cudaMalloc((void**)p, sizeof(T) * (size_t)(n > 0 ? n : 1)));
  return PSK_OK;
}

#define PSK_TRY(x)          \
  do {                      \
    int _r = (x);           \
    if (_r != PSK_OK) return _r; \
  } while (0)

uint64_t bucket_count_for(int64_t records) {
  uint64_t b = 1024;
  while (b < (uint64_t)records * 2) b <<= 1;
  return b;
}

int alloc_records(psk_pool* p, int64_t records) {
  Dev& d = p->d;
  PSK_TRY(dmalloc(&d.rec_id, records));
  PSK_TRY(dmalloc(&d.rec_parent_id, records));
  PSK_TRY(dmalloc(&d.rec_parent_slot, records));
  PSK_TRY(dmalloc(&d.rec_ns, records));
  PSK_TRY(dmalloc(&d.rec_ref, records));
  PSK_TRY(dmalloc(&d.rec_child, records));
  PSK_TRY(dmalloc(&d.rec_last, records));
  PSK_TRY(dmalloc(&d.rec_hash, records));
  PSK_TRY(dmalloc(&d.rec_tokens, records * d.bs));
  PSK_TRY(dmalloc(&d.free_stack, records));
  PSK_TRY(dmalloc(&p->d_cand_last, records));
  PSK_TRY(dmalloc(&p->d_cand_id, records));
  PSK_TRY(dmalloc(&p->d_cand_slot, records));
  uint64_t nb = bucket_count_for(records);
  PSK_TRY(dmalloc(&d.buckets, (int64_t)nb));
  PSK_CUDA_TRY(cudaMemset(d.buckets, 0xff, sizeof(int32_t) * nb));
  d.bucket_mask = nb - 1;
  d.records = records;
  return PSK_OK;
}

void free_records(Dev& d, psk_pool* p) {
  cudaFree(d.rec_id); cudaFree(d.rec_parent_id); cudaFree(d.rec_parent_slot);
  cudaFree(d.rec_ns); cudaFree(d.rec_ref); cudaFree(d.rec_child); cudaFree(d.rec_last);
  cudaFree(d.rec_hash); cudaFree(d.rec_tokens); cudaFree(d.free_stack); cudaFree(d.buckets);
  cudaFree(p->d_cand_last); cudaFree(p->d_cand_id); cudaFree(p->d_cand_slot);
}

psk::pool::OpIO make_io(psk_pool* p, int32_t ns, const int64_t* tokens, int64_t n, int64_t now) {
  psk::pool::OpIO io;
  io.tokens = tokens;
  io.n_tokens = n;
  io.ns = ns;
  io.now = now;
  io.found = p->d_found;
  io.hashes = p->d_hashes;
  io.out_slots_host = p->m_out_slots;
  io.out_ids_host = p->m_out_ids;
  io.out_slots_dev = p->d_out_slots;
  io.in_slots = p->d_in_slots;
  io.in_ids = p->d_in_ids;
  io.n_handles = 0;
  io.res = p->m_res;
  return io;
}

psk::pool::Cand gcand(psk_pool* p) {
  psk::pool::Cand c;
  c.last = p->d_cand_last;
  c.id = p->d_cand_id;
  c.slot = p->d_cand_slot;
  return c;
}

int finish(psk_pool* p, cudaStream_t s) {
  PSK_LAUNCH_CHECK();
  PSK_CUDA_TRY(cudaStreamSynchronize(s));
  return (int)p->h_res->status;
}

int stage_tokens(psk_pool* p, const int64_t* tokens_dev, int64_t n, cudaStream_t s,
                 const int64_t** out) {
  PSK_CHECK_ARG(n >= 0 && n <= p->max_q, "token count %lld exceeds staging (%lld)",
                (long long)n, (long long)p->max_q);
  if (tokens_dev) {
    *out = tokens_dev;
    return PSK_OK;
  }
  if (n > 0)
    PSK_CUDA_TRY(cudaMemcpyAsync(p->d_tokens, p->h_tokens, sizeof(int64_t) * n,
                                 cudaMemcpyHostToDevice, s));
  *out = p->d_tokens;
  return PSK_OK;
}

}  // namespace

extern "C" {

int psk_pool_create(psk_pool** out, int64_t capacity_blocks, int32_t block_size, int64_t records,
                    int64_t max_query_tokens, int device) {
  PSK_CHECK_ARG(out && capacity_blocks >= 0 && block_size >= 1 && records >= 1 &&
                    max_query_tokens >= 1 && records < (1ll << 31),
                "psk_pool_create: bad args");
  PSK_CUDA_TRY(cudaSetDevice(device));
  psk_pool* p = (psk_pool*)calloc(1, sizeof(psk_pool));
  p->device = device;
  p->d.capacity = capacity_blocks;
  p->d.bs = block_size;
  p->max_q = max_query_tokens;
  PSK_TRY(alloc_records(p, records));
  PSK_TRY(dmalloc(&p->d.st, 1));
  State st0;
  memset(&st0, 0, sizeof(st0));
  st0.free_top = records;
  PSK_CUDA_TRY(cudaMemcpy(p->d.st, &st0, sizeof(State), cudaMemcpyHostToDevice));
  // free stack: slot 0 is popped first (LIFO top = records-1 -> store reversed)
  int32_t* fs = (int32_t*)malloc(sizeof(int32_t) * records);
  for (int64_t i = 0; i < records; ++i) fs[i] = (int32_t)(records - 1 - i);
  PSK_CUDA_TRY(cudaMemcpy(p->d.free_stack, fs, sizeof(int32_t) * records, cudaMemcpyHostToDevice));
  free(fs);
  psk::pool::init_records_kernel<<<148, 256>>>(p->d, 0);
  PSK_LAUNCH_CHECK();
  const int64_t mq = max_query_tokens;
  PSK_TRY(dmalloc(&p->d_tokens, mq));
  PSK_TRY(dmalloc(&p->d_found, mq));
  PSK_TRY(dmalloc(&p->d_hashes, mq));
  PSK_TRY(dmalloc(&p->d_out_slots, mq));
  PSK_TRY(dmalloc(&p->d_in_slots, mq));
  PSK_TRY(dmalloc(&p->d_in_ids, mq));
  unsigned fl = cudaHostAllocMapped;
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_tokens, sizeof(int64_t) * mq, cudaHostAllocDefault));
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_in_slots, sizeof(int32_t) * mq, cudaHostAllocDefault));
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_in_ids, sizeof(int64_t) * mq, cudaHostAllocDefault));
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_out_slots, sizeof(int32_t) * mq, fl));
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_out_ids, sizeof(int64_t) * mq, fl));
  PSK_CUDA_TRY(cudaHostAlloc((void**)&p->h_res, sizeof(psk_pool_result), fl));
  memset(p->h_res, 0, sizeof(psk_pool_result));
  PSK_CUDA_TRY(cudaHostGetDevicePointer((void**)&p->m_out_slots, p->h_out_slots, 0));
  PSK_CUDA_TRY(cudaHostGetDevicePointer((void**)&p->m_out_ids, p->h_out_ids, 0));
  PSK_CUDA_TRY(cudaHostGetDevicePointer((void**)&p->m_res, p->h_res, 0));
  PSK_CUDA_TRY(cudaFuncSetAttribute(psk::pool::insert_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)psk::pool::kCandSmem));
  PSK_CUDA_TRY(cudaFuncSetAttribute(psk::pool::evict_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)psk::pool::kCandSmem));
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  *out = p;
  return PSK_OK;
}

int psk_pool_destroy(psk_pool* p) {
  if (!p) return PSK_OK;
  cudaSetDevice(p->device);
  free_records(p->d, p);
  cudaFree(p->d.st);
  cudaFree(p->d_tokens); cudaFree(p->d_found); cudaFree(p->d_hashes); cudaFree(p->d_out_slots);
  cudaFree(p->d_in_slots); cudaFree(p->d_in_ids);
  cudaFreeHost(p->h_tokens); cudaFreeHost(p->h_in_slots); cudaFreeHost(p->h_in_ids);
  cudaFreeHost(p->h_out_slots); cudaFreeHost(p->h_out_ids); cudaFreeHost(p->h_res);
  free(p);
  return PSK_OK;
}

int64_t psk_pool_records(const psk_pool* p) { return p ? p->d.records : 0; }

int psk_pool_reserve(psk_pool* p, int64_t records) {
  PSK_CHECK_ARG(p != nullptr && records < (1ll << 31), "psk_pool_reserve: bad args");
  if (records <= p->d.records) return PSK_OK;
  PSK_CUDA_TRY(cudaSetDevice(p->device));
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  Dev old = p->d;
  psk_pool tmp = *p;
  PSK_TRY(alloc_records(p, records));
  const int64_t n = old.records;
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_id, old.rec_id, 8 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_parent_id, old.rec_parent_id, 8 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_parent_slot, old.rec_parent_slot, 4 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_ns, old.rec_ns, 4 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_ref, old.rec_ref, 4 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_child, old.rec_child, 4 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_last, old.rec_last, 8 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_hash, old.rec_hash, 8 * n, cudaMemcpyDeviceToDevice));
  PSK_CUDA_TRY(cudaMemcpy(p->d.rec_tokens, old.rec_tokens, 8 * n * old.bs, cudaMemcpyDeviceToDevice));
  psk::pool::init_records_kernel<<<148, 256>>>(p->d, n);
  PSK_LAUNCH_CHECK();
  // free stack: old free slots keep their order at the bottom, new slots on
  // top so the lowest new slot is popped first.
  State st;
  PSK_CUDA_TRY(cudaMemcpy(&st, old.st, sizeof(State), cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(p->d.free_stack, old.free_stack, 4 * st.free_top, cudaMemcpyDeviceToDevice));
  const int64_t add = records - n;
  int32_t* fs = (int32_t*)malloc(sizeof(int32_t) * add);
  for (int64_t i = 0; i < add; ++i) fs[i] = (int32_t)(records - 1 - i);
  PSK_CUDA_TRY(cudaMemcpy(p->d.free_stack + st.free_top, fs, 4 * add, cudaMemcpyHostToDevice));
  free(fs);
  st.free_top += add;
  PSK_CUDA_TRY(cudaMemcpy(p->d.st, &st, sizeof(State), cudaMemcpyHostToDevice));
  psk::pool::rebuild_kernel<<<148, 256>>>(p->d);
  PSK_LAUNCH_CHECK();
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  free_records(old, &tmp);
  return PSK_OK;
}

int psk_pool_host_buffers(psk_pool* p, int64_t** tokens, int32_t** in_slots, int64_t** in_ids,
                          int32_t** out_slots, int64_t** out_ids, psk_pool_result** result) {
  PSK_CHECK_ARG(p != nullptr, "null pool");
  if (tokens) *tokens = p->h_tokens;
  if (in_slots) *in_slots = p->h_in_slots;
  if (in_ids) *in_ids = p->h_in_ids;
  if (out_slots) *out_slots = p->h_out_slots;
  if (out_ids) *out_ids = p->h_out_ids;
  if (result) *result = p->h_res;
  return PSK_OK;
}

int psk_pool_device_out_slots(psk_pool* p, int32_t** out) {
  PSK_CHECK_ARG(p && out, "null arg");
  *out = p->d_out_slots;
  return PSK_OK;
}

int psk_pool_lookup(psk_pool* p, int32_t ns, const int64_t* tokens_dev, int64_t n, int64_t now,
                    int32_t pin, void* stream) {
  PSK_CHECK_ARG(p && ns >= 0 && ns < psk::pool::kMaxNs, "psk_pool_lookup: bad args");
  cudaStream_t s = psk::as_stream(stream);
  const int64_t* toks;
  PSK_TRY(stage_tokens(p, tokens_dev, n, s, &toks));
  auto io = make_io(p, ns, toks, n, now);
  psk::pool::lookup_kernel<<<1, psk::pool::kThreads, 0, s>>>(p->d, io, pin);
  return finish(p, s);
}

int psk_pool_insert(psk_pool* p, int32_t ns, const int64_t* tokens_dev, int64_t n, int64_t now,
                    void* stream) {
  PSK_CHECK_ARG(p && ns >= 0 && ns < psk::pool::kMaxNs, "psk_pool_insert: bad args");
  cudaStream_t s = psk::as_stream(stream);
  const int64_t* toks;
  PSK_TRY(stage_tokens(p, tokens_dev, n, s, &toks));
  auto io = make_io(p, ns, toks, n, now);
  psk::pool::insert_kernel<<<1, psk::pool::kThreads, psk::pool::kCandSmem, s>>>(p->d, io, gcand(p));
  return finish(p, s);
}

int psk_pool_evict_until(psk_pool* p, int64_t need, void* stream) {
  PSK_CHECK_ARG(p != nullptr, "null pool");
  cudaStream_t s = psk::as_stream(stream);
  if (need > p->d.capacity) {
    p->h_res->status = PSK_ECAPACITY_NEED;
    p->h_res->count = 0;
    p->h_res->evicted = 0;
    return PSK_ECAPACITY_NEED;
  }
  psk::pool::evict_kernel<<<1, psk::pool::kThreads, psk::pool::kCandSmem, s>>>(p->d, need, p->m_res,
                                                                              gcand(p));
  return finish(p, s);
}

static int handle_op(psk_pool* p, int64_t n, int64_t now, void* stream, bool is_pin) {
  PSK_CHECK_ARG(p && n >= 0 && n <= p->max_q, "pin/release: bad handle count");
  cudaStream_t s = psk::as_stream(stream);
  if (n > 0) {
    PSK_CUDA_TRY(cudaMemcpyAsync(p->d_in_slots, p->h_in_slots, 4 * n, cudaMemcpyHostToDevice, s));
    PSK_CUDA_TRY(cudaMemcpyAsync(p->d_in_ids, p->h_in_ids, 8 * n, cudaMemcpyHostToDevice, s));
  }
  auto io = make_io(p, 0, nullptr, 0, now);
  io.n_handles = n;
  if (is_pin)
    psk::pool::pin_kernel<<<1, psk::pool::kThreads, 0, s>>>(p->d, io);
  else
    psk::pool::release_kernel<<<1, psk::pool::kThreads, 0, s>>>(p->d, io);
  return finish(p, s);
}

int psk_pool_pin(psk_pool* p, int64_t n, int64_t now, void* stream) {
  return handle_op(p, n, now, stream, true);
}

int psk_pool_release(psk_pool* p, int64_t n, void* stream) {
  return handle_op(p, n, 0, stream, false);
}

int psk_pool_footprint(psk_pool* p, int32_t ns, int64_t* footprint, int64_t* peak) {
  PSK_CHECK_ARG(p && ns >= 0 && ns < psk::pool::kMaxNs, "psk_pool_footprint: bad args");
  PSK_CUDA_TRY(cudaSetDevice(p->device));
  if (footprint)
    PSK_CUDA_TRY(cudaMemcpy(footprint, &p->d.st->footprint[ns], 8, cudaMemcpyDeviceToHost));
  if (peak) PSK_CUDA_TRY(cudaMemcpy(peak, &p->d.st->peak[ns], 8, cudaMemcpyDeviceToHost));
  return PSK_OK;
}

int psk_pool_snapshot(psk_pool* p, int64_t* block_id, int64_t* parent_id, int32_t* ns,
                      int32_t* ref_count, int32_t* child_count, int64_t* last_access,
                      int64_t* tokens) {
  PSK_CHECK_ARG(p != nullptr, "null pool");
  PSK_CUDA_TRY(cudaSetDevice(p->device));
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  const int64_t n = p->d.records;
  if (block_id) PSK_CUDA_TRY(cudaMemcpy(block_id, p->d.rec_id, 8 * n, cudaMemcpyDeviceToHost));
  if (parent_id) PSK_CUDA_TRY(cudaMemcpy(parent_id, p->d.rec_parent_id, 8 * n, cudaMemcpyDeviceToHost));
  if (ns) PSK_CUDA_TRY(cudaMemcpy(ns, p->d.rec_ns, 4 * n, cudaMemcpyDeviceToHost));
  if (ref_count) PSK_CUDA_TRY(cudaMemcpy(ref_count, p->d.rec_ref, 4 * n, cudaMemcpyDeviceToHost));
  if (child_count) PSK_CUDA_TRY(cudaMemcpy(child_count, p->d.rec_child, 4 * n, cudaMemcpyDeviceToHost));
  if (last_access) PSK_CUDA_TRY(cudaMemcpy(last_access, p->d.rec_last, 8 * n, cudaMemcpyDeviceToHost));
  if (tokens) PSK_CUDA_TRY(cudaMemcpy(tokens, p->d.rec_tokens, 8 * n * p->d.bs, cudaMemcpyDeviceToHost));
  return PSK_OK;
}

int psk_pool_read_record(psk_pool* p, int32_t slot, int64_t* fields, int64_t* tokens) {
  PSK_CHECK_ARG(p && fields && slot >= 0 && slot < p->d.records, "psk_pool_read_record: bad args");
  PSK_CUDA_TRY(cudaSetDevice(p->device));
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  int32_t i32[4];
  PSK_CUDA_TRY(cudaMemcpy(&fields[0], p->d.rec_id + slot, 8, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&fields[1], p->d.rec_parent_id + slot, 8, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&i32[0], p->d.rec_ns + slot, 4, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&i32[1], p->d.rec_ref + slot, 4, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&i32[2], p->d.rec_child + slot, 4, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&fields[5], p->d.rec_last + slot, 8, cudaMemcpyDeviceToHost));
  PSK_CUDA_TRY(cudaMemcpy(&i32[3], p->d.rec_parent_slot + slot, 4, cudaMemcpyDeviceToHost));
  fields[2] = i32[0];
  fields[3] = i32[1];
  fields[4] = i32[2];
  fields[6] = i32[3];
  if (tokens)
    PSK_CUDA_TRY(cudaMemcpy(tokens, p->d.rec_tokens + (int64_t)slot * p->d.bs, 8 * p->d.bs,
                            cudaMemcpyDeviceToHost));
  return PSK_OK;
}

}  // extern "C"
