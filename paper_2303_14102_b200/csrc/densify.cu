// densify.cu -- K0: first-appearance dense cluster ids on the device.
//
// Replaces validate_and_densify's label remapping (dataset.cpp:41-51, 63-68):
// dense id = rank of a raw label's first row in dataset order.
//
// A global open-addressing table maps raw label -> first row.  Its keys and values
// carry the call's epoch in the high 32 bits (key = epoch:label, value =
// epoch:~row, merged with atomicMax), so a slot from an earlier call reads as empty
// and the table is never cleared between calls.
//   collect: each block dedups a contiguous row range in a shared-memory table and
//            merges (label, min row) into the global table (late blocks' rows lose
//            the max-merge without contention: the first rows come from early blocks)
//   finish : (single GPU, <= kSmallK labels) one block compacts the current-epoch
//            slots, ranks them by first row, writes the dense order and per-slot ids
//   map    : every row -> dense id through the table
// The sharded protocol instead orders the dictionary across ranks on the host
// (densify_collect + densify_assign_and_map).
#include <algorithm>
#include <vector>

#include "device_util.cuh"
#include "fsil_internal.cuh"

namespace fsil {
namespace {

constexpr int kSmemSlots = 1024;
constexpr int kMapSmemSlots = 8192;  // map: tables up to this many slots live in shared memory (96 KB)
constexpr int kSmallK = 2048;    // finish kernel: dictionary held in shared memory

__device__ __forceinline__ unsigned long long ekey(uint32_t epoch, int32_t lab) {
  return (static_cast<unsigned long long>(epoch) << 32) | static_cast<uint32_t>(lab);
}
__device__ __forceinline__ unsigned long long evalue(uint32_t epoch, uint32_t row) {
  return (static_cast<unsigned long long>(epoch) << 32) | (0xffffffffu - row);
}
__device__ __forceinline__ uint32_t value_row(unsigned long long v) {
  return 0xffffffffu - static_cast<uint32_t>(v);
}

__device__ bool global_insert(unsigned long long* keys, unsigned long long* vals, uint32_t mask,
                              uint32_t epoch, int32_t lab, uint32_t row) {
  const unsigned long long key = ekey(epoch, lab), val = evalue(epoch, row);
  uint32_t h = hash32(static_cast<uint32_t>(lab)) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    unsigned long long cur = keys[h];
    while (static_cast<uint32_t>(cur >> 32) != epoch) {  // stale slot: claim it
      const unsigned long long prev = atomicCAS(keys + h, cur, key);
      if (prev == cur) {
        cur = key;
        break;
      }
      cur = prev;
    }
    if (cur == key) {
      if (val > vals[h]) atomicMax(vals + h, val);  // stale values lose to any current one
      return true;
    }
    h = (h + 1) & mask;
  }
  return false;
}

// `coherent`: through L2 (a table written earlier in the same kernel)
template <bool coherent = false>
__device__ int64_t find_slot(const unsigned long long* keys, uint32_t mask, uint32_t epoch, int32_t lab) {
  const unsigned long long key = ekey(epoch, lab);
  uint32_t h = hash32(static_cast<uint32_t>(lab)) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    const unsigned long long cur = coherent ? __ldcg(keys + h) : keys[h];
    if (cur == key) return h;
    if (static_cast<uint32_t>(cur >> 32) != epoch) return -1;
    h = (h + 1) & mask;
  }
  return -1;
}

// Per-block shared-memory dedup of a contiguous row range.
__device__ __forceinline__ void collect_body(const int32_t* __restrict__ labels, int64_t n, int64_t chunk,
                                             unsigned long long* gkeys, unsigned long long* gvals, uint32_t mask,
                                             uint32_t epoch, int* overflow, int nslots) {
  // nslots (a power of two, dynamic shared memory): ~4x the expected label count, so the
  // bounded probe sequences rarely spill to the global table
  extern __shared__ __align__(8) unsigned long long skeys[];
  uint32_t* svals = reinterpret_cast<uint32_t*>(skeys + nslots);
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) {
    skeys[i] = 0;
    svals[i] = 0xffffffffu;
  }
  __syncthreads();
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  constexpr int U = 4;
  for (int64_t base = r0; base < r1; base += static_cast<int64_t>(blockDim.x) * U) {
    int32_t lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x + threadIdx.x;
      lab[u] = i < r1 ? __ldg(labels + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x + threadIdx.x;
      const bool valid = i < r1;
      if (!valid) continue;
      // every lane probes for itself: once a label sits in the block's table with a first row
      // below this one (always, after the chunk's first few rows) the lookup is two shared
      // loads and no atomic; lanes with equal labels read the same words (broadcast)
      const unsigned long long key = label_key(lab[u]);
      const uint32_t row = static_cast<uint32_t>(i);
      uint32_t h = hash32(static_cast<uint32_t>(lab[u])) & (nslots - 1);
      bool done = false;
      for (int probe = 0; probe < 16; ++probe) {  // bounded: overflow goes global
        unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(skeys + h);
        if (cur == 0) {
          const unsigned long long prev = atomicCAS(skeys + h, 0ull, key);
          cur = prev == 0 ? key : prev;
        }
        if (cur == key) {
          if (row < *reinterpret_cast<volatile uint32_t*>(svals + h)) atomicMin(svals + h, row);
          done = true;
          break;
        }
        h = (h + 1) & (nslots - 1);
      }
      if (!done && !global_insert(gkeys, gvals, mask, epoch, lab[u], row)) atomicExch(overflow, 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nslots; i += blockDim.x) {
    const unsigned long long key = skeys[i];
    if (key != 0 &&
        !global_insert(gkeys, gvals, mask, epoch, static_cast<int32_t>(static_cast<uint32_t>(key)), svals[i]))
      atomicExch(overflow, 1);
  }
}

__global__ void __launch_bounds__(256) densify_collect_kernel(const int32_t* __restrict__ labels, int64_t n,
                                                              int64_t chunk, unsigned long long* gkeys,
                                                              unsigned long long* gvals, uint32_t mask,
                                                              uint32_t epoch, int* overflow, int nslots) {
  griddep_wait();
  collect_body(labels, n, chunk, gkeys, gvals, mask, epoch, overflow, nslots);
}

// Single block: compact the current-epoch slots, rank by first row, write the dense
// order (sorted_labels) and the per-slot dense id.  More than kSmallK labels: flag
// counters[1] and leave the ordering to the multi-block kernels.
__device__ __forceinline__ void finish_body(const unsigned long long* keys, const unsigned long long* vals,
                                            uint32_t cap, uint32_t epoch, int32_t* sorted_labels, int32_t* slot_dense,
                                            int* counters, HostSummary* hsum, int32_t k_spec, bool spec_big) {
  __shared__ int32_t s_lab[kSmallK];
  __shared__ uint32_t s_row[kSmallK];
  __shared__ uint32_t s_slot[kSmallK];
  __shared__ int s_count;
  if (threadIdx.x == 0) s_count = 0;
  __syncthreads();
  constexpr int B = 8;  // slots in flight per thread
  for (uint32_t i0 = 0; i0 < cap; i0 += B * blockDim.x) {
    unsigned long long kk[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
      kk[u] = i < cap ? __ldcg(keys + i) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const uint32_t i = i0 + u * blockDim.x + threadIdx.x;
      if (i >= cap || static_cast<uint32_t>(kk[u] >> 32) != epoch) continue;
      const int j = atomicAdd(&s_count, 1);
      if (j < kSmallK) {
        s_lab[j] = static_cast<int32_t>(static_cast<uint32_t>(kk[u]));
        s_row[j] = value_row(__ldcg(vals + i));
        s_slot[j] = i;
      }
    }
  }
  __syncthreads();
  const int cnt = s_count;
  if (cnt <= kSmallK) {
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t my = s_row[i];
      int rank = 0;
      for (int j = 0; j < cnt; ++j) rank += s_row[j] < my;  // first rows are distinct
      sorted_labels[rank] = s_lab[i];
      slot_dense[s_slot[i]] = rank;
    }
  }
  if (threadIdx.x == 0) {
    counters[1] = cnt > kSmallK ? 1 : 0;  // needs the multi-block ordering
    // speculated K (k_spec > 0): raise the miss flag the scoring kernels check at entry
    const int over = __ldcg(counters);  // raised by any block (atomics)
    if (k_spec > 0 && (cnt != k_spec || over != 0 || (cnt > kSmallK && !spec_big))) counters[kAbortWord] = 1;
    *reinterpret_cast<unsigned long long*>(counters + 2) = static_cast<unsigned long long>(cnt);
    if (hsum) {
      hsum->overflow = over;
      hsum->count = cnt;
      hsum->pad = counters[1];
    }
  }
}

__global__ void __launch_bounds__(1024) densify_finish_kernel(const unsigned long long* __restrict__ keys,
                                                              const unsigned long long* __restrict__ vals,
                                                              uint32_t cap, uint32_t epoch, int32_t* sorted_labels,
                                                              int32_t* slot_dense, int* counters, HostSummary* hsum,
                                                              int32_t k_spec = 0, bool spec_big = false) {
  griddep_wait();
  finish_body(keys, vals, cap, epoch, sorted_labels, slot_dense, counters, hsum, k_spec, spec_big);
}

// Row -> dense id through the global table (per-slot dense ids; L1/L2 resident).
template <bool coherent = false>
__device__ __forceinline__ void map_body(const int32_t* __restrict__ labels, int64_t n,
                                         const unsigned long long* gkeys, const int32_t* slot_dense, uint32_t mask,
                                         uint32_t epoch, int32_t k_lim, int32_t* dense, int* missing) {
  // k_lim: the K the following kernels are launched for (the speculated K, or INT_MAX when
  // the host waits for the count).  An id outside [0, k_lim) -- only possible when the
  // speculation misses -- is stored as 0 and flagged, so every later kernel stays in bounds.
  // Tables of <= kMapSmemSlots slots are copied to shared memory first (every lookup then
  // probes shared memory); U rows per thread are looked up independently.
  extern __shared__ __align__(8) unsigned long long tkeys[];
  const bool local = mask + 1 <= static_cast<uint32_t>(kMapSmemSlots);
  int32_t* tdense = reinterpret_cast<int32_t*>(tkeys + (mask + 1));
  if (local) {
    for (uint32_t i = threadIdx.x; i <= mask; i += blockDim.x) {
      const unsigned long long key = coherent ? __ldcg(gkeys + i) : gkeys[i];
      tkeys[i] = key;
      if (static_cast<uint32_t>(key >> 32) == epoch) tdense[i] = coherent ? __ldcg(slot_dense + i) : slot_dense[i];
    }
    __syncthreads();
  }
  constexpr int U = 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    int32_t lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      lab[u] = i < n ? __ldg(labels + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) break;
      int32_t dj;
      if (local) {
        const int64_t slot = find_slot<false>(tkeys, mask, epoch, lab[u]);
        dj = slot >= 0 ? tdense[slot] : -1;
      } else {
        const int64_t slot = find_slot<coherent>(gkeys, mask, epoch, lab[u]);
        dj = slot >= 0 ? (coherent ? __ldcg(slot_dense + slot) : slot_dense[slot]) : -1;
      }
      if (dj < 0 || dj >= k_lim) {
        atomicExch(missing, 1);
        dj = 0;
      }
      dense[i] = dj;
    }
  }
}

__global__ void __launch_bounds__(256) densify_map_kernel(const int32_t* __restrict__ labels, int64_t n,
                                                          const unsigned long long* __restrict__ gkeys,
                                                          const int32_t* __restrict__ slot_dense, uint32_t mask,
                                                          uint32_t epoch, int32_t k_lim, int32_t* dense,
                                                          int* missing) {
  griddep_wait();
  map_body(labels, n, gkeys, slot_dense, mask, epoch, k_lim, dense, missing);
}


__global__ void densify_compact_kernel(const unsigned long long* __restrict__ keys,
                                       const unsigned long long* __restrict__ vals, uint32_t cap, uint32_t epoch,
                                       int64_t row_offset, int32_t* out_labels, int64_t* out_rows,
                                       int32_t* out_slot, unsigned long long* count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  const unsigned long long key = keys[i];
  if (static_cast<uint32_t>(key >> 32) != epoch) return;
  const unsigned long long j = atomicAdd(count, 1ull);
  out_labels[j] = static_cast<int32_t>(static_cast<uint32_t>(key));
  out_rows[j] = row_offset + static_cast<int64_t>(value_row(vals[i]));
  if (out_slot) out_slot[j] = static_cast<int32_t>(i);
}

// Multi-block ordering (K > kSmallK): dense id = rank of the entry's first row.
__global__ void __launch_bounds__(256) densify_rank_kernel(const int32_t* __restrict__ labels,
                                                           const int64_t* __restrict__ rows,
                                                           const int32_t* __restrict__ slots,
                                                           const unsigned long long* count,
                                                           int32_t* sorted_labels, int32_t* slot_dense) {
  __shared__ int64_t tile[1024];
  const int64_t cnt = static_cast<int64_t>(*count);
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= cnt) return;  // block-uniform
  const int64_t my = i < cnt ? rows[i] : INT64_MAX;
  int64_t rank = 0;
  for (int64_t b = 0; b < cnt; b += 1024) {
    __syncthreads();
    for (int t = threadIdx.x; t < 1024; t += blockDim.x) tile[t] = b + t < cnt ? rows[b + t] : INT64_MAX;
    __syncthreads();
    const int lim = static_cast<int>(cnt - b < 1024 ? cnt - b : 1024);
    for (int t = 0; t < lim; ++t) rank += tile[t] < my;
  }
  if (i < cnt) {
    sorted_labels[rank] = labels[i];
    slot_dense[slots[i]] = static_cast<int32_t>(rank);
  }
}

// Sharded protocol: dense id j for the j-th label of the globally ordered dictionary.
__global__ void densify_assign_kernel(const unsigned long long* __restrict__ keys, uint32_t mask, uint32_t epoch,
                                      const int32_t* __restrict__ raw, int32_t k, int32_t* slot_dense) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t slot = find_slot(keys, mask, epoch, raw[j]);
  if (slot >= 0) slot_dense[slot] = j;
}

// Device-side dictionary exchange (sharded protocol without host round trips).
// Local entries -> a fixed-capacity buffer of (label, first global row) int64 pairs,
// unused entries row = -1; the last entry carries row = -2 if this rank's labels did
// not fit (every rank then fails the merge the same way).
__global__ void densify_xcompact_kernel(const unsigned long long* __restrict__ keys,
                                        const unsigned long long* __restrict__ vals, uint32_t cap, uint32_t epoch,
                                        int64_t row_offset, int64_t* xbuf, int64_t cap_x, unsigned long long* count,
                                        const int* overflow) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && *overflow) {  // local table overflow: poison the exchange
    xbuf[2 * (cap_x - 1)] = 0;
    xbuf[2 * (cap_x - 1) + 1] = -2;
  }
  if (i >= cap) return;
  const unsigned long long key = keys[i];
  if (static_cast<uint32_t>(key >> 32) != epoch) return;
  const unsigned long long j = atomicAdd(count, 1ull);
  if (static_cast<int64_t>(j) >= cap_x - 1) {  // the last slot is the header
    xbuf[2 * (cap_x - 1)] = 0;
    xbuf[2 * (cap_x - 1) + 1] = -2;
    return;
  }
  xbuf[2 * j] = static_cast<int32_t>(static_cast<uint32_t>(key));
  xbuf[2 * j + 1] = row_offset + static_cast<int64_t>(value_row(vals[i]));
}

// Every rank's gathered entries -> one table (label -> min first global row).
__global__ void densify_xinsert_kernel(const int64_t* __restrict__ gathered, int64_t total,
                                       unsigned long long* keys, unsigned long long* vals, uint32_t mask,
                                       uint32_t epoch, int* overflow) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t row = gathered[2 * e + 1];
  if (row == -2) atomicExch(overflow, 1);
  if (row < 0) return;
  if (row >= 0xffffffffll || !global_insert(keys, vals, mask, epoch, static_cast<int32_t>(gathered[2 * e]),
                                             static_cast<uint32_t>(row)))
    atomicExch(overflow, 1);
}

int grid_for(int64_t n, int threads, int num_sms, int per_sm) {
  const int64_t want = (n + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(num_sms) * per_sm)));
}

// Table of `cap` slots for this call: a new epoch; (re)allocation zeroes it once.
uint32_t prepare_table(fsil_context* c, int64_t cap) {
  c->counters.ensure(64);
  if (cap != c->ht_alloc_cap || c->ht_epoch == 0xffffffffu) {
    c->ht_keys.ensure(cap * sizeof(unsigned long long));
    c->ht_vals.ensure(cap * sizeof(unsigned long long));
    c->ht_dense.ensure(cap * sizeof(int32_t));
    FSIL_CUDA(cudaMemsetAsync(c->ht_keys.p, 0, cap * sizeof(unsigned long long), c->stream));
    FSIL_CUDA(cudaMemsetAsync(c->ht_vals.p, 0, cap * sizeof(unsigned long long), c->stream));
    c->ht_alloc_cap = cap;
    c->ht_epoch = 0;
  }
  FSIL_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));
  return ++c->ht_epoch;
}

void launch_collect(fsil_context* c, int64_t cap, uint32_t epoch) {
  if (c->n == 0) return;
  const int grid = grid_for(c->n, 1024, c->num_sms, 4);
  const int64_t chunk = (c->n + grid - 1) / grid;
  // shared-memory dedup slots: ~4x the previous call's label count (1024 .. 4096)
  int nslots = kSmemSlots;
  while (nslots < 4096 && nslots < 4 * c->k_last) nslots <<= 1;
  const size_t smem = static_cast<size_t>(nslots) * (sizeof(unsigned long long) + sizeof(uint32_t));
  static bool attr = false;
  if (!attr) {
    FSIL_CUDA(cudaFuncSetAttribute(densify_collect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * 12));
    attr = true;
  }
  launch_pdl(c, densify_collect_kernel, grid, 256, smem, c->labels, c->n, chunk, c->ht_keys.as<unsigned long long>(),
             c->ht_vals.as<unsigned long long>(), static_cast<uint32_t>(cap - 1), epoch, c->counters.as<int>(), nslots);
}

// The map launch: a table of <= kMapSmemSlots slots is staged in shared memory by every
// block, so the grid is persistent (two blocks per SM) to keep those copies few.
template <typename... Args>
void launch_map(fsil_context* c, bool pdl, int64_t cap, Args... args) {
  const bool local = cap <= kMapSmemSlots;
  const size_t smem = local ? static_cast<size_t>(cap) * (sizeof(unsigned long long) + sizeof(int32_t)) : 0;
  static bool attr = false;
  if (!attr) {
    FSIL_CUDA(cudaFuncSetAttribute(densify_map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kMapSmemSlots * 12));
    attr = true;
  }
  int grid = grid_for(c->n, 256, c->num_sms, 8);
  if (local) grid = std::min(grid, 2 * c->num_sms);
  if (pdl) {
    launch_pdl(c, densify_map_kernel, grid, 256, smem, args...);
  } else {
    densify_map_kernel<<<grid, 256, smem, c->stream>>>(args...);
    FSIL_LAUNCHED(c);
  }
}

}  // namespace

// Sharded protocol, pass 1: local (label, first global row) dictionary.
void densify_collect(fsil_context* c) {
  if (c->n >= (int64_t(1) << 32) - 1)
    fail(FSIL_ERR_INVALID_ARGUMENT, "shard too large: a rank holds at most 2^32-2 rows");
  int64_t cap = std::max<int64_t>(c->ht_cap, 8192);
  for (;;) {
    const uint32_t epoch = prepare_table(c, cap);
    launch_collect(c, cap, epoch);
    int h_over = 0;
    FSIL_CUDA(cudaMemcpyAsync(&h_over, c->counters.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    if (h_over) {
      cap *= 4;
      continue;
    }
    c->ht_cap = cap;
    c->dict_labels.ensure(cap * sizeof(int32_t));
    c->dict_rows.ensure(cap * sizeof(int64_t));
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
    densify_compact_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->ht_keys.as<unsigned long long>(), c->ht_vals.as<unsigned long long>(), static_cast<uint32_t>(cap), epoch,
        c->row_offset, c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), nullptr, count);
    FSIL_LAUNCHED(c);
    unsigned long long h_count = 0;
    FSIL_CUDA(cudaMemcpyAsync(&h_count, count, sizeof(h_count), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    c->n_distinct = static_cast<int64_t>(h_count);
    if (c->n_distinct * 2 > cap) c->ht_cap = cap * 2;  // keep probes short next call
    return;
  }
}

// Single GPU: collect -> finish (one block) -> map, one host sync (K decides the
// kernels that follow); many labels take the multi-block ordering instead.
void densify_local(fsil_context* c) {
  if (c->n >= (int64_t(1) << 31) - 1)
    fail(FSIL_ERR_INVALID_ARGUMENT, "too many rows for one device call (2^31-2)");
  int64_t cap = std::max<int64_t>(c->ht_cap, 8192);
  bool big = c->k_last > kSmallK;  // the previous call's K predicts the ordering path
  // Speculation: launch everything after the dictionary for the previous call's K instead
  // of waiting for this call's count; finish() checks the count (one host sync per call)
  // and the call is redone without speculation when it differs.
  const bool spec = c->speculate && !c->spec_block_once && c->k_last >= 2;
  c->spec_block_once = false;
  // A small speculated dictionary gets a 1024-slot table (12 KB): every map block stages the
  // table in shared memory and finish scans all of it, so its size is most of their cost when
  // N is small (C1, C2).  More labels than expected: the speculation misses and the repeat
  // takes the full-size table.
  if (spec && c->k_last <= 256) cap = 1024;
  for (;;) {
    const uint32_t epoch = prepare_table(c, cap);
    c->dict_sorted.ensure(cap * (2 * sizeof(int32_t)));
    c->dense.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
    int32_t* sorted_labels = reinterpret_cast<int32_t*>(c->dict_sorted.p) + cap;
    int* counters = c->counters.as<int>();
    const uint32_t mask = static_cast<uint32_t>(cap - 1);
    launch_collect(c, cap, epoch);
    launch_pdl(c, densify_finish_kernel, 1, 1024, 0, c->ht_keys.as<unsigned long long>(),
               c->ht_vals.as<unsigned long long>(), static_cast<uint32_t>(cap), epoch, sorted_labels,
               c->ht_dense.as<int32_t>(), counters, c->dsum, spec ? static_cast<int32_t>(c->k_last) : 0, big);
    if (big) {
      c->dict_labels.ensure(cap * sizeof(int32_t));
      c->dict_rows.ensure(cap * sizeof(int64_t));
      int32_t* slots = reinterpret_cast<int32_t*>(c->dict_sorted.p);
      unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
      FSIL_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), c->stream));
      densify_compact_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
          c->ht_keys.as<unsigned long long>(), c->ht_vals.as<unsigned long long>(), static_cast<uint32_t>(cap), epoch,
          0, c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), slots, count);
      FSIL_LAUNCHED(c);
      densify_rank_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
          c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), slots, count, sorted_labels,
          c->ht_dense.as<int32_t>());
      FSIL_LAUNCHED(c);
    }
    if (c->n > 0) {
      launch_map(c, true, cap, c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_dense.as<int32_t>(), mask,
                 epoch, spec ? static_cast<int32_t>(c->k_last) : INT32_MAX, c->dense.as<int32_t>(), counters + 4);
    }
    if (spec) {
      c->k_spec = true;
      c->spec_big = big;
      c->n_distinct = c->k_last;
      c->k = static_cast<int32_t>(c->k_last);
      c->dict_sorted_labels = sorted_labels;
      return;
    }
    FSIL_CUDA(cudaStreamSynchronize(c->stream));  // K decides the kernels
    const volatile HostSummary* hs = c->hsum;
    const int64_t over = hs->overflow, cnt = hs->count;
    const bool needs_big = hs->pad != 0;
    if (over) {
      cap *= 4;
      continue;
    }
    c->k_last = cnt;
    if (needs_big && !big) {  // more labels than the one-block path holds: redo, ordered
      big = true;
      continue;
    }
    c->ht_cap = cnt * 2 > cap ? cap * 2 : cap;
    c->n_distinct = cnt;
    c->k = static_cast<int32_t>(cnt);
    c->dict_sorted_labels = sorted_labels;
    return;
  }
}

// Sharded protocol, pass 2: dense ids from the globally ordered dictionary, then rows.
void densify_assign_and_map(fsil_context* c, const int32_t* raw_in_dense_order, int32_t k) {
  const int64_t cap = c->ht_cap;
  const uint32_t epoch = c->ht_epoch;
  c->ht_dense.ensure(cap * sizeof(int32_t));
  c->dense.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
  c->dict_labels.ensure(std::max<int64_t>(k, 1) * sizeof(int32_t));
  int32_t* d_raw = c->dict_labels.as<int32_t>();
  FSIL_CUDA(cudaMemcpyAsync(d_raw, raw_in_dense_order, k * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  densify_assign_kernel<<<(k + 255) / 256, 256, 0, c->stream>>>(c->ht_keys.as<unsigned long long>(),
                                                                static_cast<uint32_t>(cap - 1), epoch, d_raw, k,
                                                                c->ht_dense.as<int32_t>());
  FSIL_LAUNCHED(c);
  FSIL_CUDA(cudaMemsetAsync(c->counters.as<int>() + 4, 0, sizeof(int), c->stream));  // missing
  if (c->n > 0) {
    launch_map(c, false, cap, c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_dense.as<int32_t>(),
               static_cast<uint32_t>(cap - 1), epoch, k, c->dense.as<int32_t>(), c->counters.as<int>() + 4);
  }
  // `missing` is checked by the caller at the end of the call (no extra sync here).
}

}  // namespace fsil

namespace fsil {

// Sharded protocol, device exchange, pass 1: local dictionary into the exchange buffer
// (no host sync).  Returns the buffer (cap_x entries of two int64).
int64_t* densify_exchange_begin(fsil_context* c, int64_t cap_x) {
  if (c->n >= (int64_t(1) << 32) - 1)
    fail(FSIL_ERR_INVALID_ARGUMENT, "shard too large: a rank holds at most 2^32-2 rows");
  const int64_t cap = std::max<int64_t>(c->ht_cap, 8192);
  const uint32_t epoch = prepare_table(c, cap);
  launch_collect(c, cap, epoch);
  c->xbuf.ensure(static_cast<size_t>(cap_x) * 2 * sizeof(int64_t));
  FSIL_CUDA(cudaMemsetAsync(c->xbuf.p, 0xff, static_cast<size_t>(cap_x) * 2 * sizeof(int64_t), c->stream));
  unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
  densify_xcompact_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
      c->ht_keys.as<unsigned long long>(), c->ht_vals.as<unsigned long long>(), static_cast<uint32_t>(cap), epoch,
      c->row_offset, c->xbuf.as<int64_t>(), cap_x, count, c->counters.as<int>());
  FSIL_LAUNCHED(c);
  return c->xbuf.as<int64_t>();
}

// After an exchange overflow: the repeat gets a larger exchange buffer and local table.
void exchange_grow(fsil_context* c, int64_t cap_x) {
  c->k_global_last = std::max<int64_t>(c->k_global_last, cap_x) * 4;
  c->ht_cap = std::max<int64_t>(c->ht_cap, 8192) * 4;
  c->spec_block_once = true;
}

// Pass 2: merge the gathered buffers of `nranks` ranks into the global dictionary
// (first-appearance order), dense ids for this rank's rows; one host sync for K.
void densify_exchange_set(fsil_context* c, const int64_t* gathered, int nranks, int64_t cap_x) {
  int64_t cap = 1024;
  while (cap < 2 * static_cast<int64_t>(nranks) * cap_x && cap < (int64_t(1) << 28)) cap *= 2;
  // the global dictionary gets its own epoch-tagged table (the local one keeps its size:
  // neither is re-zeroed from call to call)
  if (cap != c->xt_cap || c->xt_epoch == 0xffffffffu) {
    c->xt_keys.ensure(cap * sizeof(unsigned long long));
    c->xt_vals.ensure(cap * sizeof(unsigned long long));
    c->xt_dense.ensure(cap * sizeof(int32_t));
    FSIL_CUDA(cudaMemsetAsync(c->xt_keys.p, 0, cap * sizeof(unsigned long long), c->stream));
    FSIL_CUDA(cudaMemsetAsync(c->xt_vals.p, 0, cap * sizeof(unsigned long long), c->stream));
    c->xt_cap = cap;
    c->xt_epoch = 0;
  }
  const uint32_t epoch = ++c->xt_epoch;
  unsigned long long* keys = c->xt_keys.as<unsigned long long>();
  unsigned long long* vals = c->xt_vals.as<unsigned long long>();
  int32_t* slot_dense = c->xt_dense.as<int32_t>();
  int* counters = c->counters.as<int>();
  FSIL_CUDA(cudaMemsetAsync(counters, 0, 64, c->stream));
  const uint32_t mask = static_cast<uint32_t>(cap - 1);
  c->dict_sorted.ensure(cap * (2 * sizeof(int32_t)));
  c->dense.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
  int32_t* sorted_labels = reinterpret_cast<int32_t*>(c->dict_sorted.p) + cap;
  const int64_t total = static_cast<int64_t>(nranks) * cap_x;
  densify_xinsert_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, c->stream>>>(
      gathered, total, keys, vals, mask, epoch, counters);
  FSIL_LAUNCHED(c);
  // Speculation (as in densify_local): every rank holds the same previous global K, so all
  // speculate alike and all see the same miss at finish (FSIL_AGAIN: repeat the protocol).
  const bool spec = c->speculate && !c->spec_block_once && c->k_global_last >= 2;
  c->spec_block_once = false;
  int64_t cnt = c->k_global_last;
  bool big = c->k_global_last > kSmallK;
  densify_finish_kernel<<<1, 1024, 0, c->stream>>>(keys, vals, static_cast<uint32_t>(cap), epoch, sorted_labels,
                                                   slot_dense, counters, c->dsum,
                                                   spec ? static_cast<int32_t>(c->k_global_last) : 0, big);
  FSIL_LAUNCHED(c);
  if (!spec) {
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    const volatile HostSummary* hs = c->hsum;
    if (hs->overflow) {  // some rank's dictionary outgrew the exchange: every rank sees it
      exchange_grow(c, cap_x);
      fail(FSIL_AGAIN, "device dictionary exchange: more distinct labels than its capacity (" +
                           std::to_string(cap_x - 1) + " per rank); repeat with a larger one");
    }
    cnt = hs->count;
    big = hs->pad != 0;
  }
  c->k_spec = spec;
  c->spec_big = big;
  c->spec_cap_x = cap_x;
  if (big) {  // more labels than the one-block ordering holds: multi-block
    c->dict_labels.ensure(cap * sizeof(int32_t));
    c->dict_rows.ensure(cap * sizeof(int64_t));
    int32_t* slots = reinterpret_cast<int32_t*>(c->dict_sorted.p);
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
    FSIL_CUDA(cudaMemsetAsync(count, 0, sizeof(unsigned long long), c->stream));
    densify_compact_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        keys, vals, static_cast<uint32_t>(cap), epoch, 0, c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(),
        slots, count);
    FSIL_LAUNCHED(c);
    densify_rank_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), slots, count, sorted_labels, slot_dense);
    FSIL_LAUNCHED(c);
  }
  FSIL_CUDA(cudaMemsetAsync(counters + 4, 0, sizeof(int), c->stream));  // missing
  if (c->n > 0) {
    launch_map(c, false, static_cast<int64_t>(mask) + 1, c->labels, c->n, keys, slot_dense, mask, epoch,
               spec ? static_cast<int32_t>(c->k_global_last) : INT32_MAX, c->dense.as<int32_t>(), counters + 4);
  }
  c->ht_cap = std::max<int64_t>(c->ht_cap, 8192);
  c->n_distinct = cnt;
  c->k = static_cast<int32_t>(cnt);
  c->dict_sorted_labels = sorted_labels;
}

}  // namespace fsil
