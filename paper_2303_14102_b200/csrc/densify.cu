// densify.cu -- K0: first-appearance dense cluster ids on the device.
//
// Replaces validate_and_densify's label remapping (dataset.cpp:41-51,
// 63-68): dense id = rank of a raw label's first row in dataset order.
// Pass 1 dedups labels per block in a shared-memory hash table and merges
// (label, min row) into a global open-addressing table; the host orders the
// (few) distinct labels by first row -- merging across ranks first in the
// sharded protocol -- and pass 2 maps every row to its dense id.
#include <algorithm>
#include <vector>

#include "device_util.cuh"
#include "fsil_internal.cuh"

namespace fsil {
namespace {

constexpr int kSmemSlots = 1024;

__device__ bool global_insert(unsigned long long* keys, uint32_t* vals, uint32_t cap_mask,
                              unsigned long long key, uint32_t row) {
  uint32_t h = hash32(static_cast<uint32_t>(key)) & cap_mask;
  for (uint32_t probe = 0; probe <= cap_mask; ++probe) {
    unsigned long long cur = keys[h];
    if (cur == 0) {
      const unsigned long long prev = atomicCAS(keys + h, 0ull, key);
      cur = prev == 0 ? key : prev;
    }
    if (cur == key) {
      if (row < vals[h]) atomicMin(vals + h, row);
      return true;
    }
    h = (h + 1) & cap_mask;
  }
  return false;
}

__global__ void __launch_bounds__(256) densify_collect_kernel(const int32_t* __restrict__ labels,
                                                              int64_t n,
                                                              unsigned long long* gkeys,
                                                              uint32_t* gvals, uint32_t cap_mask,
                                                              int* overflow) {
  __shared__ unsigned long long skeys[kSmemSlots];
  __shared__ uint32_t svals[kSmemSlots];
  for (int i = threadIdx.x; i < kSmemSlots; i += blockDim.x) {
    skeys[i] = 0;
    svals[i] = 0xffffffffu;
  }
  __syncthreads();
  // Four rows per thread per step (independent loads in flight); within a warp only the
  // lowest lane of each run of equal labels (= the lowest row) touches the table.
  const int lane = threadIdx.x & 31;
  constexpr int U = 4;
  const int64_t bstride = static_cast<int64_t>(gridDim.x) * blockDim.x * U;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * U; base < n; base += bstride) {
    int32_t lab[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x + threadIdx.x;
      lab[u] = i < n ? __ldg(labels + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x + threadIdx.x;
      const bool valid = i < n;
      const unsigned long long key = valid ? label_key(lab[u]) : 0ull;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (!valid || (__ffs(peers) - 1) != lane) continue;
      const uint32_t row = static_cast<uint32_t>(i);
      uint32_t h = hash32(static_cast<uint32_t>(key)) & (kSmemSlots - 1);
      bool done = false;
      for (int probe = 0; probe < 16; ++probe) {  // bounded: overflow goes global
        unsigned long long cur = skeys[h];
        if (cur == 0) {
          const unsigned long long prev = atomicCAS(skeys + h, 0ull, key);
          cur = prev == 0 ? key : prev;
        }
        if (cur == key) {
          if (row < svals[h]) atomicMin(svals + h, row);
          done = true;
          break;
        }
        h = (h + 1) & (kSmemSlots - 1);
      }
      if (!done && !global_insert(gkeys, gvals, cap_mask, key, row)) atomicExch(overflow, 1);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kSmemSlots; i += blockDim.x) {
    const unsigned long long key = skeys[i];
    if (key != 0 && !global_insert(gkeys, gvals, cap_mask, key, svals[i])) atomicExch(overflow, 1);
  }
}

__global__ void densify_compact_kernel(const unsigned long long* __restrict__ gkeys,
                                       const uint32_t* __restrict__ gvals, uint32_t cap,
                                       int64_t row_offset, int32_t* out_labels,
                                       int64_t* out_rows, unsigned long long* count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  const unsigned long long key = gkeys[i];
  if (key == 0) return;
  const unsigned long long j = atomicAdd(count, 1ull);
  out_labels[j] = static_cast<int32_t>(static_cast<uint32_t>(key));
  out_rows[j] = row_offset + static_cast<int64_t>(gvals[i]);
}

// Dense id j for the j-th distinct label in first-row order (entries past `count`
// are padding with first row INT64_MAX).
__global__ void densify_assign_sorted_kernel(const unsigned long long* __restrict__ gkeys,
                                             uint32_t cap_mask, const int32_t* __restrict__ raw,
                                             const unsigned long long* count, int32_t* gdense);

__device__ int64_t find_slot(const unsigned long long* gkeys, uint32_t cap_mask,
                             unsigned long long key) {
  uint32_t h = hash32(static_cast<uint32_t>(key)) & cap_mask;
  for (uint32_t probe = 0; probe <= cap_mask; ++probe) {
    const unsigned long long cur = gkeys[h];
    if (cur == key) return h;
    if (cur == 0) return -1;
    h = (h + 1) & cap_mask;
  }
  return -1;
}

__global__ void densify_assign_kernel(const unsigned long long* __restrict__ gkeys,
                                      uint32_t cap_mask, const int32_t* __restrict__ raw,
                                      int32_t k, int32_t* gdense) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const int64_t slot = find_slot(gkeys, cap_mask, label_key(raw[j]));
  if (slot >= 0) gdense[slot] = j;
}

__global__ void __launch_bounds__(256) densify_map_kernel(const int32_t* __restrict__ labels,
                                                          int64_t n,
                                                          const unsigned long long* __restrict__ gkeys,
                                                          const int32_t* __restrict__ gdense,
                                                          uint32_t cap_mask, int32_t* dense,
                                                          int* missing, const int* counters,
                                                          HostSummary* hsum) {
  if (hsum && blockIdx.x == 0 && threadIdx.x == 0) {  // K and overflow for the host (final here)
    hsum->overflow = counters[0];
    hsum->count = static_cast<int64_t>(*reinterpret_cast<const unsigned long long*>(counters + 2));
  }
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t slot = find_slot(gkeys, cap_mask, label_key(labels[i]));
    const int32_t dj = slot >= 0 ? gdense[slot] : -1;
    if (dj < 0) atomicExch(missing, 1);
    dense[i] = dj;
  }
}

__global__ void densify_assign_sorted_kernel(const unsigned long long* __restrict__ gkeys,
                                             uint32_t cap_mask, const int32_t* __restrict__ raw,
                                             const unsigned long long* count, int32_t* gdense) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= static_cast<int64_t>(*count)) return;
  const int64_t slot = find_slot(gkeys, cap_mask, label_key(raw[j]));
  if (slot >= 0) gdense[slot] = static_cast<int32_t>(j);
}

__global__ void densify_init_kernel(unsigned long long* keys, uint32_t* vals, int32_t* gdense,
                                    int64_t* dict_rows, uint32_t cap, int* counters) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cap) {
    keys[i] = 0;
    vals[i] = 0xffffffffu;
    gdense[i] = -1;
    dict_rows[i] = INT64_MAX;
  }
  if (i < 16) counters[i] = 0;
}

// Compaction that also records each entry's hash slot.
__global__ void densify_compact_slot_kernel(const unsigned long long* __restrict__ gkeys,
                                            const uint32_t* __restrict__ gvals, uint32_t cap,
                                            int32_t* out_labels, int64_t* out_rows, int32_t* out_slot,
                                            unsigned long long* count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap) return;
  const unsigned long long key = gkeys[i];
  if (key == 0) return;
  const unsigned long long j = atomicAdd(count, 1ull);
  out_labels[j] = static_cast<int32_t>(static_cast<uint32_t>(key));
  out_rows[j] = static_cast<int64_t>(gvals[i]);
  out_slot[j] = static_cast<int32_t>(i);
}

// Dense id = rank of the entry's first row among all distinct labels (first rows
// are unique); writes the dense order and the per-slot dense id in one pass.
__global__ void __launch_bounds__(256) densify_rank_kernel(const int32_t* __restrict__ labels,
                                                           const int64_t* __restrict__ rows,
                                                           const int32_t* __restrict__ slots,
                                                           const unsigned long long* count,
                                                           int32_t* sorted_labels, int32_t* gdense) {
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
    gdense[slots[i]] = static_cast<int32_t>(rank);
  }
}

int grid_for(int64_t n, int threads, int num_sms, int per_sm) {
  const int64_t want = (n + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(num_sms) * per_sm)));
}

}  // namespace

void densify_collect(fsil_context* c) {
  if (c->n >= (int64_t(1) << 32) - 1)
    fail(FSIL_ERR_INVALID_ARGUMENT, "shard too large: a rank holds at most 2^32-2 rows");
  int64_t cap = std::max<int64_t>(c->ht_cap, 8192);
  c->counters.ensure(64);
  for (;;) {
    c->ht_keys.ensure(cap * sizeof(unsigned long long));
    c->ht_vals.ensure(cap * sizeof(uint32_t));
    FSIL_CUDA(cudaMemsetAsync(c->ht_keys.p, 0, cap * sizeof(unsigned long long), c->stream));
    FSIL_CUDA(cudaMemsetAsync(c->ht_vals.p, 0xff, cap * sizeof(uint32_t), c->stream));
    FSIL_CUDA(cudaMemsetAsync(c->counters.p, 0, 64, c->stream));
    int* overflow = c->counters.as<int>();
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
    if (c->n > 0) {
      densify_collect_kernel<<<grid_for(c->n, 256, c->num_sms, 4), 256, 0, c->stream>>>(
          c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_vals.as<uint32_t>(),
          static_cast<uint32_t>(cap - 1), overflow);
      FSIL_LAUNCHED(c);
    }
    int h_over = 0;
    FSIL_CUDA(cudaMemcpyAsync(&h_over, overflow, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    if (h_over) {
      cap *= 4;
      continue;
    }
    c->ht_cap = cap;
    // Compact occupied slots into (label, first global row) pairs.
    c->dict_labels.ensure(cap * sizeof(int32_t));
    c->dict_rows.ensure(cap * sizeof(int64_t));
    densify_compact_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->ht_keys.as<unsigned long long>(), c->ht_vals.as<uint32_t>(), static_cast<uint32_t>(cap),
        c->row_offset, c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), count);
    FSIL_LAUNCHED(c);
    unsigned long long h_count = 0;
    FSIL_CUDA(cudaMemcpyAsync(&h_count, count, sizeof(h_count), cudaMemcpyDeviceToHost, c->stream));
    FSIL_CUDA(cudaStreamSynchronize(c->stream));
    c->n_distinct = static_cast<int64_t>(h_count);
    if (c->n_distinct * 2 > cap) c->ht_cap = cap * 2;  // keep probes short next call
    return;
  }
}

// Single-GPU densify with one host sync: init -> collect -> compact -> rank by first
// row (dense order) + per-slot dense ids -> per-row map; then read K and overflow.
void densify_local(fsil_context* c) {
  if (c->n >= (int64_t(1) << 31) - 1)
    fail(FSIL_ERR_INVALID_ARGUMENT, "too many rows for one device call (2^31-2)");
  int64_t cap = std::max<int64_t>(c->ht_cap, 8192);
  c->counters.ensure(64);
  for (;;) {
    c->ht_keys.ensure(cap * sizeof(unsigned long long));
    c->ht_vals.ensure(cap * sizeof(uint32_t));
    c->ht_dense.ensure(cap * sizeof(int32_t));
    c->dict_labels.ensure(cap * sizeof(int32_t));
    c->dict_rows.ensure(cap * sizeof(int64_t));
    c->dict_sorted.ensure(cap * (2 * sizeof(int32_t)));
    c->dense.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
    int* overflow = c->counters.as<int>();
    int* missing = c->counters.as<int>() + 4;
    unsigned long long* count = reinterpret_cast<unsigned long long*>(c->counters.as<char>() + 8);
    const uint32_t mask = static_cast<uint32_t>(cap - 1);
    int32_t* slots = reinterpret_cast<int32_t*>(c->dict_sorted.p);
    int32_t* sorted_labels = slots + cap;
    densify_init_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->ht_keys.as<unsigned long long>(), c->ht_vals.as<uint32_t>(), c->ht_dense.as<int32_t>(),
        c->dict_rows.as<int64_t>(), static_cast<uint32_t>(cap), c->counters.as<int>());
    FSIL_LAUNCHED(c);
    densify_collect_kernel<<<grid_for(c->n, 256, c->num_sms, 2), 256, 0, c->stream>>>(
        c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_vals.as<uint32_t>(), mask,
        overflow);
    FSIL_LAUNCHED(c);
    densify_compact_slot_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->ht_keys.as<unsigned long long>(), c->ht_vals.as<uint32_t>(), static_cast<uint32_t>(cap),
        c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), slots, count);
    FSIL_LAUNCHED(c);
    densify_rank_kernel<<<static_cast<unsigned>((cap + 255) / 256), 256, 0, c->stream>>>(
        c->dict_labels.as<int32_t>(), c->dict_rows.as<int64_t>(), slots, count, sorted_labels,
        c->ht_dense.as<int32_t>());
    FSIL_LAUNCHED(c);
    densify_map_kernel<<<grid_for(c->n, 256, c->num_sms, 8), 256, 0, c->stream>>>(
        c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_dense.as<int32_t>(), mask,
        c->dense.as<int32_t>(), missing, c->counters.as<int>(), c->dsum);
    FSIL_LAUNCHED(c);
    FSIL_CUDA(cudaStreamSynchronize(c->stream));  // the one host sync: K decides the kernels
    const volatile HostSummary* hs = c->hsum;
    const int64_t over = hs->overflow, cnt = hs->count;
    if (over) {
      cap *= 4;
      continue;
    }
    c->ht_cap = cnt * 2 > cap ? cap * 2 : cap;
    c->n_distinct = cnt;
    c->k = static_cast<int32_t>(cnt);
    c->dict_sorted_labels = sorted_labels;
    return;
  }
}

void densify_assign_and_map(fsil_context* c, const int32_t* raw_in_dense_order, int32_t k) {
  const int64_t cap = c->ht_cap;
  c->ht_dense.ensure(cap * sizeof(int32_t));
  c->dense.ensure(std::max<int64_t>(c->n, 1) * sizeof(int32_t));
  int32_t* d_raw = c->dict_labels.as<int32_t>();  // reuse: host order -> device
  c->dict_labels.ensure(std::max<int64_t>(k, 1) * sizeof(int32_t));
  d_raw = c->dict_labels.as<int32_t>();
  FSIL_CUDA(cudaMemcpyAsync(d_raw, raw_in_dense_order, k * sizeof(int32_t), cudaMemcpyHostToDevice,
                            c->stream));
  FSIL_CUDA(cudaMemsetAsync(c->ht_dense.p, 0xff, cap * sizeof(int32_t), c->stream));
  densify_assign_kernel<<<(k + 255) / 256, 256, 0, c->stream>>>(
      c->ht_keys.as<unsigned long long>(), static_cast<uint32_t>(cap - 1), d_raw, k,
      c->ht_dense.as<int32_t>());
  FSIL_LAUNCHED(c);
  int* missing = c->counters.as<int>() + 4;
  FSIL_CUDA(cudaMemsetAsync(missing, 0, sizeof(int), c->stream));
  if (c->n > 0) {
    densify_map_kernel<<<grid_for(c->n, 256, c->num_sms, 8), 256, 0, c->stream>>>(
        c->labels, c->n, c->ht_keys.as<unsigned long long>(), c->ht_dense.as<int32_t>(),
        static_cast<uint32_t>(cap - 1), c->dense.as<int32_t>(), missing, nullptr, nullptr);
    FSIL_LAUNCHED(c);
  }
  // `missing` is checked by the caller at the end of the call (no extra sync here).
}

}  // namespace fsil
