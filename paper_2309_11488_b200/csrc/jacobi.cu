// Block-Jacobi relaxation of the preconditioner matrix on the device
// (bs/jacobi.py:111-147): drop every block coupling two partitions (the
// diagonal always survives), record the retained slots as the copy plan,
// and refresh the relaxed values from the full matrix with one gather.
// Used by the slab-partitioned multi-GPU solver (one partition per GPU)
// and by SolverConfig.jacobi_partitions.
#include <cub/cub.cuh>

#include "common.cuh"

namespace b2s {

__global__ void k_keep_count(int n, const int32_t* __restrict__ rp,
                             const int32_t* __restrict__ ci, const int32_t* __restrict__ part,
                             int32_t* cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int pi = part[i];
    int c = 0;
    for (int q = rp[i]; q < rp[i + 1]; ++q) c += (part[ci[q]] == pi) ? 1 : 0;
    cnt[i] = c;
  }
}

__global__ void k_keep_fill(int n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const int32_t* __restrict__ part, const int32_t* __restrict__ nrp,
                            int32_t* nci, int32_t* idx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int pi = part[i];
    int d = nrp[i];
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      const int c = ci[q];
      if (part[c] == pi) { nci[d] = c; idx[d] = q; ++d; }
    }
  }
}

inline int grid_for(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > kSms * 32) g = kSms * 32;
  return (int)g;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// Pass 1: new row pointers (n+1) and the retained block count to host.
int b2s_jacobi_pattern(int n, const int32_t* rp, const int32_t* ci, const int32_t* part,
                       int32_t* new_rp, int32_t* kept_host, cudaStream_t st) {
  *kept_host = 0;
  if (n < 0) return B2S_SHAPE;
  if (n == 0) {
    B2S_CHECK(cudaMemsetAsync(new_rp, 0, sizeof(int32_t), st));
    return B2S_OK;
  }
  int32_t* cnt = nullptr;
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (n + 1), st));
  B2S_CHECK(cudaMemsetAsync(cnt + n, 0, sizeof(int32_t), st));
  k_keep_count<<<grid_for(n), 256, 0, st>>>(n, rp, ci, part, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, new_rp, n + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, new_rp, n + 1, st);
  B2S_LAUNCH_CHECK();
  B2S_CHECK(cudaMemcpyAsync(kept_host, new_rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  return B2S_OK;
}

// Pass 2: retained columns and their source slots (the CopyPlan indices).
int b2s_jacobi_fill(int n, const int32_t* rp, const int32_t* ci, const int32_t* part,
                    const int32_t* new_rp, int32_t* new_ci, int32_t* indices, cudaStream_t st) {
  if (n < 0) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  k_keep_fill<<<grid_for(n), 256, 0, st>>>(n, rp, ci, part, new_rp, new_ci, indices);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

}  // extern "C"

// ---- the greedy partitioner (bs/jacobi.py:61-108), host side ---------------
//
// Region growing along the heaviest frontier edge is a strictly sequential
// priority-queue walk, so it stays on the host (as in the reference), but in
// C++ instead of Python: the same min-heap on (-w, cell) -- pops are fully
// determined by that key, so the assignment is the reference's exactly.
#include <queue>
#include <utility>
#include <vector>

extern "C" int b2s_partition_greedy(long long n, long long nedges, const long long* lo,
                                    const long long* hi, const double* w, long long k,
                                    long long* part) {
  if (n < 0 || nedges < 0 || k < 1 || k > (n > 0 ? n : 1)) return B2S_SHAPE;
  std::vector<long long> deg(n + 1, 0);
  for (long long e = 0; e < nedges; ++e) {
    if (lo[e] < 0 || hi[e] >= n || lo[e] >= hi[e]) return B2S_SHAPE;
    ++deg[lo[e] + 1];
    ++deg[hi[e] + 1];
  }
  for (long long i = 0; i < n; ++i) deg[i + 1] += deg[i];
  std::vector<long long> pos(deg.begin(), deg.end() - 1), adj(2 * nedges);
  std::vector<double> aw(2 * nedges);
  for (long long e = 0; e < nedges; ++e) {
    adj[pos[lo[e]]] = hi[e]; aw[pos[lo[e]]++] = w[e];
    adj[pos[hi[e]]] = lo[e]; aw[pos[hi[e]]++] = w[e];
  }
  for (long long i = 0; i < n; ++i) part[i] = -1;
  typedef std::pair<double, long long> Item;   // (-w, cell): heapq's order
  std::priority_queue<Item, std::vector<Item>, std::greater<Item>> heap;
  const long long base = n / k, rem = n % k;
  long long seed = 0;
  for (long long q = 0; q < k; ++q) {
    const long long want = base + (q < rem ? 1 : 0);
    long long got = 0;
    while (!heap.empty()) heap.pop();
    while (got < want) {
      long long cell;
      if (!heap.empty()) {
        cell = heap.top().second;
        heap.pop();
        if (part[cell] >= 0) continue;
      } else {
        while (part[seed] >= 0) ++seed;
        cell = seed;
      }
      part[cell] = q;
      ++got;
      for (long long t = deg[cell]; t < deg[cell + 1]; ++t)
        if (part[adj[t]] < 0) heap.push(Item(-aw[t], adj[t]));
    }
  }
  return B2S_OK;
}
