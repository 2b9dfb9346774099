// Block ILU0 factorisation (bs/ilu0.py:145-201) as a sync-free wavefront.
//
// Phase 1, symbolic (value independent): for every strict-lower slot k of
// permuted row i (column r) list the update pairs (p, q) -- slot p of row i
// and slot q of row r with equal columns j > r.  These are exactly the
// targets of the reference's `A_ij -= L_ir A_rj` (the searchsorted merge of
// bs/ilu0.py:183-195), precomputed so that the numeric phase has nothing
// but value loads left on its critical path.  On a 7-point stencil every
// list holds one pair (the diagonal).
//
// Phase 2, numeric: rows are claimed slice by slice in plan order through an
// atomic ticket; a row processes its lower slots in ascending column order
// (the reference's order), waiting on a per-row "finished" flag for each
// pivot row r, then L_ir = A_ir inv(U_rr), A_ip -= L_ir A_rq over its pairs,
// and finally inv(A_ii) with the reference's singularity rule.  A warp keeps
// polling while any of its lanes still waits, so lanes of one slice may even
// depend on each other (user-built plans) without deadlock.
#include <cstdlib>

#include <cub/cub.cuh>

#include "sell.cuh"

namespace b2s {

constexpr int kFast = 3;   // lower entries handled by the one-round fast path

struct Tickets2 {
  unsigned int next, finished;
};

__device__ __forceinline__ long long claim_slice(Tickets2* tk, int nslices) {
  const int lane = threadIdx.x & 31;
  unsigned int t = 0;
  if (lane == 0) t = atomicAdd(&tk->next, 1u);
  t = __shfl_sync(0xffffffffu, t, 0);
  if (t < (unsigned)nslices) return t;
  if (lane == 0) {
    const unsigned int total = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(&tk->finished, 1u) == total - 1) {
      tk->next = 0;
      tk->finished = 0;
      __threadfence();
    }
  }
  return -1;
}

__device__ __forceinline__ int ld_flag_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_flag_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- symbolic phase: count (pairs == nullptr) or fill the update pairs
__global__ void k_factor_pairs(int n, const int32_t* __restrict__ rp,
                               const int32_t* __restrict__ ci, const int32_t* __restrict__ diag,
                               int32_t* __restrict__ cnt, const int32_t* __restrict__ ptr,
                               int2* __restrict__ pairs) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int end = rp[i + 1];
    for (int k = rp[i]; k < diag[i]; ++k) {
      const int r = ci[k];
      int m = 0, p = k + 1;
      const int out = pairs ? ptr[k] : 0;
      const int rend = rp[r + 1];
      for (int q = diag[r] + 1; q < rend && p < end; ++q) {
        const int j = ci[q];
        while (p < end && ci[p] < j) ++p;
        if (p < end && ci[p] == j) {
          if (pairs) pairs[out + m] = make_int2(p, q);
          ++m;
        }
      }
      if (!pairs) cnt[k] = m;
    }
  }
}

// ---- per-row "simple" mark: <= kFast lower entries, each with at most one
// update pair, every pair landing on the row's own diagonal.  The upper
// blocks of a simple row are never modified by the factorisation, so its
// consumers may read them before the row is finished.
__global__ void k_factor_simple(int n, const int32_t* __restrict__ rp,
                                const int32_t* __restrict__ diag,
                                const int32_t* __restrict__ pptr,
                                const int2* __restrict__ pairs, int8_t* simple,
                                int* nonsimple) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int k0 = rp[i], d = diag[i];
    bool ok = d - k0 <= kFast;
    for (int k = k0; ok && k < d; ++k) {
      const int b0 = pptr[k], b1 = pptr[k + 1];
      if (b1 - b0 > 1 || (b1 > b0 && pairs[b0].x != d)) ok = false;
    }
    simple[i] = ok ? 1 : 0;
    if (!ok) atomicAdd(nonsimple, 1);
  }
}

// ---- numeric phase
template <int B>
__global__ void __launch_bounds__(256) k_factor_numeric(
    SliceMap map, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
    const int32_t* __restrict__ diag, const int32_t* __restrict__ pptr,
    const int2* __restrict__ pairs, const int8_t* __restrict__ simple_row, double* w,
    double* invd, int* flag, int* bad, Tickets2* tk, int sleep_ns, int all_simple) {
  constexpr int BB = B * B;
  const int lane = threadIdx.x & 31;
  for (;;) {
    const long long s = claim_slice(tk, map.nslices);
    if (s < 0) break;
    const int i = map.row0[s] + lane;
    bool done = lane >= map.nrows[s];
    int k = 0, dpos = 0;
    int r = -1, pb = 0, pe = 0;
    int2 pq0 = make_int2(0, 0);
    // fast path: the row and all its pivots are "simple" (see k_factor_simple).
    // Everything static (own blocks, the pivots' upper blocks) is prefetched
    // at claim time; the only thing waited for is the pivots' inverse
    // diagonals, polled directly (sentinel-initialised) -- one L2 round trip
    // per dependency level, no flag, no fence on the consumer side.
    bool simple = false;
    int fr[kFast], nl = 0;
    double wik[kFast][BB], urq[kFast][BB], inv_r[kFast][BB], dblk[BB];
    if (!done) {
      k = rp[i];
      dpos = diag[i];
      nl = dpos - k;
      simple = simple_row[i] != 0;
#pragma unroll
      for (int t = 0; t < kFast; ++t) {
        fr[t] = 0;
        if (simple && t < nl) {
          fr[t] = ci[k + t];
          if (!simple_row[fr[t]]) simple = false;
        }
      }
      if (simple) {
#pragma unroll
        for (int t = 0; t < kFast; ++t) {
          const int b0 = t < nl ? pptr[k + t] : 0, b1 = t < nl ? pptr[k + t + 1] : 0;
          const int q = b1 > b0 ? pairs[b0].y : -1;
#pragma unroll
          for (int e = 0; e < BB; ++e) {
            wik[t][e] = t < nl ? w[(long long)(k + t) * BB + e] : 0.0;
            urq[t][e] = q >= 0 ? __ldcg(w + (long long)q * BB + e) : 0.0;
            inv_r[t][e] = 0.0;
          }
        }
#pragma unroll
        for (int e = 0; e < BB; ++e) dblk[e] = w[(long long)dpos * BB + e];
      } else if (k < dpos) {  // static data of the first pivot (general path)
        r = ci[k]; pb = pptr[k]; pe = pptr[k + 1];
        if (pb < pe) pq0 = pairs[pb];
      }
    }
    unsigned int fpend = simple ? ((1u << nl) - 1u) : 0u;
    for (;;) {
      if (!done && simple) {
        const unsigned int todo = fpend;
#pragma unroll
        for (int t = 0; t < kFast; ++t)
          if (todo & (1u << t)) {
#pragma unroll
            for (int e = 0; e < BB; ++e) inv_r[t][e] = ld_relaxed_f64(invd + (long long)fr[t] * BB + e);
          }
#pragma unroll
        for (int t = 0; t < kFast; ++t) {
          bool miss = false;
#pragma unroll
          for (int e = 0; e < BB; ++e) miss |= is_sentinel(inv_r[t][e]);
          if ((todo & (1u << t)) && !miss) fpend &= ~(1u << t);
        }
        if (!fpend) {
#pragma unroll
          for (int t = 0; t < kFast; ++t) {
            if (t < nl) {
              double l[BB], prod[BB];
              matmul<B>(wik[t], inv_r[t], l);  // L_ir = A_ir inv(U_rr)
#pragma unroll
              for (int e = 0; e < BB; ++e) w[(long long)(k + t) * BB + e] = l[e];
              matmul<B>(l, urq[t], prod);      // A_ii -= L_ir U_ri (zero block: no pair)
#pragma unroll
              for (int e = 0; e < BB; ++e) dblk[e] -= prod[e];
            }
          }
          double inv[BB];
#pragma unroll
          for (int e = 0; e < BB; ++e) w[(long long)dpos * BB + e] = dblk[e];
          if (!invert_block<B>(dblk, inv)) atomicMin(bad, i);
#pragma unroll
          for (int e = 0; e < BB; ++e) st_relaxed_f64(invd + (long long)i * BB + e, canon(inv[e]));
          // for general-path consumers (none when every row is simple: the
          // release fence is then skipped)
          if (!all_simple) st_flag_release(flag + i, 1);
          done = true;
        }
      }
      if (!done && !simple) {
        while (k < dpos) {
          if (ld_flag_relaxed(flag + r) == 0) break;
          // every value load of this pivot step is independent: one round trip
          double inv_r[BB], wik[BB], urq[BB], wip[BB], l[BB], prod[BB];
#pragma unroll
          for (int e = 0; e < BB; ++e) {
            inv_r[e] = __ldcg(invd + (long long)r * BB + e);
            wik[e] = w[(long long)k * BB + e];
          }
          if (pb < pe) {
#pragma unroll
            for (int e = 0; e < BB; ++e) {
              urq[e] = __ldcg(w + (long long)pq0.y * BB + e);
              wip[e] = w[(long long)pq0.x * BB + e];
            }
          }
          matmul<B>(wik, inv_r, l);  // L_ir = A_ir inv(U_rr)
#pragma unroll
          for (int e = 0; e < BB; ++e) w[(long long)k * BB + e] = l[e];
          if (pb < pe) {
            matmul<B>(l, urq, prod);  // A_ip -= L_ir U_rq
#pragma unroll
            for (int e = 0; e < BB; ++e) w[(long long)pq0.x * BB + e] = wip[e] - prod[e];
            for (int t = pb + 1; t < pe; ++t) {  // further pairs (not on stencils)
              const int2 pq = pairs[t];
#pragma unroll
              for (int e = 0; e < BB; ++e) urq[e] = __ldcg(w + (long long)pq.y * BB + e);
              matmul<B>(l, urq, prod);
#pragma unroll
              for (int e = 0; e < BB; ++e) w[(long long)pq.x * BB + e] -= prod[e];
            }
          }
          ++k;
          if (k < dpos) {
            r = ci[k]; pb = pptr[k]; pe = pptr[k + 1];
            if (pb < pe) pq0 = pairs[pb];
          }
        }
        if (k >= dpos) {
          double dblk[BB], inv[BB];
#pragma unroll
          for (int e = 0; e < BB; ++e) dblk[e] = w[(long long)dpos * BB + e];
          if (!invert_block<B>(dblk, inv)) atomicMin(bad, i);
#pragma unroll
          for (int e = 0; e < BB; ++e) st_relaxed_f64(invd + (long long)i * BB + e, canon(inv[e]));
          st_flag_release(flag + i, 1);  // publishes this row's L, U and inverse
          done = true;
        }
      }
      if (__all_sync(0xffffffffu, done)) break;
      if (sleep_ns) __nanosleep(sleep_ns);   // back off while the pivots are pending
    }
  }
}

template <int B>
int launch_numeric(SliceMap map, const int32_t* rp, const int32_t* ci, const int32_t* diag,
                   const int32_t* pptr, const int2* pairs, const int8_t* simple, double* w,
                   double* invd, int* flag,
                   int* bad, Tickets2* tk, int all_simple, cudaStream_t st) {
  int per_sm = 0, dev = 0, sms = kSms;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_factor_numeric<B>, 256, 0);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one CTA of 4 warps per SM: fewer spinning warps leave L2 to the rows in
  // progress (measured on C4 level plans: 8 warps 3.2 ms, 4 warps 2.6 ms,
  // 2 warps 2.8 ms for the whole factorisation)
  int g = (per_sm < 1 ? 1 : per_sm) * sms;
  int threads = 128, sleep_ns = 0;
  if (const char* e = getenv("B2S_FACTOR_SLEEP")) sleep_ns = atoi(e);
  if (const char* e = getenv("B2S_FACTOR_WARPS")) threads = 32 * atoi(e);
  if (const char* e = getenv("B2S_FACTOR_CTAS_PER_SM")) g = atoi(e) * sms;
  k_factor_numeric<B><<<g, threads, 0, st>>>(map, rp, ci, diag, pptr, pairs, simple, w, invd,
                                             flag, bad, tk, sleep_ns, all_simple);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

int fill_sentinel(long long m, double* v, cudaStream_t st);  // ilu0.cu

inline int grid_rows(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > kSms * 16) g = kSms * 16;
  return (int)g;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// Symbolic half of the factorisation (pattern only): the update pairs of
// every lower entry and the rows whose pivots are all "simple".  Allocates
// stream-ordered device buffers behind an opaque handle (freed by
// b2s_ilu0_symbolic_free); synchronises for the pair count.
struct IluSym {
  int n = 0, nnz = 0, npairs = 0, all_simple = 0;
  int32_t* pptr = nullptr;
  int2* pairs = nullptr;
  int8_t* simple = nullptr;
};

int b2s_ilu0_symbolic(int n, int b, const int32_t* rp, const int32_t* ci, const int32_t* diag,
                      void** handle, cudaStream_t st) {
  *handle = nullptr;
  if (n < 0 || b < 1) return B2S_SHAPE;
  if (b > 4) return B2S_UNSUPPORTED;
  IluSym* h = new IluSym();
  h->n = n;
  if (n == 0) { *handle = h; return B2S_OK; }
  int32_t nnz = 0;
  B2S_CHECK(cudaMemcpyAsync(&nnz, rp + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  h->nnz = nnz;
  int32_t* cnt = nullptr;
  B2S_CHECK(cudaMallocAsync(&cnt, sizeof(int32_t) * (nnz + 1), st));
  B2S_CHECK(cudaMallocAsync(&h->pptr, sizeof(int32_t) * (nnz + 1), st));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (nnz + 1), st));
  k_factor_pairs<<<grid_rows(n), 256, 0, st>>>(n, rp, ci, diag, cnt, nullptr, nullptr);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, h->pptr, nnz + 1, st);
  void* tmp = nullptr;
  B2S_CHECK(cudaMallocAsync(&tmp, tb, st));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, h->pptr, nnz + 1, st);
  int32_t npairs = 0;
  B2S_CHECK(cudaMemcpyAsync(&npairs, h->pptr + nnz, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  h->npairs = npairs;
  B2S_CHECK(cudaMallocAsync(&h->pairs, sizeof(int2) * (npairs > 0 ? npairs : 1), st));
  k_factor_pairs<<<grid_rows(n), 256, 0, st>>>(n, rp, ci, diag, nullptr, h->pptr, h->pairs);
  B2S_CHECK(cudaMallocAsync(&h->simple, n, st));
  B2S_CHECK(cudaMemsetAsync(cnt, 0, sizeof(int32_t), st));   // (cnt is free again)
  k_factor_simple<<<grid_rows(n), 256, 0, st>>>(n, rp, diag, h->pptr, h->pairs, h->simple, cnt);
  int32_t nonsimple = 1;
  B2S_CHECK(cudaMemcpyAsync(&nonsimple, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(tmp, st));
  B2S_CHECK(cudaFreeAsync(cnt, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  h->all_simple = nonsimple == 0 ? 1 : 0;
  B2S_LAUNCH_CHECK();
  *handle = h;
  return B2S_OK;
}

int b2s_ilu0_symbolic_free(void* handle, cudaStream_t st) {
  IluSym* h = reinterpret_cast<IluSym*>(handle);
  if (!h) return B2S_OK;
  if (h->pptr) cudaFreeAsync(h->pptr, st);
  if (h->pairs) cudaFreeAsync(h->pairs, st);
  if (h->simple) cudaFreeAsync(h->simple, st);
  delete h;
  return B2S_OK;
}

// Numeric half: factor the permuted block-CSR values in place (combined
// L\U) and write the inverse diagonal blocks (row-major, n*b*b).  The slice
// map gives the claim order (plan order).  bad_dev null: synchronises and
// reports the smallest failing *permuted* row in bad_row_host
// (B2S_SINGULAR_PIVOT); bad_dev given (device int, INT32_MAX on entry): the
// row lands there, stream-ordered, no host read.
int b2s_ilu0_numeric(const void* handle, int b, int nslices, const int32_t* row0,
                     const int32_t* nrows, const int32_t* rp, const int32_t* ci,
                     const int32_t* diag, double* vals, double* inv_diag, int* bad_dev,
                     int32_t* bad_row_host, cudaStream_t st) {
  if (bad_row_host) *bad_row_host = -1;
  const IluSym* h = reinterpret_cast<const IluSym*>(handle);
  if (!h || b < 1) return B2S_SHAPE;
  if (b > 4) return B2S_UNSUPPORTED;
  const int n = h->n;
  if (n == 0) return B2S_OK;
  int* flag = nullptr;
  int* bad = bad_dev;
  Tickets2* tk = nullptr;
  B2S_CHECK(cudaMallocAsync(&flag, sizeof(int) * n, st));
  B2S_CHECK(cudaMallocAsync(&tk, sizeof(Tickets2), st));
  B2S_CHECK(cudaMemsetAsync(flag, 0, sizeof(int) * n, st));
  B2S_CHECK(cudaMemsetAsync(tk, 0, sizeof(Tickets2), st));
  const int big = 0x7fffffff;
  if (!bad) {
    B2S_CHECK(cudaMallocAsync(&bad, sizeof(int), st));
    B2S_CHECK(cudaMemcpyAsync(bad, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  }
  // the inverse diagonals double as the fast path's "ready" marks
  if (int rcf = fill_sentinel((long long)n * b * b, inv_diag, st)) return rcf;
  B2S_LAUNCH_CHECK();
  SliceMap map{nslices, row0, nrows};
  int rc;
  switch (b) {
    case 1: rc = launch_numeric<1>(map, rp, ci, diag, h->pptr, h->pairs, h->simple, vals, inv_diag, flag, bad, tk, h->all_simple, st); break;
    case 2: rc = launch_numeric<2>(map, rp, ci, diag, h->pptr, h->pairs, h->simple, vals, inv_diag, flag, bad, tk, h->all_simple, st); break;
    case 3: rc = launch_numeric<3>(map, rp, ci, diag, h->pptr, h->pairs, h->simple, vals, inv_diag, flag, bad, tk, h->all_simple, st); break;
    default: rc = launch_numeric<4>(map, rp, ci, diag, h->pptr, h->pairs, h->simple, vals, inv_diag, flag, bad, tk, h->all_simple, st); break;
  }
  if (rc != B2S_OK) return rc;
  B2S_CHECK(cudaFreeAsync(flag, st));
  B2S_CHECK(cudaFreeAsync(tk, st));
  if (bad_dev) return B2S_OK;
  int hb = big;
  B2S_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(bad, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  if (hb != big) {
    if (bad_row_host) *bad_row_host = hb;
    return B2S_SINGULAR_PIVOT;
  }
  return B2S_OK;
}

// Both halves (the original entry point): on a singular pivot the smallest
// failing *permuted* row goes to bad_row_host (B2S_SINGULAR_PIVOT).
int b2s_ilu0_factor(int n, int b, int nslices, const int32_t* row0, const int32_t* nrows,
                    const int32_t* rp, const int32_t* ci, const int32_t* diag, double* vals,
                    double* inv_diag, int32_t* bad_row_host, cudaStream_t st) {
  *bad_row_host = -1;
  if (n < 0 || b < 1) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  if (b > 4) return B2S_UNSUPPORTED;
  void* h = nullptr;
  int rc = b2s_ilu0_symbolic(n, b, rp, ci, diag, &h, st);
  if (rc == B2S_OK)
    rc = b2s_ilu0_numeric(h, b, nslices, row0, nrows, rp, ci, diag, vals, inv_diag, nullptr,
                          bad_row_host, st);
  b2s_ilu0_symbolic_free(h, st);
  return rc;
}

}  // extern "C"
