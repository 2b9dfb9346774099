// ILU0 of a two-colour plan straight into the SELL layouts (bs/ilu0.py:
// 145-201 specialised to 2 independent groups).
//
// In plan order a colouring with two groups puts every off-diagonal entry of
// a colour-0 row in colour 1 (higher plan index) and every off-diagonal
// entry of a colour-1 row in colour 0 (lower), so the IKJ elimination
// degenerates exactly:
//   colour 0:  U_ii = A_ii                       (no strict-lower entries)
//   colour 1:  L_ik = A_ik inv(U_kk)  for its lower entries k (ascending),
//              U_ii = A_ii - sum_k L_ik A_ki     (every update lands on the
//              diagonal: two colour-0 rows are never coupled)
//   U_ij = A_ij off the diagonal                 (never updated).
// Per-row arithmetic is the general factor kernel's (factor.cu: matmul, then
// subtract, ascending k; Gauss-Jordan inverse with the reference's
// singularity rule), so results are bit-identical to it -- tested.
//
// The operator itself is filled into its SELL layout directly from the
// input-order values through the permutation's source map (no plan-order
// CSR copy), the factor reads that layout and writes the strict-lower SELL
// and the inverse-diagonal tiles; U is the operator's colour-0 rows (the
// fused Krylov pass reads them there).  The plan-order CSR of L\U is only
// materialised if the caller asks for it (k_f2c_combined).
#include "sell.cuh"

namespace b2s {

// rows of group g are consecutive in plan order and sliced from the group's
// first slice: plan row i -> (slice, lane)
__device__ __forceinline__ void f2c_where(long long i, int goff1, int gs1, long long& s, int& lane) {
  if (i < goff1) { s = i >> 5; lane = (int)(i & 31); }
  else { s = gs1 + ((i - goff1) >> 5); lane = (int)((i - goff1) & 31); }
}

template <int B>
__global__ void __launch_bounds__(256) k_f2c_colour0(int s1, int goff1, SliceMap map, Sell a,
                                                     double* __restrict__ inv,
                                                     double* __restrict__ dtiles, int* bad,
                                                     int* shape_bad) {
  constexpr int BB = B * B;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < s1; s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = a.sp[s];
    const int width = (a.sp[s + 1] - slot0) >> 5;
    double out[BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) out[e] = 0.0;
    if (ok) {
      bool shape = a.cols[slot0 + lane] != i;    // entry 0 must be the diagonal
      for (int k = 1; k < width; ++k) {
        const int c = a.cols[slot0 + 32 * k + lane];
        shape |= c >= 0 && c < goff1;             // off-diagonals all in colour 1
      }
      if (shape) atomicExch(shape_bad, 1);
      double d[BB];
#pragma unroll
      for (int e = 0; e < BB; ++e) d[e] = a.vals[vidx(slot0, 0, e, lane, BB)];
      if (!invert_block<B>(d, out)) atomicMin(bad, (int)i);
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        out[e] = canon(out[e]);
        inv[i * BB + e] = out[e];
      }
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dtiles[((long long)s * BB + e) * 32 + lane] = out[e];
  }
}

template <int B>
__global__ void __launch_bounds__(256) k_f2c_colour1(int s1, int nslices, int goff1, SliceMap map,
                                                     Sell a, Sell lo, double* __restrict__ inv,
                                                     double* __restrict__ udiag,
                                                     double* __restrict__ dtiles, int* bad,
                                                     int* shape_bad) {
  constexpr int BB = B * B;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = s1 + gw; s < nslices; s += nw) {
    const bool ok = lane < map.nrows[s];
    const long long i = (long long)map.row0[s] + lane;
    const int slot0 = a.sp[s];
    const int width = (a.sp[s + 1] - slot0) >> 5;
    const int lslot0 = lo.sp[s];
    const int lwidth = (lo.sp[s + 1] - lslot0) >> 5;
    double outv[BB];
#pragma unroll
    for (int e = 0; e < BB; ++e) outv[e] = 0.0;
    int cnt = 0;
    if (ok) {
      while (cnt < width && a.cols[slot0 + 32 * cnt + lane] >= 0) ++cnt;
      bool shape = cnt < 1 || a.cols[slot0 + 32 * (cnt - 1) + lane] != i;  // diagonal last
      double d[BB];
#pragma unroll
      for (int e = 0; e < BB; ++e) d[e] = shape ? 0.0 : a.vals[vidx(slot0, cnt - 1, e, lane, BB)];
      for (int k = 0; k + 1 < cnt && !shape; ++k) {
        const int c = a.cols[slot0 + 32 * k + lane];
        if (c >= goff1) { shape = true; break; }   // lower entries all in colour 0
        double aik[BB], ic[BB], l[BB], urq[BB], prod[BB];
#pragma unroll
        for (int e = 0; e < BB; ++e) {
          aik[e] = a.vals[vidx(slot0, k, e, lane, BB)];
          ic[e] = inv[(long long)c * BB + e];
        }
        // A_ci: row c (colour 0) holds column i among its entries 1..
        long long sc;
        int lc;
        f2c_where(c, goff1, s1, sc, lc);
        const int cs0 = a.sp[sc], cw = (a.sp[sc + 1] - cs0) >> 5;
        int m = 1;
        while (m < cw && a.cols[cs0 + 32 * m + lc] != i) ++m;
        if (m >= cw) { shape = true; break; }     // unsymmetric pattern: general path
#pragma unroll
        for (int e = 0; e < BB; ++e) urq[e] = a.vals[vidx(cs0, m, e, lc, BB)];
        matmul<B>(aik, ic, l);                     // L_ic = A_ic inv(U_cc)
#pragma unroll
        for (int e = 0; e < BB; ++e) const_cast<double*>(lo.vals)[vidx(lslot0, k, e, lane, BB)] = l[e];
        const_cast<int32_t*>(lo.cols)[lslot0 + 32 * k + lane] = c;
        matmul<B>(l, urq, prod);                   // A_ii -= L_ic U_ci
#pragma unroll
        for (int e = 0; e < BB; ++e) d[e] -= prod[e];
      }
      if (shape) atomicExch(shape_bad, 1);
#pragma unroll
      for (int e = 0; e < BB; ++e) udiag[(i - goff1) * BB + e] = d[e];
      if (!invert_block<B>(d, outv)) atomicMin(bad, (int)i);
#pragma unroll
      for (int e = 0; e < BB; ++e) {
        outv[e] = canon(outv[e]);
        inv[i * BB + e] = outv[e];
      }
    }
    for (int k = ok ? cnt - 1 : 0; k < lwidth; ++k) {   // padding of the lower layout
      const_cast<int32_t*>(lo.cols)[lslot0 + 32 * k + lane] = -1;
#pragma unroll
      for (int e = 0; e < BB; ++e) const_cast<double*>(lo.vals)[vidx(lslot0, k, e, lane, BB)] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < BB; ++e) dtiles[((long long)s * BB + e) * 32 + lane] = outv[e];
  }
}

// plan-order CSR of the combined factors (the reference's `combined`)
template <int B>
__global__ void k_f2c_combined(int n, int goff1, int s1, const int32_t* __restrict__ rp, Sell a,
                               Sell lo, const double* __restrict__ udiag, double* __restrict__ lu) {
  constexpr int BB = B * B;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    long long s;
    int lane;
    f2c_where(i, goff1, s1, s, lane);
    const int q0 = rp[i], cnt = rp[i + 1] - q0;
    for (int k = 0; k < cnt; ++k) {
      double* dst = lu + (long long)(q0 + k) * BB;
      if (i < goff1) {             // colour 0: U row = A row (diagonal first)
#pragma unroll
        for (int e = 0; e < BB; ++e) dst[e] = a.vals[vidx(a.sp[s], k, e, lane, BB)];
      } else if (k + 1 < cnt) {    // colour 1: L entries, then U_ii
#pragma unroll
        for (int e = 0; e < BB; ++e) dst[e] = lo.vals[vidx(lo.sp[s], k, e, lane, BB)];
      } else {
#pragma unroll
        for (int e = 0; e < BB; ++e) dst[e] = udiag[(i - goff1) * BB + e];
      }
    }
  }
}

inline int f2c_grid(long long work) {
  long long g = (work + 255) / 256;
  if (g < 1) g = 1;
  if (g > kSms * 16) g = kSms * 16;
  return (int)g;
}

template <int B>
int f2c_factor_b(int n, int goff1, int s1, int nslices, SliceMap map, Sell a, Sell lo,
                 double* inv, double* udiag, double* dtiles, int* flags, cudaStream_t st) {
  if (s1 > 0)
    k_f2c_colour0<B><<<f2c_grid((long long)s1 * 32), 256, 0, st>>>(s1, goff1, map, a, inv, dtiles,
                                                                   flags, flags + 1);
  if (nslices > s1)
    k_f2c_colour1<B><<<f2c_grid((long long)(nslices - s1) * 32), 256, 0, st>>>(
        s1, nslices, goff1, map, a, lo, inv, udiag, dtiles, flags, flags + 1);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// Two-colour factorisation on the operator's SELL layout (see top).  s1 =
// first slice of colour 1, goff1 = its first plan row.  lo: the strict-lower
// SELL offsets (b2s_sell_offsets sel 1 on the plan-order pattern) with
// cols/vals to fill.  inv: n*b*b row-major inverses (plan order); udiag:
// (n-goff1)*b*b U_ii of colour 1; dtiles: per-slice inverse tiles.
// B2S_SINGULAR_PIVOT with the smallest failing plan row in *bad_row_host;
// B2S_UNSUPPORTED when the pattern is not a two-colour structure (caller
// falls back to the general factorisation).
static int f2c_launch(int n, int b, int goff1, int s1, int nslices, const int32_t* row0,
                      const int32_t* nrows, const int32_t* a_sp, const int32_t* a_cols,
                      const double* a_vals, const int32_t* l_sp, int32_t* l_cols, double* l_vals,
                      double* inv, double* udiag, double* dtiles, int* flags, cudaStream_t st) {
  SliceMap map{nslices, row0, nrows};
  Sell a{a_sp, a_cols, a_vals};
  Sell lo{l_sp, l_cols, l_vals};
  switch (b) {
    case 1: return f2c_factor_b<1>(n, goff1, s1, nslices, map, a, lo, inv, udiag, dtiles, flags, st);
    case 2: return f2c_factor_b<2>(n, goff1, s1, nslices, map, a, lo, inv, udiag, dtiles, flags, st);
    case 3: return f2c_factor_b<3>(n, goff1, s1, nslices, map, a, lo, inv, udiag, dtiles, flags, st);
    case 4: return f2c_factor_b<4>(n, goff1, s1, nslices, map, a, lo, inv, udiag, dtiles, flags, st);
  }
  return B2S_UNSUPPORTED;
}

int b2s_factor_2colour(int n, int b, int goff1, int s1, int nslices, const int32_t* row0,
                       const int32_t* nrows, const int32_t* a_sp, const int32_t* a_cols,
                       const double* a_vals, const int32_t* l_sp, int32_t* l_cols,
                       double* l_vals, double* inv, double* udiag, double* dtiles,
                       int32_t* bad_row_host, cudaStream_t st) {
  *bad_row_host = -1;
  if (n <= 0 || b < 1 || b > 4 || goff1 < 0 || goff1 > n || s1 < 0 || s1 > nslices)
    return B2S_SHAPE;
  int* flags = nullptr;
  B2S_CHECK(cudaMallocAsync(&flags, 2 * sizeof(int), st));
  const int init[2] = {0x7fffffff, 0};
  B2S_CHECK(cudaMemcpyAsync(flags, init, sizeof(init), cudaMemcpyHostToDevice, st));
  const int rc = f2c_launch(n, b, goff1, s1, nslices, row0, nrows, a_sp, a_cols, a_vals, l_sp,
                            l_cols, l_vals, inv, udiag, dtiles, flags, st);
  if (rc) return rc;
  int h[2];
  B2S_CHECK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st));
  B2S_CHECK(cudaFreeAsync(flags, st));
  B2S_CHECK(cudaStreamSynchronize(st));
  if (h[1]) return B2S_UNSUPPORTED;
  if (h[0] != 0x7fffffff) {
    *bad_row_host = h[0];
    return B2S_SINGULAR_PIVOT;
  }
  return B2S_OK;
}

// The same without the host read: flags_dev (2 ints, device) must hold
// {INT32_MAX, 0} on entry and receives {smallest singular plan row or
// INT32_MAX, 1 if the pattern is not a two-colour structure}; the caller
// reads them at a later synchronisation (stream-ordered, no sync here).
int b2s_factor_2colour_async(int n, int b, int goff1, int s1, int nslices, const int32_t* row0,
                             const int32_t* nrows, const int32_t* a_sp, const int32_t* a_cols,
                             const double* a_vals, const int32_t* l_sp, int32_t* l_cols,
                             double* l_vals, double* inv, double* udiag, double* dtiles,
                             int* flags_dev, cudaStream_t st) {
  if (n <= 0 || b < 1 || b > 4 || goff1 < 0 || goff1 > n || s1 < 0 || s1 > nslices || !flags_dev)
    return B2S_SHAPE;
  return f2c_launch(n, b, goff1, s1, nslices, row0, nrows, a_sp, a_cols, a_vals, l_sp, l_cols,
                    l_vals, inv, udiag, dtiles, flags_dev, st);
}

int b2s_factor_2colour_combined(int n, int b, int goff1, int s1, const int32_t* rp,
                                const int32_t* a_sp, const int32_t* a_cols, const double* a_vals,
                                const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                                const double* udiag, double* lu, cudaStream_t st) {
  if (n < 0 || b < 1 || b > 4) return B2S_SHAPE;
  if (n == 0) return B2S_OK;
  Sell a{a_sp, a_cols, a_vals}, lo{l_sp, l_cols, const_cast<double*>(l_vals)};
  const int g = f2c_grid(n);
  switch (b) {
    case 1: k_f2c_combined<1><<<g, 256, 0, st>>>(n, goff1, s1, rp, a, lo, udiag, lu); break;
    case 2: k_f2c_combined<2><<<g, 256, 0, st>>>(n, goff1, s1, rp, a, lo, udiag, lu); break;
    case 3: k_f2c_combined<3><<<g, 256, 0, st>>>(n, goff1, s1, rp, a, lo, udiag, lu); break;
    case 4: k_f2c_combined<4><<<g, 256, 0, st>>>(n, goff1, s1, rp, a, lo, udiag, lu); break;
  }
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

}  // extern "C"
