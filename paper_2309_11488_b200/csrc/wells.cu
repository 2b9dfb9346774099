// Well terms applied separately after the SpMV (bs/wells.py:125-162,
// bs/krylov.py:84-94): y -= C^T (D^-1 (B x)) for every standard well (D^-1
// stored) and every multi-segment well (D applied through its pivoted dense
// LU factors, scipy lu_factor layout).
//
// Two passes, both deterministic:
//   1. one warp per well: t1 = B x accumulated entry by entry (the
//      reference's einsum / np.add.at order over perforations), then
//      t2 = D^-1 t1 (standard: the stored inverse; multi-segment: row
//      interchanges, unit-lower and upper triangular solves, LAPACK getrs);
//   2. one thread per perforated cell: y[cell] -= C_e^T t2(well of e) for the
//      cell's entries in well order (all standard wells first, then the
//      multi-segment ones, as WellSet.apply_contributions does), so a cell
//      shared by several wells sees the reference's subtraction order.
#include "common.cuh"
#include "sell.cuh"

namespace b2s {

struct WellsDev {
  int nwells, nb;               // wells (standard then multi-segment), cell block size N
  const int32_t* kind;          // [nwells] 0 standard, 1 multi-segment
  const int32_t* M;             // [nwells] well-equation block height
  const int32_t* nseg;          // [nwells] segments (1 for standard wells)
  const int32_t* bptr;          // [nwells+1] B entries of well w
  const int32_t* bcell;         // [nbent] perforated cell of B entry e
  const int32_t* bseg;          // [nbent] segment of B entry e
  const int64_t* boff;          // [nbent] offset of B entry e's MxN block in bvals
  const double* bvals;
  const int64_t* doff;          // [nwells] D^-1 (standard) or LU (multi-segment) offset
  const double* dvals;
  const int64_t* pivoff;        // [nwells] pivot offset (multi-segment)
  const int32_t* piv;           // scipy/LAPACK row interchanges (0-based)
  const int64_t* toff;          // [nwells] offset of t2 (nseg*M doubles) in the scratch
  int ncells;                   // distinct cells touched by some C entry
  const int32_t* cells;         // [ncells]
  const int32_t* cptr;          // [ncells+1] C entries of each cell, in well order
  const int64_t* ccoff;         // [ncent] offset of the MxN C block in cvals
  const int64_t* ct2;           // [ncent] offset of the entry's M-vector of t2
  const int32_t* cM;            // [ncent] its M
  const double* cvals;
};


// pass 1: t2 of well w (one warp)
__global__ void k_wells_t2(WellsDev W, const double* __restrict__ x, double* __restrict__ t2,
                           const int* done) {
  griddep_wait();   // programmatic launch inside the Krylov graph
  griddep_launch();
  if (done && *done) return;
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= W.nwells) return;
  const int M = W.M[w], S = W.nseg[w] * M, N = W.nb;
  double* t = t2 + W.toff[w];
  if (W.kind[w] == 0 && M <= 8) {
    // standard well: lane j computes B_e x_cell of entry e = e0 + j (the
    // loads of all perforations in flight at once, not one dependent chain
    // per entry), then every lane sums the entries' vectors in entry order
    // through shuffles -- the same additions in the same order as the
    // sequential loop below, so t1 is bit-identical
    const int e0 = W.bptr[w], e1 = W.bptr[w + 1];
    double acc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc[m] = 0.0;
    for (int eb = e0; eb < e1; eb += 32) {
      const int e = eb + lane;
      double sv[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) sv[m] = 0.0;
      if (e < e1) {
        const double* blk = W.bvals + W.boff[e];
        const double* xc = x + (long long)W.bcell[e] * N;
        double xv[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) xv[c] = c < N ? xc[c] : 0.0;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (m < M) {
            double sm = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c)
              if (c < N) sm = fma(blk[m * N + c], xv[c], sm);
            sv[m] = sm;
          }
        }
      }
      const int cnt = e1 - eb < 32 ? e1 - eb : 32;
      for (int j = 0; j < cnt; ++j) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const double v = __shfl_sync(0xffffffffu, sv[m], j);
          if (m < M) acc[m] += v;
        }
      }
    }
    // t2 = D^-1 t1 (one lane per row)
    double r = 0.0;
    const double* dinv = W.dvals + W.doff[w];
    if (lane < M) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < M) r = fma(dinv[lane * M + c], acc[c], r);
      t[lane] = r;
    }
    return;
  }
  // t1: lane q owns entries q, q+32, ... of the nseg*M vector; entries of B
  // are visited in order, each adds its M-vector B_e x_cell
  for (int q = lane; q < S; q += 32) t[q] = 0.0;
  __syncwarp();
  for (int e = W.bptr[w]; e < W.bptr[w + 1]; ++e) {
    const double* blk = W.bvals + W.boff[e];
    const double* xc = x + (long long)W.bcell[e] * N;
    const int base = W.bseg[e] * M;
    for (int m = lane; m < M; m += 32) {
      double s = 0.0;
      for (int c = 0; c < N; ++c) s = fma(blk[m * N + c], xc[c], s);
      t[base + m] += s;
    }
    __syncwarp();
  }
  if (W.kind[w] == 0) {   // standard: t2 = D^-1 t1 (M <= 32: one lane per row)
    double r = 0.0;
    const double* dinv = W.dvals + W.doff[w];
    if (lane < M)
      for (int c = 0; c < M; ++c) r = fma(dinv[lane * M + c], t[c], r);
    __syncwarp();
    if (lane < M) t[lane] = r;
    __syncwarp();
    return;
  }
  // multi-segment: getrs with the packed LU (row-major S x S) and pivots
  const double* lu = W.dvals + W.doff[w];
  const int32_t* pv = W.piv + W.pivoff[w];
  if (lane == 0) {
    for (int i = 0; i < S; ++i) {          // row interchanges
      const int p = pv[i];
      if (p != i) { const double tmp = t[i]; t[i] = t[p]; t[p] = tmp; }
    }
  }
  __syncwarp();
  for (int i = 0; i < S; ++i) {            // L y = P t (unit lower)
    double s = 0.0;
    for (int c = lane; c < i; c += 32) s = fma(lu[(long long)i * S + c], t[c], s);
    s = warp_sum(s);
    if (lane == 0) t[i] -= s;
    __syncwarp();
  }
  for (int i = S - 1; i >= 0; --i) {       // U z = y
    double s = 0.0;
    for (int c = i + 1 + lane; c < S; c += 32) s = fma(lu[(long long)i * S + c], t[c], s);
    s = warp_sum(s);
    if (lane == 0) t[i] = (t[i] - s) / lu[(long long)i * S + i];
    __syncwarp();
  }
}

// pass 2: y[cell] -= C_e^T t2 for the cell's entries in well order
__global__ void k_wells_apply(WellsDev W, const double* __restrict__ t2, double* y) {
  const int N = W.nb;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W.ncells; q += gridDim.x * blockDim.x) {
    double* yc = y + (long long)W.cells[q] * N;
    for (int e = W.cptr[q]; e < W.cptr[q + 1]; ++e) {
      const double* blk = W.cvals + W.ccoff[e];
      const double* tv = t2 + W.ct2[e];
      const int M = W.cM[e];
      for (int c = 0; c < N; ++c) {
        double s = 0.0;
        for (int m = 0; m < M; ++m) s = fma(blk[m * N + c], tv[m], s);
        yc[c] -= s;
      }
    }
  }
}

// inside the device Krylov loop: corr[q] = sum of the cell's C_e^T t2 in
// well order; the SpMV epilogue subtracts it (sell.cuh WellFix)
__global__ void k_wells_corr(WellsDev W, const double* __restrict__ t2, double* __restrict__ corr,
                             const int* done) {
  griddep_wait();   // programmatic launch inside the Krylov graph
  griddep_launch();
  if (done && *done) return;
  const int N = W.nb;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < W.ncells; q += gridDim.x * blockDim.x) {
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (int e = W.cptr[q]; e < W.cptr[q + 1]; ++e) {
      const double* blk = W.cvals + W.ccoff[e];
      const double* tv = t2 + W.ct2[e];
      const int M = W.cM[e];
      for (int c = 0; c < N; ++c) {
        double s = 0.0;
        for (int m = 0; m < M; ++m) s = fma(blk[m * N + c], tv[m], s);
        tot[c] += s;
      }
    }
    for (int c = 0; c < N; ++c) corr[(long long)q * N + c] = tot[c];
  }
}

static WellsDev wells_dev(const b2s_wells* w) {
  return WellsDev{w->nwells, w->nb,  w->kind,   w->M,    w->nseg,  w->bptr,  w->bcell,
                  w->bseg,   w->boff, w->bvals, w->doff, w->dvals, w->pivoff, w->piv,
                  w->toff,   w->ncells, w->cells, w->cptr, w->ccoff, w->ct2,  w->cM,
                  w->cvals};
}

int launch_wells_corr(const b2s_wells* w, const double* x, double* scratch, double* corr,
                      const int* done, cudaStream_t st, bool pdl) {
  if (!w || w->nwells < 0 || w->nb < 1 || w->nb > 4) return B2S_SHAPE;
  if (w->nwells == 0) return B2S_OK;
  const WellsDev W = wells_dev(w);
  launch_k(k_wells_t2, dim3((w->nwells + 7) / 8), dim3(256), 0, st, pdl, W, x, scratch, done);
  const int g = (w->ncells + 255) / 256;
  launch_k(k_wells_corr, dim3(g < 1 ? 1 : g), dim3(256), 0, st, pdl, W, (const double*)scratch,
           corr, done);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

// Fused 2-colour passes with wells: the colour-0 rows of v (t) were written by
// the fused backward+SpMV pass before p^ (s^) was complete, so their well
// terms are subtracted here, after launch_wells_corr, together with the
// change of that pass's dot-product partials (one CTA, one partial slot):
// mode 1: gamma += r^.(v_new - v_old); mode 2: t.t += t_new^2 - t_old^2,
// t.s += s.(t_new - t_old).  Colour-1 rows get theirs in the SpMV epilogue.
__global__ void k_wells_patch(const int32_t* __restrict__ cells, int ncells, int nb, int goff1,
                              const double* __restrict__ corr, double* v,
                              const double* __restrict__ w, int mode, double* p0, double* p1,
                              const int* done, SImgPatch sp) {
  __shared__ double red[8];
  griddep_wait();   // programmatic launch inside the Krylov graph
  griddep_launch();
  if (done && *done) return;
  double a0 = 0.0, a1 = 0.0;
  for (int q = threadIdx.x; q < ncells; q += blockDim.x) {
    const long long row = cells[q];
    if (row >= goff1) continue;
    double vr[4];
    for (int c = 0; c < nb; ++c) {
      const double vo = v[row * nb + c];
      const double vn = vo - corr[(long long)q * nb + c];
      v[row * nb + c] = vn;
      vr[c] = vn;
      const double wv = w[row * nb + c];
      if (mode == 1) a0 += wv * vn - wv * vo;
      else { a0 += vn * vn - vo * vo; a1 += wv * vn - wv * vo; }
    }
    if (sp.u) {   // s-image: u_i = inv(A_ii) v_i again for the patched row
      int lo = 0, hi = sp.nslices - 1;   // the slice holding the row (row0 ascending)
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sp.row0[mid] <= row) lo = mid; else hi = mid - 1;
      }
      const long long lane = row - sp.row0[lo];
      const int bb = nb * nb;
      for (int e = 0; e < nb; ++e) {
        double acc = 0.0;
        for (int c = 0; c < nb; ++c)
          acc = fma(sp.dtiles[((long long)lo * bb + e * nb + c) * 32 + lane], vr[c], acc);
        sp.u[row * nb + e] = acc;
      }
    }
  }
  const double t0 = block_sum(a0, red);
  if (threadIdx.x == 0) *p0 = t0;
  if (mode == 2) {
    const double t1 = block_sum(a1, red);
    if (threadIdx.x == 0) *p1 = t1;
  }
}

int launch_wells_patch(const b2s_wells* w, int goff1, const double* corr, double* v,
                       const double* wv, int mode, double* p0, double* p1, const int* done,
                       cudaStream_t st, SImgPatch sp, bool pdl) {
  launch_k(k_wells_patch, dim3(1), dim3(256), 0, st, pdl, (const int32_t*)w->cells, w->ncells,
           w->nb, goff1, corr, v, wv, mode, p0, p1, done, sp);
  return cudaGetLastError() == cudaSuccess ? B2S_OK : B2S_CUDA_ERROR;
}

}  // namespace b2s

using namespace b2s;

extern "C" {

// y -= sum over wells of C^T D^-1 B x  (x, y: block vectors of the cells)
int b2s_wells_apply(const b2s_wells* w, const double* x, double* y, double* scratch,
                    cudaStream_t st) {
  if (!w || w->nwells < 0 || w->nb < 1) return B2S_SHAPE;
  if (w->nwells == 0) return B2S_OK;
  const WellsDev W = wells_dev(w);
  const int warps = w->nwells;
  k_wells_t2<<<(warps + 7) / 8, 256, 0, st>>>(W, x, scratch, nullptr);
  const int g = (w->ncells + 255) / 256;
  k_wells_apply<<<g < 1 ? 1 : g, 256, 0, st>>>(W, scratch, y);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

}  // extern "C"
