// Right-preconditioned BiCGStab (bs/krylov.py:140-244), device resident.
//
// One iteration is a fixed sequence of stream-ordered kernels captured once
// into a CUDA graph and replayed; the host only polls a pinned "done" word a
// couple of iterations behind the GPU, so the device never idles on the
// host.  Control decisions (breakdown floors, convergence tests, half-step
// counting, the order of the reference's exits) run in the last CTA of the
// kernel that produces the partial sums they need (ctl.cuh): that CTA is the
// only writer of the solver state; every kernel reads `state->done` first
// and becomes a no-op once the solve has ended, which reproduces the
// reference's early exits exactly even though later kernels of the
// iteration are already queued.  Nine kernels per iteration, no 1-CTA
// control kernels in between.
//
// Vector passes per iteration (fused so each vector is touched as few times
// as possible; partial sums go to fixed per-CTA slots and are reduced in a
// fixed order, so every run is bit-identical):
//   p  = r + beta (p - omega v)                       (1 kernel)
//   p^ = M^-1 p                                       (fwd + bwd sweep)
//   v  = A p^,  gamma partials r^.v                   (SpMV epilogue)
//   s  = r - alpha v,  x += alpha p^,  |s|^2 partials (1 kernel)
//   s^ = M^-1 s                                       (fwd + bwd sweep)
//   t  = A s^,  (t.t, t.s) partials                   (SpMV epilogue)
//   x += omega s^, r = s - omega t, |r|^2 and r^.r partials (1 kernel)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cstring>
#include <mutex>
#include <vector>
#include <cuda.h>

#include "ctl.cuh"
#include "sell.cuh"

namespace b2s {

int launch_spmv(int b, int mode, int nparts, SliceMap map, Sell a, const double* x, double* y,
                const double* w, double* p0, double* p1, const int* done, Ctl ctl,
                cudaStream_t st, bool pdl = false, WellFix wf = WellFix{});
int launch_sweeps(int b, int kc, SliceMap map, Sell lo, Sell up, const double* dt,
                  const double* r, double* y, double* z, int reset_y, int flags, void* tickets,
                  const int* done, cudaStream_t st);
int fill_sentinel(long long m, double* v, cudaStream_t st);
int launch_phased(int b, int kc, int ngroups, const int32_t* gslice_host, int goff1, SliceMap map,
                  Sell lo, Sell up, const double* dt, const double* r, double* y, double* z,
                  const int* done, cudaStream_t st, bool skip_g0, bool pdl = false);
int launch_spmv_range(int b, int mode, int nparts, SliceMap map, int s0, int s1, int poff, Sell a,
                      const double* x, double* y, const double* w, double* p0, double* p1,
                      const int* done, Ctl ctl, cudaStream_t st, bool pdl = false,
                      WellFix wf = WellFix{});
int launch_wells_corr(const b2s_wells* w, const double* x, double* scratch, double* corr,
                      const int* done, cudaStream_t st, bool pdl = false);
int launch_wells_patch(const b2s_wells* w, int goff1, const double* corr, double* v,
                       const double* wv, int mode, double* p0, double* p1, const int* done,
                       cudaStream_t st, SImgPatch sp = SImgPatch{}, bool pdl = false);
int launch_bwd_spmv(int b, int mode, int nparts, SliceMap map, int s1, Sell a, const double* dt,
                    const double* yin, double* z, double* v, const double* w, double* p0,
                    double* p1, const int* done, int* grid_out, cudaStream_t st,
                    bool pdl = false, int pre = kPreNone, const PreIn* pre_in = nullptr,
                    double* uimg = nullptr);
int launch_simg(int b, int stage, int nparts, SliceMap map, int s0, int s1, int poff, Sell m_,
                const double* dt, const double* in0, const double* in1, double* out0,
                double* out1, double* parts, const int* done, Ctl ctl, int goff1,
                const double* u, double* fv, long long mlen, const State* st, cudaStream_t q,
                bool pdl, WellFix wf = WellFix{});
int launch_fwd_pre(int b, int nparts, SliceMap map, int s0, int s1, Sell lo, const double* dt,
                   double* z, const int* done, int* grid_out, cudaStream_t st, bool pdl, int pre,
                   const PreIn* pre_in);
int launch_tiled(int b, const void* handle, const double* r, double* y, double* z, int reset_y,
                 const int* done, cudaStream_t st);
int launch_gw(int b, const void* handle, const double* r, double* z, const int* done,
              cudaStream_t st, bool pdl);

// deterministic sum of np partials by one CTA of 256 threads
__device__ double reduce_parts(const double* parts, int np, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += parts[i];
  return block_sum(v, red);  // valid in thread 0
}

__global__ void k_ctl_init(State* st, const double* prr, int np, double tol, int maxit,
                           int* host_done, MeshDev mesh) {
  __shared__ double red[8];
  double s = reduce_parts(prr, np, red);
  if (threadIdx.x == 0) {
    if (!mesh.mbox) { st->cseq = 0; st->pub = 0; }
    bool ok = true;
    if (mesh.mbox) {   // sharded: |r0|^2 over every rank
      double unused = 0.0;
      ok = mesh_sum(mesh, mesh.seq_base + (++st->cseq), kSlotInit, s, unused);
    }
    const double n0 = sqrt(s);
    st->rho = 0.0; st->rho_prev = 1.0; st->alpha = 1.0; st->omega = 1.0; st->beta = 0.0;
    st->xpend = 0;
    st->norm0 = n0; st->target = tol * n0; st->final_norm = n0; st->its = 0.0;
    st->k = 0; st->maxit = maxit; st->reason = kRunning;
    st->done = 0;
    if (!ok) { st->done = 1; st->reason = kAborted; }
    else if (!isfinite(n0)) { st->done = 1; st->reason = kNumerical; }
    else if (n0 <= st->target || n0 == 0.0) { st->done = 1; st->reason = kConverged; }
    // top of iteration 0 (maxit >= 1): rho_0 = rhat.r0 = the same partials
    else if (fabs(s) < kBreakdown) { st->done = 1; st->reason = kBreakdownR; }
    else st->rho = s;
    // no iteration needed: let the host's replay loop stop at its first check
    st->init_exit = st->done;
    if (st->done && host_done) *reinterpret_cast<volatile int*>(host_done) = 1;
  }
}

// ---- sharded solves: ghost rows straight from the owners' vectors
struct MeshHalo {
  int rank, nranks, nghost, nnbr;
  const int32_t* nbr;
  const int32_t* ghost_owner;
  const int32_t* ghost_row;
  double* const* peer_vec[3];   // x, phat, shat of every rank
  long long* flags;             // posted by peers: "vector #seq is ready"
  long long* const* peer_flags;
  long long seq_base;
  double* mbox;                 // this rank's mailbox (its abort word) ...
  double* const* peer_mbox;     // ... and every rank's
  long long timeout_ns;
};

__global__ void k_zero_words(unsigned* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0u;
}

__global__ void k_mesh_raise_abort(MeshDev m) { mesh_raise_abort(m.peer_mbox, m.nranks); }

__global__ void k_mesh_reset(State* st) {
  st->done = 0;
  st->pub = 0;
  st->cseq = 0;
}

// one thread: this rank's vector (the kernels before it in the stream) is
// complete -- post the sequence number into every rank's flags
__global__ void k_mesh_publish(State* st, MeshHalo h, const int* done) {
  if (done && *done) return;
  const long long seq = h.seq_base + (++st->pub);
  __threadfence_system();
  for (int q = 0; q < h.nranks; ++q) st_release_sys(h.peer_flags[q] + h.rank, seq);
}
// one CTA: wait until every neighbour posted the same vector (a separate
// kernel, so waiting never holds more than one SM); a neighbour that does
// not post in time (or an abort raised anywhere) ends the solve on every
// rank: the kernels after this one no-op, the host sees kAborted
__global__ void k_mesh_wait(State* st, MeshHalo h, const int* done, int* host_done) {
  if (done && *done) return;
  const long long seq = h.seq_base + st->pub;
  bool ok = true;
  for (int k = threadIdx.x; k < h.nnbr; k += blockDim.x) {
    const long long* f = h.flags + h.nbr[k];
    ok &= wait_ge(f, seq, h.mbox, h.nranks, h.timeout_ns);
  }
  if (__syncthreads_or(!ok) && threadIdx.x == 0) {
    mesh_raise_abort(h.peer_mbox, h.nranks);
    st->reason = kAborted;
    st->done = 1;
    __threadfence();
    if (host_done) *reinterpret_cast<volatile int*>(host_done) = 1;
  }
}
// ghost rows of vector `which` (0 x, 1 phat, 2 shat) -> dst (after the owned rows)
__global__ void k_mesh_pull(MeshHalo h, int which, int b, double* dst, const int* done) {
  if (done && *done) return;
  const long long total = (long long)h.nghost * b;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long g = t / b;
    const int c = (int)(t - g * b);
    const double* src = h.peer_vec[which][h.ghost_owner[g]];
    dst[t] = __ldcg(src + (long long)h.ghost_row[g] * b + c);
  }
}
// all-reduce of a local partial array (or of a flag) into out[0]
__global__ void k_mesh_scalar(State* st, MeshDev mesh, int slot, const double* parts, int np,
                              const int* flag, double* out) {
  __shared__ double red[8];
  double v = 0.0;
  if (parts) v = reduce_parts(parts, np, red);
  if (threadIdx.x == 0) {
    if (flag) v = *flag ? 1.0 : 0.0;
    double unused = 0.0;
    if (mesh.mbox && !mesh_sum(mesh, mesh.seq_base + (++st->cseq), slot, v, unused))
      st->reason = kAborted;   // v is NaN; b2s_bicgstab reports B2S_PEER_TIMEOUT
    out[0] = v;
  }
}

// Sharded 2-colour solves: the fused passes ran on the local block; add the
// ghost couplings of the boundary rows (pulled just before) and their share
// of the fused dot products, then run the control step over every partial
// (the local kernels' at [0, poff), these at [poff, poff + grid)).  The
// ghost entries are the last ones of their rows, so the row sum simply
// continues in column order.  kResidual: y = w - A_loc x already, subtract
// the ghost products (the r0 / final true residuals).
template <int B, int MODE>
__global__ void __launch_bounds__(256) k_ghost_correct(int nb, const int32_t* __restrict__ brow,
                                                       const int32_t* __restrict__ bptr,
                                                       const int32_t* __restrict__ bcol,
                                                       const double* __restrict__ bval,
                                                       const double* __restrict__ xg, double* y,
                                                       const double* __restrict__ w,
                                                       double* part0, double* part1, int poff,
                                                       const int* done, Ctl ctl) {
  constexpr int BB = B * B;
  __shared__ double red[8];
  if (done && *done) return;
  double p0 = 0.0, p1 = 0.0;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nb; q += gridDim.x * blockDim.x) {
    const long long row = brow[q];
    double yl[B], acc[B];
#pragma unroll
    for (int c = 0; c < B; ++c) acc[c] = yl[c] = y[row * B + c];
    for (int e = bptr[q]; e < bptr[q + 1]; ++e) {
      const long long g = bcol[e];
      double blk[BB], xv[B], pr[B];
#pragma unroll
      for (int k = 0; k < BB; ++k) blk[k] = bval[(long long)e * BB + k];
#pragma unroll
      for (int c = 0; c < B; ++c) xv[c] = __ldcg(xg + g * B + c);
      matvec<B>(blk, xv, pr);
#pragma unroll
      for (int c = 0; c < B; ++c) acc[c] = MODE == kResidual ? acc[c] - pr[c] : acc[c] + pr[c];
    }
#pragma unroll
    for (int c = 0; c < B; ++c) {
      y[row * B + c] = acc[c];
      const double d = acc[c] - yl[c];
      if (MODE == kResidual) p0 = fma(d, acc[c] + yl[c], p0);   // r.r: new^2 - old^2
      if (MODE == kDotW) p0 = fma(w[row * B + c], d, p0);
      if (MODE == kSelfAndW) {
        p0 = fma(d, acc[c] + yl[c], p0);   // t.t: new^2 - old^2
        p1 = fma(w[row * B + c], d, p1);
      }
    }
  }
  const double t0 = block_sum(p0, red);
  if (threadIdx.x == 0) part0[poff + blockIdx.x] = t0;
  if (MODE == kSelfAndW) {
    const double t1 = block_sum(p1, red);
    if (threadIdx.x == 0) part1[poff + blockIdx.x] = t1;
  }
  if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, part0, part1, poff + gridDim.x, red);
}
constexpr int kCorrCtas = 32;

template <int MODE>
void launch_ghost_correct(int b, const b2s_mesh* m, const double* xg, double* y, const double* w,
                          double* p0, double* p1, int poff, const int* done, Ctl ctl,
                          cudaStream_t st) {
  switch (b) {
    case 1: k_ghost_correct<1, MODE><<<kCorrCtas, 256, 0, st>>>(m->nbnd, m->bnd_row, m->bnd_ptr, m->bnd_col, m->bnd_val, xg, y, w, p0, p1, poff, done, ctl); break;
    case 2: k_ghost_correct<2, MODE><<<kCorrCtas, 256, 0, st>>>(m->nbnd, m->bnd_row, m->bnd_ptr, m->bnd_col, m->bnd_val, xg, y, w, p0, p1, poff, done, ctl); break;
    case 3: k_ghost_correct<3, MODE><<<kCorrCtas, 256, 0, st>>>(m->nbnd, m->bnd_row, m->bnd_ptr, m->bnd_col, m->bnd_val, xg, y, w, p0, p1, poff, done, ctl); break;
    default: k_ghost_correct<4, MODE><<<kCorrCtas, 256, 0, st>>>(m->nbnd, m->bnd_row, m->bnd_ptr, m->bnd_col, m->bnd_val, xg, y, w, p0, p1, poff, done, ctl); break;
  }
}

#define GRID_STRIDE(t, m) \
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (m); \
       t += (long long)gridDim.x * blockDim.x)

// Vector passes: 16-byte loads (double2) and two pairs in flight per thread
// per step (all loads of a step issued before its arithmetic); an odd tail
// element goes to thread 0 of CTA 0.  Callers guarantee 16-byte aligned
// vectors (workspace sub-buffers are 256-byte aligned; torch allocations
// 512-byte).  The per-thread accumulation order is fixed by (m, grid), so
// the partial sums are deterministic.
constexpr int kU = 2;   // element pairs in flight per thread in the vector passes

__device__ __forceinline__ double2 ld2(const double* p, long long j) {
  return __ldcs(reinterpret_cast<const double2*>(p) + j);
}
__device__ __forceinline__ void st2(double* p, long long j, double a, double b) {
  reinterpret_cast<double2*>(p)[j] = make_double2(a, b);
}

__global__ void __launch_bounds__(256, 4) k_p_update(long long m, const State* st,
                                                  const double* __restrict__ r,
                                                  const double* __restrict__ v, double* p) {
  griddep_wait();
  griddep_launch();
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, omega = st->omega;
  const long long m2 = m >> 1, T = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (k == 0) {
    for (; j < m2; j += T) {
      const double2 a = ld2(r, j);
      st2(p, j, a.x, a.y);
    }
    if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[m - 1] = r[m - 1];
    return;
  }
  for (; j < m2; j += kU * T) {
    double2 rr[kU], pp[kU], vv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2) { rr[u] = ld2(r, q); pp[u] = ld2(p, q); vv[u] = ld2(v, q); }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2)
        st2(p, q, bicg_p(rr[u].x, pp[u].x, vv[u].x, beta, omega),
            bicg_p(rr[u].y, pp[u].y, vv[u].y, beta, omega));
    }
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    p[m - 1] = bicg_p(r[m - 1], p[m - 1], v[m - 1], beta, omega);
}

// s = r - alpha v ; x += alpha p^ ; |s|^2 partials ; optionally p^ <- sentinel
__device__ __forceinline__ void s_elem(double rv, double vv, double ph, double& xo, double& so,
                                       double alpha, double& acc) {
  so = bicg_axpy(rv, alpha, vv);
  xo = bicg_xupd(xo, alpha, ph);
  acc = fma(so, so, acc);
}

// XU = false: x is left alone (x += alpha p^ deferred to the r-update,
// State.xpend): two vectors fewer to stream
template <bool XU>
__global__ void __launch_bounds__(256, 4) k_s_update(long long m, const State* st,
                                                  const double* __restrict__ r,
                                                  const double* __restrict__ v, double* phat,
                                                  double* __restrict__ x,
                                                  double* __restrict__ s, double* pss,
                                                  int reset, Ctl ctl) {
  __shared__ double red[8];
  griddep_wait();
  griddep_launch();
  if (st->done) return;
  const double alpha = st->alpha;
  double acc = 0.0;
  const long long m2 = m >> 1, T = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // kU pairs per thread in flight (every load issued before any store), in
  // the same per-thread order j, j+T, j+2T, ... as a plain grid-stride loop
  for (; j < m2; j += kU * T) {
    double2 rv[kU], vv[kU], ph[kU], xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        rv[u] = ld2(r, q); vv[u] = ld2(v, q);
        if (XU) {
          ph[u] = ld2(phat, q);
          xv[u] = reinterpret_cast<const double2*>(x)[q];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        double s0, s1;
        if (XU) {
          s_elem(rv[u].x, vv[u].x, ph[u].x, xv[u].x, s0, alpha, acc);
          s_elem(rv[u].y, vv[u].y, ph[u].y, xv[u].y, s1, alpha, acc);
          st2(x, q, xv[u].x, xv[u].y);
        } else {
          s0 = bicg_axpy(rv[u].x, alpha, vv[u].x);
          acc = fma(s0, s0, acc);
          s1 = bicg_axpy(rv[u].y, alpha, vv[u].y);
          acc = fma(s1, s1, acc);
        }
        st2(s, q, s0, s1);
        if (reset) st2(phat, q, sentinel(), sentinel());
      }
    }
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double s0;
    if (XU) {
      s_elem(r[m - 1], v[m - 1], phat[m - 1], x[m - 1], s0, alpha, acc);
    } else {
      s0 = bicg_axpy(r[m - 1], alpha, v[m - 1]);
      acc = fma(s0, s0, acc);
    }
    s[m - 1] = s0;
    if (reset) phat[m - 1] = sentinel();
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) pss[blockIdx.x] = tot;
  if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, pss, nullptr, gridDim.x, red);
}

// x += omega s^ ; r = s - omega t ; |r|^2 and r^.r partials ; s^ <- sentinel
__device__ __forceinline__ void r_elem(double sh, double tv, double sv, double rh, double& xo,
                                       double& ro, double omega, double& a0, double& a1) {
  xo = bicg_xupd(xo, omega, sh);
  ro = bicg_axpy(sv, omega, tv);
  a0 = fma(ro, ro, a0);
  a1 = fma(rh, ro, a1);
}

// XA (fused vector passes): x += alpha p^ happens here too, x = (x + alpha
// p^) + omega s^ with the same roundings as the two separate updates
template <bool XA>
__global__ void __launch_bounds__(256, 4) k_r_update(long long m, const State* st, double* shat,
                                                  const double* __restrict__ tv,
                                                  const double* __restrict__ s,
                                                  const double* __restrict__ rhat,
                                                  double* __restrict__ x,
                                                  double* __restrict__ r, double* prr,
                                                  double* prho, int reset, Ctl ctl,
                                                  const double* __restrict__ phat) {
  __shared__ double red[8];
  griddep_wait();
  griddep_launch();
  if (st->done) return;
  const double omega = st->omega, alpha = st->alpha;
  double a0 = 0.0, a1 = 0.0;
  const long long m2 = m >> 1, T = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; j < m2; j += kU * T) {
    double2 sh[kU], t2[kU], sv[kU], rh[kU], xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        sh[u] = ld2(shat, q); t2[u] = ld2(tv, q); sv[u] = ld2(s, q); rh[u] = ld2(rhat, q);
        xv[u] = reinterpret_cast<const double2*>(x)[q];
        if (XA) {
          const double2 ph = ld2(phat, q);
          xv[u].x = bicg_xupd(xv[u].x, alpha, ph.x);
          xv[u].y = bicg_xupd(xv[u].y, alpha, ph.y);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long long q = j + u * T;
      if (q < m2) {
        double r0, r1;
        r_elem(sh[u].x, t2[u].x, sv[u].x, rh[u].x, xv[u].x, r0, omega, a0, a1);
        r_elem(sh[u].y, t2[u].y, sv[u].y, rh[u].y, xv[u].y, r1, omega, a0, a1);
        st2(x, q, xv[u].x, xv[u].y);
        st2(r, q, r0, r1);
        if (reset) st2(shat, q, sentinel(), sentinel());
      }
    }
  }
  if ((m & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double r0;
    if (XA) x[m - 1] = bicg_xupd(x[m - 1], alpha, phat[m - 1]);
    r_elem(shat[m - 1], tv[m - 1], s[m - 1], rhat[m - 1], x[m - 1], r0, omega, a0, a1);
    r[m - 1] = r0;
    if (reset) shat[m - 1] = sentinel();
  }
  const double t0 = block_sum(a0, red);
  if (threadIdx.x == 0) prr[blockIdx.x] = t0;
  const double t1 = block_sum(a1, red);
  if (threadIdx.x == 0) prho[blockIdx.x] = t1;
  if (ctl.st && last_cta(ctl.counter)) ctl_run(ctl, prr, prho, gridDim.x, red);
}

// the fused vector passes end a solve between the s half-step and the
// r-update without x += alpha p^ (State.xpend): add it once, after the loop
__global__ void k_x_fixup(long long m, const State* st, const double* __restrict__ phat,
                          double* __restrict__ x) {
  if (!st->xpend) return;
  const double alpha = st->alpha;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m;
       t += (long long)gridDim.x * blockDim.x)
    x[t] = bicg_xupd(x[t], alpha, phat[t]);
}

template <class... P>
inline bool misaligned16(const P*... p) {
  return ((reinterpret_cast<uintptr_t>(p) | ...) & 15) != 0;
}

__global__ void k_copy(long long m, const double* __restrict__ a, double* __restrict__ b) {
  GRID_STRIDE(t, m) b[t] = a[t];
}

// per-CTA partials of a.b (fixed assignment: deterministic)
__global__ void __launch_bounds__(256) k_dot_parts(long long m, const double* __restrict__ a,
                                                   const double* __restrict__ b, double* parts) {
  __shared__ double red[8];
  double acc = 0.0;
  GRID_STRIDE(t, m) acc = fma(a[t], b[t], acc);
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) parts[blockIdx.x] = tot;
}

__global__ void k_reduce_parts(const double* parts, int np, double* out) {
  __shared__ double red[8];
  const double s = reduce_parts(parts, np, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_all_finite(long long m, const double* __restrict__ a, int* bad) {
  int local = 0;
  GRID_STRIDE(t, m) local |= !isfinite(a[t]);
  if (__any_sync(0xffffffffu, local) && (threadIdx.x & 31) == 0) atomicExch(bad, 1);
}


}  // namespace b2s

using namespace b2s;

namespace {
// Mapped page-locked words the host polls (one 64-byte line each), kept for
// the life of the process: a cudaHostAlloc + cudaFreeHost pair per solve
// measured 1-36 ms of host time inside the solve once the process holds a
// large device working set (the wavefront records), against 0.01 ms without.
std::mutex g_done_mu;
std::vector<int*> g_done_free;
int* done_acquire() {
  std::lock_guard<std::mutex> lk(g_done_mu);
  if (g_done_free.empty()) {
    char* blk = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&blk), 4096,
                      cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return nullptr;
    for (int i = 4096 / 64 - 1; i >= 0; --i) g_done_free.push_back(reinterpret_cast<int*>(blk + 64 * i));
  }
  int* w = g_done_free.back();
  g_done_free.pop_back();
  return w;
}
void done_release(int* w) {
  if (!w) return;
  std::lock_guard<std::mutex> lk(g_done_mu);
  g_done_free.push_back(w);
}

// A finished solve's graph, streams and events are destroyed at the start of
// the thread's next solve instead of at its end: the ~0.2 ms of host
// teardown then overlaps the caller's next device work instead of leaving
// the device idle between the loop and the caller's follow-up kernels.
struct Leftovers {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t streams[2] = {nullptr, nullptr};
  cudaEvent_t events[10] = {};
  int nev = 0;
  void destroy() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (cudaStream_t& s : streams)
      if (s) { cudaStreamDestroy(s); s = nullptr; }
    for (int i = 0; i < nev; ++i)
      if (events[i]) cudaEventDestroy(events[i]);
    exec = nullptr;
    graph = nullptr;
    nev = 0;
  }
};
thread_local Leftovers t_left;
}  // namespace

extern "C" {

static long long vec_doubles_g(int n, int nghost, int b) {
  long long m = (long long)(n + nghost) * b;
  return (m + 31) / 32 * 32;  // 256-byte aligned sub-buffers
}


long long b2s_bicgstab_workspace_bytes(int n, int b, int nparts) {
  return b2s_bicgstab_workspace_bytes_mesh(n, 0, b, nparts);
}

long long b2s_bicgstab_workspace_bytes_mesh(int n, int nghost, int b, int nparts) {
  const long long m = vec_doubles_g(n, nghost, b);
  // r rhat p v phat s shat t y x0  + 6 partial arrays (2 x nparts: the fused
  // 2-colour passes split a dot product over two kernels) + state + tickets
  return (10 * m + 6 * 2 * (long long)((nparts + 31) / 32 * 32)) * 8 + 256 + 64;
}

int b2s_bicgstab(const b2s_bicg_args* a, b2s_bicg_result* res) {
  res->converged = 0; res->reason = 0; res->graph_launches = 0; res->kernels_per_iteration = 0;
  res->iterations = 0.0; res->initial_norm = 0.0; res->final_norm = 0.0;
  if (a->n < 0 || a->b < 1 || a->nparts < 1 || a->maxit < 1) return B2S_SHAPE;
  if (a->b > 4) return B2S_UNSUPPORTED;
  // the vector passes use 16-byte loads
  if ((reinterpret_cast<uintptr_t>(a->x) | reinterpret_cast<uintptr_t>(a->rhs) |
       reinterpret_cast<uintptr_t>(a->work)) & 15)
    return B2S_SHAPE;
  t_left.destroy();   // the previous solve's graph and streams (this thread)
  // B2S_SOLVE_TIMING=1: host-side phase times of each solve on stderr
  static const bool tmg = getenv("B2S_SOLVE_TIMING") && getenv("B2S_SOLVE_TIMING")[0] == '1';
  using clk = std::chrono::steady_clock;
  clk::time_point tp[9];
  int ntp = 0;
  auto mark = [&]() { if (tmg && ntp < 9) tp[ntp++] = clk::now(); };
  mark();
  if (tmg) { cudaDeviceSynchronize(); mark(); }
  const long long m = (long long)a->n * a->b;
  const b2s_mesh* mesh = a->mesh;
  const int nghost = mesh ? mesh->nghost : 0;
  const long long mv = vec_doubles_g(a->n, nghost, a->b);
  const long long npv = 2 * ((a->nparts + 31) / 32 * 32);
  double* w = a->work;
  double *r = w, *rhat = w + mv, *p = w + 2 * mv, *v = w + 3 * mv, *phat = w + 4 * mv,
         *s = w + 5 * mv, *shat = w + 6 * mv, *t = w + 7 * mv, *y = w + 8 * mv,
         *x0 = w + 9 * mv;
  double* parts = w + 10 * mv;
  double *prr = parts, *prho = parts + npv, *pg = parts + 2 * npv, *pss = parts + 3 * npv,
         *ptt = parts + 4 * npv, *pts = parts + 5 * npv;
  State* state = reinterpret_cast<State*>(parts + 6 * npv);
  void* tickets = reinterpret_cast<char*>(state) + 256;  // 2 sweep ticket pairs (16 B)
  unsigned* counters = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(tickets) + 32);
  const bool ilu = a->precond == 1;
  const bool phased = ilu && !a->tiles && a->ngroups >= 2 && a->gslice_host;
  // 2 colours + colour-0 rows of A == [diag, U row] (b2s_fuse_check): the
  // backward pass of colour 0 and the SpMV rows of colour 0 share one read
  // (sharded: the SpMV needs the owners' ghost rows of p^ between the two)
  // sharded + fused: the operator passed is the local block, the boundary
  // rows' ghost couplings come separately (b2s_mesh bnd_*)
  const bool mesh_local = mesh && mesh->bnd_ptr != nullptr;
  // separately applied wells: the well terms of p^ (s^) are computed right
  // before each SpMV and subtracted in its epilogue; with the fused colour
  // passes (which produce v's colour-0 rows before p^ is complete) the
  // colour-0 rows are patched after the terms are known (k_wells_patch)
  const bool wells = a->wells != nullptr && a->wells->nwells > 0;
  if (wells && (mesh || !a->well_slice || !a->well_lane || !a->well_corr || !a->well_scratch))
    return mesh ? B2S_UNSUPPORTED : B2S_SHAPE;
  const WellFix wf = wells ? WellFix{a->well_slice, a->well_lane, a->well_corr} : WellFix{};
  auto well_terms = [&](const double* xin, const int* dn, cudaStream_t q, bool pd = false) {
    return wells ? launch_wells_corr(a->wells, xin, a->well_scratch, a->well_corr, dn, q, pd) : 0;
  };
  const bool fused = phased && a->ngroups == 2 && a->fuse && (!mesh || mesh_local);
  // fused vector passes on top of the fused colour passes: 7 kernels per
  // iteration instead of 9.  They move the same bytes (the separate p-update
  // largely hits L2), so they pay where the iteration is launch-bound --
  // measured 65.9 vs 71.0 us per iteration at 48k cells, 388.8 vs 384.7 us at
  // 1M (profiles/r02/vec_fusion.txt).  The unfused passes take the s-image
  // below, which wins from ~100k cells on (350k: 152.8 vs 165.4 us, 113k
  // even, 48k: 57.1 vs 56.4; profiles/r02/simg.txt): on up to 100k cells by
  // default; B2S_FUSE_VEC=1/0 forces it
  const char* fv_env = getenv("B2S_FUSE_VEC");
  const bool vecf = fused && (fv_env ? fv_env[0] == '1' : a->n <= 100000);
  // sync-free sweeps need sentinel-filled outputs (not the wavefront sweeps)
  const int reset = (ilu && !phased && !a->gw) ? 1 : 0;
  // x += alpha p^ deferred from the s-update to the r-update (one x pass per
  // iteration instead of two, the same two roundings; k_x_fixup after a
  // half-step exit) -- not with sync-free sweeps (their s-update refills p^)
  const char* xd_env = getenv("B2S_XDEFER");
  const bool xdefer = ilu && !vecf && !reset && !(xd_env && xd_env[0] == '0');
  // s-image (fused.cu): the s^ forward sweep of a 2-colour plan replaced by
  // F(s) = F(r) - alpha F(v), both images computed in passes that stream the
  // same blocks anyway (F(r) in y's colour-1 rows, u = inv(A_kk) v and F(v)
  // in t, which is dead until the s-phase); B2S_SIMG=0 turns it off
  const char* si_env = getenv("B2S_SIMG");
  const bool simg = fused && !vecf && xdefer && !mesh && !(si_env && si_env[0] == '0');
  MeshDev md{};
  MeshHalo mh{};
  if (mesh && !ilu) return B2S_UNSUPPORTED;   // sharded solves are block-Jacobi ILU0
  if (mesh) {
    if (mesh->nranks < 1 || mesh->rank < 0 || mesh->rank >= mesh->nranks || !mesh->mbox ||
        !mesh->peer_mbox || !mesh->flags || !mesh->peer_flags)
      return B2S_SHAPE;
    const char* to_env = getenv("B2S_MESH_TIMEOUT_MS");
    const long long timeout_ns = mesh->timeout_ns > 0 ? mesh->timeout_ns
                                 : (to_env ? atoll(to_env) * 1000000ll : 60000000000ll);
    md = MeshDev{mesh->rank, mesh->nranks, mesh->mbox, mesh->peer_mbox, mesh->seq_base, timeout_ns};
    mh.rank = mesh->rank; mh.nranks = mesh->nranks; mh.nghost = mesh->nghost;
    mh.nnbr = mesh->nnbr; mh.nbr = mesh->nbr;
    mh.ghost_owner = mesh->ghost_owner; mh.ghost_row = mesh->ghost_row;
    mh.peer_vec[0] = mesh->peer_x; mh.peer_vec[1] = mesh->peer_phat;
    mh.peer_vec[2] = mesh->peer_shat;
    mh.flags = mesh->flags; mh.peer_flags = mesh->peer_flags; mh.seq_base = mesh->seq_base;
    mh.mbox = mesh->mbox; mh.peer_mbox = mesh->peer_mbox; mh.timeout_ns = md.timeout_ns;
  }
  const int np = a->nparts;
  SliceMap map{a->nslices, a->row0, a->nrows};
  Sell A{a->a_sp, a->a_cols, a->a_vals};
  // residuals: the whole operator when given, else the local block + the
  // residual-mode ghost correction (np + kCorrCtas partials)
  const bool res_corr = mesh_local && !mesh->full_vals;
  const Sell Afull = (mesh && mesh->full_vals)
                         ? Sell{mesh->full_sp, mesh->full_cols, mesh->full_vals} : A;
  const int np_res = res_corr ? np + kCorrCtas : np;
  Sell L{a->l_sp, a->l_cols, a->l_vals}, U{a->u_sp, a->u_cols, a->u_vals};
  const int* done = &state->done;
  cudaStream_t user = a->stream;
  const int grid_v = np;

  // mapped pinned word the exiting CTA (or the init kernel) sets; the host
  // polls it `lag` replays behind the device
  int* host_done = nullptr;
  int* dev_done = nullptr;
  if (!(host_done = done_acquire())) return B2S_CUDA_ERROR;
  mark();
  *host_done = 0;
  if (cudaHostGetDevicePointer(&dev_done, host_done, 0) != cudaSuccess) {
    done_release(host_done);
    return B2S_CUDA_ERROR;
  }

  // publish this rank's vector, wait for the neighbours', pull the ghosts
  auto halo = [&](cudaStream_t q, int which, double* vec, const int* dn) {
    k_mesh_publish<<<1, 1, 0, q>>>(state, mh, dn);
    k_mesh_wait<<<1, 32, 0, q>>>(state, mh, dn, dev_done);
    if (mh.nghost > 0) {
      long long g = ((long long)mh.nghost * a->b + 255) / 256;
      if (g > kSms * 2) g = kSms * 2;
      k_mesh_pull<<<(int)g, 256, 0, q>>>(mh, which, a->b, vec + m, dn);
    }
  };

  // ---- setup on the caller's stream: r0 = b - A x0, |r0|, r^ = r0, rho_0
  // partials.  Launched after the iteration graph is captured and
  // instantiated (host work that may synchronise the device implicitly --
  // sharded solves on one GPU must not do that while another shard's kernel
  // waits for this one); the initial state is read back once, after the solve.
  auto setup = [&]() -> int {
    int rc = B2S_OK;
    k_zero_words<<<1, 32, 0, user>>>(reinterpret_cast<unsigned*>(tickets), 16);
    k_copy<<<grid_v, 256, 0, user>>>(m, a->x, x0);
    // the readiness/mailbox sequences restart from seq_base: clear `done`
    // and the counters the halo kernels read before k_ctl_init runs
    if (mesh) k_mesh_reset<<<1, 1, 0, user>>>(state);
    if (a->x0_zero) {   // r0 = b - A 0 = b: a copy and the |r0|^2 partials
      k_copy<<<grid_v, 256, 0, user>>>(m, a->rhs, r);
      k_dot_parts<<<np, 256, 0, user>>>(m, r, r, prr);
    } else {
      if (mesh) halo(user, 0, a->x, &state->done);
      rc = well_terms(a->x, nullptr, user);
      if (rc == B2S_OK)
        rc = launch_spmv(a->b, 3, np, map, Afull, a->x, r, a->rhs, prr, nullptr, nullptr, Ctl{},
                         user, false, wf);
      if (res_corr)
        launch_ghost_correct<kResidual>(a->b, mesh, a->x + m, r, nullptr, prr, nullptr, np,
                                        nullptr, Ctl{}, user);
    }
    if (a->x0_zero && res_corr)   // the correction's partial slots stay zero
      k_zero_words<<<1, 32, 0, user>>>(reinterpret_cast<unsigned*>(prr + np), 2 * kCorrCtas);
    if (rc == B2S_OK) {
      k_ctl_init<<<1, 256, 0, user>>>(state, prr, np_res, a->tol, a->maxit, dev_done, md);
      k_copy<<<grid_v, 256, 0, user>>>(m, r, rhat);
      k_copy<<<grid_v, 256, 0, user>>>(m, r, v);  // v is only read for k > 0
      if (ilu && !phased && !a->gw) {
        rc = fill_sentinel(m, y, user);
        if (!rc) rc = fill_sentinel(m, phat, user);
        if (!rc) rc = fill_sentinel(m, shat, user);
      }
    }
    if (rc == B2S_OK && cudaGetLastError() != cudaSuccess) rc = B2S_CUDA_ERROR;
    return rc;
  };
  // a peer's host thread that failed (its callback returns nonzero) must not
  // leave this shard spinning: raise the mesh-wide abort and leave
  bool barrier_failed = false;
  auto peer_barrier = [&]() {
    if (mesh && mesh->host_barrier && mesh->host_barrier(mesh->host_barrier_ctx) != 0)
      barrier_failed = true;
    return !barrier_failed;
  };
  State hs;
  bool tail_queued = false;

  // ---- capture one iteration
  cudaStream_t cs;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
    done_release(host_done);
    return B2S_CUDA_ERROR;
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int status = B2S_OK;
  int kernels = 0;
  // Sharded solves: overlapping the halo with the colour-1 SpMV (a side
  // branch of the captured graph) hides the cross-GPU flag and pull latency,
  // but the fork's event nodes break the programmatic-launch chain: on one
  // GPU it measured slower (two shards 15.4 -> 16.5 ms), so it is on by
  // default only for ranks with ghost rows on their own GPU.
  // B2S_MESH_OVERLAP=1/0 forces it.
  const char* ov_env = getenv("B2S_MESH_OVERLAP");
  const bool overlap = mesh && (ov_env ? ov_env[0] == '1'
                                       : (!mesh->shared_device && mesh->nghost > 0));
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (overlap && (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess ||
                  cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming) != cudaSuccess ||
                  cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming) != cudaSuccess)) {
    done_release(host_done);
    cudaStreamDestroy(cs);
    return B2S_CUDA_ERROR;
  }
  auto fork_halo = [&](int which, double* vec) {
    if (!overlap) return;
    cudaEventRecord(ev_fork, cs);
    cudaStreamWaitEvent(side, ev_fork, 0);
    halo(side, which, vec, &state->done);
    cudaEventRecord(ev_join, side);
  };
  auto join_halo = [&](int which, double* vec) {
    if (overlap) cudaStreamWaitEvent(cs, ev_join, 0);
    else halo(cs, which, vec, &state->done);
  };
  do {
    mark();
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      status = B2S_CUDA_ERROR; break;
    }
    // programmatic dependent launch between the iteration's kernels
    // (B2S_PDL=0 turns it off)
    const char* pdl_env = getenv("B2S_PDL");
    // (shards sharing one GPU: a programmatically launched kernel would hold
    // SMs while its predecessor's last CTA waits for another shard)
    // (wavefront loops: no programmatic launches at all.  Their sweep tiles
    // spin on each other, and with any kernel of the loop launched
    // programmatically some C4 level steps stalled to 20-40 ms against 14.0:
    // bench means 15.3-16.1 ms vs 13.95-14.06 with PDL off; plain launches of
    // the sweeps alone did not cure it; profiles/r02/level_pdl.txt)
    const bool pdl = !(pdl_env && pdl_env[0] == '0') && !(mesh && mesh->shared_device) && !a->gw;
    double* ph = ilu ? phat : p;
    double* sh = ilu ? shat : s;
    const int reset_y = a->refill_y ? 0 : 1;
    const int s1c = fused ? a->gslice_host[1] : 0;
    if (vecf) {
      // fused vector passes (7 kernels): p and s are formed inside the colour
      // passes, the half-step |s| test moves to the omega control step, and
      // x += alpha p^ + omega s^ is one update in the r-pass
      PreIn inP{state, r, v, p, nullptr};
      int gF = np, g0 = np;
      launch_fwd_pre(a->b, np, map, s1c, map.nslices, L, a->dinv_tiles, phat, done, &gF, cs, pdl,
                     kPreP, &inP);
      launch_bwd_spmv(a->b, 1, np, map, s1c, A, a->dinv_tiles, nullptr, phat, v, rhat, pg,
                      nullptr, done, &g0, cs, pdl, kPreP, &inP);
      const Ctl ca{state, counters + 0, dev_done, kCtlAlpha, md};
      if (mesh) fork_halo(1, phat);
      if (wells) {
        well_terms(phat, done, cs, pdl);
        launch_wells_patch(a->wells, a->goff1, a->well_corr, v, rhat, 1, pg + g0, nullptr, done, cs, SImgPatch{}, pdl);
        kernels += 3;
        ++g0;
      }
      launch_spmv_range(a->b, 1, np, map, s1c, map.nslices, g0, A, phat, v, rhat, pg, nullptr,
                        done, mesh ? Ctl{} : ca, cs, pdl, wf);
      kernels += 3;
      if (mesh) {
        join_halo(1, phat);
        launch_ghost_correct<kDotW>(a->b, mesh, phat + m, v, rhat, pg, nullptr, g0 + np, done, ca,
                                    cs);
        kernels += mh.nghost > 0 ? 4 : 3;
      }
      PreIn inS{state, r, v, s, pss};
      launch_fwd_pre(a->b, np, map, s1c, map.nslices, L, a->dinv_tiles, shat, done, &gF, cs, pdl,
                     kPreS, &inS);
      PreIn inS0{state, r, v, s, pss + gF};
      launch_bwd_spmv(a->b, 2, np, map, s1c, A, a->dinv_tiles, nullptr, shat, t, s, ptt, pts,
                      done, &g0, cs, pdl, kPreS, &inS0);
      const Ctl co{state, counters + 2, dev_done, kCtlOmegaS, md, pss, gF + g0};
      if (mesh) fork_halo(2, shat);
      if (wells) {
        well_terms(shat, done, cs, pdl);
        launch_wells_patch(a->wells, a->goff1, a->well_corr, t, s, 2, ptt + g0, pts + g0, done, cs, SImgPatch{}, pdl);
        kernels += 3;
        ++g0;
      }
      launch_spmv_range(a->b, 2, np, map, s1c, map.nslices, g0, A, shat, t, s, ptt, pts, done,
                        mesh ? Ctl{} : co, cs, pdl, wf);
      kernels += 3;
      if (mesh) {
        join_halo(2, shat);
        launch_ghost_correct<kSelfAndW>(a->b, mesh, shat + m, t, s, ptt, pts, g0 + np, done, co,
                                        cs);
        kernels += mh.nghost > 0 ? 4 : 3;
      }
      launch_k(k_r_update<true>, dim3(grid_v), dim3(256), 0, cs, pdl, m, (const State*)state,
               shat, (const double*)t, (const double*)s, (const double*)rhat, a->x, r, prr, prho,
               reset, Ctl{state, counters + 3, dev_done, kCtlEndBegin, md},
               (const double*)phat);
      ++kernels;
    } else {
      launch_k(k_p_update, dim3(grid_v), dim3(256), 0, cs, pdl, m, (const State*)state,
               (const double*)r, (const double*)v, p);
      ++kernels;
      if (simg) {
        // p^ colour 1 + F(r); colour 0 + v + u; colour-1 SpMV + F(v) + alpha
        launch_simg(a->b, 0, np, map, s1c, map.nslices, 0, L, a->dinv_tiles, p, r, phat, y,
                    nullptr, done, Ctl{}, a->goff1, nullptr, nullptr, m, state, cs, pdl);
        int g0 = np;
        launch_bwd_spmv(a->b, 1, np, map, s1c, A, a->dinv_tiles, p, phat, v, rhat, pg, nullptr,
                        done, &g0, cs, pdl, kPreNone, nullptr, t);
        if (wells) {   // p^ complete: the well terms; colour-0 rows of v (and u) patched
          well_terms(phat, done, cs, pdl);
          launch_wells_patch(a->wells, a->goff1, a->well_corr, v, rhat, 1, pg + g0, nullptr, done,
                             cs, SImgPatch{t, map.row0, map.nslices, a->dinv_tiles}, pdl);
          kernels += 3;
          ++g0;
        }
        launch_simg(a->b, 1, np, map, s1c, map.nslices, g0, A, nullptr, phat, rhat, v, nullptr, pg,
                    done, Ctl{state, counters + 0, dev_done, kCtlAlpha, md}, a->goff1, t, t, m,
                    state, cs, pdl, wf);
        kernels += 3;
      } else if (fused) {
        launch_phased(a->b, a->kc, 2, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles, p, y,
                      phat, done, cs, true, pdl);
        int g0 = np;
        launch_bwd_spmv(a->b, 1, np, map, s1c, A, a->dinv_tiles, p, phat, v, rhat, pg, nullptr,
                        done, &g0, cs, pdl);
        const Ctl ca{state, counters + 0, dev_done, kCtlAlpha, md};
        // sharded: p^ is complete here -- its halo (publish, wait, pull) runs on
        // a side branch of the graph, overlapped with the colour-1 SpMV (which
        // reads only local columns), and joins before the ghost correction
        if (mesh) fork_halo(1, phat);
        if (wells) {   // p^ complete: the well terms, colour-0 rows patched
          well_terms(phat, done, cs, pdl);
          launch_wells_patch(a->wells, a->goff1, a->well_corr, v, rhat, 1, pg + g0, nullptr, done,
                             cs, SImgPatch{}, pdl);
          kernels += 3;
          ++g0;
        }
        launch_spmv_range(a->b, 1, np, map, s1c, map.nslices, g0, A, phat, v, rhat, pg, nullptr,
                          done, mesh ? Ctl{} : ca, cs, pdl, wf);
        kernels += 3;
        if (mesh) {   // the boundary rows' ghost couplings + alpha
          join_halo(1, phat);
          launch_ghost_correct<kDotW>(a->b, mesh, phat + m, v, rhat, pg, nullptr, g0 + np, done, ca,
                                      cs);
          kernels += mh.nghost > 0 ? 4 : 3;
        }
      } else if (phased) {
        launch_phased(a->b, a->kc, a->ngroups, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles,
                      p, y, phat, done, cs, false, pdl);
        kernels += 2 * (a->ngroups - 1);
      } else if (ilu) {
        if (a->refill_y && !a->gw) { fill_sentinel(m, y, cs); ++kernels; }
        if (a->gw) launch_gw(a->b, a->gw, p, phat, done, cs, pdl);
        else if (a->tiles) launch_tiled(a->b, a->tiles, p, y, phat, reset_y, done, cs);
        else launch_sweeps(a->b, a->kc, map, L, U, a->dinv_tiles, p, y, phat, reset_y, a->sweep_flags,
                           tickets, done, cs);
        kernels += 2;
      }
      if (mesh && !fused) { halo(cs, 1, ph, done); kernels += mh.nghost > 0 ? 3 : 2; }
      if (!fused) {
        if (wells) { well_terms(ph, done, cs, pdl); kernels += 2; }
        launch_spmv(a->b, 1, np, map, A, ph, v, rhat, pg, nullptr, done,
                    Ctl{state, counters + 0, dev_done, kCtlAlpha, md}, cs, pdl, wf);
        ++kernels;
      }
      if (simg)   // s, |s|^2, the half-step test, and colour 1's s^ from the images
        launch_simg(a->b, 2, grid_v, map, s1c, map.nslices, 0, Sell{}, a->dinv_tiles, r, v, s,
                    shat, pss, done, Ctl{state, counters + 1, dev_done, kCtlS, md}, a->goff1, y, t,
                    m, state, cs, pdl);
      else
        launch_k(xdefer ? k_s_update<false> : k_s_update<true>, dim3(grid_v), dim3(256), 0, cs,
                 pdl, m, (const State*)state, (const double*)r, (const double*)v, ph, a->x, s, pss,
                 reset, Ctl{state, counters + 1, dev_done, kCtlS, md});
      ++kernels;
      if (fused) {
        if (simg)
          --kernels;   // no forward pass: the pair below counts as three
        else
          launch_phased(a->b, a->kc, 2, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles, s, y,
                        shat, done, cs, true, pdl);
        int g0 = np;
        launch_bwd_spmv(a->b, 2, np, map, s1c, A, a->dinv_tiles, s, shat, t, s, ptt, pts, done,
                        &g0, cs, pdl);
        const Ctl co{state, counters + 2, dev_done, kCtlOmega, md};
        if (mesh) fork_halo(2, shat);
        if (wells) {
          well_terms(shat, done, cs, pdl);
          launch_wells_patch(a->wells, a->goff1, a->well_corr, t, s, 2, ptt + g0, pts + g0, done,
                             cs, SImgPatch{}, pdl);
          kernels += 3;
          ++g0;
        }
        launch_spmv_range(a->b, 2, np, map, s1c, map.nslices, g0, A, shat, t, s, ptt, pts, done,
                          mesh ? Ctl{} : co, cs, pdl, wf);
        kernels += 3;
        if (mesh) {
          join_halo(2, shat);
          launch_ghost_correct<kSelfAndW>(a->b, mesh, shat + m, t, s, ptt, pts, g0 + np, done, co,
                                          cs);
          kernels += mh.nghost > 0 ? 4 : 3;
        }
      } else if (phased) {
        launch_phased(a->b, a->kc, a->ngroups, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles,
                      s, y, shat, done, cs, false, pdl);
        kernels += 2 * (a->ngroups - 1);
      } else if (ilu) {
        if (a->refill_y && !a->gw) { fill_sentinel(m, y, cs); ++kernels; }
        if (a->gw) launch_gw(a->b, a->gw, s, shat, done, cs, pdl);
        else if (a->tiles) launch_tiled(a->b, a->tiles, s, y, shat, reset_y, done, cs);
        else launch_sweeps(a->b, a->kc, map, L, U, a->dinv_tiles, s, y, shat, reset_y, a->sweep_flags,
                           tickets, done, cs);
        kernels += 2;
      }
      if (mesh && !fused) { halo(cs, 2, sh, done); kernels += mh.nghost > 0 ? 3 : 2; }
      if (!fused) {
        if (wells) { well_terms(sh, done, cs, pdl); kernels += 2; }
        launch_spmv(a->b, 2, np, map, A, sh, t, s, ptt, pts, done,
                    Ctl{state, counters + 2, dev_done, kCtlOmega, md}, cs, pdl, wf);
        ++kernels;
      }
      launch_k(xdefer ? k_r_update<true> : k_r_update<false>, dim3(grid_v), dim3(256), 0, cs, pdl,
               m, (const State*)state, sh, (const double*)t, (const double*)s,
               (const double*)rhat, a->x, r, prr, prho, reset,
               Ctl{state, counters + 3, dev_done, kCtlEndBegin, md},
               xdefer ? (const double*)ph : (const double*)nullptr);
      ++kernels;
    }
    if (cudaStreamEndCapture(cs, &graph) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    mark();
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    mark();
    // shards sharing one GPU replay on their own (caller's) stream: every
    // extra stream risks sharing a hardware work queue with a peer's stream,
    // i.e. a false dependency behind a kernel that waits for that very peer
    cudaStream_t rs = (mesh && mesh->shared_device) ? user : cs;
    if (!peer_barrier()) {   // a peer's host side failed before its loop
      k_mesh_raise_abort<<<1, 1, 0, user>>>(md);
      status = B2S_PEER_TIMEOUT;
      cudaStreamSynchronize(user);
      break;
    }
    if ((status = setup()) != B2S_OK) { cudaStreamSynchronize(user); break; }
    // order the graph after the setup work on the caller's stream
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    cudaEventRecord(ev, user);
    cudaStreamWaitEvent(rs, ev, 0);
    cudaEventDestroy(ev);
    // ---- replay: the host stays `lag` iterations behind the device
    const int lag = a->check_lag > 0 ? a->check_lag : 2;
    const int total = a->maxit + 1;  // every exit sets done; the spare replay only no-ops
    cudaEvent_t ring[8];
    for (int q = 0; q < 8; ++q) cudaEventCreateWithFlags(&ring[q], cudaEventDisableTiming);
    int launched = 0;
    for (int it = 0; it < total; ++it) {
      if (cudaGraphLaunch(exec, rs) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
      cudaEventRecord(ring[it & 7], rs);
      ++launched;
      if (it >= lag) {
        cudaEventSynchronize(ring[(it - lag) & 7]);
        if (*reinterpret_cast<volatile int*>(host_done)) break;
      }
    }
    res->graph_launches = launched;
    mark();
    // leave the caller's stream ordered after the solve
    cudaEvent_t fin;
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, rs);
    cudaStreamWaitEvent(user, fin, 0);
    cudaEventDestroy(fin);
    if (status == B2S_OK) {
      // the solve's tail goes on the device before the host tears the graph
      // down (that host work overlapped nothing before: ~0.3 ms idle at C4)
      if (vecf || xdefer)   // an exit between the s half-step and the r-update: x += alpha p^
        k_x_fixup<<<grid_v, 256, 0, user>>>(m, state, phat, a->x);
      tail_queued = cudaMemcpyAsync(&hs, state, sizeof(State), cudaMemcpyDeviceToHost, user) ==
                    cudaSuccess;
    }
    if (cudaStreamSynchronize(rs) != cudaSuccess) status = B2S_CUDA_ERROR;
    for (int q = 0; q < 8; ++q) t_left.events[t_left.nev++] = ring[q];
    peer_barrier();   // no shard tears down while another still runs
  } while (0);
  t_left.exec = exec;
  t_left.graph = graph;
  t_left.streams[0] = cs;
  t_left.streams[1] = side;
  if (ev_fork) t_left.events[t_left.nev++] = ev_fork;
  if (ev_join) t_left.events[t_left.nev++] = ev_join;
  // (sharded solves tear down at once: their peers' kernels may be spinning
  // on this device, and nothing of theirs should wait behind our teardown)
  if (mesh) t_left.destroy();
  mark();
  done_release(host_done);
  host_done = nullptr;
  dev_done = nullptr;   // (read by reference in halo(): the late halo below must not set it)
  mark();
  if (tmg && ntp == 9) {
    auto ms = [&](int i) { return std::chrono::duration<double, std::milli>(tp[i + 1] - tp[i]).count(); };
    fprintf(stderr, "b2s_bicgstab host ms: device sync %.3f host alloc %.3f prologue %.3f capture %.3f "
            "instantiate %.3f loop %.3f teardown %.3f free host %.3f (%d graphs)\n", ms(0), ms(1),
            ms(2), ms(3), ms(4), ms(5), ms(6), ms(7), res->graph_launches);
  }
  if (status != B2S_OK) return status;
  res->kernels_per_iteration = kernels;

  if (!tail_queued) return B2S_CUDA_ERROR;
  B2S_CHECK(cudaStreamSynchronize(user));
  if (hs.reason == kAborted || barrier_failed) return B2S_PEER_TIMEOUT;
  res->initial_norm = hs.norm0;
  if (hs.init_exit) {  // zero or non-finite initial residual, rho_0 breakdown: no iteration
    res->converged = hs.reason == kConverged;
    res->reason = hs.reason;
    res->final_norm = hs.norm0;
    return B2S_OK;
  }
  res->iterations = hs.its;
  res->reason = hs.reason == kRunning ? kBudget : hs.reason;
  if (hs.reason == kConverged) {
    res->converged = 1;
    res->final_norm = hs.final_norm;
    return B2S_OK;
  }
  // not converged: true residual of the current x, then x0 if x is not finite
  // (bs/krylov.py:242-244)
  // (sharded: x's ghost rows first, and both results all-reduced, so every
  // rank reports the global norm and restores x0 together; on one GPU the
  // shards first rendezvous again -- a peer still tearing down its graph or
  // freeing its host flag would otherwise wait for these waiting kernels)
  if (mesh) {
    if (!peer_barrier()) {
      k_mesh_raise_abort<<<1, 1, 0, user>>>(md);
      cudaStreamSynchronize(user);
      return B2S_PEER_TIMEOUT;
    }
    halo(user, 0, a->x, nullptr);
  }
  int rc = well_terms(a->x, nullptr, user);
  if (rc) return rc;
  rc = launch_spmv(a->b, 3, np, map, Afull, a->x, t, a->rhs, pg, nullptr, nullptr, Ctl{}, user,
                   false, wf);
  if (rc) return rc;
  if (res_corr)
    launch_ghost_correct<kResidual>(a->b, mesh, a->x + m, t, nullptr, pg, nullptr, np, nullptr,
                                    Ctl{}, user);
  if (mesh) k_mesh_scalar<<<1, 256, 0, user>>>(state, md, kSlotFinal, pg, np_res, nullptr, pss);
  else k_reduce_parts<<<1, 256, 0, user>>>(pg, np, pss);
  int* bad = reinterpret_cast<int*>(ptt);
  k_zero_words<<<1, 32, 0, user>>>(reinterpret_cast<unsigned*>(bad), 1);
  k_all_finite<<<grid_v, 256, 0, user>>>(m, a->x, bad);
  if (mesh) k_mesh_scalar<<<1, 256, 0, user>>>(state, md, kSlotFinite, nullptr, 0, bad, pts);
  B2S_LAUNCH_CHECK();
  double fin2 = 0.0, gbad = 0.0;
  int hbad = 0;
  B2S_CHECK(cudaMemcpyAsync(&fin2, pss, sizeof(double), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, user));
  if (mesh) B2S_CHECK(cudaMemcpyAsync(&gbad, pts, sizeof(double), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaStreamSynchronize(user));
  if (mesh) {   // an abort raised by a peer during these last all-reduces
    State h2;
    B2S_CHECK(cudaMemcpy(&h2, state, sizeof(State), cudaMemcpyDeviceToHost));
    if (h2.reason == kAborted) return B2S_PEER_TIMEOUT;
  }
  res->final_norm = sqrt(fin2);
  if (mesh) hbad = gbad != 0.0;
  if (hbad) {
    k_copy<<<grid_v, 256, 0, user>>>(m, x0, a->x);
    B2S_LAUNCH_CHECK();
  }
  return B2S_OK;
}

long long b2s_mesh_mbox_bytes(int nranks) {
  // kMboxSlots x nranks x 4 doubles, then the abort word (ctl.cuh abort_word)
  return nranks < 1 ? 0 : (long long)kMboxSlots * nranks * 4 * 8 + 64;
}

int b2s_bicgstab_workspace_layout(int n, int nghost, int b, long long* phat_off,
                                  long long* shat_off) {
  if (n < 0 || nghost < 0 || b < 1) return B2S_SHAPE;
  const long long mv = vec_doubles_g(n, nghost, b);
  *phat_off = 4 * mv;
  *shat_off = 6 * mv;
  return B2S_OK;
}

int b2s_ipc_handle(const void* ptr, unsigned char* handle64, long long* offset) {
  // the allocation's base through the driver entry point (no libcuda link
  // dependency: the library must load on hosts without a driver)
  using range_fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fp)
    return B2S_CUDA_ERROR;
  CUdeviceptr base = 0;
  size_t size = 0;
  if (reinterpret_cast<range_fn>(fp)(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) !=
      CUDA_SUCCESS)
    return B2S_CUDA_ERROR;
  cudaIpcMemHandle_t h;
  B2S_CHECK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  memcpy(handle64, &h, sizeof(h));
  *offset = (long long)(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return B2S_OK;
}

int b2s_ipc_open(const unsigned char* handle64, long long offset, void** ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  B2S_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *ptr_out = static_cast<char*>(base) + offset;
  return B2S_OK;
}

int b2s_ipc_close(void* base) {
  B2S_CHECK(cudaIpcCloseMemHandle(base));
  return B2S_OK;
}

// ---- standalone reductions and vector helpers for the Python layer
int b2s_dot(long long m, const double* a, const double* b, int nparts, double* parts,
            double* out, cudaStream_t st) {
  if (m < 0 || nparts < 1) return B2S_SHAPE;
  k_dot_parts<<<nparts, 256, 0, st>>>(m, a, b, parts);
  k_reduce_parts<<<1, 256, 0, st>>>(parts, nparts, out);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

const char* b2s_version(void) { return "b200solve 0.1.0 sm_100a"; }

// Keep freed stream-ordered scratch (cudaMallocAsync) in the device's default
// pool instead of returning it to the driver at every synchronisation; the
// setup path allocates and frees scratch per call.
int b2s_retain_pool_memory(int device) {
  cudaMemPool_t pool;
  B2S_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = ~0ull;
  B2S_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  return B2S_OK;
}

// ---- fused BiCGStab vector steps with host-provided scalars (the
//      multi-GPU loop, paper_2309_11488_b200/distributed.py, drives these and
//      all-reduces the partial sums between them).  A 2-double "scalars"
//      record is staged on the device so the same kernels serve both paths.
static State* stage_state(double* scratch, int k, double alpha, double beta, double omega,
                          cudaStream_t st, int* rc) {
  State h{};
  h.alpha = alpha; h.beta = beta; h.omega = omega; h.k = k; h.done = 0;
  State* d = reinterpret_cast<State*>(scratch);
  *rc = cudaMemcpyAsync(d, &h, sizeof(State), cudaMemcpyHostToDevice, st) == cudaSuccess
            ? B2S_OK : B2S_CUDA_ERROR;
  return d;
}

// p = r (k == 0) or r + beta (p - omega v); scratch >= 128 bytes device
int b2s_vec_p(long long m, int k, double beta, double omega, const double* r, const double* v,
              double* p, double* scratch, cudaStream_t st) {
  if (misaligned16(r, v, p)) return B2S_SHAPE;
  int rc;
  State* s = stage_state(scratch, k, 0.0, beta, omega, st, &rc);
  if (rc) return rc;
  k_p_update<<<kSms * 4, 256, 0, st>>>(m, s, r, v, p);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// s = r - alpha v ; x += alpha phat ; partials |s|^2 (nparts CTAs)
int b2s_vec_s(long long m, double alpha, const double* r, const double* v, double* phat,
              double* x, double* s, double* parts, int nparts, int reset, double* scratch,
              cudaStream_t st) {
  if (misaligned16(r, v, phat, x, s)) return B2S_SHAPE;
  int rc;
  State* d = stage_state(scratch, 0, alpha, 0.0, 0.0, st, &rc);
  if (rc) return rc;
  k_s_update<true><<<nparts, 256, 0, st>>>(m, d, r, v, phat, x, s, parts, reset, Ctl{});
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// x += omega shat ; r = s - omega t ; partials |r|^2 and rhat.r
int b2s_vec_r(long long m, double omega, double* shat, const double* t, const double* s,
              const double* rhat, double* x, double* r, double* prr, double* prho, int nparts,
              int reset, double* scratch, cudaStream_t st) {
  if (misaligned16(shat, t, s, rhat, x, r)) return B2S_SHAPE;
  int rc;
  State* d = stage_state(scratch, 0, 0.0, 0.0, omega, st, &rc);
  if (rc) return rc;
  k_r_update<false><<<nparts, 256, 0, st>>>(m, d, shat, t, s, rhat, x, r, prr, prho, reset, Ctl{},
                                            nullptr);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// out[0] = fixed-order sum of parts[0..np)
int b2s_reduce(const double* parts, int np, double* out, cudaStream_t st) {
  k_reduce_parts<<<1, 256, 0, st>>>(parts, np, out);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

int b2s_all_finite(long long m, const double* a, int* bad_dev, cudaStream_t st) {
  if (m < 0) return B2S_SHAPE;
  B2S_CHECK(cudaMemsetAsync(bad_dev, 0, sizeof(int), st));
  if (m == 0) return B2S_OK;
  long long g = (m + 255) / 256;
  if (g > kSms * 8) g = kSms * 8;
  k_all_finite<<<(int)g, 256, 0, st>>>(m, a, bad_dev);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

}  // extern "C"
