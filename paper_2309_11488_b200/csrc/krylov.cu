// Right-preconditioned BiCGStab (bs/krylov.py:140-244), device resident.
//
// One iteration is a fixed sequence of stream-ordered kernels captured once
// into a CUDA graph and replayed; the host only polls a pinned "done" word a
// couple of iterations behind the GPU, so the device never idles on the
// host.  Control decisions (breakdown floors, convergence tests, half-step
// counting, the order of the reference's exits) run in four 1-CTA control
// kernels that are the only writers of the solver state; every other kernel
// reads `state->done` first and becomes a no-op once the solve has ended,
// which reproduces the reference's early exits exactly even though later
// kernels of the iteration are already queued.
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
#include <cmath>

#include "sell.cuh"

namespace b2s {

int launch_spmv(int b, int mode, int nparts, SliceMap map, Sell a, const double* x, double* y,
                const double* w, double* p0, double* p1, const int* done, cudaStream_t st);
int launch_sweeps(int b, int kc, SliceMap map, Sell lo, Sell up, const double* dt,
                  const double* r, double* y, double* z, int reset_y, int flags, void* tickets,
                  const int* done, cudaStream_t st);
int fill_sentinel(long long m, double* v, cudaStream_t st);
int launch_phased(int b, int kc, int ngroups, const int32_t* gslice_host, int goff1, SliceMap map,
                  Sell lo, Sell up, const double* dt, const double* r, double* y, double* z,
                  const int* done, cudaStream_t st);
int launch_tiled(int b, const void* handle, const double* r, double* y, double* z, int reset_y,
                 const int* done, cudaStream_t st);

constexpr double kBreakdown = 1e-60;  // bs/krylov.py:27

enum Reason { kRunning = 0, kConverged = 1, kBreakdownR = 2, kNumerical = 3, kBudget = 4 };

struct State {
  double rho, rho_prev, alpha, omega, beta;
  double norm0, target, final_norm, its;
  int k, maxit, done, reason;
};

// deterministic sum of np partials by one CTA of 256 threads
__device__ double reduce_parts(const double* parts, int np, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += parts[i];
  return block_sum(v, red);  // valid in thread 0
}

__global__ void k_ctl_init(State* st, const double* prr, int np, double tol, int maxit) {
  __shared__ double red[8];
  const double s = reduce_parts(prr, np, red);
  if (threadIdx.x == 0) {
    const double n0 = sqrt(s);
    st->rho = 0.0; st->rho_prev = 1.0; st->alpha = 1.0; st->omega = 1.0; st->beta = 0.0;
    st->norm0 = n0; st->target = tol * n0; st->final_norm = n0; st->its = 0.0;
    st->k = 0; st->maxit = maxit; st->reason = kRunning;
    st->done = 0;
    if (!isfinite(n0)) { st->done = 1; st->reason = kNumerical; }
    else if (n0 <= st->target || n0 == 0.0) { st->done = 1; st->reason = kConverged; }
  }
}

// top of iteration k: previous |r| test (k > 0), budget, rho, beta
__global__ void k_ctl_begin(State* st, const double* prr, const double* prho, int np) {
  __shared__ double red[8];
  if (st->done) return;
  const double rr = reduce_parts(prr, np, red);
  const double rho = reduce_parts(prho, np, red);
  if (threadIdx.x != 0) return;
  const int k = st->k;
  if (k > 0) {
    const double nr = sqrt(rr);
    if (!isfinite(nr)) { st->done = 1; st->reason = kNumerical; return; }
    if (nr <= st->target) { st->done = 1; st->reason = kConverged; st->final_norm = nr; return; }
    st->rho_prev = st->rho;
  }
  if (k >= st->maxit) { st->done = 1; st->reason = kBudget; return; }
  if (fabs(rho) < kBreakdown) { st->done = 1; st->reason = kBreakdownR; return; }
  st->rho = rho;
  if (k > 0) st->beta = (rho / st->rho_prev) * (st->alpha / st->omega);
}

__global__ void k_ctl_alpha(State* st, const double* pg, int np) {
  __shared__ double red[8];
  if (st->done) return;
  const double gamma = reduce_parts(pg, np, red);
  if (threadIdx.x != 0) return;
  if (fabs(gamma) < kBreakdown) { st->done = 1; st->reason = kBreakdownR; return; }
  st->alpha = st->rho / gamma;
}

__global__ void k_ctl_s(State* st, const double* pss, int np) {
  __shared__ double red[8];
  if (st->done) return;
  const double ss = reduce_parts(pss, np, red);
  if (threadIdx.x != 0) return;
  st->its += 0.5;  // the x update of this half step has happened
  const double ns = sqrt(ss);
  if (!isfinite(ns)) { st->done = 1; st->reason = kNumerical; return; }
  if (ns <= st->target) { st->done = 1; st->reason = kConverged; st->final_norm = ns; }
}

__global__ void k_ctl_omega(State* st, const double* ptt, const double* pts, int np) {
  __shared__ double red[8];
  if (st->done) return;
  const double tt = reduce_parts(ptt, np, red);
  const double ts = reduce_parts(pts, np, red);
  if (threadIdx.x != 0) return;
  if (tt < kBreakdown) { st->done = 1; st->reason = kBreakdownR; return; }
  const double om = ts / tt;
  if (fabs(om) < kBreakdown) { st->done = 1; st->reason = kBreakdownR; return; }
  st->omega = om;
}

// after the second half step: its, k
__global__ void k_ctl_end(State* st) {
  if (st->done) return;
  st->its += 0.5;
  st->k += 1;
}

#define GRID_STRIDE(t, m) \
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (m); \
       t += (long long)gridDim.x * blockDim.x)

__global__ void __launch_bounds__(256) k_p_update(long long m, const State* st,
                                                  const double* __restrict__ r,
                                                  const double* __restrict__ v, double* p) {
  if (st->done) return;
  const int k = st->k;
  const double beta = st->beta, omega = st->omega;
  if (k == 0) {
    GRID_STRIDE(t, m) p[t] = r[t];
  } else {
    GRID_STRIDE(t, m) p[t] = r[t] + beta * (p[t] - omega * v[t]);
  }
}

// s = r - alpha v ; x += alpha p^ ; |s|^2 partials ; optionally p^ <- sentinel
__global__ void __launch_bounds__(256) k_s_update(long long m, const State* st,
                                                  const double* __restrict__ r,
                                                  const double* __restrict__ v, double* phat,
                                                  double* __restrict__ x,
                                                  double* __restrict__ s, double* pss,
                                                  int reset) {
  __shared__ double red[8];
  if (st->done) return;
  const double alpha = st->alpha;
  double acc = 0.0;
  GRID_STRIDE(t, m) {
    const double sv = r[t] - alpha * v[t];
    const double ph = phat[t];
    s[t] = sv;
    x[t] += alpha * ph;
    acc = fma(sv, sv, acc);
    if (reset) phat[t] = sentinel();
  }
  const double tot = block_sum(acc, red);
  if (threadIdx.x == 0) pss[blockIdx.x] = tot;
}

// x += omega s^ ; r = s - omega t ; |r|^2 and r^.r partials ; s^ <- sentinel
__global__ void __launch_bounds__(256) k_r_update(long long m, const State* st, double* shat,
                                                  const double* __restrict__ tv,
                                                  const double* __restrict__ s,
                                                  const double* __restrict__ rhat,
                                                  double* __restrict__ x,
                                                  double* __restrict__ r, double* prr,
                                                  double* prho, int reset) {
  __shared__ double red[8];
  if (st->done) return;
  const double omega = st->omega;
  double a0 = 0.0, a1 = 0.0;
  GRID_STRIDE(t, m) {
    const double sh = shat[t];
    x[t] += omega * sh;
    const double rv = s[t] - omega * tv[t];
    r[t] = rv;
    a0 = fma(rv, rv, a0);
    a1 = fma(rhat[t], rv, a1);
    if (reset) shat[t] = sentinel();
  }
  const double t0 = block_sum(a0, red);
  if (threadIdx.x == 0) prr[blockIdx.x] = t0;
  const double t1 = block_sum(a1, red);
  if (threadIdx.x == 0) prho[blockIdx.x] = t1;
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

__global__ void k_copy_done(const State* st, int* host_done) { *host_done = st->done; }

}  // namespace b2s

using namespace b2s;

extern "C" {

static long long vec_doubles(int n, int b) {
  long long m = (long long)n * b;
  return (m + 31) / 32 * 32;  // 256-byte aligned sub-buffers
}

long long b2s_bicgstab_workspace_bytes(int n, int b, int nparts) {
  const long long m = vec_doubles(n, b);
  // r rhat p v phat s shat t y x0  + 6 partial arrays + state + tickets
  return (10 * m + 6 * (long long)((nparts + 31) / 32 * 32)) * 8 + 256 + 64;
}

int b2s_bicgstab(const b2s_bicg_args* a, b2s_bicg_result* res) {
  res->converged = 0; res->reason = 0; res->graph_launches = 0; res->kernels_per_iteration = 0;
  res->iterations = 0.0; res->initial_norm = 0.0; res->final_norm = 0.0;
  if (a->n < 0 || a->b < 1 || a->nparts < 1 || a->maxit < 1) return B2S_SHAPE;
  if (a->b > 4) return B2S_UNSUPPORTED;
  const long long m = (long long)a->n * a->b;
  const long long mv = vec_doubles(a->n, a->b);
  const long long npv = (a->nparts + 31) / 32 * 32;
  double* w = a->work;
  double *r = w, *rhat = w + mv, *p = w + 2 * mv, *v = w + 3 * mv, *phat = w + 4 * mv,
         *s = w + 5 * mv, *shat = w + 6 * mv, *t = w + 7 * mv, *y = w + 8 * mv,
         *x0 = w + 9 * mv;
  double* parts = w + 10 * mv;
  double *prr = parts, *prho = parts + npv, *pg = parts + 2 * npv, *pss = parts + 3 * npv,
         *ptt = parts + 4 * npv, *pts = parts + 5 * npv;
  State* state = reinterpret_cast<State*>(parts + 6 * npv);
  void* tickets = reinterpret_cast<char*>(state) + 256;
  const bool ilu = a->precond == 1;
  const bool phased = ilu && !a->tiles && a->ngroups >= 2 && a->gslice_host;
  const int reset = (ilu && !phased) ? 1 : 0;  // sync-free sweeps need sentinel-filled outputs
  const int np = a->nparts;
  SliceMap map{a->nslices, a->row0, a->nrows};
  Sell A{a->a_sp, a->a_cols, a->a_vals};
  Sell L{a->l_sp, a->l_cols, a->l_vals}, U{a->u_sp, a->u_cols, a->u_vals};
  const int* done = &state->done;
  cudaStream_t user = a->stream;
  const int grid_v = np;

  // ---- setup on the caller's stream: r0 = b - A x0, |r0|, r^ = r0, rho_0 partials
  B2S_CHECK(cudaMemsetAsync(tickets, 0, 64, user));
  k_copy<<<grid_v, 256, 0, user>>>(m, a->x, x0);
  int rc = launch_spmv(a->b, 3, np, map, A, a->x, r, a->rhs, prr, nullptr, nullptr, user);
  if (rc) return rc;
  k_ctl_init<<<1, 256, 0, user>>>(state, prr, np, a->tol, a->maxit);
  k_copy<<<grid_v, 256, 0, user>>>(m, r, rhat);
  k_copy<<<grid_v, 256, 0, user>>>(m, r, v);  // v is only read for k > 0
  B2S_CHECK(cudaMemcpyAsync(prho, prr, sizeof(double) * np, cudaMemcpyDeviceToDevice, user));
  if (ilu && !phased) {
    if ((rc = fill_sentinel(m, y, user))) return rc;
    if ((rc = fill_sentinel(m, phat, user))) return rc;
    if ((rc = fill_sentinel(m, shat, user))) return rc;
  }
  B2S_LAUNCH_CHECK();
  State hs;
  B2S_CHECK(cudaMemcpyAsync(&hs, state, sizeof(State), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaStreamSynchronize(user));
  res->initial_norm = hs.norm0;
  if (hs.done) {  // non-finite or zero initial residual: no iteration
    res->converged = hs.reason == kConverged;
    res->reason = hs.reason;
    res->final_norm = hs.norm0;
    return B2S_OK;
  }

  // ---- capture one iteration
  cudaStream_t cs;
  B2S_CHECK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  int* host_done = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int status = B2S_OK;
  int kernels = 0;
  do {
    if (cudaHostAlloc(&host_done, sizeof(int), cudaHostAllocMapped) != cudaSuccess) {
      status = B2S_CUDA_ERROR; break;
    }
    *host_done = 0;
    int* dev_done = nullptr;
    if (cudaHostGetDevicePointer(&dev_done, host_done, 0) != cudaSuccess) {
      status = B2S_CUDA_ERROR; break;
    }
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      status = B2S_CUDA_ERROR; break;
    }
    double* ph = ilu ? phat : p;
    double* sh = ilu ? shat : s;
    k_ctl_begin<<<1, 256, 0, cs>>>(state, prr, prho, np); ++kernels;
    k_p_update<<<grid_v, 256, 0, cs>>>(m, state, r, v, p); ++kernels;
    const int reset_y = a->refill_y ? 0 : 1;
    if (phased) {
      launch_phased(a->b, a->kc, a->ngroups, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles,
                    p, y, phat, done, cs);
      kernels += 2 * (a->ngroups - 1);
    } else if (ilu) {
      if (a->refill_y) { fill_sentinel(m, y, cs); ++kernels; }
      if (a->tiles) launch_tiled(a->b, a->tiles, p, y, phat, reset_y, done, cs);
      else launch_sweeps(a->b, a->kc, map, L, U, a->dinv_tiles, p, y, phat, reset_y, a->sweep_flags,
                         tickets, done, cs);
      kernels += 2;
    }
    launch_spmv(a->b, 1, np, map, A, ph, v, rhat, pg, nullptr, done, cs); ++kernels;
    k_ctl_alpha<<<1, 256, 0, cs>>>(state, pg, np); ++kernels;
    k_s_update<<<grid_v, 256, 0, cs>>>(m, state, r, v, ph, a->x, s, pss, reset); ++kernels;
    k_ctl_s<<<1, 256, 0, cs>>>(state, pss, np); ++kernels;
    if (phased) {
      launch_phased(a->b, a->kc, a->ngroups, a->gslice_host, a->goff1, map, L, U, a->dinv_tiles,
                    s, y, shat, done, cs);
      kernels += 2 * (a->ngroups - 1);
    } else if (ilu) {
      if (a->refill_y) { fill_sentinel(m, y, cs); ++kernels; }
      if (a->tiles) launch_tiled(a->b, a->tiles, s, y, shat, reset_y, done, cs);
      else launch_sweeps(a->b, a->kc, map, L, U, a->dinv_tiles, s, y, shat, reset_y, a->sweep_flags,
                         tickets, done, cs);
      kernels += 2;
    }
    launch_spmv(a->b, 2, np, map, A, sh, t, s, ptt, pts, done, cs); ++kernels;
    k_ctl_omega<<<1, 256, 0, cs>>>(state, ptt, pts, np); ++kernels;
    k_r_update<<<grid_v, 256, 0, cs>>>(m, state, sh, t, s, rhat, a->x, r, prr, prho, reset); ++kernels;
    k_ctl_end<<<1, 1, 0, cs>>>(state); ++kernels;
    k_copy_done<<<1, 1, 0, cs>>>(state, dev_done); ++kernels;
    if (cudaStreamEndCapture(cs, &graph) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    // order the graph after the setup work on the caller's stream
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
    cudaEventRecord(ev, user);
    cudaStreamWaitEvent(cs, ev, 0);
    cudaEventDestroy(ev);
    // ---- replay: the host stays `lag` iterations behind the device
    const int lag = a->check_lag > 0 ? a->check_lag : 2;
    const int total = a->maxit + 1;  // +1: the final k_ctl_begin does the last |r| / budget test
    cudaEvent_t ring[8];
    for (int q = 0; q < 8; ++q) cudaEventCreateWithFlags(&ring[q], cudaEventDisableTiming);
    int launched = 0;
    for (int it = 0; it < total; ++it) {
      if (cudaGraphLaunch(exec, cs) != cudaSuccess) { status = B2S_CUDA_ERROR; break; }
      cudaEventRecord(ring[it & 7], cs);
      ++launched;
      if (it >= lag) {
        cudaEventSynchronize(ring[(it - lag) & 7]);
        if (*reinterpret_cast<volatile int*>(host_done)) break;
      }
    }
    res->graph_launches = launched;
    // leave the caller's stream ordered after the solve
    cudaEvent_t fin;
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, cs);
    cudaStreamWaitEvent(user, fin, 0);
    cudaEventDestroy(fin);
    if (cudaStreamSynchronize(cs) != cudaSuccess) status = B2S_CUDA_ERROR;
    for (int q = 0; q < 8; ++q) cudaEventDestroy(ring[q]);
  } while (0);
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  cudaStreamDestroy(cs);
  if (host_done) cudaFreeHost(host_done);
  if (status != B2S_OK) return status;
  res->kernels_per_iteration = kernels;

  B2S_CHECK(cudaMemcpyAsync(&hs, state, sizeof(State), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaStreamSynchronize(user));
  res->iterations = hs.its;
  res->reason = hs.reason == kRunning ? kBudget : hs.reason;
  if (hs.reason == kConverged) {
    res->converged = 1;
    res->final_norm = hs.final_norm;
    return B2S_OK;
  }
  // not converged: true residual of the current x, then x0 if x is not finite
  // (bs/krylov.py:242-244)
  rc = launch_spmv(a->b, 3, np, map, A, a->x, t, a->rhs, pg, nullptr, nullptr, user);
  if (rc) return rc;
  k_reduce_parts<<<1, 256, 0, user>>>(pg, np, pss);
  int* bad = reinterpret_cast<int*>(ptt);
  B2S_CHECK(cudaMemsetAsync(bad, 0, sizeof(int), user));
  k_all_finite<<<grid_v, 256, 0, user>>>(m, a->x, bad);
  B2S_LAUNCH_CHECK();
  double fin2 = 0.0;
  int hbad = 0;
  B2S_CHECK(cudaMemcpyAsync(&fin2, pss, sizeof(double), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, user));
  B2S_CHECK(cudaStreamSynchronize(user));
  res->final_norm = sqrt(fin2);
  if (hbad) {
    k_copy<<<grid_v, 256, 0, user>>>(m, x0, a->x);
    B2S_LAUNCH_CHECK();
  }
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
  int rc;
  State* d = stage_state(scratch, 0, alpha, 0.0, 0.0, st, &rc);
  if (rc) return rc;
  k_s_update<<<nparts, 256, 0, st>>>(m, d, r, v, phat, x, s, parts, reset);
  B2S_LAUNCH_CHECK();
  return B2S_OK;
}

// x += omega shat ; r = s - omega t ; partials |r|^2 and rhat.r
int b2s_vec_r(long long m, double omega, double* shat, const double* t, const double* s,
              const double* rhat, double* x, double* r, double* prr, double* prho, int nparts,
              int reset, double* scratch, cudaStream_t st) {
  int rc;
  State* d = stage_state(scratch, 0, 0.0, 0.0, omega, st, &rc);
  if (rc) return rc;
  k_r_update<<<nparts, 256, 0, st>>>(m, d, shat, t, s, rhat, x, r, prr, prho, reset);
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
