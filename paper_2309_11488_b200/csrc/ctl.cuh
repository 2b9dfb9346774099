// BiCGStab control state and the "last CTA" control steps (bs/krylov.py:
// 171-244 semantics).  The kernel that produces a set of per-CTA partial
// sums also finishes the reduction: every CTA publishes its partial, takes a
// ticket, and the CTA that arrives last reduces all partials in a fixed
// order (deterministic, no fp64 atomics) and runs the scalar logic of that
// point of the iteration.  So no 1-CTA control kernel sits between the
// bandwidth kernels of an iteration.
#pragma once
#include "common.cuh"

namespace b2s {

constexpr double kBreakdown = 1e-60;  // bs/krylov.py:27

// BiCGStab's vector updates with explicit roundings (no contraction choice
// left to the compiler), so every kernel that forms one -- the plain vector
// passes and the fused colour passes that form p and s on the fly -- gets
// the same bits.
__device__ __forceinline__ double bicg_p(double r, double p, double v, double beta,
                                         double omega) {
  return __fma_rn(beta, __fma_rn(-omega, v, p), r);   // r + beta (p - omega v)
}
__device__ __forceinline__ double bicg_axpy(double y, double a, double x) {
  return __fma_rn(-a, x, y);                           // y - a x
}
__device__ __forceinline__ double bicg_xupd(double x, double a, double d) {
  return __fma_rn(a, d, x);                            // x + a d
}

enum Reason { kRunning = 0, kConverged = 1, kBreakdownR = 2, kNumerical = 3, kBudget = 4,
              kAborted = 5 /* sharded: a peer did not answer in time, or aborted */ };

struct State {
  double rho, rho_prev, alpha, omega, beta;
  double norm0, target, final_norm, its;
  int k, maxit, done, reason;
  int init_exit;   // finished by k_ctl_init (no iteration): zero/non-finite r0, rho_0 breakdown
  int xpend;       // fused vector passes: x still lacks alpha p^ (added with omega s^ in the
                   // r-update, or by k_x_fixup when the solve ends in between)
  long long cseq;  // mesh: control points passed (mailbox sequence)
  long long pub;   // mesh: vectors published (readiness-flag sequence)
};

// Sharded solves: the all-reduce mailbox of this rank and every rank's
// (b2s_mesh in b200solve.h).  mbox == nullptr: single system.
constexpr int kMboxSlots = B2S_MBOX_SLOTS;
enum MboxSlot { kSlotInit = 0, kSlotFinal = 5, kSlotFinite = 6 };
struct MeshDev {
  int rank, nranks;
  double* mbox;
  double* const* peer_mbox;
  long long seq_base;
  long long timeout_ns;   // bound on every wait for a peer
};

__device__ __forceinline__ void st_relaxed_sys(double* p, double v) {
  asm volatile("st.relaxed.sys.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
  double v;
  asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Every rank's mailbox ends with an abort word (b2s_mesh_mbox_bytes): any
// rank whose wait for a peer times out -- a dead, hung or misconfigured
// peer -- raises it on every rank, so the whole mesh leaves its loop
// (reason kAborted -> B2S_PEER_TIMEOUT) instead of spinning forever.
__device__ __forceinline__ long long* abort_word(double* mbox, int nranks) {
  return reinterpret_cast<long long*>(mbox + (long long)kMboxSlots * nranks * 4);
}
__device__ __forceinline__ void mesh_raise_abort(double* const* peer_mbox, int nranks) {
  __threadfence_system();
  for (int h = 0; h < nranks; ++h) st_release_sys(abort_word(peer_mbox[h], nranks), 1);
}
// spin until *f >= seq; false once the abort word is up or timeout_ns passed
__device__ __forceinline__ bool wait_ge(const long long* f, long long seq, double* mbox,
                                        int nranks, long long timeout_ns) {
  const long long* ab = abort_word(mbox, nranks);
  unsigned long long t0 = 0;
  for (int it = 0;; ++it) {
    if (ld_acquire_sys(f) >= seq) return true;
    if (ld_acquire_sys(ab) != 0) return false;
    const unsigned long long now = global_ns();
    if (it == 0) t0 = now;
    else if ((long long)(now - t0) > timeout_ns) return false;
    __nanosleep(64);
  }
}

// All-reduce of (a, b) over the mesh, one thread: post the local sums into
// slot `slot` of every rank's mailbox, wait for every rank's post of this
// sequence number, sum them in rank order.  Every rank computes the same
// bits.  A slot is reused only after every rank has read it: a rank posts
// into slot s again only after passing the control points in between, which
// need every other rank's later posts.  Returns false (abort raised on every
// rank) when some rank does not post in time.
__device__ __forceinline__ bool mesh_sum3(const MeshDev& m, long long seq, int slot, double& a,
                                          double& b, double& c) {
  const int N = m.nranks;
  for (int h = 0; h < N; ++h) {
    double* e = m.peer_mbox[h] + ((long long)slot * N + m.rank) * 4;
    st_relaxed_sys(e, a);
    st_relaxed_sys(e + 1, b);
    st_relaxed_sys(e + 3, c);
  }
  __threadfence_system();
  for (int h = 0; h < N; ++h)
    st_release_sys(reinterpret_cast<long long*>(m.peer_mbox[h] + ((long long)slot * N + m.rank) * 4 + 2),
                   seq);
  double sa = 0.0, sb = 0.0, sc = 0.0;
  for (int h = 0; h < N; ++h) {
    const double* e = m.mbox + ((long long)slot * N + h) * 4;
    if (!wait_ge(reinterpret_cast<const long long*>(e + 2), seq, m.mbox, N, m.timeout_ns)) {
      mesh_raise_abort(m.peer_mbox, N);
      a = b = c = __longlong_as_double(0x7FF8000000000000ll);
      return false;
    }
    sa += ld_relaxed_sys(e);
    sb += ld_relaxed_sys(e + 1);
    sc += ld_relaxed_sys(e + 3);
  }
  a = sa;
  b = sb;
  c = sc;
  return true;
}
__device__ __forceinline__ bool mesh_sum(const MeshDev& m, long long seq, int slot, double& a,
                                         double& b) {
  double c = 0.0;
  return mesh_sum3(m, seq, slot, a, b, c);
}

enum Pre { kPreNone = 0, kPreP = 1, kPreS = 2 };

struct PreIn {
  const State* st;
  const double* r;
  const double* v;
  double* io;      // kPreP: p (old in, new out); kPreS: s (out)
  double* pss;     // kPreS: one |s|^2 partial per CTA
};

// kCtlOmegaS: the fused vector passes form s together with s^ and t, so the
// half-step exit test on |s| runs here, before omega (same order of tests as
// the reference: |s| finite, |s| <= target, then t.t and omega breakdowns)
enum CtlStep { kCtlNone = 0, kCtlAlpha = 1, kCtlS = 2, kCtlOmega = 3, kCtlEndBegin = 4,
               kCtlOmegaS = 5 };

struct Ctl {
  State* st;            // solver state (nullptr: no control step)
  unsigned* counter;    // arrival ticket of this call site (self-resetting)
  int* host_done;       // mapped pinned word the host polls (may be nullptr)
  int step;             // CtlStep
  MeshDev mesh;         // sharded solve: all-reduce the sums first
  const double* p2;     // kCtlOmegaS: the |s|^2 partials ...
  int np2;              // ... and their count
};

// deterministic sum of np partials by one CTA (L2 loads: written by other SMs)
__device__ __forceinline__ double reduce_parts_cg(const double* parts, int np, double* red) {
  double v = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v += __ldcg(parts + i);
  return block_sum(v, red);  // valid in thread 0
}

// true in every thread of the CTA that arrived last; call after thread 0
// stored this CTA's partials.  Resets the ticket for the next launch.
__device__ __forceinline__ bool last_cta(unsigned* counter) {
  __shared__ int am_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
    if (am_last) *counter = 0u;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__device__ __forceinline__ void ctl_finish(State* st, int* host_done, int reason) {
  st->done = 1;
  st->reason = reason;
  if (host_done) *reinterpret_cast<volatile int*>(host_done) = 1;
}

// The scalar logic after each reduction point; whole CTA calls, thread 0 writes.
// The state fields a step reads are loaded before the reductions, and the
// two or three partial arrays are summed in one pass with one shared-memory
// round (per-thread order and tree exactly reduce_parts_cg's): the control
// step is the serial tail of its kernel.
__device__ __forceinline__ void ctl_run(const Ctl& c, const double* p0, const double* p1, int np,
                                        double* red) {
  (void)red;
  State* st = c.st;
  __shared__ double red3[3][32];
  const bool two = c.step == kCtlOmega || c.step == kCtlEndBegin || c.step == kCtlOmegaS;
  const bool three = c.step == kCtlOmegaS;
  const double rho = st->rho, alpha = st->alpha, omega = st->omega;
  const double target = st->target, its = st->its;
  const int k = st->k, maxit = st->maxit;
  double v0 = 0.0, v1 = 0.0, v2 = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    v0 += __ldcg(p0 + i);
    if (two) v1 += __ldcg(p1 + i);
  }
  if (three)
    for (int i = threadIdx.x; i < c.np2; i += blockDim.x) v2 += __ldcg(c.p2 + i);
  v0 = warp_sum(v0);
  if (two) v1 = warp_sum(v1);
  if (three) v2 = warp_sum(v2);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { red3[0][w] = v0; red3[1][w] = v1; red3[2][w] = v2; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int nw = blockDim.x >> 5;
  double a = warp_sum(l < nw ? red3[0][l] : 0.0);
  double b = two ? warp_sum(l < nw ? red3[1][l] : 0.0) : 0.0;
  double c2 = three ? warp_sum(l < nw ? red3[2][l] : 0.0) : 0.0;
  if (threadIdx.x != 0) return;
  const int slot = c.step == kCtlOmegaS ? kCtlOmega : c.step;
  if (c.mesh.mbox && !mesh_sum3(c.mesh, c.mesh.seq_base + (++st->cseq), slot, a, b, c2)) {
    ctl_finish(st, c.host_done, kAborted);
    return;
  }
  switch (c.step) {
    case kCtlAlpha: {  // gamma = rhat.v  (bs/krylov.py:206-210)
      if (fabs(a) < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      st->alpha = rho / a;
      return;
    }
    case kCtlS: {  // test |s|  (bs/krylov.py:211-220); x advanced by alpha p^ here or,
                   // deferred, in the r-update (k_x_fixup after an exit in between)
      st->its = its + 0.5;
      st->xpend = 1;
      const double ns = sqrt(a);
      if (!isfinite(ns)) { ctl_finish(st, c.host_done, kNumerical); return; }
      if (ns <= target) { st->final_norm = ns; ctl_finish(st, c.host_done, kConverged); }
      return;
    }
    case kCtlOmega: {  // tt, ts  (bs/krylov.py:223-229)
      if (a < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      const double om = b / a;
      if (fabs(om) < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      st->omega = om;
      return;
    }
    case kCtlOmegaS: {  // |s| (bs/krylov.py:211-220), then tt, ts (:223-229)
      st->its = its + 0.5;
      st->xpend = 1;   // x += alpha p^ is deferred to the r-update (or k_x_fixup)
      const double ns = sqrt(c2);
      if (!isfinite(ns)) { ctl_finish(st, c.host_done, kNumerical); return; }
      if (ns <= target) { st->final_norm = ns; ctl_finish(st, c.host_done, kConverged); return; }
      if (a < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      const double om = b / a;
      if (fabs(om) < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      st->omega = om;
      return;
    }
    case kCtlEndBegin: {  // end of iteration k, then the top of k+1 (bs/krylov.py:195-200,230-240)
      st->xpend = 0;   // the r-update advanced x by alpha p^ + omega s^
      st->its = its + 0.5;
      const double nr = sqrt(a);
      if (!isfinite(nr)) { ctl_finish(st, c.host_done, kNumerical); return; }
      if (nr <= target) { st->final_norm = nr; ctl_finish(st, c.host_done, kConverged); return; }
      st->rho_prev = rho;
      st->k = k + 1;
      if (k + 1 >= maxit) { ctl_finish(st, c.host_done, kBudget); return; }
      if (fabs(b) < kBreakdown) { ctl_finish(st, c.host_done, kBreakdownR); return; }
      st->rho = b;
      st->beta = (b / rho) * (alpha / omega);
      return;
    }
    default:
      return;
  }
}

}  // namespace b2s
