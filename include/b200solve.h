/*
 * b200solve.h -- C ABI of libb200solve.so, the sm_100a kernels behind the
 * drop-in replacement for the reference `blocksolve` ILU0-BiCGStab path.
 *
 * The reference (/root/reference/pkg/src/blocksolve, "bs/") is pure Python
 * and has no FFI of its own; each entry point below replaces the body of the
 * reference function cited beside it, and the Python layer
 * (paper_2309_11488_b200/) keeps the reference's names, argument meaning and
 * exceptions on top (binding: paper_2309_11488_b200/_lib.py, ctypes).
 *
 * Conventions
 *   - every pointer is DEVICE memory unless its name ends in `_host`;
 *   - indices are int32 (the reference uses int64, bs/blockcore.py:83-84),
 *     values fp64, block vectors interleaved [row][b], blocks row-major;
 *   - all work is ordered on the caller's `stream`; functions that must
 *     report a data-dependent result (missing diagonal, singular pivot,
 *     sizes) synchronise that stream before returning;
 *   - the library keeps no global mutable state: independent solves may run
 *     concurrently on different streams;
 *   - return value: B2S_OK or one of the error codes below, which the Python
 *     layer maps onto the reference's exceptions (bs/errors.py).
 */
#ifndef B200SOLVE_H
#define B200SOLVE_H

#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2S_OK 0
#define B2S_SHAPE 1            /* -> ShapeError            (bs/errors.py:8-9)   */
#define B2S_MISSING_DIAGONAL 2 /* -> MissingDiagonal(row)  (bs/errors.py:20-25) */
#define B2S_SINGULAR_PIVOT 3   /* -> SingularPivot(row)    (bs/errors.py:28-33) */
#define B2S_CUDA_ERROR 4       /* -> RuntimeError                              */
#define B2S_UNSUPPORTED 5      /* block size outside 1..4                      */
#define B2S_PEER_TIMEOUT 6     /* sharded solve: a peer did not answer within
                                  b2s_mesh.timeout_ns (or aborted) -> PeerTimeout */

/* ---- analysis (bs/analysis.py) ------------------------------------------ */

/* diagonal slot per row (-1 if absent); replaces SparsityPattern.
 * diagonal_positions (bs/blockcore.py:127-134) and the missing-diagonal scans
 * (bs/analysis.py:79-82, bs/ilu0.py:159-161): B2S_MISSING_DIAGONAL with the
 * first such row in *first_missing_host. */
int b2s_find_diagonal(int n, const int32_t* rp, const int32_t* ci, int32_t* diag_pos,
                      int32_t* first_missing_host, cudaStream_t stream);

/* level_schedule (bs/analysis.py:85-100): row_group[i] = level, bit-exact. */
int b2s_level_schedule(int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                       int32_t* ngroups_host, cudaStream_t stream);

/* graph_color (bs/analysis.py:103-145): greedy first-fit colours, bit-exact. */
int b2s_graph_color(int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                    int32_t* ngroups_host, cudaStream_t stream);

/* The same two plans with a grid hint (nx, ny of a natural-order stencil;
 * nx <= 0: none): the closed-form plan (level = ix+iy+iz, colour = parity) is
 * checked against every row's defining equation in one pass -- a plan that
 * satisfies them all is, by induction over the rows, the reference's plan --
 * and the sync-free wavefront runs only if some row violates it.
 * *used_hint = 1 when the checked guess was taken. */
int b2s_level_schedule_hint(int n, const int32_t* rp, const int32_t* ci, int nx, int ny,
                            int32_t* row_group, int32_t* ngroups_host, int* used_hint,
                            cudaStream_t stream);
int b2s_graph_color_hint(int n, const int32_t* rp, const int32_t* ci, int nx, int ny,
                         int32_t* row_group, int32_t* ngroups_host, int* used_hint,
                         cudaStream_t stream);

/* debug: rerun the level (kind 0) / colour (1) kernel recording each row's
 * publication time (%globaltimer, ns) in trace[n] */
int b2s_analysis_trace(int kind, int n, const int32_t* rp, const int32_t* ci, int32_t* row_group,
                       unsigned long long* trace, cudaStream_t stream);

/* _plan_from_groups (bs/analysis.py:61-71): perm (old->new), iperm (new->old,
 * stable), offsets (ngroups+1). */
int b2s_plan_from_groups(int n, const int32_t* row_group, int ngroups, int32_t* perm,
                         int32_t* iperm, int32_t* offsets, cudaStream_t stream);

/* apply_permutation (bs/analysis.py:162-197): new row k = old row take[k],
 * columns through cmap, re-sorted.  Forward: cmap = perm, take = iperm.
 * out_src (optional) receives the source slot of every output block. */
int b2s_permute_bsr(int n, int b, const int32_t* rp, const int32_t* ci, const double* vals,
                    const int32_t* cmap, const int32_t* take, int32_t* out_rp, int32_t* out_ci,
                    double* out_vals, int32_t* out_src, cudaStream_t stream);

/* apply_permutation_vec (bs/analysis.py:153-159): out[i] = in[src[i]]. */
int b2s_gather_rows(int n, int b, const int32_t* src, const double* in, double* out,
                    cudaStream_t stream);

/* int64 -> int32 index narrowing on the device; *overflow_host = 1 when a
 * value does not fit (the host raises; synchronises the stream).  A null
 * overflow_host skips the check and the synchronisation: for indices already
 * validated on the host (a SparsityPattern whose n and nnz fit int32). */
int b2s_narrow_index(long long m, const int64_t* in, int32_t* out, int* overflow_host,
                     cudaStream_t stream);

/* block gather out[q] = in[src[q]] (refresh_values, bs/jacobi.py:139-147). */
int b2s_gather_blocks(long long nblk, int b, const int32_t* src, const double* in, double* out,
                      cudaStream_t stream);

/* ---- SELL-32 device layouts (no reference counterpart: the device form of
 *      the BLOCK_ROW_MAJOR values, bs/blockcore.py:26-44, and of the
 *      per-sweep _Phase packing, bs/ilu0.py:204-236) ----------------------- */

int b2s_slices_plain(int n, int32_t* row0, int32_t* nrows, cudaStream_t stream);
int b2s_slices_grouped_count(int ngroups, const int32_t* offsets, int32_t* base,
                             int32_t* nslices_host, cudaStream_t stream);
int b2s_slices_grouped_fill(int ngroups, int nslices, const int32_t* offsets,
                            const int32_t* base, int32_t* row0, int32_t* nrows,
                            cudaStream_t stream);
/* sel: 0 = all blocks, 1 = strict lower, 2 = strict upper */
int b2s_sell_offsets(int nslices, const int32_t* row0, const int32_t* nrows, const int32_t* rp,
                     const int32_t* ci, int sel, int32_t* sp, long long* slots_host,
                     cudaStream_t stream);
/* the same, plus the widest slice in entries per row (one readback) */
int b2s_sell_offsets_ex(int nslices, const int32_t* row0, const int32_t* nrows, const int32_t* rp,
                        const int32_t* ci, int sel, int32_t* sp, long long* slots_host,
                        int* width_host, cudaStream_t stream);
/* goff/ngroups (optional, plan group offsets): entries of a triangular
 * selection whose column lies in the row's own group are encoded -(c+2),
 * "read the value from before the sweep" -- the reference updates a whole
 * group at once (bs/ilu0.py:125-142). */
int b2s_sell_fill(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                  const int32_t* rp, const int32_t* ci, const double* vals, int sel,
                  const int32_t* sp, const int32_t* goff, int ngroups, int32_t* cols,
                  double* svals, cudaStream_t stream);
/* as b2s_sell_fill, with the values of pattern slot q read from input slot
 * src[q] (the permutation's source map): a plan-order layout filled straight
 * from the unpermuted matrix */
int b2s_sell_fill_src(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                      const int32_t* rp, const int32_t* ci, const double* vals, int sel,
                      const int32_t* sp, const int32_t* goff, int ngroups, int32_t* cols,
                      double* svals, const int32_t* src, cudaStream_t stream);
int b2s_diag_tiles(int nslices, int b, const int32_t* row0, const int32_t* nrows,
                   const double* inv, double* tiles, cudaStream_t stream);
int b2s_slice_conflicts(int nslices, const int32_t* row0, const int32_t* nrows,
                        const int32_t* rp, const int32_t* ci, int* conflict_host,
                        cudaStream_t stream);

/* ---- SpMV (bs/blockcore.py:342-376 spmv_array / residual) --------------- */

/* mode 0: y = A x; 1: + partials w.y; 2: + partials y.y and y.w;
 * 3: y = w - A x (residual) + partials y.y.  One partial per CTA (nparts). */
int b2s_spmv(int b, int mode, int nparts, int nslices, const int32_t* row0,
             const int32_t* nrows, const int32_t* sp, const int32_t* cols, const double* vals,
             const double* x, double* y, const double* w, double* part0, double* part1,
             const int* done, cudaStream_t stream);

/* ---- ILU0 (bs/ilu0.py) --------------------------------------------------- */

/* decompose (bs/ilu0.py:145-201) on an already permuted matrix, in place;
 * B2S_SINGULAR_PIVOT with the smallest failing permuted row. */
int b2s_ilu0_factor(int n, int b, int nslices, const int32_t* row0, const int32_t* nrows,
                    const int32_t* rp, const int32_t* ci, const int32_t* diag, double* vals,
                    double* inv_diag, int32_t* bad_row_host, cudaStream_t stream);
/* The same in two halves.  Symbolic (pattern only; may synchronise): the
 * update pairs of every lower entry behind an opaque handle, freed
 * stream-ordered by b2s_ilu0_symbolic_free.  Numeric: values in place; with
 * bad_dev (device int, INT32_MAX on entry) the smallest failing permuted row
 * is left there with no host read, else as b2s_ilu0_factor. */
int b2s_ilu0_symbolic(int n, int b, const int32_t* rp, const int32_t* ci, const int32_t* diag,
                      void** handle, cudaStream_t stream);
int b2s_ilu0_numeric(const void* handle, int b, int nslices, const int32_t* row0,
                     const int32_t* nrows, const int32_t* rp, const int32_t* ci,
                     const int32_t* diag, double* vals, double* inv_diag, int* bad_dev,
                     int32_t* bad_row_host, cudaStream_t stream);
int b2s_ilu0_symbolic_free(void* handle, cudaStream_t stream);

/* decompose (bs/ilu0.py:145-201) for a plan of two independent groups
 * (a 2-colouring), straight into SELL layouts on the group-aligned slice map
 * (csrc/factor2c.cu): reads the operator's SELL (a_*), writes the strict-
 * lower SELL (l_cols/l_vals on offsets l_sp), the plan-order inverse
 * diagonals inv (n*b*b), colour 1's U_ii (udiag, (n-goff1)*b*b) and the
 * per-slice inverse tiles.  s1/goff1: first slice / plan row of colour 1.
 * B2S_SINGULAR_PIVOT (smallest failing plan row in *bad_row_host), or
 * B2S_UNSUPPORTED when the pattern is not a 2-colour structure.  Results are
 * bit-identical to b2s_ilu0_factor. */
int b2s_factor_2colour(int n, int b, int goff1, int s1, int nslices, const int32_t* row0,
                       const int32_t* nrows, const int32_t* a_sp, const int32_t* a_cols,
                       const double* a_vals, const int32_t* l_sp, int32_t* l_cols,
                       double* l_vals, double* inv, double* udiag, double* dtiles,
                       int32_t* bad_row_host, cudaStream_t stream);
/* The same, stream-ordered with no host read (the solve path checks later):
 * flags_dev (device, 2 ints) holds {INT32_MAX, 0} on entry and receives
 * {smallest singular plan row or INT32_MAX, 1 if not a 2-colour structure}. */
int b2s_factor_2colour_async(int n, int b, int goff1, int s1, int nslices, const int32_t* row0,
                             const int32_t* nrows, const int32_t* a_sp, const int32_t* a_cols,
                             const double* a_vals, const int32_t* l_sp, int32_t* l_cols,
                             double* l_vals, double* inv, double* udiag, double* dtiles,
                             int* flags_dev, cudaStream_t stream);
/* the plan-order CSR values of combined L\U from the layouts above (rp =
 * the plan-order row pointers); materialised only on request */
int b2s_factor_2colour_combined(int n, int b, int goff1, int s1, const int32_t* rp,
                                const int32_t* a_sp, const int32_t* a_cols, const double* a_vals,
                                const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                                const double* udiag, double* lu, cudaStream_t stream);

/* Ilu0Factorization.apply_permuted_array (bs/ilu0.py:105-142). */
int b2s_ilu0_apply(int n, int b, int kc, int nslices, const int32_t* row0, const int32_t* nrows,
                   const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                   const int32_t* u_sp, const int32_t* u_cols, const double* u_vals,
                   const double* dinv_tiles, const double* r, double* y, double* z, int reset_y,
                   int flags, void* tickets, cudaStream_t stream);
int b2s_fill_sentinel(long long m, double* v, cudaStream_t stream);

/* Phased application (same result as b2s_ilu0_apply, bit for bit) for plans
 * of 2..32 independent groups with no same-group entries -- every colouring:
 * 2(G-1) data-parallel passes, no polling, no sentinel preconditions.
 * gslice_host[0..G]: first slice of each group of the group-aligned slice
 * map (HOST memory); goff1: first plan row of group 1. */
int b2s_ilu0_apply_phased(int n, int b, int kc, int ngroups, const int32_t* gslice_host,
                          int goff1, const int32_t* row0, const int32_t* nrows,
                          const int32_t* l_sp, const int32_t* l_cols, const double* l_vals,
                          const int32_t* u_sp, const int32_t* u_cols, const double* u_vals,
                          const double* dinv_tiles, const double* r, double* y, double* z,
                          cudaStream_t stream);

/* Tiled level-scheduled sweeps (csrc/tiles.cu): rows split into px*py column
 * patches of an nx x ny natural-order grid (px > 0) or T contiguous input-row
 * ranges; one co-resident CTA per tile walks the tile's rows one plan group
 * ("step") at a time -- a producer warp streams each step's packed record
 * into a shared-memory ring with TMA bulk copies, consumer warps resolve
 * in-tile dependencies from shared memory and poll only cross-tile ones.
 * rp/ci/diag/lu: combined L\U in plan order; inv: inverse diagonal blocks.
 * B2S_UNSUPPORTED when T exceeds the SMs or the ring does not fit. */
int b2s_tiles_create(int n, int b, int T, int nx, int ny, int px, int py, const int32_t* iperm,
                     const int32_t* rp, const int32_t* ci, const int32_t* diag, const double* lu,
                     const double* inv, const int32_t* goff, int ngroups, void** handle_out,
                     cudaStream_t stream);
int b2s_tiles_destroy(void* handle);
/* debug: per-step event times of the step kernels into buf[2][T][1024][4];
 * dbg != 0 only for timing experiments (results are then wrong) */
int b2s_tiles_trace(void* handle, unsigned long long* buf, int dbg);
int b2s_tiles_apply(int b, const void* handle, const double* r, double* y, double* z,
                    int reset_y, cudaStream_t stream);

/* ---- wavefront sweeps for natural-order 7-point grids (csrc/gridwave.cu) --
 * Deep plans (level schedules, the sequential plan) of an nx*ny*nz grid: one
 * warp per tile of wx*wy <= 32 columns walks the levels, in-tile
 * dependencies through warp shuffles, tile edges through sentinel-checked
 * edge buffers.  create checks that every row of the plan-order pattern
 * (perm old->plan, iperm plan->old) is a stencil row of the plan --
 * B2S_UNSUPPORTED otherwise (keep the sync-free sweeps) -- and fill packs the
 * factor's values into the warp's step records.  apply: z = U^-1 L^-1 r in
 * plan order, bit-identical to b2s_ilu0_apply.  Replaces
 * Ilu0Factorization.apply (bs/ilu0.py:105-142). */
long long b2s_gw_workspace_bytes(int n, int b, int nx, int ny, int nz, int wx, int wy);
/* pattern phase (rp/ci: the plan-order pattern; synchronises once) */
int b2s_gw_create(int n, int b, int nx, int ny, int nz, int wx, int wy, const int32_t* perm,
                  const int32_t* iperm, const int32_t* rp, const int32_t* ci, void* workspace,
                  long long ws_bytes, void** handle_out, cudaStream_t stream);
/* value phase, stream-ordered: lu = combined L\U on that pattern, inv = inverse diagonals */
int b2s_gw_fill(void* handle, const double* lu, const double* inv, cudaStream_t stream);
int b2s_gw_destroy(void* handle);
/* ILU0 of the handle's grid straight into its step records (wavefront
 * factorisation, bit-identical to b2s_ilu0_factor on these patterns): rp/ci/
 * diag = plan-order pattern, vsrc = plan slot -> input slot (null: identity
 * plan), vals = input values; writes the plan-order inverse diagonals (invd)
 * and U_ii (dvals); the smallest singular plan row goes to *bad_dev (device,
 * INT32_MAX on entry).  Stream-ordered, no host read; B2S_UNSUPPORTED when
 * the tiles cannot be co-resident (factorise the general way). */
long long b2s_gw_factor_workspace_bytes(const void* handle);
int b2s_gw_factor(void* handle, const int32_t* rp, const int32_t* ci, const int32_t* diag,
                  const int32_t* vsrc, const double* vals, double* invd, double* dvals,
                  int* bad_dev, void* workspace, long long workspace_bytes, cudaStream_t stream);
/* the combined L\U CSR values from the records (lu holds the plan-order
 * operator values on entry) -- materialised only on request */
int b2s_gw_unpack_lu(const void* handle, const int32_t* diag, const double* dvals, double* lu,
                     cudaStream_t stream);
int b2s_gw_apply(int b, const void* handle, const double* r, double* z, cudaStream_t stream);
/* debug (B2S_GW_TRACE set at create): the last apply's per-step end times,
 * [2][T][S] ns; shape = {TX, TY, S, wx, wy} */
int b2s_gw_trace(const void* handle, unsigned long long* host, long long cap, long long* count,
                 int* shape);

/* ---- reductions (bs/krylov.py:30-60) ------------------------------------ */

int b2s_dot(long long m, const double* a, const double* b, int nparts, double* parts,
            double* out, cudaStream_t stream);
int b2s_all_finite(long long m, const double* a, int* bad, cudaStream_t stream);
/* Inner product in the reference's exact summation order (bs/krylov.py:30-47,
 * REDUCTION_CHUNK = 64): parts[c] = numpy's np.add.reduceat of a*b over the
 * c-th 64-element chunk (ceil(m/64) doubles), *total = np.cumsum(parts)[-1]
 * (skipped when total is NULL).  Bit-identical to the reference
 * (csrc/refdot.cu); used by the public dot/norm/dot_partials and the
 * reported initial residual norm, not by the Krylov loop. */
int b2s_dot_chunked(long long m, const double* a, const double* b, double* parts,
                    double* total, cudaStream_t stream);
int b2s_reduce(const double* parts, int np, double* out, cudaStream_t stream);

/* BiCGStab vector steps with host scalars (multi-GPU loop; bs/krylov.py:201-233):
 * scratch = >= 128 device bytes for the staged scalars. */
int b2s_vec_p(long long m, int k, double beta, double omega, const double* r, const double* v,
              double* p, double* scratch, cudaStream_t stream);
int b2s_vec_s(long long m, double alpha, const double* r, const double* v, double* phat,
              double* x, double* s, double* parts, int nparts, int reset, double* scratch,
              cudaStream_t stream);
int b2s_vec_r(long long m, double omega, double* shat, const double* t, const double* s,
              const double* rhat, double* x, double* r, double* prr, double* prho, int nparts,
              int reset, double* scratch, cudaStream_t stream);

/* ---- BiCGStab (bs/krylov.py:140-244) ------------------------------------ */

/* 2-colour plans: *ok_host = 1 when every colour-0 row of the operator
 * (slices [0, s1) of the group-aligned map) is its diagonal block followed
 * by exactly the factor's U row (same columns, bitwise-equal blocks) -- then
 * the backward sweep of colour 0 and the SpMV of colour 0 share one read of
 * those blocks (csrc/fused.cu). */
int b2s_fuse_check(int s1, int b, const int32_t* row0, const int32_t* nrows, const int32_t* a_sp,
                   const int32_t* a_cols, const double* a_vals, const int32_t* u_sp,
                   const int32_t* u_cols, const double* u_vals, int* ok_host,
                   cudaStream_t stream);

/* Sharded solves (one shard per rank): peer-memory communication.  Every
 * pointer is device memory valid in this process -- another process's
 * buffers opened with b2s_ipc_open (NVLink P2P), or another shard's buffers
 * on the same GPU.  Ghost rows (the columns of owned rows that other ranks
 * own) are appended after the n owned rows of x, phat and shat; before each
 * SpMV they are pulled straight from the owners' vectors.  Dot products are
 * all-reduced through per-rank mailboxes (kMboxSlots x nranks x 4 doubles):
 * the last CTA of each reducing kernel posts its local sums into every
 * rank's mailbox and sums all ranks' posts in rank order (deterministic). */
typedef struct {
  int rank, nranks;
  int nghost;                      /* ghost rows after the n owned rows */
  const int32_t* ghost_owner;      /* [nghost] owning rank */
  const int32_t* ghost_row;        /* [nghost] plan-order row on the owner */
  int nnbr;
  const int32_t* nbr;              /* [nnbr] ranks this one pulls ghosts from */
  double* const* peer_x;           /* [nranks] every rank's x / phat / shat */
  double* const* peer_phat;
  double* const* peer_shat;
  long long* flags;                /* [nranks] readiness flags peers post here */
  long long* const* peer_flags;    /* [nranks] every rank's flags */
  double* mbox;                    /* this rank's mailbox */
  double* const* peer_mbox;        /* [nranks] every rank's mailbox */
  long long seq_base;              /* strictly increasing per solve, equal on all ranks */
  int shared_device;               /* shards share one GPU: no programmatic launch overlap */
  /* optional: called (by every shard's host thread) once all host-side
   * preparation is done and again after the device loop -- shards on one GPU
   * rendezvous there, so no implicitly synchronising host call (host/device
   * allocation, graph instantiation) runs while a peer's kernel waits */
  int (*host_barrier)(void*);   /* returns 0; nonzero: this host thread failed */
  void* host_barrier_ctx;
  /* Optional, 2-colour plans: run the fused colour passes on the local block
   * (b2s_bicg_args' operator = the owned columns only) and add the ghost
   * couplings afterwards -- they are the last entries of their rows, so the
   * row sums continue in column order.  bnd_*: the rows with ghost couplings
   * (plan order) as CSR over ghost indices; full_*: the whole operator (ghost
   * columns included) on the same slice map, for the r0 / final residuals. */
  int nbnd;
  const int32_t* bnd_row;
  const int32_t* bnd_ptr;
  const int32_t* bnd_col;
  const double* bnd_val;
  const int32_t* full_sp;
  const int32_t* full_cols;
  const double* full_vals;
  /* bound on every device-side wait for a peer (0: $B2S_MESH_TIMEOUT_MS, else
   * 60 s); a wait that expires raises the abort word in every rank's mailbox
   * (the last 64 bytes of b2s_mesh_mbox_bytes), every rank leaves its loop
   * and b2s_bicgstab returns B2S_PEER_TIMEOUT */
  long long timeout_ns;
} b2s_mesh;

#define B2S_MBOX_SLOTS 8
/* bytes of one rank's mailbox */
long long b2s_mesh_mbox_bytes(int nranks);
/* double offsets of phat and shat inside the b2s_bicgstab workspace */
int b2s_bicgstab_workspace_layout(int n, int nghost, int b, long long* phat_off,
                                  long long* shat_off);
long long b2s_bicgstab_workspace_bytes_mesh(int n, int nghost, int b, int nparts);
/* CUDA IPC of a device buffer (any pointer inside a cudaMalloc allocation):
 * 64-byte handle + offset from the allocation base; open maps it here. */
int b2s_ipc_handle(const void* ptr, unsigned char* handle64, long long* offset);
int b2s_ipc_open(const unsigned char* handle64, long long offset, void** ptr_out);
int b2s_ipc_close(void* base);

/* Device description of a WellSet (standard wells first, then multi-segment
 * ones, in list order); every pointer is device memory, offsets in doubles.
 * Built by paper_2309_11488_b200/wells.py (DeviceWells). */
typedef struct {
  int nwells, nb;
  const int32_t *kind, *M, *nseg, *bptr, *bcell, *bseg;
  const int64_t* boff;
  const double* bvals;
  const int64_t* doff;
  const double* dvals;
  const int64_t* pivoff;
  const int32_t* piv;
  const int64_t* toff;
  int ncells;
  const int32_t *cells, *cptr;
  const int64_t *ccoff, *ct2;
  const int32_t* cM;
  const double* cvals;
} b2s_wells;

typedef struct {
  int n, b, nparts, precond /* 0 none, 1 ilu0 */, kc, maxit, check_lag;
  int refill_y; /* 1: U has same-group entries, refill the sweep scratch each apply */
  int sweep_flags; /* bit 0: nanosleep back-off while polling */
  double tol;
  int nslices;
  const int32_t *row0, *nrows;
  const int32_t *a_sp, *a_cols;
  const double* a_vals;
  const int32_t *l_sp, *l_cols;
  const double* l_vals;
  const int32_t *u_sp, *u_cols;
  const double* u_vals;
  const double* dinv_tiles;
  const void* tiles; /* optional b2s_tiles_create() handle: tiled sweeps */
  const double* rhs;
  double* x;    /* x0 on entry, solution on exit */
  double* work; /* b2s_bicgstab_workspace_bytes() */
  cudaStream_t stream;
  /* phased sweeps (b2s_ilu0_apply_phased) when ngroups >= 2 */
  int ngroups, goff1;
  const int32_t* gslice_host;
  /* 2 colours and b2s_fuse_check() passed: fused colour-0 backward + SpMV */
  int fuse;
  /* sharded solve over peer memory (NULL: single system); x is then
   * (n + mesh->nghost) * b long and the workspace sized by
   * b2s_bicgstab_workspace_bytes_mesh */
  const b2s_mesh* mesh;
  /* 1: x0 is all zeros (the caller passed no initial guess): r0 = b - A 0 is
   * b itself (bs/krylov.py:171 up to the sign of zero), so the initial
   * residual SpMV (and, sharded, its ghost pull) is skipped */
  int x0_zero;
  /* Optional separately applied wells (bs/krylov.py:84-94, NULL: none): the
   * operator is A - sum_w C_w^T D_w^-1 B_w.  Before each operator
   * application the well terms of its input go into well_corr (compact
   * perforated cells, b doubles each; well_scratch: sum over wells of nseg*M
   * doubles) and the SpMV subtracts them before its dot-product epilogue.
   * well_slice[s]: base of slice s's 32 entries in well_lane, or -1;
   * well_lane[base + l]: compact cell of row row0[s] + l, or -1.  The wells'
   * cells are in the operator's (plan) row order.  Not with fuse or mesh. */
  const b2s_wells* wells;
  const int32_t* well_slice;
  const int32_t* well_lane;
  double* well_corr;
  double* well_scratch;
  /* optional b2s_gw_create() handle: the preconditioner applications use the
   * wavefront sweeps of a natural-order grid (takes precedence over tiles) */
  const void* gw;
} b2s_bicg_args;

typedef struct {
  int converged, reason /* 1 converged 2 breakdown 3 numerical 4 budget */;
  int graph_launches, kernels_per_iteration;
  double iterations, initial_norm, final_norm;
} b2s_bicg_result;

long long b2s_bicgstab_workspace_bytes(int n, int b, int nparts);
int b2s_bicgstab(const b2s_bicg_args* args, b2s_bicg_result* result);

/* ---- wells applied separately (bs/wells.py:125-162, bs/krylov.py:84-94) --- */



/* y -= sum_w C_w^T D_w^-1 B_w x; scratch: sum over wells of nseg*M doubles.
 * Replaces WellSet.apply_contributions_array (bs/wells.py:196-202). */
int b2s_wells_apply(const b2s_wells* wells, const double* x, double* y, double* scratch,
                    cudaStream_t stream);

/* ---- Block-Jacobi copy plan (bs/jacobi.py:111-147) ---------------------- */

/* The greedy heaviest-edge region growing of bs/jacobi.py:61-108 on the host:
 * undirected edges lo[e] < hi[e] with weights w[e]; part[n] receives the
 * partition of every cell (k balanced parts, seeds = lowest unassigned
 * cells, heap order (-w, cell) as heapq) -- the reference's assignment. */
int b2s_partition_greedy(long long n, long long nedges, const long long* lo, const long long* hi,
                         const double* w, long long k, long long* part);
int b2s_jacobi_pattern(int n, const int32_t* rp, const int32_t* ci, const int32_t* part,
                       int32_t* new_rp, int32_t* kept_host, cudaStream_t stream);
int b2s_jacobi_fill(int n, const int32_t* rp, const int32_t* ci, const int32_t* part,
                    const int32_t* new_rp, int32_t* new_ci, int32_t* indices,
                    cudaStream_t stream);

/* ---- library identity / process configuration --------------------------- */
const char* b2s_version(void);
/* keep freed cudaMallocAsync scratch in the default pool (setup speed) */
int b2s_retain_pool_memory(int device);

#ifdef __cplusplus
}
#endif
#endif /* B200SOLVE_H */
