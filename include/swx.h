/*
 * swx.h -- C ABI of the B200-native REXI hot path (libswx.so).
 *
 * Drop-in boundary for the reference package `swerexi` (arXiv 1805.06557,
 * /root/reference/pkg/src/swerexi).  The reference is pure Python; its seam
 * for this path is the solver duck type returned by
 *     get_solver(token, dt, params)                       solvers.py:259-261
 * with warm/solve_stacked/solve_stacked_batch/apply_stacked (solvers.py:188-256),
 * the pole reduction tree_sum + realify_stacked (steppers.py:157-185) that every
 * caller applies after solve_stacked_batch (steppers.py:231-234, 264-266;
 * parallel.py:140-169), and the spectral transforms / tendencies of the N term
 * (sphere.py:297-430, swe.py:188-279).  Each entry point below names the
 * reference interface it replaces.
 *
 * Conventions
 *   - complex128 values are `swx_c128` = {re, im} (layout of numpy complex128
 *     and CUDA double2).
 *   - Spectral state = 3 fields [phi', vort, div], each packed m-major over the
 *     triangle l >= m (the reference's mode_index_map, solvers.py:288-290):
 *     slot(l, m) = m*(T+1) - m*(m-1)/2 + (l - m);  ncoef = (T+1)(T+2)/2.
 *     A state is 3*ncoef contiguous swx_c128, field-major.
 *   - Pointers named d_* are device pointers; h_* are host pointers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *     stream-ordered and allocation-free after *_create; nothing synchronises
 *     unless documented.
 *   - Return value: SWX_OK or an SWX_ERR_* code; swx_last_error() gives the
 *     message.  SWX_ERR_SOLVER maps to swerexi.errors.SolverError (errors.py:24),
 *     SWX_ERR_CONFIG to ConfigurationError (errors.py:8), SWX_ERR_DATA to
 *     DataError (errors.py:12).
 */
#ifndef SWX_H
#define SWX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWX_OK 0
#define SWX_ERR_CONFIG 1
#define SWX_ERR_SOLVER 2
#define SWX_ERR_DATA 3
#define SWX_ERR_CUDA 4

#define SWX_GROUP_LG 0 /* gravity terms only: diagonal 2x2 per (l,m)      */
#define SWX_GROUP_L 1  /* gravity + Coriolis: two tridiagonal chains per m */

#define SWX_TEND_LC 1 /* linear Coriolis atom (swe.py:188-211)          */
#define SWX_TEND_N 2  /* nonlinear atom (swe.py:214-251)                */

typedef struct swx_c128 {
  double re, im;
} swx_c128;

typedef struct swx_solver_s *swx_solver;
typedef struct swx_sht_s *swx_sht;

/* ---- library ------------------------------------------------------------ */
int swx_version(void);
const char *swx_last_error(void);

/* ---- shifted solvers: replaces ShiftedLinearSolver / get_solver ----------
 * solvers.py:57-81 (construction), 259-261 (get_solver).  group is
 * SWX_GROUP_LG or SWX_GROUP_L; dt > 0; phibar > 0 (swe.py:78-87).            */
int swx_solver_create(swx_solver *out, int group, int trunc, double dt,
                      double phibar, double radius, double omega);
int swx_solver_destroy(swx_solver s);

/* warm(alphas), solvers.py:188-194 (+ the guards of 95-104 and 176-184).
 * Uploads the N shifts and validates every (pole, l|m) system: a singular
 * gravity block (|det| <= 1e-13 (|a|^2 + dt^2 phibar kappa)), alpha == 0, or a
 * chain pivot with (||dt L_m||_1 + |a|) / |pivot| > 1e13 returns
 * SWX_ERR_SOLVER with *err_pole = n and *err_index = l (lg) or m (l).
 * Synchronises `stream`.                                                     */
int swx_solver_warm(swx_solver s, const swx_c128 *h_alphas, int n_poles,
                    int *err_pole, int *err_index, void *stream);

/* Workspace for swx_rexi_sum over [pole_begin, pole_end) with n_rhs RHS.    */
size_t swx_rexi_workspace_bytes(swx_solver s, int n_rhs, int pole_begin,
                                int pole_end);

/* Fused REXI pole sum -- replaces solve_stacked_batch + beta weighting +
 * tree_sum + realify_stacked (steppers.py:214-235, 262-267; parallel.py:140-169):
 *   d_out[r] = sum_{n in [pole_begin, pole_end)} d_betas[r*n_poles + n] *
 *              (dt L + alpha_n)^{-1} d_rhs[r]            for r < n_rhs (<= 2)
 * without materialising the (N, 3, n, n) batch.  Poles are reduced in the
 * reference's fixed pairwise tree order; for power-of-two pole counts the
 * result over a block equals the block's subtree of tree_sum, so per-rank
 * partials combined by swx_tree_combine are bitwise independent of the rank
 * count.  realify != 0 zeroes Im of the m = 0 column (steppers.py:175-185);
 * pass 0 for partial sums that are reduced across ranks afterwards.
 * d_betas is device memory (n_rhs * n_poles); d_rhs / d_out hold n_rhs states. */
int swx_rexi_sum(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                 const swx_c128 *d_betas, int pole_begin, int pole_end,
                 int realify, swx_c128 *d_out, void *d_workspace,
                 size_t workspace_bytes, void *stream);

/* Prepared pole sums.  For the gravity group the per-(pole, l) factors
 * (beta folded, solvers.py:93-107 with the reciprocals hoisted) depend only
 * on the shifts, the weights and l, so a caller that reuses one weight set
 * (every ETD2RK step, rexi_step at fixed dt) builds them once with
 * swx_rexi_prepare into a buffer of swx_rexi_prepared_bytes and then calls
 * swx_rexi_sum_prepared (same result as swx_rexi_sum).  The Coriolis group
 * needs no preparation (0 bytes; the prepared call forwards to swx_rexi_sum). */
size_t swx_rexi_prepared_bytes(swx_solver s, int n_rhs, int pole_begin, int pole_end);
int swx_rexi_prepare(swx_solver s, int n_rhs, const swx_c128 *d_betas, int pole_begin,
                     int pole_end, void *d_prep, size_t prep_bytes, void *stream);
int swx_rexi_sum_prepared(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                          const swx_c128 *d_betas, const void *d_prep, int pole_begin,
                          int pole_end, int realify, swx_c128 *d_out, void *d_workspace,
                          size_t workspace_bytes, void *stream);
/* The same sum with the ETD2RK combination fused into its epilogue:
 * d_out = d_base + scale * (realified) sum, per state -- the
 * `psi0 u + dt psi1 N(u)` and `a + dt psi2 (N(a) - N(u))` updates of
 * etdrk2_step (steppers.py:259-269), bitwise equal to swx_rexi_sum_prepared
 * followed by swx_state_axpy.  d_base has the layout of d_out.              */
int swx_rexi_sum_prepared_axpy(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                               const swx_c128 *d_betas, const void *d_prep, int pole_begin,
                               int pole_end, int realify, const swx_c128 *d_base,
                               double scale, swx_c128 *d_out, void *d_workspace,
                               size_t workspace_bytes, void *stream);

/* The prepared sum (d_base may be null: plain sum) started from a table
 * analysis' column counters instead of stream order: d_ready is the address
 * returned by swx_sht_set_done_signal for the SH plan whose signalled
 * tendency immediately precedes this call on the stream.  The pole-sum items
 * (degree l, 32 modes) wait for their columns (generation x item count;
 * the counters only grow), so the sum overlaps the tail of the analysis.
 * One stream per SH plan.  Same arithmetic as
 * swx_rexi_sum_prepared(_axpy) (bitwise).  Replaces the stream-ordered
 * `etdrk2_generic` pole sums of steppers.py:259-269 on the device step.     */
int swx_rexi_sum_prepared_ready(swx_solver s, int n_rhs, const swx_c128 *d_rhs,
                                const swx_c128 *d_betas, const void *d_prep, int pole_begin,
                                int pole_end, int realify, const swx_c128 *d_base,
                                double scale, swx_c128 *d_out, void *d_workspace,
                                size_t workspace_bytes, int *d_ready, void *stream);

/* Forward operator (dt L + alpha) x -- apply_stacked, solvers.py:252-256.   */
int swx_apply(swx_solver s, swx_c128 alpha, const swx_c128 *d_x,
              swx_c128 *d_out, void *stream);

/* ---- reductions / state algebra ------------------------------------------ */
/* d_out = realify?( tree_sum(d_parts[0..n_parts)) ), each part n_states*3*ncoef
 * values -- the cross-rank / cross-block reduce of parallel.py:161-169.     */
int swx_tree_combine(int trunc, int n_states, int n_parts,
                     const swx_c128 *d_parts, int realify, swx_c128 *d_out,
                     void *stream);
/* d_out[i] = tree_sum(d_parts[p * n_values + i], p < n_parts) for i < n_values,
 * no realify: the per-slice combine of the tree-order reduce-scatter
 * (PoleComm, parallel.py:161-169) -- every rank combines its 1/K slice of
 * all ranks' block partials, then the slices are all-gathered.            */
int swx_tree_combine_flat(size_t n_values, int n_parts, const swx_c128 *d_parts,
                          swx_c128 *d_out, void *stream);
/* d_out = d_x + s * d_y over n_states packed states (PrognosticState
 * __add__/__mul__, swe.py:135-157).  d_out may alias d_x.                    */
int swx_state_axpy(int trunc, int n_states, const swx_c128 *d_x, double s,
                   const swx_c128 *d_y, swx_c128 *d_out, void *stream);

/* ---- spherical-harmonic transforms + tendencies --------------------------
 * Plan = SpherePlan (sphere.py:163-223) for a Gauss-Legendre x equiangular
 * grid; h_sinlat / h_weights are the nlat Gauss nodes (ascending) and weights
 * (sphere.py:31-58).  Legendre functions are generated on the fly from the
 * reference recurrence (sphere.py:72-112); h_seed holds the sectoral seeds
 * Pbar_m^m(x_j) as an (T+1) x nlat row-major table (m-major).              */
int swx_sht_create(swx_sht *out, int trunc, int nlat, int nlon, double radius,
                   double omega, const double *h_sinlat, const double *h_weights,
                   const double *h_seed);
int swx_sht_destroy(swx_sht p);
size_t swx_sht_workspace_bytes(swx_sht p);

/* synthesis of n_fields real-origin fields: packed coeffs -> (nlat, nlon)
 * grids (sphere.py:318-339).                                                */
int swx_sht_synthesis(swx_sht p, int n_fields, const swx_c128 *d_coeffs,
                      double *d_grid, void *d_workspace, size_t ws_bytes,
                      void *stream);
/* analysis of n_fields real grids -> packed coeffs (sphere.py:297-315).     */
int swx_sht_analysis(swx_sht p, int n_fields, const double *d_grid,
                     swx_c128 *d_coeffs, void *d_workspace, size_t ws_bytes,
                     void *stream);
/* u, v grids from packed vort/div (sphere.py:375-402).                      */
int swx_sht_uv(swx_sht p, const swx_c128 *d_vort, const swx_c128 *d_div,
               double *d_u, double *d_v, void *d_workspace, size_t ws_bytes,
               void *stream);
/* Vorticity and divergence coefficients from grid winds, vortdiv_from_uv
 * (sphere.py:405-430): d_u, d_v are (nlat, nlon) float64 grids; needs the
 * plan's Legendre table (SWX_ERR_CONFIG above T ~700).                     */
int swx_sht_vortdiv(swx_sht p, const double *d_u, const double *d_v, swx_c128 *d_vort,
                    swx_c128 *d_div, void *d_workspace, size_t ws_bytes, void *stream);
/* tendency_group for atoms in `atoms` (SWX_TEND_LC | SWX_TEND_N), swe.py:254-279:
 * d_out = sum of the selected atom tendencies of d_state (one packed state).  */
int swx_sht_tendency(swx_sht p, int atoms, const swx_c128 *d_state,
                     swx_c128 *d_out, void *d_workspace, size_t ws_bytes,
                     void *stream);
/* Record `event` (cudaEvent_t; null clears) on the tendency's stream right
 * after the synthesis stage of every following swx_sht_tendency[_sub] call,
 * so independent work on another stream can overlap the lighter grid and
 * analysis stages instead of the FP64-bound synthesis.                      */
int swx_sht_set_synth_event(swx_sht p, void *event);
/* Column hand-off to a following lg pole sum: while on, the tendency's table
 * analysis bumps a generation counter (d_counters[T+1]) before it lets
 * dependent kernels launch and counts each completed item in per-column
 * counters d_counters[m]; *d_counters receives their address (pass it to
 * swx_rexi_sum_prepared_ready).  Needs the table analysis (the fused-stage
 * plans).  No reference counterpart (device scheduling).                    */
int swx_sht_set_done_signal(swx_sht p, int on, int **d_counters);
/* d_out = tendency(d_state) - d_sub, the difference N(a) - N(u) of the
 * ETD2RK stage (steppers.py:262-266) fused into the analysis epilogue;
 * bitwise equal to swx_sht_tendency followed by swx_state_axpy(-1).        */
int swx_sht_tendency_sub(swx_sht p, int atoms, const swx_c128 *d_state,
                         const swx_c128 *d_sub, swx_c128 *d_out, void *d_workspace,
                         size_t ws_bytes, void *stream);

/* The three stages of swx_sht_tendency[_sub] separately, on a column range:
 * stage 0 synthesises columns [m0, m1) of d_state into the workspace's grid
 * stage rows, stage 1 runs the fused grid stage (every latitude pair; needs
 * all columns synthesised), stage 2 the analysis of columns [m0, m1) into
 * d_out (minus d_sub when non-null).  Column blocks of stages 0 and 2 are
 * independent, so a caller can pipeline them with the per-column pole sums
 * (the ETD2RK engine's analysis -> psi_k -> synthesis chain).  Fused-grid
 * (table) plans only.                                                       */
int swx_sht_tendency_part(swx_sht p, int stage, int atoms, int m0, int m1,
                          const swx_c128 *d_state, const swx_c128 *d_sub, swx_c128 *d_out,
                          void *d_workspace, size_t ws_bytes, void *stream);
/* 1 when the plan has the separable (fused-grid, table) tendency stages.    */
int swx_sht_has_stages(swx_sht p);

/* ---- column-sharded N term over ranks -----------------
 * The reference evaluates the non-linear tendency on every worker (the
 * paper's replicated "no communication" non-linearities, parallel.py:185-214,
 * PAPER.md:849-853).  Here rank r of K owns the zonal columns
 * [m_bounds[r], m_bounds[r+1]) -- balanced by column length, so the Legendre
 * synthesis/analysis and the lg pole sums split evenly -- and the latitude
 * pairs [p_bounds[r], p_bounds[r+1]) of the padded pair range [0, nt16) for
 * the longitude transforms and grid products.  One tendency is three stages
 * separated by two all-to-all exchanges the caller performs (NCCL
 * all_to_all_single with the byte counts of swx_sht_shard_counts):
 *   stage 0: synthesis of the own columns for all pairs; packs exchange 0
 *            (Fourier rows of every peer's pairs, own columns) into d_send;
 *   stage 1: unpacks exchange 0 from d_recv; fused grid stage of the own
 *            pairs; packs exchange 1 (prepared analysis rows of every peer's
 *            columns, own pairs) into d_send;
 *   stage 2: unpacks exchange 1; analysis of the own columns into the own
 *            columns' slots of d_out (d_out - d_sub with d_sub).
 * Slabs are ordered by peer rank; the self slab is empty (it stays in the
 * workspace).  With K = 1 the stages run exactly the kernels of
 * swx_sht_tendency; for any K every coefficient is computed by the same
 * kernel arithmetic, so the sharded result is bitwise equal to it.
 * Needs the fused grid path (Legendre table, nlon_t <= 1024).               */
#define SWX_MAX_RANKS 64
typedef struct swx_shard {
  int nranks, rank;
  int m_bounds[SWX_MAX_RANKS + 1]; /* columns of rank r: [m_bounds[r], m_bounds[r+1])   */
  int p_bounds[SWX_MAX_RANKS + 1]; /* padded latitude pairs of rank r (last ends at nt16) */
} swx_shard;
/* Balanced bounds (host only, no device needed).                            */
int swx_shard_init(swx_shard *sh, int trunc, int nlat, int nranks, int rank);
/* Per-peer byte counts of `exchange` (0 or 1) for atoms; h_send/h_recv hold
 * nranks entries.  Returns max(total send, total recv) bytes (0 on error).  */
size_t swx_sht_shard_counts(swx_sht p, const swx_shard *sh, int exchange, int atoms,
                            size_t *h_send, size_t *h_recv);
int swx_sht_tendency_shard(swx_sht p, int stage, int atoms, const swx_shard *sh,
                           const swx_c128 *d_state, const swx_c128 *d_sub, swx_c128 *d_out,
                           const void *d_recv, void *d_send, void *d_workspace,
                           size_t ws_bytes, void *stream);
/* Column-sharded plain transforms (the cfg4 T1279 round trip): synthesis
 * stage 0 synthesises the own columns of n_fields (<= 4) packed fields for
 * every latitude and packs the Fourier rows of every peer's latitude pairs;
 * stage 1 unpacks the rows received and runs the longitude transforms of
 * the own pairs' rows into d_grid ((n_fields, nlat, nlon); only the own
 * rows -- south [a, b), north [nlat-b, nlat-a) of pairs [a, b) -- are
 * written).  Analysis stage 0 transforms the own rows of d_grid and packs
 * the Fourier coefficients of every peer's columns; stage 1 unpacks, folds
 * and contracts the own columns into their slots of d_coeffs (table-free
 * plans, T > ~700).  Exchange byte counts: swx_sht_transform_shard_counts
 * (which = 0 synthesis, 1 analysis).                                       */
size_t swx_sht_transform_shard_counts(swx_sht p, const swx_shard *sh, int which, int n_fields,
                                      size_t *h_send, size_t *h_recv);
int swx_sht_synthesis_shard(swx_sht p, int stage, int n_fields, const swx_shard *sh,
                            const swx_c128 *d_coeffs, double *d_grid, const void *d_recv,
                            void *d_send, void *d_workspace, size_t ws_bytes, void *stream);
int swx_sht_analysis_shard(swx_sht p, int stage, int n_fields, const swx_shard *sh,
                           const double *d_grid, swx_c128 *d_coeffs, const void *d_recv,
                           void *d_send, void *d_workspace, size_t ws_bytes, void *stream);
/* Direct exchange over peer memory (alternative to pack -> all-to-all ->
 * unpack; run the stages with null slabs): copies this rank's blocks of
 * `exchange` from d_ws into every peer's workspace h_peer_ws[r] (device
 * addresses valid on this device, e.g. a symmetric-memory rendezvous) at the
 * same offsets.  Every rank's push must complete (barrier) before stage
 * exchange + 1 runs anywhere.                                               */
int swx_sht_shard_push(swx_sht p, const swx_shard *sh, int exchange, int atoms,
                       const void *d_ws, const uint64_t *h_peer_ws, void *stream);
/* Fused exchange: the stages store straight into the owners' workspaces --
 * the synthesis epilogue writes each latitude pair's Fourier rows into the
 * pair owner's workspace, the grid stage each column's prepared rows into
 * the column owner's -- so there is no copy step at all; only a barrier
 * between the stages.  swx_sht_peer_map_create uploads the owners and the
 * ranks' workspace addresses (h_peer_ws[r], valid on this device: peer-mapped
 * symmetric memory, or co-resident workspaces); stages as in
 * swx_sht_tendency_shard.                                                   */
int swx_sht_peer_map_create(swx_sht p, const swx_shard *sh, const uint64_t *h_peer_ws,
                            void **d_map);
int swx_sht_peer_map_destroy(void *d_map);
int swx_sht_tendency_shard_peer(swx_sht p, int stage, int atoms, const swx_shard *sh,
                                const void *d_map, const swx_c128 *d_state,
                                const swx_c128 *d_sub, swx_c128 *d_out, void *d_workspace,
                                size_t ws_bytes, void *stream);
/* Restrict the pole sums of an lg solver to columns [m_begin, m_end) (the
 * column shard of the caller's rank; m_end < 0: all).  Slots of other
 * columns in d_out are left unspecified.  SWX_ERR_CONFIG for the Coriolis
 * group, whose ranks shard the poles instead (parallel.py:100-182).        */
int swx_solver_set_columns(swx_solver s, int m_begin, int m_end);
/* Bytes of the Coriolis group's warm-time pivot cache (1/den per pole, m,
 * chain position and chain: the analogue of the reference's per-(m, alpha)
 * LU cache, solvers.py:168-194); 0 when not built (lg group, truncations
 * up to T255 - served by the cache-free partition kernel -, SWX_L_CACHE=0,
 * or more than half the free device memory).                               */
size_t swx_solver_cache_bytes(swx_solver s);
/* Geometry of the Coriolis group's partition kernel (truncations up to T255)
 * for a column of n_rows = T + 1 - m chain rows: lanes per (pole, m, chain)
 * system (a power of two <= 32) and rows per lane (even, <= 8), lanes x rows
 * >= n_rows.  Host only (no device needed); SWX_ERR_CONFIG outside 1..256.
 * The per-m work split the reference leaves to LAPACK's band LU
 * (solvers.py:196-212).                                                     */
int swx_l_partition_geometry(int n_rows, int *lanes, int *rows_per_lane);

/* ---- host layout conversion (API edge) ------------------------------------
 * Dense (T+1)x(T+1) complex128 fields, C order (row l, column m) -- the
 * reference's SpectralField.coeffs (sphere.py) -- to and from packed m-major
 * states (n_fields x ncoef).  Host memory only, multithreaded; unpack writes
 * every dense entry (zeros for m > l).  Used by the swerexi-shaped stepper API
 * around each step (solvers.py:288-307 index map).                          */
int swx_host_pack(int trunc, int n_fields, const swx_c128 *const *h_dense,
                  swx_c128 *h_packed);
int swx_host_unpack(int trunc, int n_fields, const swx_c128 *h_packed,
                    swx_c128 *const *h_dense);

/* ---- measurement helpers (bench.py) ---------------------------------------
 * swx_sht_tendency with per-stage device times (ms) written to h_stage_ms[7]:
 * {synthesis, C2R FFT, grid products, R2C FFT, analysis prep, analysis,
 * total}.  Synchronises `stream`; not for the hot path.                     */
int swx_sht_tendency_profile(swx_sht p, int atoms, const swx_c128 *d_state,
                             swx_c128 *d_out, void *d_workspace, size_t ws_bytes,
                             double *h_stage_ms, void *stream);
/* FP64 FMA throughput probe: n_blocks x 256 threads, `iters` x 8 independent
 * DFMA chains each (2 flops per DFMA); d_sink receives one double per thread
 * so nothing is optimised away.  Used for the FP64 roofline denominator.   */
int swx_fp64_fma_probe(double *d_sink, int n_blocks, int iters, void *stream);
/* Per-CTA phase trace of the instrumented transform kernels (state synthesis,
 * square fused grid stage): enable 1/0 (-1: unchanged); when h_out is
 * non-null, copies n_ctas records of 8 u64 {smid, globaltimer marks (ns)}.  */
int swx_trace(int enable, unsigned long long *h_out, int n_ctas);
/* the same for the REXI pole-sum kernels (rexi.cu's trace buffer) */
int swx_trace_rexi(int enable, unsigned long long *h_out, int n_ctas);

#ifdef __cplusplus
}
#endif
#endif /* SWX_H */
