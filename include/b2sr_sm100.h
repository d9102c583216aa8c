/*
 * b2sr_sm100.h -- C ABI of the B200-native Bit-GraphBLAS hot path.
 *
 * This is the drop-in boundary under the Python API of the reference package
 * `b2sr` 0.1.0 (/root/reference/pkg/src/b2sr/__init__.py:3-96).  The Python
 * mirror (paper_2201_08560_b200/) binds these symbols with ctypes -- the FFI
 * a Python package uses -- and keeps the reference's names, argument meaning
 * and exception classes.  Each entry point below cites the reference function
 * it replaces.
 *
 * Conventions
 *  - Every function returns an int status (B2SR_OK == 0).  On failure the
 *    message is available from b2sr_last_error() (thread-local).  No C++
 *    exception crosses this boundary.
 *  - Status codes map onto the reference's exception classes
 *    (SURVEY.md §8b): B2SR_EINVAL -> ValueError, B2SR_EFORMAT -> FormatError,
 *    B2SR_ENOCONV -> RuntimeError, B2SR_ECUDA / B2SR_ENOMEM -> RuntimeError /
 *    MemoryError.
 *  - Matrices live on the device behind an opaque b2sr_matrix handle.  Their
 *    arrays use the reference's layout exactly (formats.py:3-9, 228-240):
 *    tile_row_ptr u32[ntr+1], tile_col_ind u32[T], bit_tiles word[T][dim],
 *    word = u8/u8/u16/u32 for dim 4/8/16/32, LSB = lowest column.
 *  - Vectors are caller-owned DEVICE pointers.  Bit vectors use the
 *    reference BitVector word layout (formats.py:332-357); their buffers must
 *    be padded to a multiple of 4 bytes (ceil(ntr*wordbytes/4)*4).
 *  - `stream` is a cudaStream_t passed as void*; NULL = legacy default stream.
 *    Calls are stream-ordered; functions that must return a host scalar
 *    (tile counts, iteration counts, sums) synchronise that stream.
 *  - Re-entrant: no hidden global mutable state besides the per-thread error
 *    string and a lazily initialised, internally locked memory-pool setup.
 */
#ifndef B2SR_SM100_H
#define B2SR_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    B2SR_OK = 0,
    B2SR_EINVAL = 1,   /* ValueError   */
    B2SR_EFORMAT = 2,  /* FormatError  */
    B2SR_ECUDA = 3,    /* RuntimeError (CUDA failure) */
    B2SR_ENOMEM = 4,   /* MemoryError  */
    B2SR_ENOCONV = 5   /* RuntimeError (iteration cap, algorithms.py:91-92, 195-196) */
};

enum { B2SR_RING_BOOLEAN = 0, B2SR_RING_ARITHMETIC = 1, B2SR_RING_MINPLUS = 2, B2SR_RING_MAXTIMES = 3 };

typedef struct b2sr_matrix b2sr_matrix;
typedef struct b2sr_comm b2sr_comm;          /* one rank's communicator (multi-GPU) */
typedef struct b2sr_dist_bfs b2sr_dist_bfs;  /* one rank's row-partitioned BFS plan */

/* ---- library ----------------------------------------------------------- */
const char *b2sr_last_error(void);
int b2sr_version(void);
/* Number of kernel launches issued by this process so far (evidence for
 * bench.py's "gpu_launches"). */
uint64_t b2sr_launch_count(void);
/* Measurement hook: when on, the calling thread's bin-SpMV calls bracket
 * their main streaming kernel with CUDA events on the launch stream, and
 * b2sr_last_kernel_ms returns that kernel's duration (waits for it). */
int b2sr_set_kernel_timing(int on);
int b2sr_last_kernel_ms(float *ms);

/* ---- matrices (formats.py:228-329, 444-489) ---------------------------- */
/* csr_to_b2sr (formats.py:444-464): device CSR (row_ptr u32[n+1], col_ind
 * u32[nnz], strictly increasing columns per row) -> B2SR on the device.
 * K1 (segmented tile-row count + scan) and K2 (merge/pack) kernels. */
int b2sr_from_csr(uint32_t n, uint32_t dim, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                  uint64_t nnz, void *stream, b2sr_matrix **out);
/* sample_profile (profile.py:73-127), counting step: over the m sampled
 * tile rows d_rows[] (ascending, distinct, < ceil(n/dim)) of a device CSR,
 * the tiles they would store at width dim (*tiles, the K1 merge count) and
 * their CSR entries (*nnz).  Sample selection and the estimates stay with
 * the caller (they are defined by numpy's generator). */
int b2sr_profile_rows(uint32_t n, uint32_t dim, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                      const uint32_t *d_rows, uint32_t m, uint64_t *tiles, uint64_t *nnz, void *stream);
/* Adopt existing arrays (already validated on the host, e.g. a B2srMatrix
 * built by the caller): copies from host pointers into a new device matrix. */
/* Host -> device copy of `bytes` from h_src (any host memory).  Pageable
 * sources are staged through the library's page-locked chunks, filled by
 * several host threads while the previous chunk's DMA runs; h_src may be
 * reused once the call returns.  b2sr_from_host / b2sr_block_from_host
 * upload this way. */
int b2sr_h2d(void *d_dst, const void *h_src, uint64_t bytes, void *stream);
int b2sr_from_host(uint32_t n, uint32_t dim, const uint32_t *h_trp, const uint32_t *h_tci,
                   const void *h_tiles, uint64_t num_tiles, void *stream, b2sr_matrix **out);
int b2sr_free(b2sr_matrix *m);
int b2sr_info(const b2sr_matrix *m, uint32_t *n, uint32_t *dim, uint32_t *ntr, uint64_t *num_tiles);
/* Device pointers of the three arrays (borrowed; valid until b2sr_free). */
int b2sr_arrays(const b2sr_matrix *m, const uint32_t **trp, const uint32_t **tci, const void **tiles);
/* Copy the three arrays to host buffers (sizes from b2sr_info). */
/* from_host with the B2SR invariants of formats.py:242-295 checked on the
 * device (b2sr_validate): B2SR_EFORMAT with the reference's message for the
 * first violated one (row pointer start / monotone / last, column range,
 * column order, empty tile, d=4 high nibble, padding rows, padding
 * columns).  Used by load_b2sr (the .b2sr container, formats.py:533-554). */
int b2sr_from_host_checked(uint32_t n, uint32_t dim, const uint32_t *h_trp, const uint32_t *h_tci,
                           const void *h_tiles, uint64_t num_tiles, void *stream, b2sr_matrix **out);
int b2sr_validate(const b2sr_matrix *m, void *stream);
int b2sr_to_host(const b2sr_matrix *m, uint32_t *h_trp, uint32_t *h_tci, void *h_tiles, void *stream);
/* b2sr_transpose (formats.py:477-489): K3, radix sort by tile column +
 * in-register bit transpose. */
int b2sr_transpose(const b2sr_matrix *m, void *stream, b2sr_matrix **out);
/* B2srMatrix.__eq__ (formats.py:320-329) on the device. */
int b2sr_equal(const b2sr_matrix *a, const b2sr_matrix *b, void *stream, int *equal);
/* b2sr_to_csr (formats.py:467-474), two phases: row_ptr (u32[n+1]) + nnz,
 * then col_ind (u32[nnz]) given that row_ptr. */
int b2sr_to_csr_rowptr(const b2sr_matrix *m, uint32_t *d_row_ptr, uint64_t *nnz, void *stream);
int b2sr_to_csr_fill(const b2sr_matrix *m, const uint32_t *d_row_ptr, uint32_t *d_col_ind, void *stream);
/* _drop_diagonal(b2sr_to_csr(m)) -> csr_to_b2sr (algorithms.py:96-101,111)
 * done directly in tile form. */
int b2sr_drop_diagonal(const b2sr_matrix *m, void *stream, b2sr_matrix **out);
/* Rows [row_begin, row_end) of tile rows as a row-block matrix (multi-GPU
 * 1-D partition).  Column space and n stay global. */
int b2sr_row_block(const b2sr_matrix *m, uint32_t tr_begin, uint32_t tr_end, void *stream,
                   b2sr_matrix **out);
int b2sr_row_offset(const b2sr_matrix *m, uint32_t *tr_begin);
/* A row block [tr_begin, tr_end) uploaded from host arrays (tile_row_ptr
 * local to the block, starting at 0): the multi-GPU end-to-end path, where
 * every rank copies only its own block of the caller's matrix. */
int b2sr_block_from_host(uint32_t n, uint32_t dim, uint32_t tr_begin, uint32_t tr_end, const uint32_t *h_trp,
                         const uint32_t *h_tci, const void *h_tiles, uint64_t num_tiles, void *stream,
                         b2sr_matrix **out);
/* used_columns (kernels.py:86-94): d_out u8[n] (0/1). */
int b2sr_used_columns(const b2sr_matrix *m, uint8_t *d_out, void *stream);

/* ---- bin-SpMV (kernels.py:97-249) -------------------------------------- */
/* bmv_bin_bin_bin[_masked]: y words (tile width layout) = OR_j a_ij & x_j,
 * cleared where keep is 0 (d_keep may be NULL).  For a row-block matrix, y
 * holds only the block's words. */
int b2sr_bmv_bbb(const b2sr_matrix *m, const void *d_x, const void *d_keep, void *d_y, void *stream);
/* bmv_bin_bin_full[_masked]: y f64[n] (or the block's rows) = popcounts. */
int b2sr_bmv_bbf(const b2sr_matrix *m, const void *d_x, const void *d_keep, double *d_y, void *stream);
/* bmv_bin_full_full[_masked]: semiring gather over x f64[n]; ring is one of
 * B2SR_RING_*, inc in {0,1} for minplus; d_scale (f64[n]) only with
 * ARITHMETIC.  Terms reduce per output element in ascending column order
 * (kernels.py:195-207), so ARITHMETIC is bit-identical to the reference.
 * A zero scale at a used column fails with B2SR_EINVAL and *bad_col = j. */
int b2sr_bmv_bff(const b2sr_matrix *m, const double *d_x, int ring, double inc, const double *d_scale,
                 const void *d_keep, double *d_y, int64_t *bad_col, void *stream);
/* As b2sr_bmv_bff with the semiring's add identity given explicitly
 * (Semiring.add_identity, semirings.py:18-21): every output element starts
 * from it and masked-off positions hold it (kernels.py:176, 249).
 * b2sr_bmv_bff uses the built-in identities (+inf min-plus, else 0). */
int b2sr_bmv_bff_ex(const b2sr_matrix *m, const double *d_x, int ring, double inc, double add_identity,
                    const double *d_scale, const void *d_keep, double *d_y, int64_t *bad_col, void *stream);

/* ---- bin-SpGEMM (kernels.py:298-367) ----------------------------------- */
/* bmm_bin_bin_sum: sum of all entries of A @ B (int64). */
int b2sr_bmm_sum(const b2sr_matrix *a, const b2sr_matrix *b, int64_t *out, void *stream);
/* bmm_bin_bin_sum_masked with B given TRANSPOSED (bt = transpose(b)):
 * sum over mask bits (i,j) of popc(A_row_i & Bt_row_j) per common tile col. */
int b2sr_bmm_sum_masked_bt(const b2sr_matrix *a, const b2sr_matrix *bt, const b2sr_matrix *mask,
                           int64_t *out, void *stream);

/* ---- drivers (algorithms.py:75-215) ------------------------------------ */
/* bfs (algorithms.py:75-93).  at = transpose(a) (the caller transposes, as
 * algorithms.py:78 does).  With a != NULL the driver is direction-optimizing:
 * small frontiers push over a (top-down), large ones pull over at
 * (bottom-up, masked bbb with early exit); both produce the identical
 * next frontier.  a == NULL -> pull only.  at == NULL -> push only over a
 * (d = 4, 8; no transpose needed: for a matrix that has none yet).
 * levels f64[n] (+inf unreachable);
 * *iterations counts the final empty sweep like the reference.  Env
 * B2SR_BFS_ALPHA tunes the switch, B2SR_BFS_TRACE logs levels. */
int b2sr_bfs(const b2sr_matrix *a, const b2sr_matrix *at, uint32_t src, double *d_levels, int64_t *iterations,
             void *stream);
/* The BFS sweep split into its pieces for the row-partitioned multi-GPU
 * driver (paper_2201_08560_b200/dist.py): seed, one masked pull sweep over a
 * row block (d_next = the block's words, zeroed here), and the fused
 * visited/levels/any update over the gathered global frontier. */
int b2sr_bfs_init(uint32_t n, uint32_t dim, uint32_t src, void *d_visited, void *d_frontier, double *d_levels,
                  void *stream);
int b2sr_bfs_sweep(const b2sr_matrix *at_block, const void *d_frontier, const void *d_visited, void *d_next,
                   void *stream);
int b2sr_bfs_update(uint32_t n, uint32_t dim, const void *d_frontier, void *d_visited, double *d_levels,
                    double level, int *d_any, void *stream);
/* Row-partitioned levels with the single-GPU sweep shortcuts: flags
 * B2SR_SWEEP_ACTIVE streams only the loads whose rows still hold an
 * unvisited vertex, B2SR_SWEEP_LAZY fetches tile bytes only where the
 * frontier words are non-zero (sparse frontiers).  Same output as
 * b2sr_bfs_sweep.  b2sr_bfs_update_ex also adds the frontier's vertex count
 * to *d_frontier_vertices (u64, caller-zeroed). */
#define B2SR_SWEEP_ACTIVE 1
#define B2SR_SWEEP_LAZY 2
int b2sr_bfs_sweep_ex(const b2sr_matrix *at_block, const void *d_frontier, const void *d_visited, void *d_next,
                      int flags, void *stream);
int b2sr_bfs_update_ex(uint32_t n, uint32_t dim, const void *d_frontier, void *d_visited, double *d_levels,
                       double level, int *d_any, uint64_t *d_frontier_vertices, void *stream);
/* sssp relaxation (algorithms.py:113-124) on at = transpose(drop_diag(a)). */
int b2sr_sssp(const b2sr_matrix *at, uint32_t src, double *d_dist, int64_t *iterations, void *stream);
/* pagerank (algorithms.py:127-163); a = transposed adjacency. */
int b2sr_pagerank(const b2sr_matrix *a, const double *d_out_degree, double alpha, double epsilon,
                  int64_t max_iter, double *d_rank, int64_t *iterations, int *converged,
                  int64_t *bad_col, void *stream);
/* Pieces of the drivers for the row-partitioned loops (dist.py), each the
 * exact arithmetic of the single-GPU driver:
 *   b2sr_pr_step      rank' = teleport + alpha*g (no FMA), diff = |rank'-rank|,
 *                     xs = rank'/deg (0 where deg == 0) -- algorithms.py:150-157
 *   b2sr_pairwise_sum numpy's pairwise float64 sum (the PR delta, algorithms.py:157)
 *   b2sr_min_relax    dist = np.minimum(dist, y), *changed |= any change (algorithms.py:119-122) */
int b2sr_pr_step(uint32_t count, double teleport, double alpha, const double *d_g, const double *d_deg, double *d_rank,
                 double *d_xs, double *d_diff, void *stream);
int b2sr_pairwise_sum(const double *d_a, uint64_t n, double *d_out, void *stream);
int b2sr_min_relax(uint64_t count, double *d_dist, const double *d_y, int *d_changed, void *stream);
/* connected_components (algorithms.py:166-196) on a symmetric matrix. */
int b2sr_cc(const b2sr_matrix *a, double *d_labels, int64_t *iterations, void *stream);
/* triangle_count core (algorithms.py:212-214): L = strict lower triangle in
 * B2SR; count = bmm_masked(L, transpose(L), L). */
int b2sr_tc(const b2sr_matrix *lower, int64_t *count, void *stream);
/* The same count plus W, the AND+POPC units the masked SpGEMM executed
 * (SURVEY.md §8d TC roofline; counting costs a little time). */
int b2sr_tc_work(const b2sr_matrix *lower, int64_t *count, uint64_t *work, void *stream);

/* ---- CSR utilities on the device (formats.py:96-225, algorithms.py:218) - */
/* Strict lower triangle of a device CSR (two phases like b2sr_to_csr). */
int b2sr_csr_lower_rowptr(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                          uint32_t *d_lrow_ptr, uint64_t *lnnz, void *stream);
int b2sr_csr_lower_fill(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind,
                        const uint32_t *d_lrow_ptr, uint32_t *d_lcol_ind, void *stream);
/* Degree-oriented triangle DAG of a symmetric device CSR: keep (u, v) iff
 * (deg u, u) < (deg v, v) (edges point at higher degree).  triangle_count (algorithms.py:199-215) runs its
 * masked bin-SpGEMM on this instead of the ID-ordered lower triangle: the
 * count is the same for any total vertex order, and hub rows stay short. */
int b2sr_csr_orient_rowptr(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, uint32_t *d_orow_ptr,
                           uint64_t *onnz, void *stream);
int b2sr_csr_orient_fill(uint32_t n, const uint32_t *d_row_ptr, const uint32_t *d_col_ind, const uint32_t *d_orow_ptr,
                         uint32_t *d_ocol_ind, void *stream);
/* Synthetic Graph500 R-MAT edges. */
int b2sr_rmat_edges(int scale, uint64_t m, uint64_t seed, uint32_t *d_src, uint32_t *d_dst, void *stream);
/* COO -> CSR with CsrMatrix.from_coo semantics (formats.py:156-190):
 * symmetrize / drop self-loops / sort / de-duplicate.  d_row_ptr u32[n+1];
 * d_col_ind must hold (symmetrize ? 2m : m) entries; *nnz returned. */
int b2sr_coo_to_csr(uint32_t n, uint64_t m, const uint32_t *d_src, const uint32_t *d_dst, int symmetrize,
                    int drop_loops, uint32_t *d_row_ptr, uint32_t *d_col_ind, uint64_t *nnz, void *stream);


/* ---- multi-GPU: row-partitioned drivers ---------------- */
/* The reference's only parallelism is contiguous tile-row chunks
 * (kernels.py:44-57); here the chunks are GPUs.  One communicator per rank
 * (one process per GPU, or one host thread per GPU):
 *   b2sr_comm_unique_id  rank 0 makes the NCCL id (128 bytes), the caller
 *                        ships it to the other ranks (e.g. torch.distributed)
 *   b2sr_comm_init       NCCL communicator of `rank` of `world` on the
 *                        current device (libnccl opened at run time)
 *   b2sr_comm_init_local `world` thread-ranks sharing the current device,
 *                        exchanging through device copies (tests: the same
 *                        level loop with N ranks on one GPU); outs[world]
 * Every collective is enqueued on the caller's stream. */
int b2sr_comm_unique_id(uint8_t *out128);
int b2sr_comm_init(const uint8_t *id128, int world, int rank, b2sr_comm **out);
int b2sr_comm_init_local(int world, b2sr_comm **outs);
int b2sr_comm_free(b2sr_comm *comm);
/* In-place int64 sum over ranks (NCCL all-reduce). */
int b2sr_comm_allreduce_sum_i64(b2sr_comm *comm, int64_t *d, uint64_t count, void *stream);
/* bfs (algorithms.py:75-93) over row blocks, direction-optimizing and
 * device-controlled like b2sr_bfs (d = 4, 8).  Each rank holds the rows
 * [begin, end) of a (push) and of at (pull), cut where at's tile prefix
 * crosses k/world of its tiles; frontier, visited and levels are global on
 * every rank.  Per level: push/pull over the blocks, an all-to-all-v of the
 * row contributions, OR-merge, an all-gather-v of the merged rows; the level
 * plan runs on the device from global counters, identically on every rank,
 * and the host polls a mapped snapshot ring (no sync per level).
 *   b2sr_dist_bfs_plan         from the full a / at on every rank's device
 *   b2sr_dist_bfs_plan_blocks  from this rank's blocks (not copied: keep them
 *                              alive) and the global tile_row_ptr of a / at
 *                              (device or host pointers, ntr+1 entries)
 * b2sr_dist_bfs_run: levels f64[n] on every rank, *iterations as b2sr_bfs. */
int b2sr_dist_bfs_plan(b2sr_comm *comm, const b2sr_matrix *a, const b2sr_matrix *at, void *stream,
                       b2sr_dist_bfs **out);
int b2sr_dist_bfs_plan_blocks(b2sr_comm *comm, const b2sr_matrix *a_block, const b2sr_matrix *at_block,
                              const uint32_t *tile_row_ptr_a, const uint32_t *tile_row_ptr_at, void *stream,
                              b2sr_dist_bfs **out);
int b2sr_dist_bfs_rows(const b2sr_dist_bfs *plan, uint32_t *begin, uint32_t *end);
int b2sr_dist_bfs_run(b2sr_dist_bfs *plan, uint32_t src, double *d_levels, int64_t *iterations, void *stream);
int b2sr_dist_bfs_free(b2sr_dist_bfs *plan);
/* triangle_count's masked SpGEMM (algorithms.py:199-215, kernels.py:323-367)
 * with the lower triangle L replicated and its tile rows (the mask) cut into
 * blocks of equal estimated work; one int64 all-reduce.  rows_out (world+1,
 * may be NULL) receives the cuts. */
int b2sr_dist_tc(b2sr_comm *comm, const b2sr_matrix *lower, int64_t *count, uint32_t *rows_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* B2SR_SM100_H */
