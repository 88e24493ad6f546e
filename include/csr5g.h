/*
 * csr5g.h -- C ABI of the B200-native CSR5 SpMV library (libcsr5g.so).
 *
 * Drop-in boundary for the reference's hot path (namespace csr5 in
 * /root/reference/proj/core).  Every entry point below replaces one reference
 * interface; the citation names it.  Plain pointers and sizes only: device
 * pointers are prefixed d_, host pointers h_; `stream` is a cudaStream_t
 * passed as void* (NULL = the legacy default stream).
 *
 * Errors: every function returns a CSR5G_* status.  csr5g_last_error()
 * returns the message of the last failure on the calling thread; for the
 * argument errors the text is the reference's own std::invalid_argument text.
 *
 * There is no CPU fallback: on a host without a usable sm_100 device every
 * compute entry point fails with CSR5G_ECUDA.
 */
#ifndef CSR5G_H
#define CSR5G_H

#include <stddef.h>
#include <stdint.h>

#if defined(CSR5G_BUILD)
#define CSR5G_API __attribute__((visibility("default")))
#else
#define CSR5G_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CSR5G_OK 0
#define CSR5G_EINVAL 1   /* reference: std::invalid_argument */
#define CSR5G_ERUNTIME 2 /* reference: std::runtime_error */
#define CSR5G_ERANGE 3   /* reference: std::out_of_range / unsupported size */
#define CSR5G_ECUDA 4    /* CUDA runtime failure (no device, launch error, ...) */
#define CSR5G_ENOMEM 5   /* device allocation failed */

#define CSR5G_MODE_DETERMINISTIC 0 /* reference SpmvMode::deterministic (spmv.hpp:16) */
#define CSR5G_MODE_ATOMIC 1        /* reference SpmvMode::atomic */

typedef struct csr5g_matrix_s *csr5g_matrix;

/* Reference TuningParams (tuning.hpp:13-24).  omega must be 32 (one warp
 * lane per tile column).  sigma = 0 selects sigma with the reference rule
 * select_sigma(nnz/m, <r,s,t,u>) (tuning.cpp:25-34). */
typedef struct {
  int64_t omega, sigma, r, s, t, u;
} csr5g_params;

/* Sizes of a built handle (Csr5Matrix fields, format.hpp:130-176). */
typedef struct {
  int64_t m, n, nnz;            /* global matrix */
  int64_t omega, sigma;
  int64_t p, p_complete, tail_len; /* global tile counts */
  int64_t tile_begin, tile_end; /* complete tiles held: [tile_begin, tile_end) */
  int32_t has_tail;             /* this handle owns the CSR tail */
  int32_t tile_ptr_bits, word_bits, y_offset_bits, seg_offset_bits;
  int32_t num_sms, spmv_warps;  /* persistent SpMV grid */
  int64_t tile_ptr_len;         /* tile_ptr words held (tiles + closing entry) */
  int64_t empty_offset_len;     /* empty_offset entries held */
  int64_t nnz_held;             /* col_idx/val entries held */
  int64_t metadata_bytes;       /* tile_ptr + tile_desc at stored widths (format.hpp:171) */
  int64_t device_bytes;         /* all device memory owned by the handle */
  int64_t spmv_bytes;           /* algorithmic HBM bytes of one SpMV */
  int64_t first_row, last_row;  /* rows of the first / last head held */
  int64_t own_row_begin, own_row_end; /* rows this handle writes in y (shards) */
  double build_ms, alloc_ms;    /* last build: total and allocation share */
  /* SpMV plan chosen from the sampled gather locality */
  double lines_per_gather;      /* distinct 128 B x lines per warp gather (1..32) */
  int32_t warps_per_cta, stages, smem_bytes, x_mode, x_window;
  int32_t kernel_variant;       /* 0 general, 1 VR (values with the gathers), 2 NF (no flag paths) */
  int64_t long_rows;            /* rows with partials from three or more parts (tiles, tail) */
  int64_t hot_cols;             /* x values staged per SpMV for the hot columns (0: none) */
  double hot_coverage;          /* sampled share of the gathers that read a staged value */
} csr5g_info;

/* One boundary partial of a shard: row = -1 when there is none. */
typedef struct {
  int64_t row;
  double value;
} csr5g_partial;

CSR5G_API const char *csr5g_last_error(void);
CSR5G_API const char *csr5g_version(void);

/* tuning.cpp:25-34 select_sigma (no fixed sigma). */
CSR5G_API int csr5g_select_sigma(double nnz_per_row, int64_t r, int64_t s, int64_t t, int64_t u,
                       int64_t *out);
/* descriptor.cpp:22-36 make_descriptor_layout. */
CSR5G_API int csr5g_layout(int64_t omega, int64_t sigma, int32_t *y_offset_bits, int32_t *seg_offset_bits,
                 int32_t *word_bits);

/* format.cpp:165-252 csr_to_csr5 (format.hpp:182).  Inputs are the caller's
 * device CSR (row_ptr int64[m+1], col_idx int32[nnz], val f64[nnz]); they are
 * only read.  The handle owns every CSR5 array.  Synchronises `stream`. */
CSR5G_API int csr5g_build(int device, int64_t m, int64_t n, int64_t nnz, const int64_t *d_row_ptr,
                const int32_t *d_col_idx, const double *d_val, const csr5g_params *params,
                void *stream, csr5g_matrix *out);

/* Shard build for the multi-GPU driver: holds global complete tiles
 * [tile_begin, tile_end) (and the tail when with_tail).  d_row_ptr is the
 * FULL global row_ptr; d_col_idx / d_val point at global position
 * tile_begin * omega * sigma.  sigma must be explicit (global).  The held
 * arrays equal the slices of the single-device arrays bit for bit. */
CSR5G_API int csr5g_build_shard(int device, int64_t m, int64_t n, int64_t nnz, const int64_t *d_row_ptr,
                      const int32_t *d_col_idx, const double *d_val, const csr5g_params *params,
                      int64_t tile_begin, int64_t tile_end, int32_t with_tail, void *stream,
                      csr5g_matrix *out);

CSR5G_API int csr5g_info_get(csr5g_matrix h, csr5g_info *out);

/* Copies the held arrays to host buffers, widened to the reference's 64-bit
 * types (PackedWords, format.hpp:106-124; index_t vectors).  Any pointer may
 * be NULL to skip that array.  Sizes: tile_ptr tile_ptr_len, tile_desc
 * (tile_end-tile_begin)*omega, eo_ptr (tile_end-tile_begin)+1, eo
 * empty_offset_len, col_idx/val nnz_held. */
CSR5G_API int csr5g_export(csr5g_matrix h, uint64_t *h_tile_ptr, uint64_t *h_tile_desc, int64_t *h_eo_ptr,
                 int64_t *h_eo, int64_t *h_col_idx, double *h_val);

/* spmv.cpp:224-298 spmv_csr5 (spmv.hpp:58): y = A x, y fully overwritten
 * (rows own_row_begin..own_row_end for a shard).  Stream-ordered, no sync.
 * Concurrent calls on one handle from distinct streams are safe: every
 * stream gets its own scratch (the reference's per-worker workspaces,
 * spmv.hpp:27-38). */
CSR5G_API int csr5g_spmv(csr5g_matrix h, const double *d_x, double *d_y, int32_t mode, void *stream);

/* Same, recording ev_tiles_begin / ev_tiles_end (from csr5g_event_create)
 * around the dominant tile kernel, for roofline timing. */
CSR5G_API int csr5g_spmv_evt(csr5g_matrix h, const double *d_x, double *d_y, int32_t mode, void *stream,
                   void *ev_tiles_begin, void *ev_tiles_end);

/* Shard boundary exchange.  After csr5g_spmv on a shard, d_send (device,
 * one csr5g_partial) holds the partial of a first row this shard does not
 * own (row = -1 if none).  The driver all-gathers every shard's record into
 * d_all[world] and calls csr5g_fixup, which adds, in shard order, the
 * partials of later shards whose row this shard owns. */
CSR5G_API int csr5g_shard_send_record(csr5g_matrix h, csr5g_partial **d_send);
/* Redirect the send record to caller device memory (e.g. this rank's slot of
 * an all-gather buffer); NULL restores the handle's own record. */
CSR5G_API int csr5g_set_send_buffer(csr5g_matrix h, csr5g_partial *d_send);
CSR5G_API int csr5g_fixup(csr5g_matrix h, const csr5g_partial *d_all, int32_t world, int32_t rank,
                double *d_y, void *stream);

/* NVLink P2P boundary exchange (the reference has no distributed
 * backend).  One mailbox per rank in its own HBM, exported with a CUDA IPC
 * handle and opened by every peer.  A shard that does not own its first row
 * stores that row's partial straight into the owner's mailbox (dest) from
 * its SpMV kernel, then a ready flag; an owner stream-waits on the
 * flags of its senders (the ranks sender_begin..sender_end-1 right after it
 * whose first row is its last row), adds their partials in shard order and
 * acknowledges.  No collective, no host sync per call.  Deterministic mode
 * only.  Ranks that share one GPU must separate csr5g_mg_spmv_post and
 * csr5g_mg_spmv_fixup with a host barrier (cross-process waits on one GPU
 * are not safe); on distinct GPUs csr5g_mg_spmv does both. */
#define CSR5G_IPC_HANDLE_BYTES 64
#define CSR5G_MAX_WORLD 64
typedef struct csr5g_mailbox_s *csr5g_mailbox;
/* vec_len > 0 (iterative mode, = m = n): the mailbox also holds the two x
 * buffers of the y -> x ping-pong, x_k = vector(k & 1). */
CSR5G_API int csr5g_mailbox_create(int device, int32_t world, int32_t rank, int64_t vec_len,
                                   csr5g_mailbox *out);
CSR5G_API int csr5g_mailbox_vector(csr5g_mailbox mb, int32_t which, double **d_vec);
CSR5G_API int csr5g_mailbox_ipc_handle(csr5g_mailbox mb, void *handle_out /* 64 bytes */);
/* map another process's mailbox (its csr5g_mailbox_ipc_handle bytes) */
CSR5G_API int csr5g_mailbox_open_peer(csr5g_mailbox mb, int32_t peer, const void *handle /* 64 bytes */);
/* link a mailbox of the same process (single-process emulation, tests) */
CSR5G_API int csr5g_mailbox_link_local(csr5g_mailbox mb, int32_t peer, csr5g_mailbox peer_mb);
/* protocol violations seen by this rank's fix-ups (0 = none; synchronous) */
CSR5G_API int csr5g_mailbox_errors(csr5g_mailbox mb, uint32_t *errors);
CSR5G_API int csr5g_mailbox_release(csr5g_mailbox mb);
/* active_world: ranks holding tiles (0 .. active_world-1) */
/* NVSwitch multicast (NVLS) for the fused iterative mode: every rank's x
 * ping-pong bound to one multicast object, so each mirror store is one
 * multimem.st the switch replicates (instead of G-1 peer stores).  Order:
 * rank 0 _create (exports a 64-byte fabric handle when ndev > 1), the others
 * _import it, every rank _add (its device), a barrier, every rank _bind, a
 * barrier.  After _bind, csr5g_mailbox_vector returns the bound buffers.
 * Any failure leaves the peer-store path; _release drops the object.
 * (No reference counterpart: the reference has no distributed backend.) */
CSR5G_API int csr5g_mcast_supported(int device, int32_t *out);
CSR5G_API int csr5g_mailbox_mcast_create(csr5g_mailbox mb, int32_t ndev, void *handle64);
CSR5G_API int csr5g_mailbox_mcast_import(csr5g_mailbox mb, int32_t ndev, const void *handle64);
CSR5G_API int csr5g_mailbox_mcast_add(csr5g_mailbox mb);
CSR5G_API int csr5g_mailbox_mcast_bind(csr5g_mailbox mb);
CSR5G_API int csr5g_mailbox_mcast_release(csr5g_mailbox mb);
/* test hook: multimem stores into x buffer 1's multicast mapping, then the
 * values that did not land in this rank's bound copy */
CSR5G_API int csr5g_mailbox_mcast_selftest(csr5g_mailbox mb, int64_t *mismatches);

CSR5G_API int csr5g_mg_bind(csr5g_matrix h, csr5g_mailbox mb, int32_t dest, int32_t sender_begin,
                            int32_t sender_end, int32_t active_world);
CSR5G_API int csr5g_mg_spmv_post(csr5g_matrix h, const double *d_x, double *d_y, void *stream,
                                 void *ev_tiles_begin, void *ev_tiles_end);
CSR5G_API int csr5g_mg_spmv_fixup(csr5g_matrix h, double *d_y, void *stream);
CSR5G_API int csr5g_mg_spmv(csr5g_matrix h, const double *d_x, double *d_y, void *stream,
                            void *ev_tiles_begin, void *ev_tiles_end);
/* Fused iterative step it (x_{it+1} = A x_it, square A, <= 8 active ranks):
 * waits until every active peer stored its rows of x_it here, runs the SpMV
 * from vector(it & 1) into vector((it+1) & 1), every final y value also
 * stored into each peer's vector((it+1) & 1) over NVLink by the kernels that
 * produce it, then the boundary fix-up (mirrored) and the ready signal to
 * every peer.  No all-gather.  Steps run 0, 1, 2, ... on every rank (x_0 is
 * vector(0)); anything else is EINVAL.  post/finish split as above for ranks
 * sharing one GPU (host barrier between and after). */
CSR5G_API int csr5g_mg_iter_post(csr5g_matrix h, int64_t it, void *stream, void *ev_tiles_begin,
                                 void *ev_tiles_end);
CSR5G_API int csr5g_mg_iter_finish(csr5g_matrix h, int64_t it, void *stream);
CSR5G_API int csr5g_mg_iter(csr5g_matrix h, int64_t it, void *stream, void *ev_tiles_begin,
                            void *ev_tiles_end);

/* format.cpp:254-265 csr5_to_csr: undo the tile transposition into the
 * caller's device buffers (col_idx int32[nnz_held], val f64[nnz_held]). */
CSR5G_API int csr5g_to_csr(csr5g_matrix h, int32_t *d_col_idx, double *d_val, void *stream);

/* Host-vector overloads (drop-in for the reference's std::vector API; they
 * stage through the device and synchronise -- not the timed path).
 * csr_to_csr5 from a host CSR with the reference's int64 col_idx
 * (format.hpp:182); spmv_csr5 with host x / y (spmv.hpp:58-61);
 * csr5_to_csr into host buffers (format.hpp:186).  device < 0 = the calling
 * thread's current CUDA device (the reference's API has no device argument). */
CSR5G_API int csr5g_build_host(int device, int64_t m, int64_t n, int64_t nnz,
                               const int64_t *h_row_ptr, const int64_t *h_col_idx,
                               const double *h_val, const csr5g_params *params,
                               csr5g_matrix *out);
CSR5G_API int csr5g_spmv_host(csr5g_matrix h, const double *h_x, double *h_y, int32_t mode);

/* Batch of independent SpMVs on host vectors (spmv.hpp:58-61 called `count`
 * times): y_k = A x_k for h_xs[k] (n doubles) / h_ys[k] (m doubles).  The
 * copies run as a pipeline over two device buffer pairs on the handle's own
 * streams -- x_{k+1} H2D and y_k D2H overlap SpMV k -- so pinned host buffers
 * give one PCIe transfer time per step instead of the sum.  Stream-ordered:
 * starts after work queued on `stream`, and `stream` continues after the last
 * y copy; the host buffers must stay valid until then. */
CSR5G_API int csr5g_spmv_host_batch(csr5g_matrix h, const double *const *h_xs,
                                    double *const *h_ys, int64_t count, int32_t mode,
                                    void *stream);
CSR5G_API int csr5g_to_csr_host(csr5g_matrix h, int64_t *h_col_idx, double *h_val);

/* The plain-CSR kernels the reference times CSR5 against (spmv.cpp:139-209),
 * on the device: CSR5G_CSR_SCALAR = spmv_csr_scalar (one thread per row, row
 * order -- also the summation order of dense_spmv_oracle, csr.cpp:85-98),
 * CSR5G_CSR_SEGSUM = spmv_csr_segsum (products, then a segmented sum per row).
 * They feed run_benchmark's iteration scenario (bench.cpp:86-90, t_csr).  The
 * caller's device CSR (int64 row_ptr, int32 col_idx); y fully overwritten;
 * stream-ordered. */
#define CSR5G_CSR_SCALAR 0
#define CSR5G_CSR_SEGSUM 1
CSR5G_API int csr5g_csr_spmv(int device, int32_t kernel, int64_t m, int64_t n, int64_t nnz,
                             const int64_t *d_row_ptr, const int32_t *d_col_idx,
                             const double *d_val, const double *d_x, double *d_y, void *stream);

/* Matrix files (SURVEY 8f "ingest").  matrix_market.cpp:38-96
 * read_matrix_market: parses an ASCII coordinate file (real / integer /
 * pattern, general / symmetric) into a host COO object -- 0-based indices,
 * pattern values 1.0, symmetric entries mirrored (diagonal once) -- with the
 * reference's std::runtime_error texts (CSR5G_ERUNTIME).  csr5g_coo_get copies
 * its `count` entries out (any pointer may be NULL). */
typedef struct csr5g_coo_s *csr5g_coo;
CSR5G_API int csr5g_mm_read(const char *path, csr5g_coo *out, int64_t *m, int64_t *n,
                            int64_t *count);
/* The same parser over an in-memory text (read_matrix_market(std::istream&)). */
CSR5G_API int csr5g_mm_parse(const char *text, int64_t len, csr5g_coo *out, int64_t *m,
                             int64_t *n, int64_t *count);
CSR5G_API int csr5g_coo_get(csr5g_coo c, int64_t *h_rows, int64_t *h_cols, double *h_vals);
CSR5G_API int csr5g_coo_release(csr5g_coo c);

/* csr.cpp:35-72 coo_to_csr on the device: device COO (int64 rows / cols, f64
 * values, `count` entries, any order, duplicates allowed) -> canonical CSR:
 * sorted by (row, col), duplicates summed in input order (bit-identical to the
 * reference's sums).  Outputs: d_row_ptr[m+1], d_col_idx / d_val with room
 * for `count` entries; *nnz = the unique entries written.  An out-of-range
 * entry fails with the reference's std::invalid_argument text (first such
 * entry).  Synchronises `stream`. */
CSR5G_API int csr5g_coo_to_csr(int device, int64_t m, int64_t n, int64_t count,
                               const int64_t *d_rows, const int64_t *d_cols, const double *d_vals,
                               int64_t *d_row_ptr, int32_t *d_col_idx, double *d_val,
                               int64_t *nnz, void *stream);

/* Host-staged form of csr5g_coo_to_csr (the reference's host coo_to_csr
 * signature, csr.hpp): host COO in, host CSR out with int64 col_idx; the
 * output buffers hold m+1 / count entries; device < 0 = the current device. */
CSR5G_API int csr5g_coo_to_csr_host(int device, int64_t m, int64_t n, int64_t count,
                                    const int64_t *h_rows, const int64_t *h_cols,
                                    const double *h_vals, int64_t *h_row_ptr,
                                    int64_t *h_col_idx, double *h_val, int64_t *nnz);

/* Host-staged csr-scalar / csr-segsum (spmv.hpp spmv_csr_scalar /
 * spmv_csr_segsum and csr.hpp dense_spmv_oracle take host vectors): int64
 * col_idx as in the reference; device < 0 = the current device. */
CSR5G_API int csr5g_csr_spmv_host(int device, int32_t kernel, int64_t m, int64_t n, int64_t nnz,
                                  const int64_t *h_row_ptr, const int64_t *h_col_idx,
                                  const double *h_val, const double *h_x, double *h_y);

/* Csr5Matrix::row_ptr (format.hpp:168): the handle's copy of the CSR row
 * pointer, m+1 entries, into host memory (csr5_to_csr(a5) needs nothing else). */
CSR5G_API int csr5g_export_row_ptr(csr5g_matrix h, int64_t *h_row_ptr);

/* spmv.cpp:211-222 spmv_csr5_tile (the TileContribution test hook): the
 * contributions of complete tile `tid` (a global tile id inside the handle's
 * range) for host x, computed by the SpMV tile kernel itself (its trace
 * instantiation), in the reference's emission order: per column the segments
 * sealed inside it (accumulate = head 0 only), then each head-bearing
 * column's bottom piece (accumulate).  Up to `cap` entries; *count = number
 * written (= the tile's heads). */
CSR5G_API int csr5g_spmv_tile(csr5g_matrix h, int64_t tid, const double *h_x, int64_t *h_rows,
                              double *h_vals, uint8_t *h_acc, int64_t cap, int64_t *count);

/* Implicit destruction of Csr5Matrix (value type) -> explicit release. */
CSR5G_API int csr5g_release(csr5g_matrix h);

/* Timing helpers (cudaEvent with timing) for callers without a CUDA runtime. */
CSR5G_API int csr5g_event_create(void **ev);
CSR5G_API int csr5g_event_record(void *ev, void *stream);
CSR5G_API int csr5g_event_elapsed_ms(void *ev_begin, void *ev_end, float *ms);
CSR5G_API int csr5g_event_destroy(void *ev);
/* cudaStreamSynchronize for callers without a CUDA runtime (NULL = legacy). */
CSR5G_API int csr5g_stream_synchronize(void *stream);

/* Synthetic inputs on the device (bench / tests): counter-based, so the
 * same call gives the same matrix on any GPU.  kind: 0 = 2D 5-point Laplacian
 * (a x a grid), 1 = 3D 27-point stencil (a^3 grid).  Fills caller buffers
 * sized by csr5g_stencil_size. */
CSR5G_API int csr5g_stencil_size(int32_t kind, int64_t a, int64_t *m, int64_t *nnz);
CSR5G_API int csr5g_stencil_fill(int32_t kind, int64_t a, int64_t *d_row_ptr, int32_t *d_col_idx,
                       double *d_val, void *stream);
/* Box variant for weak scaling: the outermost axis (y in 2D, z in 3D) has
 * `layers` points instead of a (layers = a is the stencil above).  Writes the
 * full row_ptr (m+1) but only the entries at global positions [pos_begin,
 * pos_end) into d_col_idx / d_val (a shard's slice: pos_begin = 0, pos_end =
 * nnz for the whole matrix). */
CSR5G_API int csr5g_stencil_box_size(int32_t kind, int64_t a, int64_t layers, int64_t *m,
                                     int64_t *nnz);
CSR5G_API int csr5g_stencil_box_fill(int32_t kind, int64_t a, int64_t layers, int64_t pos_begin,
                                     int64_t pos_end, int64_t *d_row_ptr, int32_t *d_col_idx,
                                     double *d_val, void *stream);

/* The benchmark harness's x (bench.cpp:103-105): std::mt19937_64(seed),
 * x_i = 0.5 + (rng() >> 11) * 2^-53, written into the host array h_x[n]. */
CSR5G_API int csr5g_bench_x(int64_t n, uint64_t seed, double *h_x);

/* Irregular synthetic matrices on the device (BASELINE configs 3-5).  Two
 * phases: *_create generates and sizes the matrix (m, nnz) and keeps it in a
 * generator object; csr5g_gen_fill writes the CSR into caller buffers
 * (row_ptr int64[m+1], col_idx int32[nnz], val f64[nnz]).
 *  - R-MAT, Graph500 a,b,c,d = .57,.19,.19,.05, edge_factor * 2^scale edges,
 *    duplicates removed, vertex labels permuted by a keyed bijection when
 *    `permute` is set.
 *  - mixed: m = n = 2^log2_m, rows empty with probability p_empty, n_long
 *    rows of long_len nonzeros, the rest U[min_len, max_len] nonzeros. */
typedef struct csr5g_gen_s *csr5g_gen;
CSR5G_API int csr5g_rmat_create(int32_t scale, int32_t edge_factor, uint64_t seed, int32_t permute,
                                void *stream, csr5g_gen *out, int64_t *m, int64_t *nnz);
CSR5G_API int csr5g_mixed_create(int32_t log2_m, double p_empty, int32_t n_long, int64_t long_len,
                                 int32_t min_len, int32_t max_len, uint64_t seed, void *stream,
                                 csr5g_gen *out, int64_t *m, int64_t *nnz);
CSR5G_API int csr5g_gen_fill(csr5g_gen g, int64_t *d_row_ptr, int32_t *d_col_idx, double *d_val,
                             void *stream);
/* Only the entries at global positions [pos_begin, pos_end), written at
 * position - pos_begin (a multi-GPU rank's slice), and the full row_ptr when
 * d_row_ptr is not NULL. */
CSR5G_API int csr5g_gen_fill_range(csr5g_gen g, int64_t pos_begin, int64_t pos_end,
                                   int64_t *d_row_ptr, int32_t *d_col_idx, double *d_val,
                                   void *stream);
CSR5G_API int csr5g_gen_release(csr5g_gen g);

#ifdef __cplusplus
}
#endif
#endif /* CSR5G_H */
