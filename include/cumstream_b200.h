/*
 * cumstream_b200 — C ABI of the B200-native sliding-window moment/cumulant
 * hot path (arXiv 1701.06446).  This is the drop-in boundary: the C++ API
 * of the reference (namespace cumstream, /root/reference/proj/include/
 * cumstream/{symten,moments,cumulants,gauge,stream}.hpp) is re-implemented on
 * top of these entry points
 * (paper_1701_06446_b200/cpp/), and any FFI (ctypes, cgo, JNI) binds them
 * directly.
 *
 * Conventions
 *  - Plain pointers and sizes; no C++ or torch types cross the boundary.
 *  - Every call returns a status: CSB_OK, or one of the error classes below,
 *    which map 1:1 onto the reference's exception types:
 *      CSB_EINVAL  -> std::invalid_argument   (shape / usage errors)
 *      CSB_ERANGE  -> std::out_of_range       (index errors)
 *      CSB_EDOMAIN -> std::domain_error       (degenerate maths, e.g. nu)
 *      CSB_ERUNTIME-> std::runtime_error      (CUDA / NCCL / no device)
 *    csb_last_error() returns the thread's last message.
 *  - Tensors live on the device in the reference's block storage
 *    (SymTensor, symten.hpp:85-143): for order s, dim n, block b, only
 *    blocks with non-decreasing block index are stored, lexicographically,
 *    each a dense C-order block (edge blocks truncated), one flat array.
 *    Host transfers use exactly that layout, so a host array is
 *    interchangeable with SymTensor::data() (symten.hpp:122).
 *  - There is no CPU fallback: every compute entry point needs a CUDA
 *    device (sm_100a) and fails with CSB_ERUNTIME otherwise.
 */
#ifndef CUMSTREAM_B200_H
#define CUMSTREAM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CSB_OK 0
#define CSB_EINVAL 1
#define CSB_ERANGE 2
#define CSB_EDOMAIN 3
#define CSB_ERUNTIME 4

/* Tensor orders 1..20 as in the reference (symten.hpp:87); cumulants up to
 * order 16 (set partitions, cumulants.hpp:24: larger orders are
 * CSB_EINVAL).  Moments up to order 8 and cumulants up to 6 run on the
 * specialised kernels; above that the any-order kernels take over (one
 * thread per stored element, the same arithmetic sequence; not tuned, and
 * sharding is limited to orders <= 8). */
#define CSB_MAX_ORDER 20

typedef struct csb_series csb_series; /* device-resident M_1..M_d or C_1..C_d */
typedef struct csb_stream csb_stream; /* device-resident WindowState (stream.hpp:54-60) */

/* ---- library ---------------------------------------------------------- */
int csb_version(void);
const char* csb_last_error(void);
/* Number of visible CUDA devices (0 without a GPU; never fails). */
int csb_device_count(void);
/* Select the device subsequent calls on this thread use. */
int csb_set_device(int device);
/* rows_read(): rows handed to the moment routines so far in this process;
 * replaces cumstream::rows_read (moments.hpp:46, moments.cpp:15,216). */
uint64_t csb_rows_read(void);

/* ---- layout (SymTensor ctor, symten.cpp:105-140) ------------------------ */
/* Stored doubles and block count of one order. */
int csb_layout_size(int order, int dim, int block, uint64_t* stored, uint64_t* blocks);
/* block_multiplicity (symten.cpp:227-241) of a non-decreasing block index. */
int csb_block_multiplicity(const int* block_index, int order, uint64_t* out);

/* ---- series: the device backing of MomentSeries / CumulantSeries -------- */
/* (moments.hpp:33-42, cumulants.hpp:30-39) */
int csb_series_create(int dim, int max_order, int block, csb_series** out);
int csb_series_destroy(csb_series* s);
/* Deep device copy; shapes must match (value semantics of the reference). */
int csb_series_copy(csb_series* dst, const csb_series* src);
int csb_series_shape(const csb_series* s, int* dim, int* max_order, int* block,
                     uint64_t* window_len);
int csb_series_set_window_len(csb_series* s, uint64_t window_len);
/* Stored doubles of order `order` (1-based). */
int csb_series_stored(const csb_series* s, int order, uint64_t* stored);
/* Raw device pointer of order `order` (for zero-copy interop / tests). */
int csb_series_device_ptr(const csb_series* s, int order, double** dev);
/* Host <-> device transfers of one order in block storage. count must
 * equal the stored size. */
int csb_series_upload(csb_series* s, int order, const double* host, uint64_t count);
int csb_series_download(const csb_series* s, int order, double* host, uint64_t count);
/* host[i] = order's stored element at offsets[i] (block-storage offsets,
 * SymTensor addressing): sampled reads of tensors too large to download. */
int csb_series_gather(const csb_series* s, int order, const uint64_t* offsets, uint64_t count,
                      double* host);

/* ---- hot path, host buffers ------------------------------------------------ */
/* moment_series (moments.hpp:52): M_1..M_d of x (rows x cols, row-major).
 * `out` must have been created with dim == cols; window_len := rows. */
int csb_moment_series(csb_series* out, const double* x, uint64_t rows, uint64_t cols);
/* moment_tensor (moments.hpp:49): one order into a series slot.  Only
 * order `order` of `out` is written. */
int csb_moment_tensor(csb_series* out, int order, const double* x, uint64_t rows, uint64_t cols);
/* moments_update (moments.hpp:62): M += (p/T)(M(in) - M(out)), in place.
 * Pre: rows(in) == rows(out) == p <= window_len, cols == dim. */
int csb_moments_update(csb_series* m, const double* incoming, const double* outgoing,
                       uint64_t rows, uint64_t cols);
/* moms2cums (cumulants.hpp:47): cumulants C_1..C_d of moments m.
 * `c` must have the same shape; c.window_len := m.window_len. */
int csb_moms2cums(const csb_series* m, csb_series* c);
/* combine (moments.hpp:56): out = (s1*m1 + s2*m2)/(s1+s2) elementwise. */
int csb_combine(const csb_series* m1, uint64_t s1, const csb_series* m2, uint64_t s2,
                csb_series* out);

/* ---- hot path, device buffers (inputs already resident in HBM) ---------- */
int csb_moment_series_dev(csb_series* out, const double* x_dev, uint64_t rows, uint64_t cols);
int csb_moments_update_dev(csb_series* m, const double* in_dev, const double* out_dev,
                           uint64_t rows, uint64_t cols);

/* ---- norms and gauge ------------------------------------------------------ */
/* knorm (symten.hpp:156): (sum_blocks mult * sum |e|^k)^(1/k), k >= 1. */
int csb_knorm(const csb_series* s, int order, double k, double* out);
/* nu (gauge.hpp:21): knorm(C_d,2) / knorm(C_2,2)^(d/2); CSB_EDOMAIN when
 * ||C_2|| == 0, CSB_EINVAL unless 3 <= d <= max_order. */
int csb_nu(const csb_series* c, int d, double* out);

/* WindowReport (gauge.hpp:47-60).  nu[k] holds nu_{k+3}; has_skew/kurt
 * mirror the std::optional fields. */
typedef struct {
  uint64_t window;
  uint64_t rows;
  double norm_c1;
  double norm_c2;
  double nu[CSB_MAX_ORDER];
  int n_nu;
  int has_skewness, has_kurtosis;
  double max_abs_skewness;
  double max_abs_kurtosis;
} csb_report;

/* make_window_report (gauge.hpp:57, gauge.cpp:142-154). */
int csb_window_report(const csb_series* c, uint64_t window, csb_report* out);

/* ---- sliding-window engine (stream.hpp:19-89) ---------------------------- */
typedef struct {
  int dim;               /* n */
  int max_order;         /* d */
  uint64_t window_len;   /* t */
  uint64_t update_len;   /* t_up */
  int block_size;        /* b */
  uint64_t resync_every; /* steps between recomputes; 0 disables */
  int workers;           /* accepted for API parity; host threads only */
  /* B200 extension: shard of the order-d blocks this process owns
   * (SURVEY §8e); shard_count <= 1 means the whole tensor. */
  int shard_index;
  int shard_count;
} csb_stream_config;

typedef struct {
  double update_s;    /* StepTiming::update_s (stream.hpp:63-66), device time */
  double moms2cums_s; /* StepTiming::moms2cums_s */
} csb_step_timing;

/* prime (stream.hpp:69): first.rows == window_len. */
int csb_stream_prime(const csb_stream_config* cfg, const double* first, uint64_t rows,
                     uint64_t cols, csb_stream** out);
int csb_stream_destroy(csb_stream* st);
/* step (stream.hpp:73): exchange + moments_update (or resync) + moms2cums.
 * x is a host buffer (update_len x dim).  timing and report may be NULL;
 * when report is non-NULL the window report of the new window is filled. */
int csb_stream_step(csb_stream* st, const double* x, uint64_t rows, uint64_t cols,
                    csb_step_timing* timing, csb_report* report);
/* Same as csb_stream_step with x already in device memory.  The engine
 * reads x_dev on its own stream (csb_stream_cuda_stream): the caller must
 * order the writes that produced x_dev before that stream (e.g. record an
 * event on the producing stream and cudaStreamWaitEvent the engine's), and
 * must not overwrite x_dev until the engine's stream has passed this step
 * (the call returns early when report and timing are NULL). */
int csb_stream_step_dev(csb_stream* st, const double* x_dev, uint64_t rows, uint64_t cols,
                        csb_step_timing* timing, csb_report* report);
/* Pipelined ingestion: csb_stream_upload starts the host-to-device copy of
 * the next batch (update_len x dim) on a copy stream and returns at once;
 * csb_stream_step_uploaded runs one step on the oldest uploaded batch
 * (waiting for its copy on the device, not the host).  Up to two batches may
 * be uploaded ahead, so batch k+1's copy overlaps step k.  x must stay valid
 * and unchanged until the step that consumes it returns; use pinned host
 * memory for the copy to be asynchronous. */
int csb_stream_upload(csb_stream* st, const double* x, uint64_t rows, uint64_t cols);
int csb_stream_step_uploaded(csb_stream* st, csb_step_timing* timing, csb_report* report);
/* Report of the current window (after prime: window 1). */
int csb_stream_report(csb_stream* st, csb_report* report);
/* Borrowed views of the state (owned by the stream). */
int csb_stream_moments(csb_stream* st, const csb_series** m);
int csb_stream_cumulants(csb_stream* st, const csb_series** c);
int csb_stream_window(const csb_stream* st, uint64_t* window);
/* WindowBuffer::materialize (stream.hpp:47): window rows in arrival order. */
int csb_stream_materialize(const csb_stream* st, double* host, uint64_t count);
/* Per-block partial squared norms (count = the order's block count).  For a
 * sharded stream's order d these are already reduced over the ranks
 * (collective C3), so every entry is valid and first_block is 0. */
int csb_stream_norm_partials(csb_stream* st, int order, double* host, uint64_t count,
                             uint64_t* first_block);
/* CUDA graphs: a step's launch sequence depends only on the ring head, the
 * batch's device address and whether a report is wanted, so the engine
 * captures one graph per such key on its second visit and replays it
 * afterwards (on by default; steps with timing, profiling, a resync or
 * shards run eagerly).  csb_stream_use_graphs(st, 0) turns it off;
 * csb_stream_graph_replays counts the steps run from a graph. */
int csb_stream_use_graphs(csb_stream* st, int on);
int csb_stream_graph_replays(const csb_stream* st, uint64_t* replays);
/* Device stream (cudaStream_t) the engine launches on, for interop. */
int csb_stream_cuda_stream(csb_stream* st, void** cuda_stream);

/* ---- multi-GPU: block-prefix shards + NCCL ------------------ */
/* One process per GPU.  Rank 0 makes an id, every rank passes it to
 * csb_comm_init (NCCL is loaded at run time from libnccl.so.2); a stream
 * primed with shard_count == nranks, shard_index == rank then owns a
 * contiguous range of order-d and order-(d-1) blocks (prefix (j1, j2)
 * ranges balanced by canonical weight), replicates orders <= d-2, gathers
 * M_{d-1} and reduces the order-d norm partials / diagonal with NCCL. */
int csb_comm_unique_id(unsigned char* out /* 128 bytes */);
int csb_comm_init(int nranks, int rank, const unsigned char* id /* 128 bytes */);
/* Caller-supplied collectives in place of NCCL (any transport).  Callbacks
 * return 0 on success.  allgather_ranges: rank r owns buf[off[r], off[r] +
 * cnt[r]) on entry; on return every rank holds every range.  allreduce_sum:
 * elementwise sum over ranks, in place.  host_staged != 0: buf is host
 * memory, offsets are relative to buf and cuda_stream is NULL (the engine
 * drains its stream and copies around the call); host_staged == 0: buf is
 * device memory and the callback must order its work on cuda_stream
 * (a cudaStream_t).  The ops struct is copied; ctx must outlive the
 * streams primed under it. */
typedef struct {
  void* ctx;
  int host_staged;
  int (*allgather_ranges)(void* ctx, double* buf, const uint64_t* off, const uint64_t* cnt, int nranks,
                          void* cuda_stream);
  int (*allreduce_sum)(void* ctx, double* buf, uint64_t count, void* cuda_stream);
} csb_comm_ops;
int csb_comm_init_ops(int nranks, int rank, const csb_comm_ops* ops);
/* Collective health check of the current communicator: one allgather of
 * per-rank ranges and one sum allreduce of `count` doubles on device buffers,
 * verified on the host (CSB_ERUNTIME with a message on any mismatch).  Valid
 * for any rank count, including a single rank. */
int csb_comm_selftest(uint64_t count);
/* Releases this process's communicator; streams primed under it keep their
 * reference until they are destroyed. */
int csb_comm_destroy(void);
/* Collective over the stream's communicator: every rank receives the other
 * ranks' blocks of M_d and C_d (an in-place allgather of the owners'
 * contiguous block ranges), after which csb_stream_moments / _cumulants hold
 * the whole tensors in block order on every rank -- what a tensor dump
 * (serialize.cpp:13-75, tools/cumstream.cpp:90-96 --dump-cumulants) needs.
 * The next step overwrites only the owned ranges again.  No-op on an
 * unsharded stream. */
int csb_stream_gather_shards(csb_stream* st);
/* Block and element range of one shard: which = 0 for order d, 1 for d-1. */
int csb_shard_range(int max_order, int dim, int block, int shard_index, int shard_count, int which,
                    uint64_t* blk_lo, uint64_t* blk_hi, uint64_t* elem_lo, uint64_t* elem_hi);
/* Series-level shard computations without any exchange (the caller owns the
 * assembly): the shard's blocks of orders d and d-1, all orders <= d-2. */
int csb_moments_update_shard(csb_series* m, const double* incoming, const double* outgoing,
                             uint64_t rows, uint64_t cols, int shard_index, int shard_count);
/* C_1..C_{d-1} in full and the shard's blocks of C_d (m must be complete). */
int csb_moms2cums_shard(const csb_series* m, csb_series* c, int shard_index, int shard_count);

/* ---- instrumentation (bench.py) ------------------------------------------ */
/* Kernels launched by this library so far in this process. */
uint64_t csb_launch_count(void);
/* Name of the kernel (template instantiation) that computes orders d and
 * d-1 of a window update for this shape, given 16-byte aligned rows. */
int csb_top_kernel(int dim, int max_order, int block, char* out, uint64_t cap);
/* When enabled, CUDA events bracket every kernel launch on its own stream,
 * grouped by tag: "moment_top" (the order-d/d-1 pair kernel), "moment_low"
 * (lower pairs), "moms2cums", "norms". */
int csb_profile_enable(int on);
/* Sum of the event-timed durations (ms) and launch count of one tag since the
 * last read; reading resets the tag.  Synchronizes the recorded events. */
int csb_profile_read(const char* tag, double* total_ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* CUMSTREAM_B200_H */
