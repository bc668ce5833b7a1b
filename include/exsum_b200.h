/* exsum_b200.h — C ABI of the B200-native exact float64 summation library.
 *
 * Drop-in boundary for the reference's summation path.  The
 * reference exposes a C++ class API only (no C ABI, no FFI); every entry point
 * below names the reference symbol it replaces.  Paths are relative to
 * /root/reference/proj.
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *   - Every function that can fail returns an int status (EXSUM_OK == 0) and
 *     never throws; the reference throws std::invalid_argument instead
 *     (small_accumulator.cpp:351-353, vector_ops.cpp:150-160).
 *   - Accumulators are caller-owned values (exsum_small) or opaque handles
 *     (exsum_large, exsum_context).  No global mutable state; functions are
 *     reentrant for distinct accumulators / workspaces / streams.
 *   - Device entry points (exsum_cuda_*) are stream-ordered and asynchronous:
 *     pointers prefixed d_ are device pointers, `stream` is a cudaStream_t
 *     passed as void* (0 = legacy default stream).
 */
#ifndef EXSUM_B200_H_
#define EXSUM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ----------------------------------------------------------------- status */
#define EXSUM_OK 0
#define EXSUM_EINVAL 1 /* bad argument (mean with n == 0, null pointer, length mismatch) */
#define EXSUM_ECUDA 2  /* a CUDA runtime call failed (no device, launch failure, ...) */
#define EXSUM_ENOMEM 3 /* allocation failed / workspace too small */
#define EXSUM_ENCCL 4  /* NCCL unavailable or an NCCL call failed */
#define EXSUM_EIO 5    /* file I/O or parse failure (the reference throws std::runtime_error);
                          exsum_io_error() has the reference's message */

/* -------------------------------------------------------------- geometry */
/* small_accumulator.hpp:27-35 and large_accumulator.hpp:27-29 */
#define EXSUM_SMALL_CHUNKS 67      /* kSmallChunks: chunk i weighs 2^(32 i - 1075) */
#define EXSUM_SMALL_CARRY_TERMS 2047 /* kSmallCarryTerms: adds between propagations */
#define EXSUM_LARGE_CHUNKS 4096    /* kLargeChunks: one per sign+exponent */
#define EXSUM_NO_INDEX UINT64_MAX  /* "no such special value" in exsum_partial */

/* The small superaccumulator as a plain value.  Byte-for-byte the layout of
 * exsum::SmallAccumulator (small_accumulator.hpp:99-102: chunks_, inf_bits_,
 * nan_bits_, adds_until_propagate_), standard-layout, 560 bytes. */
typedef struct exsum_small {
  int64_t chunk[EXSUM_SMALL_CHUNKS];
  uint64_t inf_bits;            /* bit pattern of an absorbed infinity, 0 if none */
  uint64_t nan_bits;            /* bit pattern of the first absorbed NaN, 0 if none */
  int32_t adds_until_propagate; /* in [0, 2047] */
  int32_t reserved_;            /* padding, keep 0 */
} exsum_small;

/* A shard's exact sum as it leaves a device: the canonical (carry-propagated)
 * small accumulator plus the index-ordered special-value record that makes the
 * Inf/NaN outcome independent of how the array was sharded.
 * Indices are GLOBAL positions in the logical array (base_index + local). */
typedef struct exsum_partial {
  exsum_small acc;        /* canonical chunks; inf/nan bits as serial add order gives */
  uint64_t first_pos_inf; /* global index of the first +Inf, EXSUM_NO_INDEX if none */
  uint64_t first_neg_inf; /* global index of the first -Inf */
  uint64_t first_nan;     /* global index of the first NaN */
  uint64_t nan_payload;   /* bit pattern of the NaN at first_nan (0 if none) */
} exsum_partial;

/* ---------------------------------------------- host small superaccumulator */
/* SmallAccumulator() — small_accumulator.hpp:49,99-102; SPEC small_new */
int exsum_small_init(exsum_small *acc);
/* SmallAccumulator::add(double) — small_accumulator.cpp:165-172; SPEC small_add */
int exsum_small_add(exsum_small *acc, double v);
/* SmallAccumulator::add(span) — small_accumulator.cpp:174-189; SPEC small_add_array */
int exsum_small_add_array(exsum_small *acc, const double *x, size_t n);
/* SmallAccumulator::add_inf_nan — small_accumulator.cpp:230-242; SPEC small_add_inf_nan */
int exsum_small_add_inf_nan(exsum_small *acc, uint64_t bits);
/* SmallAccumulator::carry_propagate — small_accumulator.cpp:244-303.  Returns the
 * index of the top nonzero chunk, -1 for an exact zero (or for acc == NULL). */
int exsum_small_carry_propagate(exsum_small *acc);
/* SmallAccumulator::merge — small_accumulator.cpp:305-328; SPEC small_merge */
int exsum_small_merge(exsum_small *dst, const exsum_small *src);
/* SmallAccumulator::round — small_accumulator.cpp:330-348; SPEC small_round */
int exsum_small_round(exsum_small *acc, double *out);
/* SmallAccumulator::mean — small_accumulator.cpp:350-421; EXSUM_EINVAL for n == 0 */
int exsum_small_mean(exsum_small *acc, uint64_t n, double *out);

/* ---------------------------------------------- host large superaccumulator */
typedef struct exsum_large exsum_large; /* opaque; ~42 KB, see large_accumulator.hpp:99-103 */
/* LargeAccumulator() — large_accumulator.cpp:22-26; SPEC large_new */
exsum_large *exsum_large_new(void);
void exsum_large_free(exsum_large *acc);
/* LargeAccumulator::add(double) — large_accumulator.hpp:47-59; SPEC large_add */
int exsum_large_add(exsum_large *acc, double v);
/* LargeAccumulator::add(span) — large_accumulator.cpp:28-32; SPEC large_add_array */
int exsum_large_add_array(exsum_large *acc, const double *x, size_t n);
/* LargeAccumulator::drain — large_accumulator.cpp:113-131; SPEC large_drain */
int exsum_large_drain(exsum_large *acc);
/* LargeAccumulator::round — large_accumulator.cpp:133-136; SPEC large_round */
int exsum_large_round(exsum_large *acc, double *out);
/* LargeAccumulator::mean — large_accumulator.cpp:138-141 */
int exsum_large_mean(exsum_large *acc, uint64_t n, double *out);
/* LargeAccumulator::small() — large_accumulator.hpp:75-76 (copy out) */
int exsum_large_small(const exsum_large *acc, exsum_small *out);
/* LargeAccumulator::counts()[ix] — large_accumulator.hpp:79-81: adds left
 * before the chunk transfers (4096 on first use, counting down), -1 = unused. */
int exsum_large_count(const exsum_large *acc, int ix, int *count);
/* LargeAccumulator::chunk_in_use(ix) — large_accumulator.hpp:82-84 (0 or 1). */
int exsum_large_chunk_in_use(const exsum_large *acc, int ix);
/* LargeAccumulator::chunk_word(ix) — large_accumulator.hpp:85-86: the wrapped
 * sum of raw bit patterns; meaningful only while the chunk is in use. */
int exsum_large_chunk_word(const exsum_large *acc, int ix, uint64_t *word);
/* LargeAccumulator::chunks_in_use — large_accumulator.cpp:143-149 */
int exsum_large_chunks_in_use(const exsum_large *acc);

/* --------------------------------------------------- sqnorm / dot (host) */
/* sqnorm(values, SumMethod::large) — vector_ops.cpp:143-146 via sum_products
 * (:72-97): the exact, correctly rounded sum of the rounded squares x[i]*x[i]. */
int exsum_sqnorm(const double *x, size_t n, double *out);
/* dot(a, b, SumMethod::large) — vector_ops.cpp:147-155: exact sum of the
 * rounded products a[i]*b[i]; EXSUM_EINVAL on length mismatch (the reference
 * throws std::invalid_argument, :150-152). */
int exsum_dot(const double *a, size_t na, const double *b, size_t nb, double *out);
/* The same sum of rounded products a[i] * b[i] (b == a: sqnorm) on `threads`
 * host threads (<= 0: all; at most one per 2^20 products) with the host kernel
 * of exsum_host_sum; exsum_sqnorm / exsum_dot call it with threads = 0. */
int exsum_host_products(const double *a, const double *b, size_t n, int threads, double *out);

/* ---------------------------------------------------- partial records (host) */
/* Exact sum of x[0..n) into a partial record (host code; the record format the
 * device path and the multi-GPU exchange use).  base_index is the global index
 * of x[0]. */
int exsum_partial_from_array(const double *x, size_t n, uint64_t base_index,
                             exsum_partial *out);
/* Merge of k partial records: the combine step of parallel_exact_sum
 * (vector_ops.cpp:64-70) with index-ordered special values.  Writes the merged
 * canonical record (may alias parts[0]) and/or the rounded result. */
int exsum_partial_merge(const exsum_partial *parts, size_t k, exsum_partial *out,
                        double *result);
/* The library's own multithreaded host exact sum (the host half of the hybrid
 * exsum_context_sum): parallel_exact_sum (vector_ops.cpp:172-186) re-designed —
 * count-free significand bins with carry-flag transfers, dynamic work claiming
 * across `threads` host threads (<= 0: all), index-ordered Inf/NaN.  Bits equal
 * exact_sum(x) (vector_ops.cpp:121-130).  Outputs: result and/or partial. */
int exsum_host_sum(const double *x, size_t n, uint64_t base_index, int threads, double *result,
                   exsum_partial *partial);
/* exact_sum(values, method) on the host, one call (vector_ops.cpp:121-130):
 * method 0 = ExactMethod::small (SmallAccumulator), 1 = ExactMethod::large (the
 * host kernel of exsum_host_sum on the calling thread; LargeAccumulator bits).
 * EXSUM_EINVAL for another method (the reference throws std::invalid_argument,
 * vector_ops.cpp:107). */
int exsum_exact_sum(const double *x, size_t n, int method, double *out);
/* Rounded value of a partial record (SmallAccumulator::round on its acc). */
int exsum_partial_round(const exsum_partial *p, double *out);

/* ----------------------------------------------------------- device path */
/* Device workspace: accumulation state that persists across the stream-ordered
 * launches of one sum (67 chunk sums, special-value indices, counters).  Zero it
 * once with exsum_cuda_workspace_init; every finalizing call leaves it zeroed. */
size_t exsum_cuda_workspace_bytes(void);
int exsum_cuda_workspace_init(void *d_ws, size_t ws_bytes, void *stream);

/* exact_sum(values, ExactMethod::large) — vector_ops.cpp:121-130, with
 * LargeAccumulator() + add(span) + drain + SmallAccumulator::round
 * (large_accumulator.cpp:22-136, small_accumulator.cpp:244-348) as ONE launch:
 * K1 streaming accumulate, K2 per-CTA flush, K3 grid combine + round.
 * d_x: n doubles (any 8-byte alignment).  base_index: global index of d_x[0]
 * (0 for a whole array; the shard offset in a multi-GPU sum).  Outputs (either
 * may be NULL): d_result (1 double), d_partial (1 exsum_partial). */
int exsum_cuda_sum(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                   exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream);

/* exsum_cuda_sum with launch flags.  EXSUM_SUM_OVERLAP: programmatic dependent
 * launch — the grid may start while the previous kernel in `stream` is still
 * finishing (it waits for that kernel before touching d_ws).  Only valid when
 * d_x is not written by the immediately preceding kernel of the stream (e.g.
 * back-to-back sums over resident data). */
#define EXSUM_SUM_OVERLAP 1u
int exsum_cuda_sum_ex(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                      exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                      unsigned flags);

/* Launch configuration (a small POD instead of global state).
 * max_ctas: cap on the persistent grid (0 = one CTA per SM, fewer for short
 * sums) — leaves SMs to concurrent work; any value gives the same bits.
 * flags: EXSUM_SUM_OVERLAP or 0. */
typedef struct exsum_launch_config {
  uint32_t max_ctas;
  uint32_t flags;
  uint32_t reserved_[6]; /* keep 0 */
} exsum_launch_config;
int exsum_cuda_sum_cfg(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                       exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                       const exsum_launch_config *cfg);

/* Two-phase plain sums: exsum_cuda_sum(_ex) of at least this many terms, with a
 * workspace of exsum_cuda_workspace_bytes(), runs a windowed pass (16 warps per
 * SM, narrow exponent ranges) and then the full kernel over what it left — two
 * launches instead of one; the bits do not depend on it.  0: disabled. */
uint64_t exsum_cuda_two_phase_min(void);

/* sqnorm / dot on the device (vector_ops.cpp:143-155): the exact sum of the
 * products rounded as the reference's x86 multiply rounds them (IEEE nearest
 * even; a NaN operand propagates quieted, x first; 0 * Inf is the x86 default
 * NaN 0xFFF8000000000000), one launch like exsum_cuda_sum.  dot reads both
 * arrays with 256-bit loads when they are co-aligned mod 32 bytes; na != nb is
 * EXSUM_EINVAL. */
int exsum_cuda_sqnorm(const double *d_x, size_t n, uint64_t base_index, double *d_result,
                      exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream);
int exsum_cuda_dot(const double *d_a, size_t na, const double *d_b, size_t nb,
                   uint64_t base_index, double *d_result, exsum_partial *d_partial, void *d_ws,
                   size_t ws_bytes, void *stream);

/* Incremental form (LargeAccumulator::add(span) across calls, large_accumulator.hpp:61):
 * accumulate d_x into the workspace without rounding; then finalize. */
int exsum_cuda_accumulate(const double *d_x, size_t n, uint64_t base_index, void *d_ws,
                          size_t ws_bytes, void *stream);
int exsum_cuda_finalize(double *d_result, exsum_partial *d_partial, void *d_ws,
                        size_t ws_bytes, void *stream);

/* One exact_sum per segment: segment i is d_x[d_offsets[i] .. d_offsets[i+1]).
 * d_offsets has nseg + 1 nondecreasing entries (a decreasing pair is read as an
 * empty segment, sum +0.0, never as a wrapped length).  No reference batch API exists;
 * semantics = exact_sum(segment_i) for every i.
 * d_partials may be NULL; otherwise nseg records, indices local to the segment.
 * With ws_bytes >= exsum_cuda_segmented_workspace_bytes(nseg) (and more segments
 * than warps) two small launches build the claim order (index order, the last
 * 4 x warps segments longest first) and a last launch rounds every segment from
 * its raw record; otherwise segments are claimed in index order and rounded in
 * the streaming launch.  The order cannot change any result.
 * exsum_cuda_workspace_init with the full ws_bytes prepares both (it zeroes the
 * order state as well). */
int exsum_cuda_sum_segmented(const double *d_x, const uint64_t *d_offsets, size_t nseg,
                             double *d_out, exsum_partial *d_partials, void *d_ws,
                             size_t ws_bytes, void *stream);
size_t exsum_cuda_segmented_workspace_bytes(size_t nseg);

/* Merge k partial records resident on the device (after an all-gather of the
 * shards' records): parallel_exact_sum's merge phase, vector_ops.cpp:64-70. */
int exsum_cuda_merge(const exsum_partial *d_parts, size_t k, double *d_result,
                     exsum_partial *d_out, void *stream);

/* ------------------------------------------------ host-buffer convenience */
/* A device context: workspace, 3-slot device staging ring, copy + compute
 * streams, and a pool of host worker threads.  exsum_context_sum is
 * exact_sum(values) (vector_ops.cpp:121-130) for a HOST array, the call a
 * reference user makes.  The array is split dynamically: the calling thread
 * streams chunks host->device (pinned memory: direct DMA; pageable: through
 * pinned bounce buffers) into the sm_100a accumulate kernel while the host
 * workers sum other chunks with exsum_host_sum's kernel; the two exact records
 * are merged (exsum_partial_merge), so the bits equal exact_sum for any split.
 * Blocking.  A context serves one sum at a time (concurrent calls on one context
 * serialise on its lock); use one context per thread for parallel sums.  A
 * failed sum leaves the context reset and reusable. */
typedef struct exsum_context exsum_context;
exsum_context *exsum_context_create(int device, size_t staging_bytes);
void exsum_context_free(exsum_context *ctx);
/* Host workers beside the device: < 0 = every hardware thread (default),
 * 0 = device only (PCIe-bound, every size), k = k threads.  With workers
 * enabled, an array (or segment list) under 2^17 terms is summed by the
 * calling thread alone: the device round trip (~35 us) costs more than the
 * whole sum on one core. */
int exsum_context_set_host_threads(exsum_context *ctx, int threads);
/* Terms the last successful sum gave the device and the host workers. */
int exsum_context_last_split(const exsum_context *ctx, uint64_t *device_terms,
                             uint64_t *host_terms);
int exsum_context_sum(exsum_context *ctx, const double *h_x, size_t n, double *h_result,
                      exsum_partial *h_partial);
/* The same for a shard whose first element has global index base_index (the
 * partial record's Inf/NaN indices are global, ready for exsum_partial_merge). */
int exsum_context_sum_at(exsum_context *ctx, const double *h_x, size_t n, uint64_t base_index,
                         double *h_result, exsum_partial *h_partial);
/* One exact_sum per segment of a HOST array (host-array form of
 * exsum_cuda_sum_segmented): segment i is h_x[h_offsets[i] .. h_offsets[i+1])
 * (a decreasing pair is an empty segment).  The device takes groups of whole
 * segments (≤ one staging chunk of values, ≤ 16384 segments) over PCIe while the
 * host workers sum other segments; h_out (nseg doubles) and h_partials (nseg
 * records, indices local to each segment; may be NULL) are bit-identical to
 * the device path whatever the split.  Blocking. */
int exsum_context_sum_segmented(exsum_context *ctx, const double *h_x,
                                const uint64_t *h_offsets, size_t nseg, double *h_out,
                                exsum_partial *h_partials);
/* exact_sum(read_values(path, format)) without materialising the array: a bin
 * file is read chunk by chunk into pinned host buffers that feed the staging
 * ring (disk read, host->device copy and accumulate overlap); a text file is
 * parsed on the host first.  *n_out (optional) receives the value count. */
int exsum_context_sum_file(exsum_context *ctx, const char *path, int format, double *h_result,
                           exsum_partial *h_partial, uint64_t *n_out);

/* ------------------------------------------ multi-GPU (NCCL over NVLink) */
/* parallel_exact_sum (vector_ops.cpp:172-186) with one shard per GPU (one
 * process per GPU).  split (vector_ops.cpp:37-49) gives each rank a contiguous
 * shard; the rank reduces it to one exsum_partial record, the records are
 * exchanged with ONE ncclAllGather (nranks x 592 B) and every rank merges them
 * (merge_partials, vector_ops.cpp:64-70, with index-ordered Inf/NaN), so every
 * rank holds the serial exact_sum bits.  NCCL is loaded on first use
 * (libnccl.so.2 already in the process, else EXSUM_NCCL_LIB, else the system
 * one); `comm` is an ncclComm_t passed as void*, e.g. one the caller already
 * owns or one from exsum_nccl_comm_init. */
#define EXSUM_NCCL_UNIQUE_ID_BYTES 128 /* sizeof(ncclUniqueId) */
/* split(n, parts)[rank] — vector_ops.cpp:37-49 (remainder to the first shards). */
int exsum_shard_bounds(uint64_t n, int nranks, int rank, uint64_t *begin, uint64_t *end);
/* 1 if NCCL can be loaded (and its version in *version if non-NULL), else 0. */
int exsum_nccl_available(int *version);
int exsum_nccl_get_unique_id(void *id /* EXSUM_NCCL_UNIQUE_ID_BYTES */);
/* ncclCommInitRank on the current CUDA device. */
int exsum_nccl_comm_init(void **comm, int nranks, const void *id, int rank);
int exsum_nccl_comm_destroy(void *comm);
/* Workspace of exsum_nccl_sum for a communicator of nranks ranks (device memory;
 * zero it once with exsum_cuda_workspace_init, every call leaves it zeroed). */
size_t exsum_nccl_workspace_bytes(int nranks);
/* This rank's shard d_shard[0..n) = logical indices [base_index, base_index + n):
 * sum kernel -> ncclAllGather of the records -> merge kernel, stream-ordered and
 * graph-capturable.  Outputs (either may be NULL) are identical on every rank.
 * flags: EXSUM_SUM_OVERLAP for the sum kernel, as for exsum_cuda_sum_ex. */
int exsum_nccl_sum(const double *d_shard, size_t n, uint64_t base_index, void *comm,
                   double *d_result, exsum_partial *d_partial, void *d_ws, size_t ws_bytes,
                   void *stream, unsigned flags);

/* ------------------------------------------------------------ value files */
/* exsum::FileFormat (io.hpp:23-29): bin = raw little-endian doubles; text =
 * one value per line, decimal or a 0x-prefixed 16-hex-digit bit pattern. */
#define EXSUM_FORMAT_BIN 0
#define EXSUM_FORMAT_TEXT 1
/* parse_format (io.cpp:71-79): "bin" | "text" -> EXSUM_FORMAT_*, -1 otherwise. */
int exsum_parse_format(const char *name);
/* read_values (io.cpp:83-131): *values is malloc'ed (free with
 * exsum_free_values), *n its length.  EXSUM_EIO on open/read/parse errors. */
int exsum_read_values(const char *path, int format, double **values, size_t *n);
void exsum_free_values(double *values);
/* write_values (io.cpp:133-159): %.17g for finite values, 0x%016llx for Inf/NaN. */
int exsum_write_values(const char *path, const double *values, size_t n, int format);
/* Message of the last EXSUM_EIO on this thread ("<path>: <what>", as the
 * reference's exception text). */
const char *exsum_io_error(void);

/* ------------------------------- multi-GPU, fused exchange over peer memory */
/* parallel_exact_sum as ONE launch per rank: the sum kernel's last CTA writes
 * the rank's 592 B record into every rank's mailbox over NVLink peer memory,
 * publishes it with a system-scope release flag carrying `epoch`, waits for
 * every rank's flag (bounded: 10 s, then the result is NaN 0x7FF80000DEAD0000
 * and the mailbox error word holds the epoch) and merges the records in place
 * — the exchange of exsum_nccl_sum without a separate collective.
 * mailboxes: host array of nranks device pointers, [r] = rank r's mailbox
 * mapped into this process (its own for r == rank; exsum_ipc_open for peers);
 * each of exsum_p2p_mailbox_bytes(nranks) bytes, zeroed once.  epoch: 1, 2, 3,
 * ... per call, the same on every rank.  nranks <= 8.  flags: EXSUM_SUM_OVERLAP
 * as for exsum_cuda_sum_ex (safe across calls: the mailboxes are double-buffered). */
size_t exsum_p2p_mailbox_bytes(int nranks);
/* A zeroed mailbox as its own cudaMalloc allocation (exportable with IPC). */
int exsum_p2p_mailbox_alloc(int nranks, void **d_mailbox);
int exsum_p2p_mailbox_free(void *d_mailbox);
int exsum_p2p_sum(const double *d_shard, size_t n, uint64_t base_index, int rank, int nranks,
                  void *const *mailboxes, uint64_t epoch, double *d_result,
                  exsum_partial *d_partial, void *d_ws, size_t ws_bytes, void *stream,
                  unsigned flags);
/* flags bit for exsum_p2p_sum: sum and publish this rank's record and flag to
 * every mailbox, but return without waiting; exsum_p2p_collect (a one-warp
 * launch, no data) later waits for every rank's flag and merges.  With it,
 * ranks that share one GPU can be run strictly one after another (tests):
 * no kernel ever waits on a kernel that is not finished. */
#define EXSUM_P2P_PUBLISH_ONLY 2u
int exsum_p2p_collect(int rank, int nranks, void *const *mailboxes, uint64_t epoch,
                      double *d_result, exsum_partial *d_partial, void *stream);
/* The same protocol with nranks emulated ranks in ONE cooperative launch on one
 * GPU (rank r sums d_x[bounds[r], bounds[r+1]); d_mailboxes: nranks contiguous
 * mailboxes; d_ws: nranks contiguous workspaces; outputs: nranks results /
 * records, all equal).  For testing the exchange where only one GPU exists. */
int exsum_p2p_emulate_sum(const double *d_x, const uint64_t *bounds, int nranks, uint64_t epoch,
                          double *d_results, exsum_partial *d_partials, void *d_mailboxes,
                          void *d_ws, size_t ws_bytes, void *stream);
/* The mailbox's error word: 0, or the epoch of a call that timed out. */
int exsum_p2p_error(const void *d_mailbox, int nranks, uint64_t *epoch_out, void *stream);
/* cudaIpcMemHandle_t (64 bytes) of a cudaMalloc'ed mailbox, and its mapping in
 * another process (cudaIpcOpenMemHandle, peer access enabled lazily). */
#define EXSUM_IPC_HANDLE_BYTES 64
int exsum_ipc_get_handle(const void *d_ptr, void *handle);
int exsum_ipc_open(const void *handle, void **d_ptr);
int exsum_ipc_close(void *d_ptr);

/* --------------------------------------------------- synthetic data (bench) */
/* Seeded counter-based generators for the BASELINE.json configs (SURVEY.md
 * §8(d)); the value at index i depends only on (config, seed, i, n), so shards
 * generate independently.  config: 1..4 (config 5 values: exsum_{cuda,host}_gen_segmented);
 * host and device produce identical bits. */
int exsum_cuda_gen(int config, uint64_t seed, uint64_t n_total, uint64_t first,
                   size_t count, double *d_out, void *stream);
int exsum_host_gen(int config, uint64_t seed, uint64_t n_total, uint64_t first,
                   size_t count, double *out);
/* Config 5: nseg segment lengths log-uniform in [lo, hi]; offsets (nseg+1);
 * values (normal * 10^k with 1e-4 specials) for global indices [first, first+count). */
int exsum_host_gen_offsets(uint64_t seed, size_t nseg, uint64_t lo, uint64_t hi,
                           uint64_t *offsets);
int exsum_cuda_gen_segmented(uint64_t seed, uint64_t first, size_t count, double *d_out,
                             void *stream);
/* The same config-5 values on the host (bit-identical to exsum_cuda_gen_segmented). */
int exsum_host_gen_segmented(uint64_t seed, uint64_t first, size_t count, double *out);

/* The paper's benchmark data (generate, generator.cpp:23-45): n/2 values
 * U1 * exp(30 U2) from the minstd stream seeded with `seed`, mirrored as -v into
 * the second half (exact sum zero), Fisher-Yates shuffled on the same stream if
 * permute.  EXSUM_EINVAL for n == 0 or odd (the reference throws
 * std::invalid_argument).  Bits equal the reference's with the same libm exp. */
int exsum_generate(uint64_t n, uint64_t seed, int permute, double *out);

/* Library build/version info: "exsum_b200 <version> sm_100a". */
const char *exsum_version(void);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* EXSUM_B200_H_ */
