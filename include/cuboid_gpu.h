/*
 * cuboid_gpu.h -- C ABI of the B200 (sm_100a) residue-table builder and (p,q)
 * pair sieve for the modulo-primes perfect-cuboid search (arXiv 1601.00636).
 *
 * The reference (/root/reference/proj) is a header-only C++20 library with no
 * FFI; the drop-in points this ABI replaces are (paths relative to
 * /root/reference/proj):
 *
 *   build_table(r)                 include/cuboid/sievetable.hpp:123-141
 *   build_table_oracle(r)          include/cuboid/sievetable.hpp:102-115
 *   SieveSet::build(primes)        include/cuboid/sievetable.hpp:159-176
 *   load_sieve(tables, index)      include/cuboid/sievetable.hpp:254-292
 *   scan(set, start, p_end, ...)   include/cuboid/engine.hpp:195-295
 *   ScanStats / ScanSink           include/cuboid/engine.hpp:97-135
 *
 * Plain pointers and sizes only; no exceptions cross this boundary. Every
 * function returns a cgpu_status: 0 on success, the reference's own scan status
 * codes 2..6 (engine.hpp:5-12) where it would throw ScanRejected{code}, and
 * negative values where it would throw another exception or where CUDA fails.
 * cgpu_last_error() returns a thread-local message for the last failure.
 *
 * Table bytes are ALWAYS the reference's packed format: per prime r, ceil(r^2/8)
 * bytes, bit i = a*r + b at byte i>>3, bit i&7 (LSB first), 1 = "Q_ab(t) has no
 * root mod r"; tables concatenated at cumulative byte offsets
 * (sievetable.hpp:1-19, 41-64).
 */
#ifndef CUBOID_GPU_H
#define CUBOID_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
	CGPU_OK = 0,
	/* 2..6: ScanRejected codes of the reference (engine.hpp:5-12, 152-161) */
	CGPU_P_BELOW_152 = 2,
	CGPU_P_ABOVE_LIMIT = 3,
	CGPU_Q_BELOW_LOW = 4,
	CGPU_Q_ABOVE_HIGH = 5,
	CGPU_NOT_LOADED = 6,
	CGPU_ERR_CUDA = -1,          /* CUDA runtime failure (see cgpu_last_error) */
	CGPU_ERR_INVALID = -2,       /* std::invalid_argument in the reference */
	CGPU_ERR_OVERFLOW = -3,      /* std::overflow_error (set exceeds 2^32 bytes) */
	CGPU_ERR_FORMAT = -4,        /* FormatError (sievetable.hpp:37-39) */
	CGPU_ERR_RANGE = -5,         /* std::out_of_range */
	CGPU_ERR_CAPACITY = -6,      /* caller's output buffer too small; sizes still reported */
	CGPU_ERR_NO_DEVICE = -7,     /* no CUDA device: this library has no CPU fallback */
	CGPU_ERR_IO = -8             /* file I/O failure (read_bytes / write_bytes, sievetable.hpp:313-332) */
} cgpu_status;

/* Row-bound modes of the sieve. REGION = the reference scan() region
 * q_low(p) <= q <= 59p (region.hpp:49-63, engine.hpp:225-227). TRIANGLE =
 * 1 <= q < p (the BASELINE configs; loop of verify_small_region,
 * engine.hpp:613-625). The filter is identical: skip q == p and gcd > 1
 * (engine.hpp:258). */
enum { CGPU_REGION = 0, CGPU_TRIANGLE = 1 };

/* Table-build algorithms. PRODUCTION = build_table's row-1 + permutation
 * (sievetable.hpp:123-141). EXHAUSTIVE = the definition over every
 * (a,b,t) in Z_r^3 (sievetable.hpp:102-115, without early exit): exactly
 * sum r^3 Q evaluations. Both emit byte-identical tables. */
enum { CGPU_BUILD_PRODUCTION = 0, CGPU_BUILD_EXHAUSTIVE = 1 };

typedef struct cgpu_ctx cgpu_ctx;

const char* cgpu_last_error(void);
const char* cgpu_version(void);

/* One context per device (one process per GPU). `stream` may be NULL (the
 * context creates its own) or a cudaStream_t owned by the caller. */
int cgpu_create(int device, void* stream, cgpu_ctx** out);
/* CUDA devices visible to this process (0 on a box without a GPU). */
int cgpu_device_count(int* n);
int cgpu_destroy(cgpu_ctx* ctx);
int cgpu_set_stream(cgpu_ctx* ctx, void* stream);
int cgpu_synchronize(cgpu_ctx* ctx);

/* ---- tables ------------------------------------------------------------ */

/* Size query mirroring SieveSet::build's validation (sievetable.hpp:159-176):
 * strictly increasing primes below 9697, total bytes below 2^32. Fills
 * offsets[n] (may be NULL) and *total_bytes. Host-only. */
int cgpu_table_layout(const uint32_t* primes, uint32_t n, uint32_t* offsets, uint64_t* total_bytes);

/* Builds the set for `primes` ON THE DEVICE and keeps it resident in ctx
 * (replaces SieveSet::build). If out_bytes != NULL the packed tables
 * (total_bytes of cgpu_table_layout) are copied back; out_offsets (n) likewise.
 * *out_evals (may be NULL) = Q evaluations performed. */
int cgpu_tables_build(cgpu_ctx* ctx, const uint32_t* primes, uint32_t n, int algorithm,
                      uint8_t* out_bytes, uint32_t* out_offsets, uint64_t* out_evals);

/* Uploads reference-format packed tables (e.g. from load_sieve or a tables
 * .bin file) and makes them resident (replaces load_sieve for the device).
 * Nonzero padding bits are a FormatError (sievetable.hpp:67-79). */
int cgpu_tables_load(cgpu_ctx* ctx, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                     uint64_t nbytes);

/* As cgpu_tables_load, from DEVICE memory on ctx's device, read by a copy on
 * ctx's stream (the bytes must be complete by then: written on that stream or
 * synchronised with it): the multi-GPU upload path, where each rank copies 1/G of the host
 * tables over PCIe and the full set is all-gathered over NVLink first
 * (parallel.py load_tables_sharded). */
int cgpu_tables_load_dev(cgpu_ctx* ctx, const uint32_t* primes, uint32_t n, const void* d_bytes,
                         uint64_t nbytes);

/* Asynchronous loads, for pipelines that upload a set every step (the e2e
 * bench, the multi-GPU sharded upload): as cgpu_tables_load /
 * cgpu_tables_load_dev, but nothing waits for the device. The probe list is
 * built from the EXPECTED per-table flags (those last verified for the same
 * prime list on this context, else the reference builder's: every table of
 * r >= 11 has a set bit, r <= 7 none) and a device check compares them with
 * the derived ones. The bytes must stay valid until the stream has consumed
 * them. Errors surface later: cgpu_load_status (waits) returns the deferred
 * FormatError (nonzero padding) or CGPU_ERR_INVALID if the flags differed
 * (the context then re-derives; launches made since the load must be
 * repeated); cgpu_sieve_results and cgpu_tables_info check it too.
 * cgpu_load_status_copy enqueues a copy of the 32-bit status word (0 = ok,
 * bit 0 padding error, bit 1 flag mismatch) to dst (device or pinned host
 * memory) on the context stream, for callers that never synchronise. */
int cgpu_tables_load_async(cgpu_ctx* ctx, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                           uint64_t nbytes);
int cgpu_tables_load_dev_async(cgpu_ctx* ctx, const uint32_t* primes, uint32_t n, const void* d_bytes,
                               uint64_t nbytes);
int cgpu_load_status(cgpu_ctx* ctx);
int cgpu_load_status_copy(cgpu_ctx* ctx, void* dst);

/* Copies the resident packed tables back (total_bytes) -- byte-identical to
 * serialize_tables (sievetable.hpp:229). */
int cgpu_tables_download(cgpu_ctx* ctx, uint8_t* out_bytes, uint64_t cap);

/* n primes resident (0 = none loaded); killable[k] = table k has a set bit. */
int cgpu_tables_info(cgpu_ctx* ctx, uint32_t* n, uint8_t* killable);

/* Stateless convenience: build on a temporary context of `device`. */
int cgpu_build_tables(int device, const uint32_t* primes, uint32_t n, int algorithm,
                      uint8_t* out_bytes, uint32_t* out_offsets, uint64_t* out_evals);

/* ---- on-disk formats (host; sievetable.hpp:229-346, proj/README.md) ---- */

/* The CUPQ v1 index of a prime list (serialize_index, sievetable.hpp:231-252):
 * 9-byte header ("CUPQ", 0x01, u32 LE count) + per prime {u16 LE prime, u32 LE
 * byte offset}. out may be NULL (size query into *out_len). */
int cgpu_index_serialize(const uint32_t* primes, uint32_t n, uint8_t* out, uint64_t cap,
                         uint64_t* out_len);

/* Validates an index exactly like load_sieve (sievetable.hpp:254-292; every
 * violation is CGPU_ERR_FORMAT) and returns its primes (up to cap; primes may
 * be NULL), the count and the tables-stream length the index implies. */
int cgpu_index_parse(const uint8_t* index, uint64_t len, uint32_t* primes, uint32_t cap,
                     uint32_t* n_out, uint64_t* tables_bytes);

/* load_sieve_files / save_sieve_files (sievetable.hpp:334-346) for the device:
 * reads a tables .bin + CUPQ index and makes the set resident; writes the
 * resident set back byte-identically. */
int cgpu_tables_load_files(cgpu_ctx* ctx, const char* tables_path, const char* index_path);
int cgpu_tables_save_files(cgpu_ctx* ctx, const char* tables_path, const char* index_path);

/* ---- sieve ------------------------------------------------------------- */

/* Sieves rows p in [p_lo, p_hi] against the resident tables (replaces the
 * inner loops of scan(), engine.hpp:225-284). Rows are restricted to the
 * block-cyclic shard (p/100) % shard_count == shard_index (shard_count 1 =
 * all rows). REGION: the first row starts at q_start (0 = q_low(p_lo));
 * TRIANGLE requires q_start == 0.
 *
 * Asynchronous: enqueues on the context stream and returns; results stay on
 * the device until cgpu_sieve_results. The survivor buffer holds up to
 * surv_cap pairs (the device counts beyond it; see CGPU_ERR_CAPACITY).
 */
int cgpu_sieve_launch(cgpu_ctx* ctx, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode,
                      uint32_t shard_count, uint32_t shard_index, uint64_t surv_cap);

/* Waits for the last launch and copies its results:
 *   counts[2]      = {pairs_tested, survivors}
 *   hist[n]        = first-killer counts by rank (ScanStats::kill_histogram)
 *   block_rmax[nb] = per p/100 block max killing prime, 1 if none, for blocks
 *                    p_lo/100 .. p_hi/100 (0 for blocks outside the shard)
 *   surv_pq[2*k]   = survivors (p, q) ascending, k = min(survivors, cap)
 * Any output pointer may be NULL. */
int cgpu_sieve_results(cgpu_ctx* ctx, uint64_t* counts, uint64_t* hist, uint32_t* block_rmax,
                       uint64_t block_cap, uint64_t* surv_pq, uint64_t surv_cap);

/* Synchronous launch + results. */
int cgpu_sieve(cgpu_ctx* ctx, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode,
               uint32_t shard_count, uint32_t shard_index, uint64_t* counts, uint64_t* hist,
               uint32_t* block_rmax, uint64_t block_cap, uint64_t* surv_pq, uint64_t surv_cap);

/* Like cgpu_sieve_launch, but results go to CALLER-OWNED device buffers on the
 * context's device and stay there (e.g. for an NCCL all-reduce across ranks):
 *   d_counts[2] = {pairs_tested, survivors}
 *   d_hist[n]   = first-killer counts by rank (n = primes in the set)
 *   d_block_rmax[block_cap >= p_hi/100 - p_lo/100 + 1], as in cgpu_sieve_results
 *   d_surv[surv_cap] = survivors as (p << 32) | q, UNSORTED; d_counts[1] may
 *                   exceed surv_cap (only the first surv_cap are stored).
 * Asynchronous on the context stream. */
int cgpu_sieve_launch_dev(cgpu_ctx* ctx, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode,
                          uint32_t shard_count, uint32_t shard_index, uint64_t* d_counts,
                          uint64_t* d_hist, uint32_t* d_block_rmax, uint64_t block_cap,
                          uint64_t* d_surv, uint64_t surv_cap);

/* A REGION span that may end mid-row: rows p_lo..p_hi, the first from q_start
 * (0 = q_low), the last up to q_end inclusive (0 = q_high). Synchronous; the
 * outputs are those of cgpu_sieve_results. This is what a scan() halted by
 * its cooperative stop flag covers (engine.hpp:248-257): the caller computes
 * the reference's stop point and sieves up to the pair before it. */
int cgpu_sieve_span(cgpu_ctx* ctx, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end,
                    uint64_t* counts, uint64_t* hist, uint32_t* block_rmax, uint64_t block_cap,
                    uint64_t* surv_pq, uint64_t surv_cap);

/* cgpu_sieve_launch_dev for a REGION span that may end mid-row (as
 * cgpu_sieve_span: rows p_lo..p_hi, the first from q_start, the last up to
 * q_end inclusive, 0 = q_high), restricted to the block-cyclic shard. */
int cgpu_sieve_launch_span_dev(cgpu_ctx* ctx, uint64_t p_lo, uint64_t q_start, uint64_t p_hi,
                               uint64_t q_end, uint32_t shard_count, uint32_t shard_index,
                               uint64_t* d_counts, uint64_t* d_hist, uint32_t* d_block_rmax,
                               uint64_t block_cap, uint64_t* d_surv, uint64_t surv_cap);

/* Cooperative stop (ScanOptions::hooks.stop, engine.hpp:137-149, 248-257) that
 * the DEVICE sees. cgpu_alloc_stop_word returns a zeroed host word in mapped,
 * portable pinned memory; after cgpu_set_stop_word(ctx, word) every sieve
 * launch of ctx polls it (each warp, every 8th row) and abandons its
 * remaining rows once it is nonzero. The results of a launch that saw the
 * word raised are INCOMPLETE: the caller discards them and sieves exactly up
 * to the reference's next stop point with a span (include/cuboid/gpu.hpp
 * does). word = NULL detaches. */
int cgpu_alloc_stop_word(uint32_t** word);
int cgpu_free_stop_word(uint32_t* word);
int cgpu_set_stop_word(cgpu_ctx* ctx, uint32_t* word);

/* Device time of the last sieve launch or table build, from CUDA events on the
 * context stream (waits for them). Sieve: ms[0] = init + first plan kernel,
 * ms[1] = sieve kernel(s), ms[2] = whole launch. Table build: ms[0] = build
 * kernels (cube, or row-1 + permute), ms[1] = device-layout derivation,
 * ms[2] = both. */
int cgpu_last_timings(cgpu_ctx* ctx, float* ms3);

/* Name of the sieve kernel the last launch ran: "k_wsieve" (the wheel sieve:
 * standard probe sets, launches of long rows) or "k_sieve" (the window sieve);
 * "" before the first launch. Results never depend on the choice
 * (CUBOID_WHEEL = 0 / 1 / 2: never / by mean row length / always). No
 * reference counterpart: profiling and the bench's roofline read it. */
const char* cgpu_last_sieve_kernel(cgpu_ctx* ctx);

/* Measured INT32 throughput of `device` in thread-ops/s: ops4[0] = LOP3 chains
 * (ALU pipe), ops4[1] = IMAD chains (FMA pipe), ops4[2] = IMAD + LOP3
 * interleaved (3 register sources each), ops4[3] = IMAD + LOP3 with
 * immediates (the issue-bound ceiling). The roofline denominators of the bench. */
int cgpu_int32_peak(int device, double* ops4);

/* Measured FP32-pipe throughput of `device`: ops2[0] = FFMA2 chains in lane
 * FMAs/s (3 register sources), ops2[1] = the exhaustive table build's
 * evaluation mix (2 FFMA2 + IMAD + min per evaluation, k_cube_f2) in
 * evaluations/s -- the table build's roofline denominator. */
int cgpu_fp32_peak(int device, double* ops2);

/* Number of kernels the last cgpu_sieve_launch / cgpu_tables_* enqueued. */
int cgpu_last_launch_count(cgpu_ctx* ctx, uint32_t* n);

/* ---- classify (K3) ------------------------------------------------------- */

/* First-killer rank for explicit pairs (verify_pair's sieve part,
 * engine.hpp:72-78): out_rank[i] = rank of the smallest-rank prime whose table
 * rejects (p_i, q_i), or -1 if no table does. pq = n pairs of u64 (p, q). */
int cgpu_classify(cgpu_ctx* ctx, const uint64_t* pq, uint64_t n, int32_t* out_rank);

/* ---- in-process multi-GPU (one process, G devices, NCCL) ------------------ */

/* The reference drives its search from ONE process (scan() on the
 * SearchController's worker thread, engine.hpp:494, 555-577); this is how that
 * process uses every GPU of the box. One cgpu_ctx and stream per device, one
 * NCCL clique from ncclCommInitAll over `devices` (NULL = 0..n-1; each device
 * at most once). Rows are sharded block-cyclically by p/100 block
 * (SURVEY.md 8(e)), so each reference r_max block lives on one device. */
typedef struct cgpu_multi cgpu_multi;

int cgpu_multi_create(int n_devices, const int* devices, cgpu_multi** out);
int cgpu_multi_destroy(cgpu_multi* m);
int cgpu_multi_size(cgpu_multi* m, int* n);
/* The i-th device's context (borrowed; it holds the full set after a load). */
int cgpu_multi_ctx(cgpu_multi* m, int i, cgpu_ctx** out);

/* As cgpu_tables_load on every device: each copies 1/G of the host bytes over
 * its own PCIe link and an in-place ncclAllGather assembles the set. */
int cgpu_multi_tables_load(cgpu_multi* m, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                           uint64_t nbytes);

/* Synchronous multi-GPU cgpu_sieve (shard arguments implied): device g sieves
 * the blocks with (p/100) % G == g; one grouped NCCL all-reduce merges the
 * counters and histogram (SUM, ScanStats::merge engine.hpp:121-134) and block
 * r_max (MAX); grouped ncclSend/ncclRecv gather the survivor lists onto the
 * first device; outputs as cgpu_sieve_results (survivors ascending). q_end != 0
 * ends a REGION span mid-row (as cgpu_sieve_span). */
int cgpu_multi_sieve(cgpu_multi* m, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end,
                     int mode, uint64_t* counts, uint64_t* hist, uint32_t* block_rmax, uint64_t block_cap,
                     uint64_t* surv_pq, uint64_t surv_cap);

/* cgpu_set_stop_word on every device's context (one portable word). */
int cgpu_multi_set_stop_word(cgpu_multi* m, uint32_t* word);

/* Device time of the last cgpu_multi_sieve, max over devices (CUDA events on
 * each device's stream, from its launch to its last result copy). */
int cgpu_multi_last_ms(cgpu_multi* m, float* ms);

/* ---- region arithmetic (host) -------------------------------------------- */

/* q_bounds (region.hpp:49-63). */
int cgpu_q_bounds(uint64_t p, uint64_t* q_low, uint64_t* q_high);

/* The pair k steps after (p, q) in the order scan() visits q (rows p,
 * q_low(p)..q_high(p); the first row from q, engine.hpp:225-247), counting
 * every q (skipped pairs too, as the stop-poll counter does, :248). CGPU_OK
 * with *out_p, *out_q, or CGPU_P_ABOVE_LIMIT (3) if row p_end ends first.
 * Host-only; O(rows). */
int cgpu_region_advance(uint64_t p, uint64_t q, uint64_t k, uint64_t p_end, uint64_t* out_p, uint64_t* out_q);

#ifdef __cplusplus
}
#endif

#endif /* CUBOID_GPU_H */
