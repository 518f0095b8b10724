// Host-side launchers for the device kernels (tables.cu, sieve.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

namespace cgpu {

// ---- K1: residue tables ------------------------------------------------------

// One prime of a set being built/derived on the device.
struct PrimeJob {
	uint32_t r;         // prime
	uint32_t m;         // barrett_m(r)
	uint32_t byte_off;  // offset of its packed table in the set
	uint32_t ext_base;  // word offset of its ext rows
	uint32_t aux_off;   // offset into per-prime scratch (row1 / inverses), sum of r
	uint32_t pad;
};

// Exhaustive cube: all (a,b,t) in Z_r^3, no early exit. `jobs` sorted by
// descending r (blockIdx.y = job); h_jobs is the host copy of d_jobs.
cudaError_t launch_cube(const PrimeJob* d_jobs, const PrimeJob* h_jobs, uint32_t njobs,
                        uint8_t* d_packed, cudaStream_t s);
uint32_t cube_launches(const PrimeJob* h_jobs, uint32_t njobs);  // kernels launch_cube issues

// Production: row 1 (t <= r/2, early exit) + modular inverses, then the
// permuted, packed r x r table.
cudaError_t launch_row1(const PrimeJob* d_jobs, uint32_t njobs, uint32_t max_r,
                        uint8_t* d_row1, uint32_t* d_inv, unsigned long long* d_evals,
                        cudaStream_t s);
cudaError_t launch_permute(const PrimeJob* d_jobs, uint32_t njobs, uint32_t max_rr,
                           const uint8_t* d_row1, const uint32_t* d_inv, uint8_t* d_packed,
                           cudaStream_t s);

// Packed reference bytes -> row-extended words + killable flags; jobs in rank
// order (killable index = job), one CTA per work item (derive_items).
// Window tables of the table probes (k_sieve's first kTabProbes register
// probes) for every row: probes[j] = {r, ext_base, S, tab base}; out holds
// `stride` masks then `stride` successor indices.
cudaError_t launch_wintab(const uint4* d_probes, uint32_t nprobes, uint32_t entries, const uint32_t* d_ext,
                          uint32_t stride, uint32_t* d_out, cudaStream_t s);

// Speculative-load check (k_load_check): *d_status = padding error | flag mismatch << 1.
cudaError_t launch_load_check(const uint32_t* d_kf, const uint8_t* d_expect, uint32_t n, uint32_t* d_status,
                              cudaStream_t s);
cudaError_t launch_derive(const PrimeJob* d_jobs, const uint4* d_items, uint32_t nitems, const uint8_t* d_packed,
                          uint32_t* d_ext, uint32_t* d_killable, int keep_row0, cudaStream_t s);
// k_derive work items {job, first row, rows, 0} of <= kDeriveItemWords output words each
std::vector<uint4> derive_items(const std::vector<uint32_t>& primes);

// Padding-bit check for uploaded tables (FormatError on nonzero padding).
cudaError_t launch_check_padding(const PrimeJob* d_jobs, uint32_t njobs, const uint8_t* d_packed,
                                 uint32_t* d_bad, cudaStream_t s);

constexpr uint32_t kCubeThreads = 256;
constexpr int kCubePairs = 4;  // (a,b) pairs per thread in k_cube
constexpr int kCubeF2Pairs = 16;  // (a,b) pairs per thread in k_cube_f2 (two per FFMA2)
#ifndef CGPU_CUBE_SCALAR
#define CGPU_CUBE_SCALAR 0
#endif
constexpr int kCubeF2Scalar = CGPU_CUBE_SCALAR;  // of them evaluated with scalar FFMA (fmalite or fmaheavy)
constexpr uint32_t kCubeF2MaxR = 2039;  // largest prime with h + 4h^2 < 2^22, h = (r-1)/2
constexpr uint32_t kPermThreads = 256;
constexpr uint32_t kRow1Threads = 128;
// 128 threads x <= 32 registers = 4096 registers per CTA: exactly what a
// resident sieve CTA (768 x 80 = 61440 of 65536) leaves free, so the next
// load's layout kernels run beside a sieve still in flight (the e2e pipeline)
constexpr uint32_t kDeriveThreads = 128;
constexpr uint32_t kDeriveMinBlocks = 16;
constexpr uint32_t kDeriveItemWords = 2048;  // output words per k_derive CTA

// ---- K2: sieve ---------------------------------------------------------------

// One 24-warp CTA per SM (80 registers x 768 threads). Measured against
// three 8-warp CTAs per SM: the warp schedulers favour the SM's oldest CTA,
// so with a static split the younger CTAs' warps finish last and the SM
// runs its tail at a third of its warps (C5: 3.34 -> 3.04 ms).
#ifndef CGPU_SIEVE_THREADS
#define CGPU_SIEVE_THREADS 768
#endif
constexpr int kSieveThreads = CGPU_SIEVE_THREADS;
#ifndef CGPU_SIEVE_MIN_BLOCKS
#define CGPU_SIEVE_MIN_BLOCKS 1
#endif
constexpr int kSieveMinBlocks = CGPU_SIEVE_MIN_BLOCKS;  // CTAs per SM the register budget targets
// Launches whose mean row has fewer windows run the short-row kernel variant
// (dispatch_row SHORT): C4's rows average 1.6k windows, C5's 6.3k.
constexpr uint32_t kShortRowWindows = 4000;
constexpr uint32_t kDefaultRowCostShort = 650;  // ... for the short-row kernel (sweep: C4 0.528 -> 0.521 ms)
constexpr uint32_t kDefaultRowCost = 800;                 // window-equivalents per row setup (measured: 500 -> 800 C4 -2%, C5 -0.5%)
constexpr int kSieveWarps = kSieveThreads / 32;
constexpr int kMaxReg2 = 8;     // leading probes held in registers with r <= 31 (2-word rows)
constexpr int kMaxReg3 = 4;     // then with 31 < r <= 63 (3-word rows), after all of 11..31
constexpr int kMaxReg = kMaxReg2 + kMaxReg3;
constexpr int kMaxFactors = 9;  // distinct prime factors of p < 2^32
#ifndef CGPU_TAB_PROBES
#define CGPU_TAB_PROBES 8
#endif
constexpr int kTabProbes = CGPU_TAB_PROBES;  // leading register probes read from a window table
#ifndef CGPU_STD_REG3
#define CGPU_STD_REG3 1
#endif
constexpr int kStdReg3 = CGPU_STD_REG3;  // 3-word register probes of the standard sets (measured best: 1)
__host__ __device__ constexpr uint32_t std_prime(int j)
{
	return j == 0 ? 11 : j == 1 ? 13 : j == 2 ? 17 : j == 3 ? 19 : j == 4 ? 23 : j == 5 ? 29 : j == 6 ? 31
	     : j == 7 ? 37 : j == 8 ? 41 : j == 9 ? 43 : 47;
}
__host__ __device__ constexpr uint32_t std_tab_entries(int j)
{
	return j <= 0 ? 0 : std_tab_entries(j - 1) + std_prime(j - 1) * std_prime(j - 1);
}
// Window tables of the table probes, all rows: sum over them of r^2 entries.
// Standard sets: 11..37 need 4640. Other sets are admitted up to
// kTabStrideGen (the host stops adding 3-word probes at that bound); any
// 8 table probes fit (11..31 and one prime below 64: 3271 + 61^2 = 6992).
constexpr uint32_t kTabStrideStd = std_tab_entries(7 + kStdReg3 < kTabProbes ? 7 + kStdReg3 : kTabProbes);
constexpr uint32_t kTabStrideGen = kTabStrideStd > 7424 ? kTabStrideStd : 7424;
constexpr int kQueue = 64;      // per-warp deep-probe work queue entries
constexpr uint32_t kPlanChunk = 1024;  // row slots per plan CTA
// per row slot: nf | even << 8 | window-weight shift << 16, the odd factors,
// then their Barrett constants
constexpr uint32_t kFacWords = 1 + 2 * kMaxFactors;
constexpr float kDefaultDrainAlpha = 12.0f;

// ---- K2w: the wheel sieve (k_wsieve), standard probe sets ----------------------
// The first three probes (11, 13, 17) are not probed per window: only the
// residue classes of q mod 2431 that all three leave alive are visited at all
// (3 * 9 * 5 = 135 of 2431 for a canonical row), as 32-bit windows of stride 2431
// (bit i = q0 + 2431 i), and their first kills are counted analytically. The
// other five register probes (19..37) read strided window tables.
constexpr uint32_t kWheelM = 2431;                 // 11 * 13 * 17
constexpr uint32_t kWheelChunk = 32 * kWheelM;     // q covered by one window of every class
constexpr uint32_t kWheelDivMul = 1766750;         // floor(x / 2431) = umulhi(x, .) for x < 2^20
constexpr uint32_t kWheelE143 = 1717, kWheelE17 = 715;  // CRT idempotents mod 2431 of (143, 17)
constexpr int kWheelFirst = 3;                     // register probes 0..2 are the wheel
constexpr int kWheelReg = 8;                       // register probes of the standard sets (11..37)
constexpr uint32_t kWheelMidMax = 37681;           // factors below: path "mid" (2 f^2 < 2^32 and f <= 31 M / 2)
// layout of the wheel tables (32-bit words; k_wheeltab builds, every CTA copies to shared memory)
constexpr uint32_t kWtKill = 0;      // [3][32] kill masks (bit b = u_r(a, b)) of the rows of 11, 13, 17
constexpr uint32_t kWtB11 = 96;      // [11][11] entry (a, d): residues t mod 11 with (d t mod 11) alive in row a
constexpr uint32_t kWtRep11 = 224;   // [11][11][5] entry (a, d): B11(a, d) repeated with period 11 over 143 bits
constexpr uint32_t kWtRep13 = 832;   // [13][13][5] likewise for 13 (bits >= 143 zero in both)
constexpr uint32_t kWtNinv143 = 1680;  // [143] x -> (-x^-1) mod 143 (0 where gcd > 1)
constexpr uint32_t kWtNinv17 = 1824;   // [17]  x -> (-x^-1) mod 17
constexpr uint32_t kWtTinyOff = 1856;  // [32] f -> word offset of the tiny-factor masks of f (f < 32 prime, not 11, 13, 17)
constexpr uint32_t kWtTiny = 1888;     // masks (f, t), t < 2f: bits i with f | t + 2431 i   (234 words)
constexpr uint32_t kWtTab = 2144;    // strided window tables of 19..37: entry (j, a, b), b < 2r:
                                     // bit i = u_r(a, (b + 2431 i) mod r)
// first entry of register probe j >= kWheelFirst. Written without recursion: nvcc evaluated the
// recursive form at run time (CALL + local-memory frames, 8% of k_wsieve's instructions).
__host__ __device__ constexpr uint32_t wheel_tab_sq(int j) { return 2 * std_prime(j) * std_prime(j); }
__host__ __device__ constexpr uint32_t wheel_tab_base(int j)
{
	return kWtTab + (j > 3 ? wheel_tab_sq(3) : 0) + (j > 4 ? wheel_tab_sq(4) : 0) + (j > 5 ? wheel_tab_sq(5) : 0) +
	       (j > 6 ? wheel_tab_sq(6) : 0) + (j > 7 ? wheel_tab_sq(7) : 0);
}
static_assert(kWheelFirst == 3 && kWheelReg == 8, "wheel_tab_base lists the table probes 3..7");
constexpr uint32_t kWtWords = wheel_tab_base(kWheelReg);
constexpr uint32_t kWtBytes = (4 * kWtWords + 15) / 16 * 16;  // the per-warp blocks after them stay 16-byte aligned
#ifndef CGPU_WHEEL_THREADS
#define CGPU_WHEEL_THREADS 1024
#endif
constexpr int kWheelThreads = CGPU_WHEEL_THREADS;  // one 32-warp CTA per SM at 64 registers (768 x 80: C5 1.66 ms,
                                                   // 896 x 72: 1.64, 1024 x 64: 1.57 -- the loop is latency-bound)
constexpr int kWheelWarps = kWheelThreads / 32;
constexpr int kWheelQueue = 64;      // per-warp queue of single q alive after the register probes
#ifndef CGPU_WHEEL_CLS
#define CGPU_WHEEL_CLS 1216
#endif
constexpr uint32_t kWheelCls = CGPU_WHEEL_CLS;  // per-warp list of alive classes (uint16 offsets below 2431), one batch
// k_wsieve's load-balance model (k_plan), in instructions, from the ncu instruction counts of C5:
// per row segment, then per loop iteration {base, per factor below 37681, per factor above}, per queued q
// per-warp shared-memory block of k_wsieve (byte offsets): deep-probe rows, loop factors, the q
// queue, the two alive-offset lists, the class list of the current batch, the first-kill counters
constexpr uint32_t kWbFac = 16 * 8;                          // after uint4 deep[kDeepPrefetch = 8]
constexpr uint32_t kWbQueue = kWbFac + 16 * kMaxFactors;
constexpr uint32_t kWbLists = kWbQueue + 4 * kWheelQueue;
constexpr uint32_t kWbCls = kWbLists + 2 * 192 + 4 * 12;     // lists, then every odd factor (uint32 x kMaxFactors, padded)
constexpr uint32_t kWbHist = (kWbCls + 2 * kWheelCls + 15) / 16 * 16;
__host__ __device__ constexpr uint32_t wheel_warp_bytes(uint32_t np) { return (kWbHist + 4 * np + 15) / 16 * 16; }
constexpr uint32_t kDefaultRowCostWheel = 130000;  // units of 1/64 instruction (~2000 instructions; sweeps r02w/r02x)
// launches whose mean row has fewer 32-q windows keep k_sieve (TRIANGLE p <= 3e4, mean 470: k_sieve 0.097 ms,
// k_wsieve 0.117; p <= 5e4, mean 780: 0.189 / 0.175; C4, mean 1.6k: 0.52 / 0.33; C5, mean 6.3k: 3.02 / 1.10)
constexpr uint32_t kWheelMinWindows = 650;
constexpr float kDefaultWheelCost[4] = {140.0f, 14.0f, 30.0f, 25.0f};

struct SieveArgs {
	const uint32_t* ext;          // row-extended tables
	uint64_t ext_words;           // (debug bounds checks)
	uint64_t n_blocks;            // block_rmax entries (debug bounds checks)
	const uint4* probes;          // per probe j: {r, m, ext_base, S}
	uint32_t np;                  // probes (killable tables, rank order)
	uint32_t nreg;                // leading probes held in registers (nreg2 + nreg3)
	uint32_t nreg2, nreg3;
	bool std_primes;              // register probes are exactly 11..31, 37 (immediates)
	uint32_t reg_r[kMaxReg], reg_m[kMaxReg], reg_base[kMaxReg], reg_delta[kMaxReg];
	uint32_t reg_tab[kMaxReg];    // first window-table entry of table probe j (prefix sum of r^2)
	uint32_t wtab_n;              // window-table entries (0: no table probes)
	const uint32_t* wintab;       // [2][stride]: entry (j, a, b) = mask of row a at offset b, then
	                              // the successor entry index (a, (b + 1024) mod r)
	const uint2* fprimes;         // {f, barrett m} primes < 2^16 for trial division
	uint32_t n_fprimes;
	// row slots: slot s -> owned block ordinal s/100, p = (blk0 + ord*G)*100 + s%100
	uint64_t p_lo, p_hi, q_start;
	uint64_t q_end;               // REGION: last q of row p_hi (0 = the whole row)
	int mode;
	uint32_t G;
	uint64_t blk0;                // first owned block of this launch
	uint32_t n_slots;
	uint32_t row_cost;            // load-balance charge per row (window-equivalents)
	float drain_alpha;            // load-balance weight of a window queued for the deep probes
	uint32_t short_rows;          // run the short-row loop-variant set (standard-prime kernel)
	// work units before slot s = prefix[s] + chunk_off[s / kPlanChunk]
	unsigned long long* prefix;        // [n_slots + 1] (chunk-local exclusive scan)
	unsigned long long* chunk_off;     // [n_chunks + 1] (exclusive scan of chunk totals)
	uint32_t g;                   // shard index (block b is owned when b % G == g)
	uint32_t init;                // k_plan: zero hist/counters and initialise block_rmax first
	uint32_t* tickets;                 // [2] last-CTA tickets (plan, sieve), zeroed per launch
	uint32_t* rowfac;                  // [n_slots][kFacWords] row factorisations (k_plan)
	// outputs
	unsigned long long* hist;          // [n primes] first-killer counts by rank
	uint32_t nprimes;
	const uint32_t* probe_rank;        // [np] rank of probe j
	unsigned long long* counters;      // [0] pairs_tested, [1] survivors
	uint32_t* block_rmax;              // [p/100 - blk_lo]
	uint64_t blk_lo;
	unsigned long long* surv;          // (p << 32) | q
	unsigned long long surv_cap;
	// cooperative stop (engine.hpp:248-257): a mapped host word; when nonzero
	// the sieve's warps abandon their remaining rows (checked every 8th row
	// slot) and the launch's results are incomplete -- the caller discards
	// them and re-sieves exactly up to the reference's next stop point
	const volatile uint32_t* stop;
	// wheel sieve (k_wsieve): 0 = k_sieve; tables from k_wheeltab
	uint32_t wheel;
	const uint32_t* wheeltab;          // [kWtWords]
	float wheel_cost[4];               // load-balance model (kDefaultWheelCost)
};

cudaError_t launch_plan(const SieveArgs& a, cudaStream_t s);
cudaError_t launch_sieve(const SieveArgs& a, int grid, cudaStream_t s);
int sieve_grid(int device, int nr2, int nr3, bool std_primes, size_t smem_bytes);
int wsieve_grid(int device, size_t smem_bytes);
__host__ __device__ size_t wsieve_smem_bytes(uint32_t np);
// wheel tables from the row-extended layout; reg_base[j] = ext word offset of register probe j
cudaError_t launch_wheeltab(const uint32_t* d_ext, const uint32_t* reg_base, uint32_t* d_out, cudaStream_t s);
__host__ __device__ size_t sieve_smem_bytes(uint32_t np, uint32_t tab_stride);
__host__ __device__ inline uint32_t plan_chunks(uint32_t n_slots) { return (n_slots + kPlanChunk - 1) / kPlanChunk; }

cudaError_t launch_init_blocks(uint32_t* d_block_rmax, uint64_t nblocks, uint64_t blk_lo,
                               uint32_t G, uint32_t g, cudaStream_t s);

// K3: first-killer rank for explicit pairs.
cudaError_t launch_classify(const uint64_t* d_pq, uint64_t n, const uint8_t* d_packed,
                            const uint32_t* d_primes, const uint32_t* d_offsets, uint32_t nprimes,
                            int32_t* d_out, cudaStream_t s);

// INT32 pipe peaks (peak.cu), thread-ops/s: {LOP3-only, IMAD-only,
// IMAD+LOP3 3-register, IMAD+LOP3 immediate forms}.
cudaError_t run_int_peak(int device, double out[4]);
// FP32 pipes (peak.cu): {FFMA2 lane-FMAs/s, k_cube_f2 evaluation-mix evals/s}.
cudaError_t run_fp_peak(int device, double out[2]);

}  // namespace cgpu
