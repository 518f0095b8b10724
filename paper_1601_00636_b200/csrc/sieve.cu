// K2: the (p,q) pair sieve for sm_100a, and K3 (classify).
//
// Replaces the inner loops of scan() (/root/reference/proj/include/cuboid/
// engine.hpp:225-284) and the TRIANGLE loop of verify_small_region
// (engine.hpp:613-625). Semantics, bit for bit:
//   * candidates: q in the row bounds, q != p, gcd(p, q) == 1 (engine.hpp:258);
//   * probes in rank order, first set bit u_r(p mod r, q mod r) kills
//     (engine.hpp:261-269); the first killer is histogrammed by rank;
//   * every candidate is killed or survives, so pairs_tested = sum(hist) +
//     survivors (engine.hpp:259-277) -- the kernel never counts pairs apart;
//   * survivors are emitted as (p << 32) | q and sorted on the host;
//   * per p/100 block, the largest killing prime (1 if none) (:229-236, 271).
//
// Design: bit-sliced. One lane owns a 32-wide window of
// consecutive q in one row p; a probe for prime r is ONE funnel shift of the
// row-extended table (row p mod r, starting at bit q0 mod r), so one probe
// answers 32 pairs. Warps own contiguous slices of the linearised
// (row, window) space, balanced by k_plan, which also factorises every p
// (segmented sieve); coprimality is then one periodic bit pattern per odd
// prime factor (the window loop is specialised on the factor count) plus a
// constant mask for f = 2. The leading probe primes (11..31, and the first in
// (31, 63]) are read from window tables resident in the CTA's shared memory
// for every row (each entry: the 32-q mask at one offset of one row, and a
// pointer to the lane's next entry), so a probe costs two LDS and no ALU work
// on offsets; they count their first kills by telescoping popcounts. One
// 24-warp CTA per SM. Windows still alive after them (a few percent) are
// pushed to a per-warp queue in shared memory and probed against the deep
// tables 32 at a time, one per lane, so the rare deep probes run at full SIMD
// width. Tables that never kill (all-zero, e.g. r = 3, 5, 7) are not probed --
// identical results.

#include <cuda/std/type_traits>

#include "../../include/cuboid_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace cgpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kStepQ = 32 * 32;  // q advance per warp iteration per lane
constexpr uint32_t kDeepPrefetch = 8;  // deep probes whose rows are prefetched per row

// The register probes of every BASELINE set and of the reference default
// (sievetable.hpp:178-179): 11..31 and 37. For them the kernel is compiled with
// the primes, their Barrett constants and per-iteration offset steps as
// immediates, so the window loop loads nothing from the constant bank.
__host__ __device__ constexpr uint32_t std_prime(int j)
{
	return j == 0 ? 11 : j == 1 ? 13 : j == 2 ? 17 : j == 3 ? 19 : j == 4 ? 23 : j == 5 ? 29 : j == 6 ? 31 : 37;
}

template <bool STD>
__device__ __forceinline__ uint32_t reg_prime(const SieveArgs& a, int j)
{
	return STD ? std_prime(j) : a.reg_r[j];
}

template <bool STD>
__device__ __forceinline__ uint32_t reg_barrett(const SieveArgs& a, int j)
{
	return STD ? static_cast<uint32_t>((1ull << 32) / std_prime(j)) : a.reg_m[j];
}

template <bool STD>
__device__ __forceinline__ uint32_t reg_step(const SieveArgs& a, int j)
{
	return STD ? (kStepQ % std_prime(j)) : a.reg_delta[j];
}

// least q >= 1 with 9 q^3 >= p (region.hpp:25-39) / q_bounds (region.hpp:49-63)
__device__ __forceinline__ uint64_t q_low_dev(uint64_t p)
{
	if (p < kRegionCrossover) {
		const uint64_t c = (p + 58) / 59;
		return c < 1 ? 1 : c;
	}
	uint64_t q = static_cast<uint64_t>(cbrt(static_cast<double>(p) / 9.0));
	if (q < 1) q = 1;
	while (q > 1 && 9 * (q - 1) * (q - 1) * (q - 1) >= p) --q;
	while (9 * q * q * q < p) ++q;
	return q;
}

struct RowBounds {
	uint64_t p;
	uint64_t qlo, qhi;  // inclusive; empty when qlo > qhi
};

__device__ __forceinline__ RowBounds slot_row(const SieveArgs& a, uint32_t s)
{
	RowBounds b;
	const uint64_t blk = a.blk0 + static_cast<uint64_t>(s / 100) * a.G;
	b.p = blk * 100 + s % 100;
	if (b.p < a.p_lo || b.p > a.p_hi || b.p == 0) {
		b.qlo = 1;
		b.qhi = 0;
		return b;
	}
	if (a.mode == CGPU_TRIANGLE) {
		b.qlo = 1;
		b.qhi = b.p - 1;
	} else {
		b.qlo = q_low_dev(b.p);
		b.qhi = 59 * b.p;
		if (b.p == a.p_lo && a.q_start) b.qlo = a.q_start;
		if (b.p == a.p_hi && a.q_end && a.q_end < b.qhi) b.qhi = a.q_end;  // a span ending mid-row
		// q == p is skipped (engine.hpp:258); for p > 1 the coprimality mask
		// removes it, for p = 1 (q_low = 1) start the row at q = 2
		if (b.p == 1 && b.qlo == 1) b.qlo = 2;
	}
	return b;
}

__device__ __forceinline__ uint64_t row_windows(const RowBounds& b)
{
	return b.qhi >= b.qlo ? (b.qhi - b.qlo + 32) / 32 : 0;
}

// Work units of a row for load balancing: its 32-q windows plus a fixed
// charge a.row_cost for the per-row setup (factor masks, register-probe rows,
// the row-end queue drain and counts). Without it the warps that own the many
// short rows at small p straggle (C4: one SM busy 5x longer than the rest).
//
// Windows are weighted by the expected share queued for the deep probes: the
// register probes kill a fixed fraction k_j of any row's pairs except when
// r_j | p (row 0 never kills), so rows that several of 11..37 divide keep up
// to ~100x more survivors (C5: median s = 3.3e-4 alive after the register
// probes, max 3.7e-2) and drain most of their windows. Unweighted, the warps
// that drew such a row ran on alone for up to +50% -- the whole tail of a
// launch with few rows per warp (a shard of 8 ranks). Weight = 1 + alpha
// (1 - exp(-c s)) (c = the window's coprime candidates, alpha =
// a.drain_alpha window-equivalents per queued window), rounded to a power of
// two 2^shift (shift <= 3, stored in the row's factor head) so that mapping
// units back to windows is a shift.
__device__ __forceinline__ uint64_t row_units(const SieveArgs& a, const RowBounds& b, uint32_t shift)
{
	const uint64_t w = row_windows(b);
	// k_wsieve: `shift` is the row's cost per window in units of 1/64 instruction (wheel_mult)
	if (a.wheel) return w ? a.row_cost + w * shift : 0;
	return w ? a.row_cost + (w << shift) : 0;
}

// k_wsieve's inverse of row_units: first window of the row at unit u. Rows that lie wholly in a
// warp's slice (nearly all) take the shortcuts; only split rows divide.
__device__ __forceinline__ uint32_t unit_window_mult(const SieveArgs& a, unsigned long long u, uint32_t mult,
                                                     uint32_t windows)
{
	if (u <= a.row_cost) return 0;
	const unsigned long long x = u - a.row_cost;
	if (x >= static_cast<unsigned long long>(windows) * mult) return windows;
	return static_cast<uint32_t>((x + mult - 1) / mult);
}

// First window of the row at unit u (the inverse of row_units; monotonic, so
// adjacent warps' unit slices map to adjacent window ranges).
__device__ __forceinline__ uint32_t unit_window(const SieveArgs& a, unsigned long long u, uint32_t shift,
                                                uint32_t windows)
{
	if (u <= a.row_cost) return 0;
	const unsigned long long w = (u - a.row_cost + (1u << shift) - 1) >> shift;
	return static_cast<uint32_t>(w < windows ? w : windows);
}

__device__ __forceinline__ unsigned long long slot_prefix(const SieveArgs& a, uint32_t s)
{
	return a.prefix[s] + a.chunk_off[s / kPlanChunk];
}

// Block-wide exclusive scan of one value per thread (blockDim.x == 1024).
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* s_warp,
                                                              unsigned long long& total)
{
	const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
	unsigned long long x = v;
#pragma unroll
	for (int d = 1; d < 32; d <<= 1) {
		const unsigned long long y = __shfl_up_sync(kFull, x, d);
		if (lane >= d) x += y;
	}
	if (lane == 31) s_warp[wid] = x;
	__syncthreads();
	if (wid == 0) {
		unsigned long long y = s_warp[lane];
#pragma unroll
		for (int d = 1; d < 32; d <<= 1) {
			const unsigned long long z = __shfl_up_sync(kFull, y, d);
			if (lane >= d) y += z;
		}
		s_warp[lane] = y;  // inclusive over warps
	}
	__syncthreads();
	total = s_warp[31];
	return x - v + (wid ? s_warp[wid - 1] : 0);
}

// Distinct prime factors of the CTA's rows for the sieve's coprimality masks,
// by a segmented sieve in shared memory instead of per-row trial division
// (which left every warp waiting on its slowest, prime, row: ~100 dependent
// Barrett steps). Slots come in runs of 100 consecutive rows (one p/100
// block each); one thread per (prime f <= sqrt(p_max), run) marks the
// multiples of f, then each row divides its marked primes out and what is
// left of p is 1 or its single prime factor above sqrt(p). Output per slot:
// out[0] = nf | even << 8, out[1..nf] = the odd prime factors that can divide
// some q of the row (<= qhi), ascending, out[1 + kMaxFactors + i] = the
// Barrett constant of factor i. Empty rows get nf = 0.
struct PlanSmem {
	float kill[kMaxReg];  // kill fraction of a nonzero row of register probe j
	uint32_t nf[kPlanChunk];
	uint16_t fi[kPlanChunk][kMaxFactors];  // indices into a.fprimes
};

__device__ __forceinline__ uint32_t factorise_chunk(const SieveArgs& a, PlanSmem& sm, uint32_t c0,
                                                    const RowBounds& rb, uint32_t* out)
{
	const uint32_t t = threadIdx.x;
	sm.nf[t] = 0;
	if (t < a.nreg) {  // row 1 of the probe (canonical rows a >= 1 share its popcount)
		const uint32_t r = a.reg_r[t], S = ext_row_words(r);
		const uint32_t* row = a.ext + a.reg_base[t] + S;
		const uint32_t lo = r < 32 ? (1u << r) - 1 : 0xffffffffu;
		const uint32_t n = __popc(row[0] & lo) + (r > 32 ? __popc(row[1] & ((1u << (r - 32)) - 1)) : 0);
		sm.kill[t] = static_cast<float>(n) / static_cast<float>(r);
	}
	// largest row of the chunk (slots ascend in p)
	const uint32_t s_last = min(c0 + kPlanChunk, a.n_slots) - 1;
	const uint64_t p_last = (a.blk0 + static_cast<uint64_t>(s_last / 100) * a.G) * 100 + s_last % 100;
	__syncthreads();
	const uint32_t run0 = c0 / 100, nrun = s_last / 100 - run0 + 1;
	for (uint32_t w = t;; w += kPlanChunk) {
		const uint32_t i = w / nrun, k = run0 + w % nrun;
		if (i >= a.n_fprimes) break;
		const uint2 fp = __ldg(a.fprimes + i);
		if (static_cast<uint64_t>(fp.x) * fp.x > p_last) break;  // i ascends with w
		const uint32_t sa = max(c0, 100 * k), sb = min(s_last + 1, 100 * k + 100);  // slots of run k
		const uint64_t P = (a.blk0 + static_cast<uint64_t>(k) * a.G) * 100;        // row of slot 100k
		const uint32_t pa = static_cast<uint32_t>(P + (sa - 100 * k));              // p < 2^32
		uint32_t rem = pa - __umulhi(pa, fp.y) * fp.x;
		if (rem >= fp.x) rem -= fp.x;
		for (uint32_t sl = sa + (rem ? fp.x - rem : 0); sl < sb; sl += fp.x) {
			const uint32_t j = atomicAdd(&sm.nf[sl - c0], 1u);
			if (j < kMaxFactors) sm.fi[sl - c0][j] = static_cast<uint16_t>(i);
		}
	}
	__syncthreads();
	if (c0 + t >= a.n_slots) return 0;
	uint32_t nf = 0, even = 0;
	// gathered while the factors are found (re-reading them from `out` afterwards waited on global memory):
	// the coprime share of the odd factors, and k_wsieve's loop factors by path
	float cop_odd = 1.0f;
	uint32_t nmid = 0, nlarge = 0;
	auto note_factor = [&](uint32_t f) {
		cop_odd -= cop_odd * __frcp_rn(static_cast<float>(f));
		if (f == a.reg_r[0] || f == a.reg_r[1] || f == a.reg_r[2]) return;  // the wheel primes drop classes instead
		if (f < kWheelMidMax) ++nmid;
		else ++nlarge;
	};
	if (rb.qhi >= rb.qlo && rb.p > 1) {
		const uint32_t n = min(sm.nf[t], static_cast<uint32_t>(kMaxFactors));
		uint16_t f[kMaxFactors];
		for (uint32_t j = 0; j < n; ++j) {  // ascending (insertion sort, n <= 9)
			uint16_t v = sm.fi[t][j];
			uint32_t k = j;
			for (; k > 0 && f[k - 1] > v; --k) f[k] = f[k - 1];
			f[k] = v;
		}
		uint32_t cof = static_cast<uint32_t>(rb.p);
		for (uint32_t j = 0; j < n; ++j) {
			const uint2 fp = __ldg(a.fprimes + f[j]);
			for (;;) {  // divide f out of the cofactor
				uint32_t qt = __umulhi(cof, fp.y), r = cof - qt * fp.x;
				if (r >= fp.x) { r -= fp.x; ++qt; }
				if (r) break;
				cof = qt;
			}
			if (fp.x == 2) {
				even = 1;
			} else if (fp.x <= rb.qhi && nf < kMaxFactors) {
				out[1 + kMaxFactors + nf] = fp.y;
				out[1 + nf++] = fp.x;
				note_factor(fp.x);
			}
		}
		if (cof > 1) {  // the prime factor above sqrt(p)
			if (cof == 2) {
				even = 1;
			} else if (cof <= rb.qhi && nf < kMaxFactors) {
				out[1 + kMaxFactors + nf] = static_cast<uint32_t>((1ull << 32) / cof);
				out[1 + nf++] = cof;
				note_factor(cof);
			}
		}
	}
	out[0] = nf | (even << 8);
	// window weight (row_units): survival after the register probes that do
	// not divide p, times the row's coprime candidates per window
	float surv = 1.0f;
	const float cop = (even ? 0.5f : 1.0f) * cop_odd;
	const uint32_t p32 = static_cast<uint32_t>(rb.p);
	for (uint32_t j = 0; j < a.nreg; ++j)
		if (mod_full(p32, a.reg_r[j], a.reg_m[j])) surv *= 1.0f - sm.kill[j];
	if (a.wheel) {
		// k_wsieve: instructions of the row's loop = iterations x (base + per factor) + queued q x
		// drain cost, spread over the row's windows in units of 1/64 instruction (16 bits). The
		// iterations step with the row length (one more window per class every 77792 q) and with
		// the alive classes of q mod 2431 (the wheel primes that divide p leave all but class 0).
		const uint64_t wn = row_windows(rb);
		uint32_t mult = 1;
		if (wn) {
			float classes = 1.0f;
			for (uint32_t j = 0; j < static_cast<uint32_t>(kWheelFirst); ++j) {
				const float r = static_cast<float>(a.reg_r[j]);
				classes *= mod_full(p32, a.reg_r[j], a.reg_m[j]) ? rintf(r * (1.0f - sm.kill[j])) : r - 1.0f;
			}
			const float q = static_cast<float>(wn) * 32.0f;
			const float nchunk = floorf((q - 1.0f) * (1.0f / kWheelChunk)) + 1.0f;
			const float iters = ceilf(classes * nchunk * (1.0f / 32.0f)) + 1.0f;
			const float cost = iters * (a.wheel_cost[0] + a.wheel_cost[1] * nmid + a.wheel_cost[2] * nlarge) +
			                   q * cop * surv * a.wheel_cost[3];
			mult = static_cast<uint32_t>(fminf(fmaxf(rintf(64.0f * cost / static_cast<float>(wn)), 1.0f), 65535.0f));
		}
		out[0] |= mult << 16;
		return mult;
	}
	const float wt = 1.0f + a.drain_alpha * (1.0f - __expf(-32.0f * cop * surv));
	const uint32_t shift = wt >= 6.0f ? 3u : wt >= 3.0f ? 2u : wt >= 1.5f ? 1u : 0u;
	out[0] |= shift << 16;
	return shift;
}

// Plan: per row slot, the work units before it. Each CTA scans kPlanChunk
// slots; the last CTA to finish scans the chunk totals.
__global__ void __launch_bounds__(kPlanChunk) k_plan(const SieveArgs a)
{
	__shared__ unsigned long long s_warp[32];
	__shared__ bool s_last;
	__shared__ PlanSmem s_fac;
	const uint32_t n = a.n_slots;
	const uint32_t s = blockIdx.x * kPlanChunk + threadIdx.x;
	if (a.init) {  // first plan of a scan: the sieve's outputs start from zero / owned blocks at 1
		const uint64_t nt = static_cast<uint64_t>(gridDim.x) * kPlanChunk;
		for (uint64_t i = s; i < a.n_blocks; i += nt) a.block_rmax[i] = ((a.blk_lo + i) % a.G == a.g) ? 1u : 0u;
		for (uint64_t i = s; i < a.nprimes; i += nt) a.hist[i] = 0;
		if (s < 2) a.counters[s] = 0;
	}
	const RowBounds rb = s < n ? slot_row(a, s) : RowBounds{0, 1, 0};
	const uint32_t shift = factorise_chunk(a, s_fac, blockIdx.x * kPlanChunk, rb,
	                                       a.rowfac + static_cast<size_t>(s) * kFacWords);
	const unsigned long long u = s < n ? row_units(a, rb, shift) : 0;
	unsigned long long total;
	const unsigned long long ex = block_excl_scan(u, s_warp, total);
	if (s < n) a.prefix[s] = ex;
	if (s == n - 1) a.prefix[n] = (n % kPlanChunk) ? ex + u : 0;
	if (threadIdx.x == 0) a.chunk_off[blockIdx.x] = total;
	__threadfence();
	__syncthreads();
	if (threadIdx.x == 0) s_last = atomicAdd(&a.tickets[0], 1u) == gridDim.x - 1;
	__syncthreads();
	if (!s_last) return;
	__threadfence();
	const uint32_t nc = gridDim.x;  // <= kPlanChunk (kMaxSlots / kPlanChunk)
	const unsigned long long v =
	    threadIdx.x < nc ? *reinterpret_cast<volatile unsigned long long*>(a.chunk_off + threadIdx.x) : 0;
	__syncthreads();
	const unsigned long long cex = block_excl_scan(v, s_warp, total);
	if (threadIdx.x < nc) a.chunk_off[threadIdx.x] = cex;
	if (threadIdx.x == 0) {
		a.chunk_off[nc] = total;
		a.tickets[0] = 0;  // ready for the next launch on this stream
	}
}

// period_mask(f) for f < 32 (bits at 0, f, 2f, ...): read by a whole warp
// at one index (the row's factor), so the constant bank broadcasts it
__constant__ uint32_t c_period_mask[32] = {
    0u,          0xffffffffu, 0x55555555u, 0x49249249u, 0x11111111u, 0x42108421u, 0x41041041u, 0x10204081u,
    0x01010101u, 0x08040201u, 0x40100401u, 0x00400801u, 0x01001001u, 0x04002001u, 0x10004001u, 0x40008001u,
    0x00010001u, 0x00020001u, 0x00040001u, 0x00080001u, 0x00100001u, 0x00200001u, 0x00400001u, 0x00800001u,
    0x01000001u, 0x02000001u, 0x04000001u, 0x08000001u, 0x10000001u, 0x20000001u, 0x40000001u, 0x80000001u};

#ifdef CGPU_DEBUG
__device__ __forceinline__ uint32_t dynamic_smem_size()
{
	uint32_t v;
	asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
	return v;
}
#endif

__device__ __forceinline__ uint32_t warp_sum(uint32_t v)
{
	return __reduce_add_sync(kFull, v);
}

// Per-warp first-kill counters in shared memory are 32-bit; a wrap is carried
// to the 64-bit global histogram by the lane that caused it (lane 0 only).
__device__ __forceinline__ void hist_add(const SieveArgs& a, uint32_t* h, uint32_t j, uint32_t c)
{
	const uint32_t old = h[j];
	const uint32_t nw = old + c;
	h[j] = nw;
	if (nw < old) atomicAdd(&a.hist[__ldg(a.probe_rank + j)], 1ull << 32);
}

struct WarpSmem {
	uint2* queue;    // [kQueue] windows alive after the register probes: {q0, alive}
	uint32_t* hist;  // [np] first-kill counts of this warp
	uint4* deep;     // [kDeepPrefetch] first deep probes of the current row: {row base, r, m, -}
	uint32_t tab0;   // shared address of the CTA's window tables (masks; successors TS words on)
};

// Warp-aggregated survivor output: one atomic per warp.
__device__ __forceinline__ void emit_survivors(const SieveArgs& a, uint32_t lane, uint32_t p,
                                               uint32_t q0, uint32_t alive)
{
	if (!__any_sync(kFull, alive)) return;
	const uint32_t n = __popc(alive);
	uint32_t x = n;
#pragma unroll
	for (int d = 1; d < 32; d <<= 1) {
		const uint32_t y = __shfl_up_sync(kFull, x, d);
		if (lane >= d) x += y;
	}
	const uint32_t total = __shfl_sync(kFull, x, 31);
	unsigned long long base = 0;
	if (lane == 31) base = atomicAdd(&a.counters[1], static_cast<unsigned long long>(total));
	base = __shfl_sync(kFull, base, 31) + (x - n);
	while (alive) {
		const uint32_t bit = __ffs(alive) - 1;
		alive &= alive - 1;
		if (base < a.surv_cap) a.surv[base] = (static_cast<unsigned long long>(p) << 32) | (q0 + bit);
		++base;
	}
}

// Probes queue entries [base, base + n) (n <= 32, one per lane) against the
// deep tables in rank order; the lanes step through the probes together and
// leave as soon as every entry is dead. kmax = 1 + deepest killing probe.
// Returns the number of candidates that entered (warp-uniform).
template <int NREG>
__device__ __forceinline__ uint32_t drain(const SieveArgs& a, const WarpSmem& w, uint32_t lane,
                                          uint32_t base, uint32_t n, uint32_t p, uint32_t& kmax)
{
	uint32_t q0 = 0, alive = 0;
	if (lane < n) {
		const uint2 e = w.queue[base + lane];
		q0 = e.x;
		alive = e.y;
	}
	const uint32_t entered = warp_sum(__popc(alive));
	for (uint32_t j = NREG; j < a.np; ++j) {
		if (!__any_sync(kFull, alive)) break;
		uint32_t c = 0;
		if (alive) {
			// probe j = {r, m, ext_base, S}; row p mod r of its ext table (the
			// first kDeepPrefetch were resolved at row setup)
			uint32_t row, r, m;
			if (j - NREG < kDeepPrefetch) {
				const uint4 e = w.deep[j - NREG];
				row = e.x;
				r = e.y;
				m = e.z;
			} else {
				const uint4 d = __ldg(a.probes + j);
				row = d.z + mod_full(p, d.x, d.y) * d.w;
				r = d.x;
				m = d.y;
			}
			const uint32_t b = mod_full(q0, r, m);
			const uint32_t* wp = a.ext + row + (b >> 5);
			CGPU_CHECK(row + (b >> 5) + 1 < a.ext_words);
			const uint32_t M = __funnelshift_r(__ldg(wp), __ldg(wp + 1), b);
			const uint32_t k = alive & M;
			alive ^= k;
			c = __popc(k);
		}
		c = warp_sum(c);
		if (c) {
			kmax = max(kmax, j + 1);
			if (lane == 0) hist_add(a, w.hist, j, c);
		}
	}
	emit_survivors(a, lane, p, q0, alive);
	return entered;
}

// Row context handed to the specialised window loop.
struct RowCtx {
	uint32_t p, qlo, qhi, w0, w1, wlast, tail, even;
	uint32_t nf;
	uint32_t fac[kMaxFactors];  // odd prime factors of p that can divide some q of the row
	uint32_t fm[kMaxFactors];   // their Barrett constants
};

// Warp-collective: the number of q in [qa, qb] coprime to p, by
// inclusion-exclusion over the prime factors of p that can divide some q of
// the row (odd ones in rc.fac, 2 when p is even); lanes split the subsets.
__device__ __forceinline__ uint32_t coprime_in(const RowCtx& rc, uint32_t lane, uint32_t qa, uint32_t qb)
{
	const uint32_t F = rc.nf + (rc.even ? 1u : 0u);
	long long part = 0;
	for (uint32_t sub = lane; sub < (1u << F); sub += 32) {
		uint64_t d = (rc.even && ((sub >> rc.nf) & 1)) ? 2 : 1;
		for (uint32_t i = 0; i < rc.nf; ++i)
			if ((sub >> i) & 1) d *= rc.fac[i];
		if (d > qb) continue;
		const uint32_t dd = static_cast<uint32_t>(d);
		const long long c = static_cast<long long>(qb / dd) - static_cast<long long>((qa - 1) / dd);
		part += (__popc(sub) & 1) ? -c : c;
	}
	for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
	return static_cast<uint32_t>(part);
}

// The window loop of one row segment, specialised on the number of odd prime
// factors NF so the coprimality masks cost exactly NF x 4 instructions.
// Returns 1 + the deepest probe that killed in this segment (0: none).
template <int NR2, int NR3, bool STD, int NF>
__device__ __forceinline__ uint32_t row_loop(const SieveArgs& a, const WarpSmem& w, uint32_t lane,
                                             const RowCtx& rc)
{
	constexpr int NREG = NR2 + NR3;  // register probes: NR2 with r <= 31, NR3 with 31 < r <= 63
	constexpr int NT = NREG < kTabProbes ? NREG : kTabProbes;  // probes read from the window tables
	constexpr uint32_t TS = STD ? kTabStrideStd : kTabStrideGen;
	// S[j] = sum over this lane's windows of popc(alive before register probe j);
	// probe j's first-kill count is S[j] - S[j+1] (telescoping: one LOP3 per
	// probe). S[0] (the candidates) is counted once per segment by
	// inclusion-exclusion over the prime factors of p, and S[NREG] only on the
	// rare path that queues a window -- 2 of 8 POPCs per window saved.
	uint32_t S[NREG + 1];
#pragma unroll
	for (int j = 0; j <= NREG; ++j) S[j] = 0;
	uint32_t kmax = 0;
	const uint32_t q0_first = rc.qlo + 32 * (rc.w0 + lane);
	uint32_t fo[NF > 0 ? NF : 1], fd[NF > 0 ? NF : 1], fpat[NF > 0 ? NF : 1], ff[NF > 0 ? NF : 1];
#pragma unroll
	for (int k = 0; k < NF; ++k) {
		if (k < static_cast<int>(rc.nf)) {
			// Barrett remainders (the factor's constant from k_plan; f < 2^31 so
			// the lazy remainder stays below 2^32) and a constant-bank mask
			const uint32_t f = rc.fac[k], m = rc.fm[k];
			const uint32_t b = mod_full(q0_first, f, m);
			ff[k] = f;
			fo[k] = b ? f - b : 0;
			fd[k] = mod_full(kStepQ, f, m);
			fpat[k] = f < 32 ? c_period_mask[f] : 1u;
		} else {  // padding slot of a wider variant: contributes no bits
			ff[k] = 1;
			fo[k] = fd[k] = fpat[k] = 0;
		}
	}
	// Register probes j >= NT: the row's period-r pattern in registers; a probe
	// is a funnel shift at the lane's offset rb, advanced by 1024 mod r.
	// A row of r <= 31 is 2 words (64 bits >= r + 31), of 31 < r <= 63 three.
	uint32_t rw0[NREG > 0 ? NREG : 1], rw1[NREG > 0 ? NREG : 1], rb[NREG > 0 ? NREG : 1];
	uint32_t rw2[NR3 > 0 ? NR3 : 1];
#pragma unroll
	for (int j = NT; j < NREG; ++j) {
		const uint32_t r = reg_prime<STD>(a, j), m = reg_barrett<STD>(a, j);
		const uint32_t S = j < NR2 ? 2 : 3;
		const uint32_t row = a.reg_base[j] + mod_full(rc.p, r, m) * S;
		CGPU_CHECK(row + S - 1 < a.ext_words);
		rw0[j] = __ldg(a.ext + row);
		rw1[j] = __ldg(a.ext + row + 1);
		if (j >= NR2) rw2[j >= NR2 ? j - NR2 : 0] = __ldg(a.ext + row + 2);
		rb[j] = mod_full(q0_first, r, m);
	}
	// Register probes j < NT: the window tables of every row of these primes
	// are resident in the CTA's shared memory (copied once per launch). Entry
	// (j, a, b) holds the 32-q mask of row a at offset b; the shared address of
	// the lane's next entry, (a, (b + 1024) mod r), sits TS words further, so a
	// probe is two LDS.32 -- no funnel shift, no offset update, no per-row setup
	// beyond locating the lane's first entry.
	uint32_t ta[NT > 0 ? NT : 1];  // shared address of this lane's current entry
#pragma unroll
	for (int j = 0; j < NT; ++j) {
		const uint32_t r = reg_prime<STD>(a, j), m = reg_barrett<STD>(a, j);
		ta[j] = w.tab0 + 4 * (a.reg_tab[j] + mod_full(rc.p, r, m) * r + mod_full(q0_first, r, m));
	}
	const uint32_t lt = (1u << lane) - 1;
	uint32_t qn = 0;  // queued windows

	// one window per lane; EDGE iterations also mask the row's partial last
	// window and lanes past the warp's slice
	auto step = [&](uint32_t it, auto edge) {
		const uint32_t wi = rc.w0 + lane + 32 * it;
		const uint32_t q0 = rc.qlo + 32 * wi;
		uint32_t nonc = rc.even;
#pragma unroll
		for (int k = 0; k < NF; ++k) {
			nonc |= shl_clamp(fpat[k], fo[k]);
			const uint32_t t = fo[k] - fd[k];
			fo[k] = min(t, t + ff[k]);
		}
		uint32_t alive = ~nonc;
		if constexpr (decltype(edge)::value) alive &= wi < rc.w1 ? (wi < rc.wlast ? kFull : rc.tail) : 0u;
#pragma unroll
		for (int j = 0; j < NREG; ++j) {
			if (j < NT) {
				uint32_t M, nx;
				asm volatile("ld.shared.u32 %0, [%1];" : "=r"(M) : "r"(ta[j < NT ? j : 0]));
				asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(nx) : "r"(ta[j < NT ? j : 0]), "n"(4 * TS));
				alive &= ~M;
				ta[j < NT ? j : 0] = nx;
			} else {
				if (j < NR2) {
					alive &= ~__funnelshift_r(rw0[j], rw1[j], rb[j]);
				} else {  // offset b in [0, 63): words (0,1) below 32, (1,2) above
					const bool lo = rb[j] < 32;
					alive &= ~__funnelshift_r(lo ? rw0[j] : rw1[j], lo ? rw1[j] : rw2[j >= NR2 ? j - NR2 : 0], rb[j]);
				}
				const uint32_t t = rb[j] + reg_step<STD>(a, j);
				rb[j] = min(t, t - reg_prime<STD>(a, j));
			}
			if (j + 1 < NREG) S[j + 1] += __popc(alive);
		}
		if (__any_sync(kFull, alive != 0)) {  // VOTE.ANY to a predicate: one test per window
			const uint32_t m = __ballot_sync(kFull, alive != 0);
			CGPU_CHECK(qn + __popc(m) <= kQueue);
			if (alive) w.queue[qn + __popc(m & lt)] = make_uint2(q0, alive);
			qn += __popc(m);
			if (qn >= 32) {
				__syncwarp();
				qn -= 32;
				const uint32_t e = drain<NREG>(a, w, lane, qn, 32, rc.p, kmax);
				if (lane == 0) S[NREG] += e;
				__syncwarp();
			}
		}
	};
	const uint32_t n_iter = (rc.w1 - rc.w0 + 31) / 32;
	const uint32_t E = min(rc.w1, rc.wlast);  // windows below E are whole and in the slice
	const uint32_t n_full = E > rc.w0 ? min((E - rc.w0) / 32, n_iter) : 0;
	uint32_t it = 0;
	for (; it < n_full; ++it) step(it, cuda::std::false_type{});
	for (; it < n_iter; ++it) step(it, cuda::std::true_type{});
	if (qn) {
		__syncwarp();
		const uint32_t e = drain<NREG>(a, w, lane, 0, qn, rc.p, kmax);
		if (lane == 0) S[NREG] += e;
		__syncwarp();
	}
	// register-probe counts of this segment (per-row sums are < 2^32: 59p < 2^32)
	if (NREG > 0) {
		const uint32_t qa = rc.qlo + 32 * rc.w0;
		const uint64_t qe = uint64_t(rc.qlo) + 32ull * rc.w1 - 1;  // 64-bit: no 2^32 wrap
		const uint32_t qb = qe < rc.qhi ? static_cast<uint32_t>(qe) : rc.qhi;
		const uint32_t tot = coprime_in(rc, lane, qa, qb);
		S[0] = lane == 0 ? tot : 0;  // warp_sum(S[0] - S[1]) below: exact mod 2^32
	}
#pragma unroll
	for (int j = 0; j < NREG; ++j) {
		const uint32_t s = warp_sum(S[j] - S[j + 1]);
		if (s) {
			kmax = max(kmax, static_cast<uint32_t>(j + 1));
			if (lane == 0) hist_add(a, w.hist, j, s);
		}
	}
	return kmax;
}

template <int NR2, int NR3, bool STD, bool SHORT>
__device__ __forceinline__ uint32_t dispatch_row(const SieveArgs& a, const WarpSmem& w, uint32_t lane,
                                                 const RowCtx& rc)
{
	// Four variants, not ten: a row uses the narrowest one with enough factor
	// slots (padding slots cost 4 instructions per window). Fewer copies of
	// the loop keep the kernel in the instruction cache when consecutive rows
	// differ in their factor count (C5: 60% of the work has <= 2 odd factors,
	// 32% has 3, 8% has 4-5). SHORT (launches of short rows, where a warp
	// switches rows every few hundred windows and instruction fetch binds --
	// C4: 28% of the stall samples): three, {2, 4, 9} slots. Measured against
	// the four (r02p_variants_ab.txt): C3 -8%, C4 -13%, TRIANGLE p <= 5e4 -16%,
	// 5e4 < p <= 1.5e5 -7%; 1e5 < p <= 2e5 +1%, C5 +5%.
	if constexpr (SHORT) {
		if (rc.nf <= 2) return row_loop<NR2, NR3, STD, 2>(a, w, lane, rc);
		if (rc.nf <= 4) return row_loop<NR2, NR3, STD, 4>(a, w, lane, rc);
		return row_loop<NR2, NR3, STD, 9>(a, w, lane, rc);
	} else {
		switch (rc.nf) {
		case 0:
		case 1:
		case 2: return row_loop<NR2, NR3, STD, 2>(a, w, lane, rc);
		case 3: return row_loop<NR2, NR3, STD, 3>(a, w, lane, rc);
		case 4:
		case 5: return row_loop<NR2, NR3, STD, 5>(a, w, lane, rc);
		default: return row_loop<NR2, NR3, STD, 9>(a, w, lane, rc);
		}
	}
}

#ifdef CGPU_WARP_CLOCKS
__device__ unsigned long long g_wclk[3 * 8192];
#endif

// STOP: polls the cooperative stop word (SieveArgs::stop). The standard-prime
// kernel, the benchmarked one, also exists without the poll: even a per-row
// test of a kernel parameter moved its code layout and cost it ~6% (C5).
template <int NR2, int NR3, bool STD, bool STOP = true, bool SHORT = false>
__global__ void __launch_bounds__(kSieveThreads, kSieveMinBlocks) k_sieve(const SieveArgs a)
{
	constexpr int NREG = NR2 + NR3;
	extern __shared__ uint4 s_dyn[];
	__shared__ bool s_last;
	__shared__ unsigned long long s_red[kSieveWarps];
	const uint32_t lane = threadIdx.x & 31;
	const uint32_t wib = threadIdx.x >> 5;
	WarpSmem w;
	uint2* q_all = reinterpret_cast<uint2*>(s_dyn);
	w.queue = q_all + wib * kQueue;
	w.deep = reinterpret_cast<uint4*>(q_all + kSieveWarps * kQueue) + wib * kDeepPrefetch;
	uint32_t* h_all = reinterpret_cast<uint32_t*>(reinterpret_cast<uint4*>(q_all + kSieveWarps * kQueue) +
	                                              kSieveWarps * kDeepPrefetch);
	w.hist = h_all + static_cast<size_t>(wib) * a.np;
	for (uint32_t j = lane; j < a.np; j += 32) w.hist[j] = 0;
	// the window tables, resident for the whole launch: masks, then successor
	// entries as shared addresses
	constexpr uint32_t TS = STD ? kTabStrideStd : kTabStrideGen;
	uint32_t* s_tab = h_all + static_cast<size_t>(kSieveWarps) * a.np;
	w.tab0 = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
	for (uint32_t e = threadIdx.x; e < a.wtab_n; e += blockDim.x) {
		s_tab[e] = __ldg(a.wintab + e);
		s_tab[TS + e] = w.tab0 + 4 * __ldg(a.wintab + kTabStrideGen + e);
	}
	__syncthreads();

	CGPU_CHECK(sieve_smem_bytes(a.np, a.wtab_n ? TS : 0) <= dynamic_smem_size());
#ifdef CGPU_WARP_CLOCKS
	unsigned long long t_start;
	asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
	const uint32_t n_chunks = plan_chunks(a.n_slots);
	const unsigned long long W = a.chunk_off[n_chunks];
	const unsigned long long nwarps = static_cast<unsigned long long>(gridDim.x) * kSieveWarps;
#ifdef CGPU_REVERSE_SLICES  // experiment: CTA b takes the slices of CTA grid-1-b (per-SM speed vs work)
	const unsigned long long gw = static_cast<unsigned long long>(gridDim.x - 1 - blockIdx.x) * kSieveWarps + wib;
#else
	const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * kSieveWarps + wib;
#endif
	unsigned long long ws = W * gw / nwarps;  // W < 2^40, nwarps < 2^20
	const unsigned long long we = W * (gw + 1) / nwarps;

	// 32-ary warp search: largest slot s with prefix(s) <= ws
	uint32_t lo = 0, hi = a.n_slots;
	if (ws < we) {
		while (hi - lo > 1) {
			const uint32_t step = (hi - lo + 31) / 32;
			const uint32_t idx = lo + step * lane;
			const bool le = idx < hi && slot_prefix(a, idx) <= ws;
			const uint32_t L = 31 - __clz(__ballot_sync(kFull, le));
			lo += step * L;
			hi = min(hi, lo + step);
		}
	}

	uint32_t slot = lo;
	while (ws < we) {
		const unsigned long long rs = slot_prefix(a, slot), re = slot_prefix(a, slot + 1);
		if (re <= ws) {
			++slot;
			continue;
		}
		// this warp's share of the row's units; the first row_cost are the
		// setup charge, the rest map to windows (unit_window)
		const unsigned long long u0 = ws - rs, u1 = min(we, re) - rs;
		ws = min(we, re);
		const uint32_t cur = slot++;
		if constexpr (STOP)  // a stop raised: abandon the launch (the caller re-sieves exactly)
			if (a.stop && (cur & 7u) == 0 && *a.stop) break;
		const uint32_t rcost = a.row_cost;
		if (u1 <= rcost) continue;
		const RowBounds rb = slot_row(a, cur);
		RowCtx rc;
		rc.p = static_cast<uint32_t>(rb.p);
		rc.qlo = static_cast<uint32_t>(rb.qlo);
		const uint32_t qhi = static_cast<uint32_t>(rb.qhi);
		rc.qhi = qhi;
		rc.wlast = (qhi - rc.qlo) / 32;
		rc.tail = (2u << (qhi - (rc.qlo + 32 * rc.wlast))) - 1;  // span 31 -> all ones

		// ---- distinct prime factors of p, factorised by k_plan ----
		// f = 2 becomes a constant mask (the q step per lane is even); odd
		// factors above qhi cannot divide any q of the row and were dropped.
		const uint32_t fw = lane < kFacWords ? __ldg(a.rowfac + static_cast<size_t>(cur) * kFacWords + lane) : 0u;
		const uint32_t head = __shfl_sync(kFull, fw, 0);
		rc.nf = head & 0xffu;
		const bool even = (head >> 8) & 1u;
		// this warp's windows of the row (row_units / unit_window)
		rc.w0 = unit_window(a, u0, (head >> 16) & 3u, rc.wlast + 1);
		rc.w1 = unit_window(a, u1, (head >> 16) & 3u, rc.wlast + 1);
		if (rc.w1 <= rc.w0) continue;

#pragma unroll
		for (int k = 0; k < kMaxFactors; ++k) {
			rc.fac[k] = __shfl_sync(kFull, fw, k + 1);
			rc.fm[k] = __shfl_sync(kFull, fw, k + 1 + kMaxFactors);
		}
		// q0 parity is fixed per lane (q advances by 32 per window): even p
		// excludes the even q of every window
		rc.even = even ? (((rc.qlo + 32 * (rc.w0 + lane)) & 1) ? 0xAAAAAAAAu : 0x55555555u) : 0u;
		// resolve the rows of the first deep probes (every drain of this row
		// walks them first) and pull them into L1 (lanes 2k, 2k+1 take the two
		// lines of probe k)
		if (NREG + lane / 2 < a.np && lane < 2 * kDeepPrefetch) {
			const uint4 d = __ldg(a.probes + NREG + lane / 2);
			const uint32_t base = d.z + mod_full(rc.p, d.x, d.y) * d.w;
			if ((lane & 1) == 0) w.deep[lane / 2] = make_uint4(base, d.x, d.y, 0);
			const uint32_t* row = a.ext + base + (lane & 1) * 32;
			if ((lane & 1) == 0 || d.w > 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(row));
		}
		__syncwarp();

		const uint32_t kk = dispatch_row<NR2, NR3, STD, SHORT>(a, w, lane, rc);  // 1 + deepest killer
		if (lane == 0 && kk) {
			const uint32_t j = kk - 1;
			uint32_t killer;
			if constexpr (NREG > 0)
				killer = j < static_cast<uint32_t>(NREG) ? a.reg_r[j] : __ldg(a.probes + j).x;
			else
				killer = __ldg(a.probes + j).x;
			CGPU_CHECK(rb.p / 100 - a.blk_lo < a.n_blocks);
			atomicMax(&a.block_rmax[rb.p / 100 - a.blk_lo], killer);
		}
		__syncwarp();
	}

#ifdef CGPU_WARP_CLOCKS
	{  // experiment hook (tools/warp_clocks.py): per-warp {start, end, smid}
		unsigned long long t_end;
		asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
		uint32_t smid;
		asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
		const uint32_t gwi = blockIdx.x * kSieveWarps + wib;
		if (lane == 0 && gwi < 8192) {
			g_wclk[3 * gwi] = t_start;
			g_wclk[3 * gwi + 1] = t_end;
			g_wclk[3 * gwi + 2] = smid;
		}
	}
#endif
	// ---- CTA flush: per-warp counters -> global histogram ----
	__syncthreads();
	for (uint32_t j = threadIdx.x; j < a.np; j += blockDim.x) {
		unsigned long long s = 0;
		for (int v = 0; v < kSieveWarps; ++v) s += h_all[static_cast<size_t>(v) * a.np + j];
		if (s) atomicAdd(&a.hist[__ldg(a.probe_rank + j)], s);
	}
	// the last CTA: pairs_tested = sum(hist) + survivors
	__threadfence();
	__syncthreads();
	if (threadIdx.x == 0) s_last = atomicAdd(&a.tickets[1], 1u) == gridDim.x - 1;
	__syncthreads();
	if (!s_last) return;
	__threadfence();
	unsigned long long s = 0;
	for (uint32_t k = threadIdx.x; k < a.nprimes; k += blockDim.x)
		s += *reinterpret_cast<volatile unsigned long long*>(a.hist + k);
	for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
	if (lane == 0) s_red[wib] = s;
	__syncthreads();
	if (threadIdx.x == 0) {
		unsigned long long t = 0;
		for (int v = 0; v < kSieveWarps; ++v) t += s_red[v];
		a.counters[0] = t + *reinterpret_cast<volatile unsigned long long*>(a.counters + 1);
		a.tickets[1] = 0;
	}
}

// ---------------------------------------------------------------------------
// K2w: the wheel sieve (standard probe sets: register probes 11..37).
//
// Same contract and row/segment bookkeeping as k_sieve, different window
// geometry. Probes 11, 13 and 17 are not probed per window at all: a row p
// leaves alive only the classes of q mod 2431 in A11(p mod 11) x A13(p mod 13)
// x A17(p mod 17) (135 of 2431 for canonical rows), listed once per row segment,
// and only those are visited -- as 32-bit windows of STRIDE 2431 (bit i of the
// window at q0 is q0 + 2431 i, all in one class). The remaining register probes
// 19..37 read strided window tables (entry (a, q0 mod r) = the 32 kill bits at
// stride 2431; rows doubled to 2r entries so the lazy Barrett remainder indexes
// them directly), coprimality is one stride-2431 periodic mask per odd prime
// factor of p other than 11, 13, 17 (those drop whole classes), and the
// first-kill counts of 11, 13, 17 come from S0 (candidates), S1 (alive after
// 11) and S2 (alive after 11 and 13), all by inclusion-exclusion over the
// factors of p (wheel_counts); S3 on is the telescoped popcount of k_sieve.
// Lanes still alive after 37 push their single q to the warp queue; the deep
// probes then run one q per lane.
// ---------------------------------------------------------------------------

struct WheelSmem {
	uint32_t* queue;  // [kWheelQueue] q alive after the register probes
	uint32_t* hist;   // [np]
	uint4* deep;      // [kDeepPrefetch] {row base, r, m, -}
	uint16_t* cls;    // [kWheelCls] alive classes of the current batch: offsets o < 2431 (q = qa + o + 2431 i)
	uint16_t* l143;   // [192] alive offsets mod 143 at [0, 143), mod 17 at [160, 177)
	uint32_t* allfac; // [kMaxFactors] every odd prime factor of p that can divide a q of the row
	uint4* fac;       // [kMaxFactors] loop factors {-f, barrett m, -(2431^-1) mod f (f < 37681), bit pattern}
	const uint32_t* tab;  // the CTA's wheel tables
	uint32_t tab0;        // ... as a shared address
};

// low z bits set, z clamped to [0, 32]
__device__ __forceinline__ uint32_t low_bits(int z)
{
	return ~shl_clamp(kFull, static_cast<uint32_t>(max(0, min(z, 32))));
}

// #{rho < y : P(rho)} for the 143-bit pattern P, y <= 143
__device__ __forceinline__ uint32_t prefix143(const uint32_t (&P)[5], uint32_t y)
{
	uint32_t c = 0;
#pragma unroll
	for (int wd = 0; wd < 5; ++wd) c += __popc(P[wd] & low_bits(static_cast<int>(y) - 32 * wd));
	return c;
}

// Warp-collective: S0 = #{q in [qa, qb] : gcd(q, p) = 1}, S1 = those of them
// alive after probe 11 (row a11), S2 = those alive after 11 and 13, by
// inclusion-exclusion over the prime factors of p that can divide a q of the
// row; lanes split the subsets. For a squarefree divisor d the multiples
// q = d t, t in [t0, t1], have q mod r = (d mod r)(t mod r): the table entry
// B(a, d mod r) is the set of t residues that stay alive, Rep its periodic
// extension over the 143 residues of t mod 143.
__device__ __forceinline__ void wheel_counts(const RowCtx& rc, const WheelSmem& w, uint32_t lane, uint32_t qa,
                                             uint32_t qb, uint32_t a11, uint32_t a13, uint32_t& s0, uint32_t& s1,
                                             uint32_t& s2)
{
	const uint32_t F = rc.nf + (rc.even ? 1u : 0u);
	uint32_t acc0 = 0, acc1 = 0, acc2 = 0;  // exact mod 2^32; the results are < 2^32
	for (uint32_t sub = lane; sub < (1u << F); sub += 32) {
		uint64_t d = (rc.even && ((sub >> rc.nf) & 1)) ? 2 : 1;
		for (uint32_t i = 0; i < rc.nf; ++i)
			if ((sub >> i) & 1) d *= w.allfac[i];
		if (d > qb) continue;
		const uint32_t dd = static_cast<uint32_t>(d);
		const uint32_t t1 = qb / dd, t0 = (qa - 1) / dd + 1;
		if (t1 < t0) continue;
		const uint32_t n = t1 - t0 + 1;
		const uint32_t d11 = dd % 11, d13 = dd % 13;
		const uint32_t B = w.tab[kWtB11 + a11 * 11 + d11];
		const uint32_t full = n / 11, rem = n - 11 * full, s = t0 % 11;
		const uint32_t c1 = full * __popc(B) + __popc(((B | (B << 11)) >> s) & ((1u << rem) - 1));
		uint32_t P[5];
		const uint32_t* r11 = w.tab + kWtRep11 + (a11 * 11 + d11) * 5;
		const uint32_t* r13 = w.tab + kWtRep13 + (a13 * 13 + d13) * 5;
#pragma unroll
		for (int wd = 0; wd < 5; ++wd) P[wd] = r11[wd] & r13[wd];
		const uint32_t tot = prefix143(P, 143);
		const uint32_t full2 = n / 143, rem2 = n - 143 * full2, sa = t0 % 143, sb = sa + rem2;  // sb <= 285
		const uint32_t ca = prefix143(P, sa);
		const uint32_t cb = sb >= 143 ? tot + prefix143(P, sb - 143) : prefix143(P, sb);
		const uint32_t c2 = full2 * tot + cb - ca;
		if (__popc(sub) & 1) {
			acc0 -= n;
			acc1 -= c1;
			acc2 -= c2;
		} else {
			acc0 += n;
			acc1 += c1;
			acc2 += c2;
		}
	}
	s0 = warp_sum(acc0);
	s1 = warp_sum(acc1);
	s2 = warp_sum(acc2);
}

// Deep probes for queue entries [base, base + n), one q per lane, in rank
// order; the lanes leave together once every q is dead. Survivors are emitted.
__device__ __forceinline__ void wheel_drain(const SieveArgs& a, const WheelSmem& w, uint32_t lane, uint32_t base,
                                            uint32_t n, uint32_t p, uint32_t& kmax)
{
	bool alive = lane < n;
	const uint32_t q = alive ? w.queue[base + lane] : 0u;
	for (uint32_t j = kWheelReg; j < a.np; ++j) {
		if (!__any_sync(kFull, alive)) break;
		bool kill = false;
		if (alive) {
			uint32_t row, r, m;
			if (j - kWheelReg < kDeepPrefetch) {
				const uint4 e = w.deep[j - kWheelReg];
				row = e.x;
				r = e.y;
				m = e.z;
			} else {
				const uint4 d = __ldg(a.probes + j);
				row = d.z + mod_full(p, d.x, d.y) * d.w;
				r = d.x;
				m = d.y;
			}
			const uint32_t b = mod_full(q, r, m);
			CGPU_CHECK(row + (b >> 5) < a.ext_words);
			kill = (__ldg(a.ext + row + (b >> 5)) >> (b & 31)) & 1u;
		}
		const uint32_t km = __ballot_sync(kFull, kill);
		if (km) {
			kmax = max(kmax, j + 1);
			if (lane == 0) hist_add(a, w.hist, j, __popc(km));
			alive = alive && !kill;
		}
	}
	const uint32_t sm = __ballot_sync(kFull, alive);
	if (sm) {
		unsigned long long sb = 0;
		if (lane == 0) sb = atomicAdd(&a.counters[1], static_cast<unsigned long long>(__popc(sm)));
		sb = __shfl_sync(kFull, sb, 0) + __popc(sm & ((1u << lane) - 1));
		if (alive && sb < a.surv_cap) a.surv[sb] = (static_cast<unsigned long long>(p) << 32) | q;
	}
}

// One row segment: q in [rc.qlo + 32 rc.w0, min(rc.qhi, rc.qlo + 32 rc.w1 - 1)].
// nfl = the loop's factor slots in w.fac (odd prime factors of p other than
// 11, 13, 17). Returns 1 + the deepest probe that killed in the segment (0: none).
__device__ __forceinline__ uint32_t wheel_row(const SieveArgs& a, const WheelSmem& w, uint32_t lane,
                                              const RowCtx& rc, uint32_t nfl, uint32_t nmid)
{
	const uint32_t qa = rc.qlo + 32 * rc.w0;
	const uint64_t qe = uint64_t(rc.qlo) + 32ull * rc.w1 - 1;  // 64-bit: no 2^32 wrap
	const uint32_t qb = qe < rc.qhi ? static_cast<uint32_t>(qe) : rc.qhi;
	const uint32_t span = qb - qa;
	const uint32_t lt = (1u << lane) - 1;
	uint32_t kmax = 0;

	// rows of the wheel primes; a class killed by one of them is dropped, and when
	// the prime divides p its class 0 holds no coprime q at all
	const uint32_t a11 = mod_full(rc.p, 11, barrett_m(11)), a13 = mod_full(rc.p, 13, barrett_m(13));
	const uint32_t a17 = mod_full(rc.p, 17, barrett_m(17));
	const uint32_t kill11 = w.tab[kWtKill + a11] | (a11 ? 0u : 1u);
	const uint32_t kill13 = w.tab[kWtKill + 32 + a13] | (a13 ? 0u : 1u);
	const uint32_t kill17 = w.tab[kWtKill + 64 + a17] | (a17 ? 0u : 1u);
	const uint32_t qa11 = mod_full(qa, 11, barrett_m(11)), qa13 = mod_full(qa, 13, barrett_m(13));
	const uint32_t qa17 = mod_full(qa, 17, barrett_m(17));
	// the segment's alive offsets mod 143 (cls[0 .. n143)) and mod 17 (cls[160 .. 160 + n17)), then
	// their CRT combinations o < 2431 with o <= span, written over the list from the top down so
	// that the two inputs (read in ascending order of ci / n17) are consumed before being overwritten
	uint32_t n143 = 0;
#pragma unroll
	for (uint32_t c0 = 0; c0 < 143; c0 += 32) {
		const uint32_t c = c0 + lane;
		const uint32_t x11 = mod_full(qa11 + c, 11, barrett_m(11)), x13 = mod_full(qa13 + c, 13, barrett_m(13));
		const bool ok = c < 143 && !((kill11 >> x11) & 1u) && !((kill13 >> x13) & 1u);
		const uint32_t bal = __ballot_sync(kFull, ok);
		CGPU_CHECK(n143 + __popc(bal) <= 143);
		if (ok) w.l143[n143 + __popc(bal & lt)] = static_cast<uint16_t>(c);
		n143 += __popc(bal);
	}
	uint32_t n17;
	{
		const uint32_t x17 = mod_full(qa17 + lane, 17, barrett_m(17));
		const bool ok = lane < 17 && !((kill17 >> x17) & 1u);
		const uint32_t bal = __ballot_sync(kFull, ok);
		if (ok) w.l143[160 + __popc(bal & lt)] = static_cast<uint16_t>(lane);
		n17 = __popc(bal);
	}
	__syncwarp();
	// S[j - kWheelFirst] = sum of popc(alive before register probe j), j = 3..7
	uint32_t S[kWheelReg - kWheelFirst];
#pragma unroll
	for (int j = 0; j < kWheelReg - kWheelFirst; ++j) S[j] = 0;
	uint32_t entered = 0, qn = 0;
	const uint32_t ntot = n143 * n17;
	const uint32_t rcp17 = 65536u / max(n17, 1u) + 1;  // floor(ci / n17) = (ci * rcp17) >> 16 for ci < 2432

	// the alive classes o < 2431 (CRT combinations of the two lists) with o <= span, kWheelCls at a
	// time (a canonical row has 135; only rows that 11 and 17 both divide exceed one batch)
	for (uint32_t cb = 0; cb < ntot; cb += kWheelCls) {
	const uint32_t cend = min(cb + kWheelCls, ntot);
	uint32_t n = 0;
	for (uint32_t c0 = cb; c0 < cend; c0 += 32) {
		const uint32_t ci = c0 + lane;
		const uint32_t i143 = (ci * rcp17) >> 16, i17 = ci - i143 * n17;
		uint32_t o = kWheelM;
		if (ci < cend)
			o = mod_full(w.l143[i143] * kWheelE143 + w.l143[160 + i17] * kWheelE17, kWheelM, barrett_m(kWheelM));
		const bool ok = ci < cend && o <= span;
		const uint32_t bal = __ballot_sync(kFull, ok);
		CGPU_CHECK(n + __popc(bal) <= kWheelCls);
		// bits 14..15: for even p, 1 + parity of the class's q (q0 + 2431 i alternates parity and the
		// windows of a class are 77792 q apart): the even q are (entry >> 14) * 0x55555555
		if (ok) w.cls[n + __popc(bal & lt)] = static_cast<uint16_t>(o | (rc.even ? (1u + ((qa + o) & 1u)) << 14 : 0u));
		n += __popc(bal);
	}
	__syncwarp();

	if (n) {
		// shared address of row (p mod r) of each strided window table
		uint32_t ta[kWheelReg - kWheelFirst];
#pragma unroll
		for (int j = kWheelFirst; j < kWheelReg; ++j) {
			const uint32_t r = std_prime(j);
			ta[j - kWheelFirst] = w.tab0 + 4 * (wheel_tab_base(j) + mod_full(rc.p, r, barrett_m(r)) * 2 * r);
		}
		const uint32_t nchunk = span / kWheelChunk + 1;
		const uint32_t total = n * nchunk;
		const uint32_t n_iter = (total + 31) / 32;
		const uint32_t kfull = (span + 1) / kWheelChunk;  // chunks lying wholly inside the segment
		const uint32_t n_full = (n * kfull) / 32;
		uint32_t k = 0, ci = lane;
		while (ci >= n) {
			ci -= n;
			++k;
		}

		// `left` counts the iterations down; the last n_edge of them touch the row's partial windows
		// or lanes past the end
		const uint32_t n_edge = n_iter - n_full;
		for (uint32_t left = n_iter; left; --left) {
			uint32_t alive, q0;
			{
				const uint32_t ce = w.cls[ci];
				const uint32_t c = ce & 0x3fffu;
				q0 = qa + c + kWheelChunk * k;
				uint32_t nonc = (ce >> 14) * 0x55555555u;
				// factors below 37681 (ascending, so they come first): the first i with f | q0 + 2431 i is
				// (q0 mod f) g mod f; pattern = period-f mask below 32, a single bit above
#pragma unroll 1
				for (uint32_t s = 0; s < nmid; ++s) {  // (not unrolled: 1.7 factors on average, code size)
					const uint4 e = w.fac[s];  // {-f, m, g, pattern}: x + umulhi(x, m) (-f) is the lazy remainder
					const uint32_t t = (q0 + __umulhi(q0, e.y) * e.x) * e.z;
					const uint32_t v = t + __umulhi(t, e.y) * e.x;
					nonc |= shl_clamp(e.w, min(v, v + e.x));
				}
#pragma unroll 1
				for (uint32_t s = nmid; s < nfl; ++s) {  // f >= 37681: at most two multiples of f in [q0, q0 + 31 * 2431]
					const uint4 e = w.fac[s];
					const uint32_t f = 0u - e.x;
					const uint32_t t = mod_full(q0, f, e.y);
					uint32_t d = t ? f - t : 0u;
#pragma unroll
					for (int rep = 0; rep < 2; ++rep) {
						const uint32_t i = __umulhi(min(d, kWheelChunk), kWheelDivMul);
						nonc |= i * kWheelM == d ? shl_clamp(1u, i) : 0u;
						d += f;
						if (d < f) d = kWheelChunk + 1;  // wrapped past 2^32: no further multiple in reach
					}
				}
				alive = ~nonc;
				if (left <= n_edge) {  // edge: the row's last chunks and lanes past the end
					uint32_t vm = 0;
					if (k < nchunk) {
						const uint32_t rem = span - kWheelChunk * k;
						if (c <= rem) vm = ~shl_clamp(kFull, __umulhi(min(rem - c, kWheelChunk - 1), kWheelDivMul) + 1);
					}
					alive &= vm;
				}
				S[0] += __popc(alive);
				const uint32_t q4 = q0 << 2;
#pragma unroll
				for (int j = kWheelFirst; j < kWheelReg; ++j) {
					const uint32_t r = std_prime(j);
					// 4 x the lazy remainder (in [0, 8r): the rows are doubled), exact mod 2^32
					const uint32_t rem4 = q4 - __umulhi(q0, barrett_m(r)) * (4 * r);
					uint32_t M;
					CGPU_CHECK(rem4 < 8 * r && ta[j - kWheelFirst] + rem4 < w.tab0 + 4 * kWtWords);
					asm volatile("ld.shared.u32 %0, [%1];" : "=r"(M) : "r"(ta[j - kWheelFirst] + rem4));
					alive &= ~M;
					if (j + 1 < kWheelReg) S[j + 1 - kWheelFirst] += __popc(alive);
				}
				ci += 32;  // next window of the lane: 32 classes on (a batch of fewer than 32 wraps more than once)
				while (ci >= n) {
					ci -= n;
					++k;
				}
			}
			uint32_t m = __ballot_sync(kFull, alive != 0);
			while (m) {  // usually one pass: a second only for a lane with two q alive
				CGPU_CHECK(qn + __popc(m) <= kWheelQueue);
				if (alive) {
					const uint32_t bit = __ffs(alive) - 1;
					w.queue[qn + __popc(m & lt)] = q0 + kWheelM * bit;
					alive &= alive - 1;
				}
				qn += __popc(m);
				if (qn >= 32) {
					__syncwarp();
					qn -= 32;
					entered += 32;
					wheel_drain(a, w, lane, qn, 32, rc.p, kmax);
					__syncwarp();
				}
				m = __ballot_sync(kFull, alive != 0);
			}
		}
		if (qn) {  // what the batch leaves
			__syncwarp();
			entered += qn;
			wheel_drain(a, w, lane, 0, qn, rc.p, kmax);
			qn = 0;
			__syncwarp();
		}
	}
	__syncwarp();
	}  // class batches
	// first-kill counts of the register probes
	uint32_t tot[kWheelReg + 1];
	wheel_counts(rc, w, lane, qa, qb, a11, a13, tot[0], tot[1], tot[2]);
#pragma unroll
	for (int j = kWheelFirst; j < kWheelReg; ++j) tot[j] = warp_sum(S[j - kWheelFirst]);
	tot[kWheelReg] = entered;
#pragma unroll
	for (int j = 0; j < kWheelReg; ++j) {
		const uint32_t s = tot[j] - tot[j + 1];
		if (s) {
			kmax = max(kmax, static_cast<uint32_t>(j + 1));
			if (lane == 0) hist_add(a, w.hist, j, s);
		}
	}
	return kmax;
}

template <bool STOP>
__global__ void __launch_bounds__(kWheelThreads, 1) k_wsieve(const SieveArgs a)
{
	extern __shared__ uint4 s_dyn[];
	__shared__ bool s_last;
	__shared__ unsigned long long s_red[kWheelWarps];
	const uint32_t lane = threadIdx.x & 31;
	const uint32_t wib = threadIdx.x >> 5;
	// shared memory: the wheel tables, then one contiguous block per warp (a single base address
	// with constant offsets: separate per-type arrays made the 64-register loop recompute five
	// addresses from the thread index every iteration)
	WheelSmem w;
	uint32_t* s_tab = reinterpret_cast<uint32_t*>(s_dyn);
	const uint32_t wstride = wheel_warp_bytes(a.np);
	unsigned char* blk = (reinterpret_cast<unsigned char*>(s_tab) + kWtBytes) + static_cast<size_t>(wib) * wstride;
	w.deep = reinterpret_cast<uint4*>(blk);
	w.fac = reinterpret_cast<uint4*>(blk + kWbFac);
	w.queue = reinterpret_cast<uint32_t*>(blk + kWbQueue);
	w.l143 = reinterpret_cast<uint16_t*>(blk + kWbLists);
	w.allfac = reinterpret_cast<uint32_t*>(blk + kWbLists + 2 * 192);
	w.cls = reinterpret_cast<uint16_t*>(blk + kWbCls);
	w.hist = reinterpret_cast<uint32_t*>(blk + kWbHist);
	w.tab = s_tab;
	w.tab0 = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
	for (uint32_t j = lane; j < a.np; j += 32) w.hist[j] = 0;
	for (uint32_t e = threadIdx.x; e < kWtWords; e += blockDim.x) s_tab[e] = __ldg(a.wheeltab + e);
	__syncthreads();
	CGPU_CHECK(wsieve_smem_bytes(a.np) <= dynamic_smem_size());

	const uint32_t n_chunks = plan_chunks(a.n_slots);
	const unsigned long long W = a.chunk_off[n_chunks];
	const unsigned long long nwarps = static_cast<unsigned long long>(gridDim.x) * kWheelWarps;
	const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * kWheelWarps + wib;
	// W gw / nwarps without the 64-bit overflow of the product (units are 1/64 instruction here)
	const unsigned long long Wq = W / nwarps, Wr = W % nwarps;
	unsigned long long ws = Wq * gw + Wr * gw / nwarps;
	const unsigned long long we = Wq * (gw + 1) + Wr * (gw + 1) / nwarps;

	// 32-ary warp search: largest slot s with prefix(s) <= ws
	uint32_t lo = 0, hi = a.n_slots;
	if (ws < we) {
		while (hi - lo > 1) {
			const uint32_t step = (hi - lo + 31) / 32;
			const uint32_t idx = lo + step * lane;
			const bool le = idx < hi && slot_prefix(a, idx) <= ws;
			const uint32_t L = 31 - __clz(__ballot_sync(kFull, le));
			lo += step * L;
			hi = min(hi, lo + step);
		}
	}

	uint32_t slot = lo;
	while (ws < we) {
		const unsigned long long rs = slot_prefix(a, slot), re = slot_prefix(a, slot + 1);
		if (re <= ws) {
			++slot;
			continue;
		}
		const unsigned long long u0 = ws - rs, u1 = min(we, re) - rs;
		ws = min(we, re);
		const uint32_t cur = slot++;
		if constexpr (STOP)  // a stop raised: abandon the launch (the caller re-sieves exactly)
			if (a.stop && (cur & 7u) == 0 && *a.stop) break;
		if (u1 <= a.row_cost) continue;
		const RowBounds rb = slot_row(a, cur);
		RowCtx rc;
		rc.p = static_cast<uint32_t>(rb.p);
		rc.qlo = static_cast<uint32_t>(rb.qlo);
		rc.qhi = static_cast<uint32_t>(rb.qhi);
		rc.wlast = (rc.qhi - rc.qlo) / 32;
		rc.tail = 0;
		const uint32_t fw = lane < kFacWords ? __ldg(a.rowfac + static_cast<size_t>(cur) * kFacWords + lane) : 0u;
		const uint32_t head = __shfl_sync(kFull, fw, 0);
		rc.nf = head & 0xffu;
		rc.even = (head >> 8) & 1u;
		rc.w0 = unit_window_mult(a, u0, head >> 16, rc.wlast + 1);
		rc.w1 = unit_window_mult(a, u1, head >> 16, rc.wlast + 1);
		if (rc.w1 <= rc.w0) continue;
		// all odd factors for the analytic counts (wheel_counts reads them from shared memory: lane
		// L = 1..nf holds factor L - 1)
		if (lane >= 1 && lane <= rc.nf) w.allfac[lane - 1] = fw;
		// the loop's factor slots: odd factors other than 11, 13, 17 (lane L = 1..nf holds factor L - 1)
		const uint32_t fmv = __shfl_down_sync(kFull, fw, kMaxFactors);  // lane L: its Barrett constant
		const bool keep = lane >= 1 && lane <= rc.nf && fw != 11 && fw != 13 && fw != 17;
		const uint32_t keepm = __ballot_sync(kFull, keep);
		if (keep) {
			uint32_t x = 0;
			if (fw < kWheelMidMax) {
				// g = -(2431^-1) mod f; 143^-1 = (1 + f k) / 143 with k = (-f^-1) mod 143, likewise 17^-1
				const uint32_t i143 = (1 + fw * w.tab[kWtNinv143 + fw % 143]) / 143;
				const uint32_t i17 = (1 + fw * w.tab[kWtNinv17 + fw % 17]) / 17;
				x = fw - mod_full(i143 * i17, fw, fmv);
			}
			w.fac[__popc(keepm & ((1u << lane) - 1))] = make_uint4(0u - fw, fmv, x, fw < 32 ? c_period_mask[fw] : 1u);
		}
		const uint32_t nmid = __popc(__ballot_sync(kFull, keep && fw < kWheelMidMax));
		const uint32_t nfl = __popc(keepm);
		// rows of the first deep probes, pulled into L1
		if (kWheelReg + lane / 2 < a.np && lane < 2 * kDeepPrefetch) {
			const uint4 d = __ldg(a.probes + kWheelReg + lane / 2);
			const uint32_t base = d.z + mod_full(rc.p, d.x, d.y) * d.w;
			if ((lane & 1) == 0) w.deep[lane / 2] = make_uint4(base, d.x, d.y, 0);
			const uint32_t* row = a.ext + base + (lane & 1) * 32;
			if ((lane & 1) == 0 || d.w > 32) asm volatile("prefetch.global.L1 [%0];" ::"l"(row));
		}
		__syncwarp();

		const uint32_t kk = wheel_row(a, w, lane, rc, nfl, nmid);
		if (lane == 0 && kk) {
			const uint32_t j = kk - 1;
			const uint32_t killer = j < static_cast<uint32_t>(kWheelReg) ? std_prime(j) : __ldg(a.probes + j).x;
			CGPU_CHECK(rb.p / 100 - a.blk_lo < a.n_blocks);
			atomicMax(&a.block_rmax[rb.p / 100 - a.blk_lo], killer);
		}
		__syncwarp();
	}

	// ---- CTA flush: per-warp counters -> global histogram ----
	__syncthreads();
	for (uint32_t j = threadIdx.x; j < a.np; j += blockDim.x) {
		unsigned long long s = 0;
		for (int v = 0; v < kWheelWarps; ++v)
			s += reinterpret_cast<const uint32_t*>((reinterpret_cast<unsigned char*>(s_tab) + kWtBytes) +
			                                       static_cast<size_t>(v) * wstride + kWbHist)[j];
		if (s) atomicAdd(&a.hist[__ldg(a.probe_rank + j)], s);
	}
	__threadfence();
	__syncthreads();
	if (threadIdx.x == 0) s_last = atomicAdd(&a.tickets[1], 1u) == gridDim.x - 1;
	__syncthreads();
	if (!s_last) return;
	__threadfence();
	unsigned long long s = 0;
	for (uint32_t k = threadIdx.x; k < a.nprimes; k += blockDim.x)
		s += *reinterpret_cast<volatile unsigned long long*>(a.hist + k);
	for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(kFull, s, d);
	if (lane == 0) s_red[wib] = s;
	__syncthreads();
	if (threadIdx.x == 0) {
		unsigned long long t = 0;
		for (int v = 0; v < kWheelWarps; ++v) t += s_red[v];
		a.counters[0] = t + *reinterpret_cast<volatile unsigned long long*>(a.counters + 1);
		a.tickets[1] = 0;
	}
}

// Wheel tables from the row-extended layout (kernels.cuh kWt*): one thread per word.
struct WheelTabArgs {
	uint32_t base[kWheelReg];  // ext word offset of register probe j's rows
};

__global__ void k_wheeltab(const uint32_t* __restrict__ ext, const WheelTabArgs t, uint32_t* __restrict__ out)
{
	auto ubit = [&](int j, uint32_t a, uint32_t x) -> uint32_t {  // u_r(a, x), x < r
		const uint32_t r = std_prime(j);
		return (ext[t.base[j] + a * ext_row_words(r) + (x >> 5)] >> (x & 31)) & 1u;
	};
	for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < kWtWords; e += gridDim.x * blockDim.x) {
		uint32_t v = 0;
		if (e < kWtB11) {  // kill masks of 11 (words 0..31), 13 (32..63), 17 (64..95)
			const int j = e >> 5;
			const uint32_t r = std_prime(j), a = e & 31;
			if (a < r)
				for (uint32_t b = 0; b < r; ++b) v |= ubit(j, a, b) << b;
		} else if (e < kWtRep11) {  // B(a, d): t residues with (d t mod 11) alive in row a of 11
			const uint32_t i = e - kWtB11;
			if (i < 121) {
				const uint32_t a = i / 11, d = i % 11;
				for (uint32_t rho = 0; rho < 11; ++rho) v |= (ubit(0, a, (d * rho) % 11) ^ 1u) << rho;
			}
		} else if (e < kWtNinv143) {  // B(a, d) of 11 / 13 repeated over the 143 residues of t, 5 words
			const int j = e < kWtRep13 ? 0 : 1;
			const uint32_t r = std_prime(j), i = e - (j ? kWtRep13 : kWtRep11);
			if (i < r * r * 5) {
				const uint32_t a = i / (5 * r), d = (i / 5) % r, wd = i % 5;
				for (uint32_t l = 0; l < 32; ++l) {
					const uint32_t rho = 32 * wd + l;
					if (rho < 143) v |= (ubit(j, a, (d * (rho % r)) % r) ^ 1u) << l;
				}
			}
		} else if (e < kWtNinv17) {  // x -> (-x^-1) mod 143
			const uint32_t x = e - kWtNinv143;
			if (x < 143)
				for (uint32_t y = 1; y < 143; ++y)
					if ((x * y) % 143 == 142) v = y;
		} else if (e < kWtTinyOff) {  // x -> (-x^-1) mod 17
			const uint32_t x = e - kWtNinv17;
			if (x < 17)
				for (uint32_t y = 1; y < 17; ++y)
					if ((x * y) % 17 == 16) v = y;
		} else if (e < kWtTab) {  // tiny-factor masks: offsets by f, then (f, t), t < 2f: bits i with f | t + 2431 i
			uint32_t off = kWtTiny;
			bool done = false;
			for (uint32_t f = 3; f < 32 && !done; f += 2) {
				bool prime = true;
				for (uint32_t dv = 3; dv * dv <= f; dv += 2) prime = prime && (f % dv != 0);
				if (!prime || f == 11 || f == 13 || f == 17) continue;
				if (e == kWtTinyOff + f) {
					v = off;
					done = true;
				} else if (e >= off && e < off + 2 * f) {
					const uint32_t t = e - off;
					for (uint32_t l = 0; l < 32; ++l)
						if ((t + kWheelM * l) % f == 0) v |= 1u << l;
					done = true;
				}
				off += 2 * f;
			}
		} else {
			int j = kWheelFirst;
			while (j + 1 < kWheelReg && e >= wheel_tab_base(j + 1)) ++j;
			const uint32_t r = std_prime(j), i = e - wheel_tab_base(j), a = i / (2 * r), b = i % (2 * r);
			// the row's words once (r <= 37: at most two hold bits below r), then 32 bits at stride 2431 mod r
			const uint32_t* row = ext + t.base[j] + a * ext_row_words(r);
			const uint32_t w0 = row[0], w1 = row[1];
			uint32_t x = b % r;
			for (uint32_t l = 0; l < 32; ++l) {
				v |= (((x < 32 ? w0 : w1) >> (x & 31)) & 1u) << l;
				x += kWheelM % r;
				if (x >= r) x -= r;
			}
		}
		out[e] = v;
	}
}

template <bool STOP>
void* wsieve_fn()
{
	return reinterpret_cast<void*>(&k_wsieve<STOP>);
}

// block r_max init: 1 for blocks owned by this shard, 0 otherwise
__global__ void k_init_blocks(uint32_t* rmax, uint64_t n, uint64_t blk_lo, uint32_t G, uint32_t g)
{
	for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
	     i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
		rmax[i] = ((blk_lo + i) % G == g) ? 1u : 0u;
}

// K3: rank-ordered first killer for explicit pairs (engine.hpp:72-78), read
// straight from the packed reference bytes (sievetable.hpp:199-205).
__global__ void k_classify(const uint64_t* __restrict__ pq, uint64_t n,
                           const uint8_t* __restrict__ packed, const uint32_t* __restrict__ primes,
                           const uint32_t* __restrict__ offsets, uint32_t nprimes,
                           int32_t* __restrict__ out)
{
	for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
	     i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
		const uint64_t p = pq[2 * i], q = pq[2 * i + 1];
		int32_t rank = -1;
		for (uint32_t k = 0; k < nprimes; ++k) {
			const uint32_t r = primes[k];
			const uint64_t idx = (p % r) * r + (q % r);
			if ((packed[offsets[k] + (idx >> 3)] >> (idx & 7)) & 1) {
				rank = static_cast<int32_t>(k);
				break;
			}
		}
		out[i] = rank;
	}
}

template <int NR2, int NR3, bool STD = false, bool STOP = true, bool SHORT = false>
void* sieve_fn()
{
	return reinterpret_cast<void*>(&k_sieve<NR2, NR3, STD, STOP, SHORT>);
}

// Instantiated: NR2 in 0..8 with NR3 = 0, and NR2 = 7 (every prime 11..31
// killable -- all BASELINE sets) with NR3 in 1..kMaxReg3; the standard-prime
// kernel with and without the stop poll, each with the long- and short-row
// loop-variant sets.
void* sieve_kernel_ptr(int nr2, int nr3, bool std_primes, bool stop = true, bool short_rows = false)
{
	if (std_primes) {
		if (short_rows) return stop ? sieve_fn<7, 1, true, true, true>() : sieve_fn<7, 1, true, false, true>();
		return stop ? sieve_fn<7, 1, true, true>() : sieve_fn<7, 1, true, false>();
	}
	if (nr2 == 7 && nr3 > 0) {
		switch (nr3) {
		case 1: return sieve_fn<7, 1>();
		case 2: return sieve_fn<7, 2>();
		case 3: return sieve_fn<7, 3>();
		default: return sieve_fn<7, 4>();
		}
	}
	switch (nr2) {
	case 0: return sieve_fn<0, 0>();
	case 1: return sieve_fn<1, 0>();
	case 2: return sieve_fn<2, 0>();
	case 3: return sieve_fn<3, 0>();
	case 4: return sieve_fn<4, 0>();
	case 5: return sieve_fn<5, 0>();
	case 6: return sieve_fn<6, 0>();
	case 7: return sieve_fn<7, 0>();
	default: return sieve_fn<8, 0>();
	}
}

}  // namespace

__host__ __device__ size_t sieve_smem_bytes(uint32_t np, uint32_t tab_stride)
{
	return sizeof(uint32_t) * static_cast<size_t>(np) * kSieveWarps + sizeof(uint2) * kQueue * kSieveWarps +
	       sizeof(uint4) * kDeepPrefetch * kSieveWarps + sizeof(uint32_t) * 2 * tab_stride;
}

int sieve_grid(int device, int nr2, int nr3, bool std_primes, size_t smem)
{
	int sms = 0, per_sm = 0;
	cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
	const void* fn = sieve_kernel_ptr(nr2, nr3, std_primes);
	// Opt in to the device's full per-block shared memory once for every
	// variant: contexts with different probe sets share the kernel, so a
	// per-launch-size attribute set for one would reject another's launch.
	int optin = 0;
	cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
	const void* variants[4] = {fn, sieve_kernel_ptr(nr2, nr3, std_primes, false),
	                           sieve_kernel_ptr(nr2, nr3, std_primes, true, true),
	                           sieve_kernel_ptr(nr2, nr3, std_primes, false, true)};
	for (const void* f : variants) {
		cudaFuncAttributes fa{};
		cudaFuncGetAttributes(&fa, f);
		cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
		                     optin - static_cast<int>(fa.sharedSizeBytes));
	}
	cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSieveThreads, smem);
	if (per_sm < 1) per_sm = 1;
	return sms * per_sm;
}

__host__ __device__ size_t wsieve_smem_bytes(uint32_t np)
{
	return kWtBytes + static_cast<size_t>(kWheelWarps) * wheel_warp_bytes(np);
}

int wsieve_grid(int device, size_t smem)
{
	int sms = 0, per_sm = 0, optin = 0;
	cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
	cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
	const void* variants[2] = {wsieve_fn<true>(), wsieve_fn<false>()};
	for (const void* f : variants) {
		cudaFuncAttributes fa{};
		cudaFuncGetAttributes(&fa, f);
		cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - static_cast<int>(fa.sharedSizeBytes));
	}
	cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, variants[0], kWheelThreads, smem);
	if (per_sm < 1) per_sm = 1;
	return sms * per_sm;
}

cudaError_t launch_wheeltab(const uint32_t* d_ext, const uint32_t* reg_base, uint32_t* d_out, cudaStream_t s)
{
	WheelTabArgs t;
	for (int j = 0; j < kWheelReg; ++j) t.base[j] = reg_base[j];
	k_wheeltab<<<(kWtWords + 127) / 128, 128, 0, s>>>(d_ext, t, d_out);
	return cudaGetLastError();
}

cudaError_t launch_plan(const SieveArgs& a, cudaStream_t s)
{
	k_plan<<<plan_chunks(a.n_slots), kPlanChunk, 0, s>>>(a);
	return cudaGetLastError();
}

cudaError_t launch_sieve(const SieveArgs& a, int grid, cudaStream_t s)
{
	const size_t smem = sieve_smem_bytes(a.np, a.wtab_n ? (a.std_primes ? kTabStrideStd : kTabStrideGen) : 0);
	void* args[] = {const_cast<SieveArgs*>(&a)};
	if (a.wheel)
		return cudaLaunchKernel(a.stop != nullptr ? wsieve_fn<true>() : wsieve_fn<false>(), dim3(grid),
		                        dim3(kWheelThreads), args, wsieve_smem_bytes(a.np), s);
	return cudaLaunchKernel(sieve_kernel_ptr(static_cast<int>(a.nreg2), static_cast<int>(a.nreg3), a.std_primes,
	                                         a.stop != nullptr, a.short_rows != 0),
	                        dim3(grid),
	                        dim3(kSieveThreads), args, smem, s);
}

cudaError_t launch_init_blocks(uint32_t* d_block_rmax, uint64_t nblocks, uint64_t blk_lo,
                               uint32_t G, uint32_t g, cudaStream_t s)
{
	if (!nblocks) return cudaSuccess;
	const uint32_t grid = static_cast<uint32_t>(nblocks > 256 * 1024 ? 1024 : (nblocks + 255) / 256);
	k_init_blocks<<<grid, 256, 0, s>>>(d_block_rmax, nblocks, blk_lo, G, g);
	return cudaGetLastError();
}

cudaError_t launch_classify(const uint64_t* d_pq, uint64_t n, const uint8_t* d_packed,
                            const uint32_t* d_primes, const uint32_t* d_offsets, uint32_t nprimes,
                            int32_t* d_out, cudaStream_t s)
{
	if (!n) return cudaSuccess;
	const uint32_t grid = static_cast<uint32_t>(n > 256 * 4096 ? 4096 : (n + 255) / 256);
	k_classify<<<grid, 256, 0, s>>>(d_pq, n, d_packed, d_primes, d_offsets, nprimes, d_out);
	return cudaGetLastError();
}

#ifdef CGPU_WARP_CLOCKS
// experiment hook: per-warp {start, end, smid} of the last k_sieve launch
extern "C" int cgpu_debug_warp_clocks(unsigned long long* out, unsigned n)
{
	return cudaMemcpyFromSymbol(out, g_wclk, sizeof(unsigned long long) * 3 * (n < 8192 ? n : 8192)) ==
	               cudaSuccess
	           ? 0
	           : -1;
}
#endif

}  // namespace cgpu
