// K1: residue-table builder for sm_100a.
//
// Replaces build_table / build_table_oracle / SieveSet::build
// (/root/reference/proj/include/cuboid/sievetable.hpp:102-176). All arithmetic
// is 32-bit with Barrett reduction (common.cuh); tables are produced directly
// in the reference's packed LSB-first format by warp ballots, so the bytes are
// identical to the CPU builder's.
//
// Grids are 2-D: blockIdx.y selects the prime (jobs sorted by descending r so
// the heaviest primes are dispatched first), blockIdx.x strides over that
// prime's work units.

#include "common.cuh"
#include "kernels.cuh"

#include <algorithm>
#include <vector>

namespace cgpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

// Coefficients c4..c0 (c[0]..c[4]) of Q_pq as a monic quintic in s = t^2,
// reduced to [0, r) -- modpoly.hpp:86-114. Any exact reduction gives the same
// canonical residues; products of residues are < r^2 < 2^27.
__device__ __forceinline__ void mod_coeffs(uint32_t p, uint32_t q, uint32_t r, uint32_t m,
                                           uint32_t c[5])
{
	auto md = [r, m](uint32_t x) { return mod_full(x, r, m); };
	const uint32_t p2 = md(p * p), q2 = md(q * q);
	const uint32_t p4 = md(p2 * p2), q4 = md(q2 * q2);
	const uint32_t p6 = md(p4 * p2), q6 = md(q4 * q2);
	const uint32_t p8 = md(p4 * p4), q8 = md(q4 * q4);
	c[0] = md(md(2 * q2 + p2) * md(3 * q2 + 2 * r - 2 * p2));
	c[1] = md(q8 + 10 * md(p2 * q6) + 4 * md(p4 * q4) + 14 * (r - md(p6 * q2)) + p8);
	const uint32_t in = md(q8 + 14 * (r - md(p2 * q6)) + 4 * md(p4 * q4) + 10 * md(p6 * q2) + p8);
	c[2] = md(r - md(md(p2 * q2) * in));
	const uint32_t f1 = md(q2 + 2 * p2), f2 = md(3 * p2 + 2 * r - 2 * q2);
	c[3] = md(r - md(md(md(p6 * q6) * f1) * f2));
	c[4] = md(r - md(md(p8 * p2) * md(q8 * q2)));
}

// Horner in s (modpoly.hpp:116-125) with lazy Barrett: every intermediate
// stays in [0, 2r), so y = v*s + c < 2r^2 + r < 2^28. Returns v in [0, 2r);
// Q = 0 mod r iff v == 0 or v == r.
__device__ __forceinline__ uint32_t horner_lazy(const uint32_t c[5], uint32_t s, uint32_t r,
                                                uint32_t m)
{
	uint32_t v = s + c[0];
	v = mod_lazy(v * s + c[1], r, m);
	v = mod_lazy(v * s + c[2], r, m);
	v = mod_lazy(v * s + c[3], r, m);
	v = mod_lazy(v * s + c[4], r, m);
	return v;
}

// Writes one ballot word covering bits [i0, i0+32) of a table (i0 % 32 == 0)
// as 4 bytes, clipped to the table's ceil(r^2/8) bytes.
__device__ __forceinline__ void store_word_bytes(uint8_t* table, uint32_t tbytes, uint32_t i0,
                                                 uint32_t word, uint32_t lane)
{
	if (lane < 4) {
		const uint32_t bi = (i0 >> 3) + lane;
		if (bi < tbytes) table[bi] = static_cast<uint8_t>(word >> (8 * lane));
	}
}

// Exhaustive cube (sievetable.hpp:102-115 semantics, every t evaluated): the
// bit of (a,b) is 1 iff Q_ab(t) != 0 mod r for all t in Z_r. Each thread owns
// kCubePairs pairs (a,b) (strided by the CTA width so every ballot covers 32
// consecutive bits of the reference's global index) and evaluates
//     Q = s^5 + c4 s^4 + c3 s^3 + c2 s^2 + c1 s + c0   (s = t^2, modpoly.hpp:3-11)
// at every t. The powers s^k mod r depend only on t, so they are tabulated
// once per CTA in shared memory and read as broadcasts; per evaluation that
// leaves four IMADs into an accumulator A = c0 + c1 s + ... + c4 s^4 < 2^24
// and ONE more IMAD for the test: for odd r, r | x iff x * r^-1 (mod 2^32) <=
// (2^32 - 1) / r (divisibility by multiplicative inverse), and
// (A + s^5) r^-1 = A r^-1 + (s^5 r^-1) with the second term tabulated per t.
// A running minimum over t decides the bit. Same value as the reference's
// Horner (modpoly.hpp:116-125) with no reduction at all in the loop.
__global__ void __launch_bounds__(kCubeThreads) k_cube(const PrimeJob* __restrict__ jobs,
                                                       uint8_t* __restrict__ packed)
{
	extern __shared__ uint4 s_pw[];  // [r] {s, s^2, s^3, s^4} then [r] s^5 r^-1 mod 2^32
	const PrimeJob job = jobs[blockIdx.y];
	const uint32_t r = job.r, m = job.m;
	const uint32_t rr = r * r;
	const uint32_t per_cta = kCubeThreads * kCubePairs;
	if (blockIdx.x * per_cta >= rr) return;
	// r^-1 mod 2^32 by Newton iteration (r odd); r = 2 uses the Barrett test
	uint32_t rinv = r;
	for (int i = 0; i < 5; ++i) rinv *= 2u - r * rinv;
	const bool odd = r & 1;
	const uint32_t lim = 0xffffffffu / r;
	uint32_t* s_p5 = reinterpret_cast<uint32_t*>(s_pw + r);
	for (uint32_t t = threadIdx.x; t < r; t += blockDim.x) {
		const uint32_t s1 = mod_full(t * t, r, m);
		const uint32_t s2 = mod_full(s1 * s1, r, m);
		const uint32_t s3 = mod_full(s2 * s1, r, m);
		const uint32_t s4 = mod_full(s3 * s1, r, m);
		s_pw[t] = make_uint4(s1, s2, s3, s4);
		s_p5[t] = mod_full(s4 * s1, r, m) * (odd ? rinv : 1u);
	}
	__syncthreads();
	const uint32_t tbytes = (rr + 7) >> 3;
	const uint32_t lane = threadIdx.x & 31;
	for (uint32_t base = blockIdx.x * per_cta; base < rr; base += gridDim.x * per_cta) {
		uint32_t c0[kCubePairs], c1[kCubePairs], c2[kCubePairs], c3[kCubePairs], c4[kCubePairs];
		uint32_t mn[kCubePairs];  // min over t of (Q r^-1 mod 2^32): a root iff <= lim
		bool valid[kCubePairs];
#pragma unroll
		for (int k = 0; k < kCubePairs; ++k) {
			const uint32_t i = base + k * kCubeThreads + threadIdx.x;
			valid[k] = i < rr;
			uint32_t a = __umulhi(i, m), b = i - a * r;
			if (b >= r) { b -= r; ++a; }
			uint32_t c[5];
			mod_coeffs(valid[k] ? a : 0, valid[k] ? b : 0, r, m, c);
			c4[k] = c[0];
			c3[k] = c[1];
			c2[k] = c[2];
			c1[k] = c[3];
			c0[k] = c[4];
			mn[k] = 0xffffffffu;
		}
		if (odd) {
#pragma unroll 2
			for (uint32_t t = 0; t < r; ++t) {
				const uint4 p = s_pw[t];
				const uint32_t p5 = s_p5[t];
#pragma unroll
				for (int k = 0; k < kCubePairs; ++k) {
					uint32_t acc = c4[k] * p.w + c0[k];
					acc = c3[k] * p.z + acc;
					acc = c2[k] * p.y + acc;
					acc = c1[k] * p.x + acc;                  // < 4r^2 + r < 2^24
					mn[k] = min(mn[k], acc * rinv + p5);       // (A + s^5) r^-1 mod 2^32
				}
			}
		} else {  // r = 2: remainder by Barrett, shifted so that 0 means a root
			for (uint32_t t = 0; t < r; ++t) {
				const uint4 p = s_pw[t];
				const uint32_t p5 = s_p5[t];
#pragma unroll
				for (int k = 0; k < kCubePairs; ++k) {
					const uint32_t acc = c4[k] * p.w + c3[k] * p.z + c2[k] * p.y + c1[k] * p.x + c0[k] + p5;
					mn[k] = min(mn[k], mod_full(acc, r, m) ? lim + 1 : 0u);
				}
			}
		}
#pragma unroll
		for (int k = 0; k < kCubePairs; ++k) {
			const uint32_t word = __ballot_sync(kFull, valid[k] && mn[k] > lim);
			const uint32_t i0 = base + k * kCubeThreads + (threadIdx.x & ~31u);
			store_word_bytes(packed + job.byte_off, tbytes, i0, word, lane);
		}
	}
}

// Packed FP32 pair helpers (sm_100 FFMA2: two FMAs per lane per instruction;
// a broadcast scalar operand costs nothing -- ptxas folds {b, b} into it).
__device__ __forceinline__ unsigned long long f32x2(float x, float y)
{
	unsigned long long r;
	asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
	return r;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, float b, unsigned long long c)
{
	unsigned long long d;
	asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(f32x2(b, b)), "l"(c));
	return d;
}

// Balanced residue of x in [0, r): the representative in [-(r-1)/2, (r-1)/2].
__device__ __forceinline__ float balanced(uint32_t x, uint32_t r)
{
	return static_cast<float>(x <= r / 2 ? static_cast<int>(x) : static_cast<int>(x) - static_cast<int>(r));
}

// Exhaustive cube on the FP32 pipes, for odd r <= kCubeF2MaxR. Same bit as
// k_cube (and modpoly.hpp:116-125): Q_ab(t) = 0 mod r for some t.
//
// With the coefficients c_k and the powers s^k mod r in balanced form (|.| <=
// h = (r-1)/2), A = c0 + c1 s + c2 s^2 + c3 s^3 + c4 s^4 is an integer with
// |A| <= h + 4h^2 < 2^22 and so is every partial sum. Accumulated on top of
// M = 1.5 * 2^23 every FMA result is an integer in (2^23, 2^24), where the
// float grid is the integers: the four FMAs are exact, and the float's bit
// pattern is 0x4B400000 + A. Two (a,b) pairs share one FFMA2 (the s^k operand
// is broadcast). The root test is then the same divisibility-by-inverse as
// k_cube on x = A + s^5 + K r >= 0 (K r >= 2^22), folded into one IMAD:
//     x r^-1 = bits(v) r^-1 + w_t,   w_t = (s^5 + K r - 0x4B400000) r^-1,
// all mod 2^32, and r | x iff x r^-1 mod 2^32 <= (2^32 - 1) / r.
// Per evaluation: 2 FFMA2 (half of four) + 1 IMAD + 1 min, against k_cube's
// 5 IMAD + 1 min on the IMAD-only half of the FMA pipes. PAIRS = 16 pairs per
// thread amortise the shared-memory loads and loop control (measured on C2:
// 4 -> 61 ms, 8 -> 60 ms, 16 -> 56 ms, at 128 registers, 2 CTAs per SM).
template <int PAIRS>
__global__ void __launch_bounds__(kCubeThreads) k_cube_f2(const PrimeJob* __restrict__ jobs,
                                                          uint8_t* __restrict__ packed)
{
	extern __shared__ float4 s_b[];  // [r] balanced {s, s^2, s^3, s^4} then [r] w_t
	const PrimeJob job = jobs[blockIdx.y];
	const uint32_t r = job.r, m = job.m;
	const uint32_t rr = r * r;
	constexpr uint32_t per_cta = kCubeThreads * PAIRS;
	if (blockIdx.x * per_cta >= rr) return;
	uint32_t rinv = r;
	for (int i = 0; i < 5; ++i) rinv *= 2u - r * rinv;
	const uint32_t lim = 0xffffffffu / r;
	const uint32_t Kr = ((1u << 22) + r - 1) / r * r;
	uint32_t* s_w = reinterpret_cast<uint32_t*>(s_b + r);
	for (uint32_t t = threadIdx.x; t < r; t += blockDim.x) {
		const uint32_t s1 = mod_full(t * t, r, m);
		const uint32_t s2 = mod_full(s1 * s1, r, m);
		const uint32_t s3 = mod_full(s2 * s1, r, m);
		const uint32_t s4 = mod_full(s3 * s1, r, m);
		const uint32_t s5 = mod_full(s4 * s1, r, m);
		s_b[t] = make_float4(balanced(s1, r), balanced(s2, r), balanced(s3, r), balanced(s4, r));
		s_w[t] = (s5 + Kr - 0x4B400000u) * rinv;
	}
	__syncthreads();
	const uint32_t tbytes = (rr + 7) >> 3;
	const uint32_t lane = threadIdx.x & 31;
	constexpr int SC = kCubeF2Scalar;      // pairs on scalar FFMA (either FMA pipe)
	constexpr int NP = (PAIRS - SC) / 2;  // FFMA2 pair slots (heavy pipe)
	for (uint32_t base = blockIdx.x * per_cta; base < rr; base += gridDim.x * per_cta) {
		unsigned long long C1[NP > 0 ? NP : 1], C2[NP > 0 ? NP : 1], C3[NP > 0 ? NP : 1], C4[NP > 0 ? NP : 1],
		    V0[NP > 0 ? NP : 1];
		float S1[SC > 0 ? SC : 1], S2[SC > 0 ? SC : 1], S3[SC > 0 ? SC : 1], S4[SC > 0 ? SC : 1],
		    W0[SC > 0 ? SC : 1];
		uint32_t mn[PAIRS];
#pragma unroll
		for (int k = 0; k < SC; ++k) {
			const uint32_t i = base + (2 * NP + k) * kCubeThreads + threadIdx.x;
			uint32_t a = __umulhi(i, m), b = i - a * r;
			if (b >= r) { b -= r; ++a; }
			uint32_t cu[5];
			mod_coeffs(i < rr ? a : 0, i < rr ? b : 0, r, m, cu);
			S4[k] = balanced(cu[0], r);
			S3[k] = balanced(cu[1], r);
			S2[k] = balanced(cu[2], r);
			S1[k] = balanced(cu[3], r);
			W0[k] = 12582912.0f + balanced(cu[4], r);
			mn[2 * NP + k] = 0xffffffffu;
		}
#pragma unroll
		for (int j = 0; j < NP; ++j) {
			float c[2][5];
#pragma unroll
			for (int h = 0; h < 2; ++h) {
				const uint32_t i = base + (2 * j + h) * kCubeThreads + threadIdx.x;
				uint32_t a = __umulhi(i, m), b = i - a * r;
				if (b >= r) { b -= r; ++a; }
				uint32_t cu[5];
				mod_coeffs(i < rr ? a : 0, i < rr ? b : 0, r, m, cu);  // c4, c3, c2, c1, c0
#pragma unroll
				for (int k = 0; k < 5; ++k) c[h][k] = balanced(cu[k], r);
				mn[2 * j + h] = 0xffffffffu;
			}
			C4[j] = f32x2(c[0][0], c[1][0]);
			C3[j] = f32x2(c[0][1], c[1][1]);
			C2[j] = f32x2(c[0][2], c[1][2]);
			C1[j] = f32x2(c[0][3], c[1][3]);
			V0[j] = f32x2(12582912.0f + c[0][4], 12582912.0f + c[1][4]);
		}
#pragma unroll 2
		for (uint32_t t = 0; t < r; ++t) {
			const float4 bp = s_b[t];
			const uint32_t w = s_w[t];
			// the NP chains are independent; ptxas interleaves them as it sees
			// fit (forcing the order with volatile asm measured no faster)
			unsigned long long v[NP];
#pragma unroll
			for (int j = 0; j < NP; ++j) v[j] = ffma2(C4[j], bp.w, V0[j]);
#pragma unroll
			for (int j = 0; j < NP; ++j) v[j] = ffma2(C3[j], bp.z, v[j]);
#pragma unroll
			for (int j = 0; j < NP; ++j) v[j] = ffma2(C2[j], bp.y, v[j]);
#pragma unroll
			for (int j = 0; j < NP; ++j) v[j] = ffma2(C1[j], bp.x, v[j]);
#pragma unroll
			for (int j = 0; j < NP; ++j) {
				mn[2 * j] = min(mn[2 * j], static_cast<uint32_t>(v[j]) * rinv + w);
				mn[2 * j + 1] = min(mn[2 * j + 1], static_cast<uint32_t>(v[j] >> 32) * rinv + w);
			}
#pragma unroll
			for (int k = 0; k < SC; ++k) {
				float x = fmaf(S4[k], bp.w, W0[k]);
				x = fmaf(S3[k], bp.z, x);
				x = fmaf(S2[k], bp.y, x);
				x = fmaf(S1[k], bp.x, x);
				mn[2 * NP + k] = min(mn[2 * NP + k], __float_as_uint(x) * rinv + w);
			}
		}
#pragma unroll
		for (int k = 0; k < PAIRS; ++k) {
			const uint32_t i = base + k * kCubeThreads + threadIdx.x;
			const uint32_t word = __ballot_sync(kFull, i < rr && mn[k] > lim);
			store_word_bytes(packed + job.byte_off, tbytes, i - lane, word, lane);
		}
	}
}

__device__ __forceinline__ uint32_t pow_mod(uint32_t a, uint32_t e, uint32_t r, uint32_t m)
{
	uint32_t x = 1 % r;
	while (e) {
		if (e & 1) x = mod_full(x * a, r, m);
		a = mod_full(a * a, r, m);
		e >>= 1;
	}
	return x;
}

// Production row 1 (sievetable.hpp:128-132 via row_solvable :91-96, t <= r/2
// with early exit) and the inverse table used by the permutation
// (primes.hpp:33-46; here by Fermat). One thread per q.
__global__ void __launch_bounds__(kRow1Threads) k_row1(const PrimeJob* __restrict__ jobs,
                                                       uint8_t* __restrict__ row1,
                                                       uint32_t* __restrict__ inv,
                                                       unsigned long long* __restrict__ evals)
{
	const PrimeJob job = jobs[blockIdx.y];
	const uint32_t r = job.r, m = job.m;
	unsigned long long n = 0;
	for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < r; q += gridDim.x * blockDim.x) {
		uint32_t c[5];
		mod_coeffs(1, q, r, m, c);
		bool solvable = false;
		for (uint32_t t = 0; t <= r / 2; ++t) {
			++n;
			const uint32_t v = horner_lazy(c, mod_full(t * t, r, m), r, m);
			if (v == 0 || v == r) {
				solvable = true;
				break;
			}
		}
		row1[job.aux_off + q] = solvable ? 0 : 1;
		inv[job.aux_off + q] = q ? pow_mod(q, r - 2, r, m) : 0;
	}
	for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(kFull, n, o);
	if ((threadIdx.x & 31) == 0 && n) atomicAdd(evals, n);
}

// Production rows a >= 1: row[a][q] = row1[a^{-1} q mod r]; row 0 is zero
// (sievetable.hpp:133-139). One thread per bit, packed by ballot.
// Row a >= 1 of the production table is row 1 permuted (homogeneity,
// sievetable.hpp:117-141): bit (a, q) = row1[a^-1 q mod r]; row 0 is zero.
// One thread per 32-bit word of the table's bit stream: it walks its 32 bits
// with the row index stepped by a^-1 (mod r) per q, reading row 1 and the
// inverses from shared memory, and stores its 4 bytes. (One thread per bit
// with a ballot per word: 200 us for the 256-prime set.)
__global__ void __launch_bounds__(kPermThreads) k_permute(const PrimeJob* __restrict__ jobs,
                                                          const uint8_t* __restrict__ row1,
                                                          const uint32_t* __restrict__ inv,
                                                          uint8_t* __restrict__ packed)
{
	extern __shared__ uint32_t s_perm[];  // [r] inverses, then [r] row-1 bytes
	const PrimeJob job = jobs[blockIdx.y];
	const uint32_t r = job.r, m = job.m;
	const uint32_t rr = r * r, tbytes = (rr + 7) >> 3, nwords = (rr + 31) >> 5;
	if (blockIdx.x * kPermThreads >= nwords) return;
	uint32_t* s_inv = s_perm;
	uint8_t* s_row1 = reinterpret_cast<uint8_t*>(s_perm + r);
	for (uint32_t k = threadIdx.x; k < r; k += blockDim.x) {
		s_inv[k] = inv[job.aux_off + k];
		s_row1[k] = row1[job.aux_off + k];
	}
	__syncthreads();
	uint8_t* table = packed + job.byte_off;
	for (uint32_t w = blockIdx.x * kPermThreads + threadIdx.x; w < nwords; w += gridDim.x * kPermThreads) {
		const uint32_t i0 = 32 * w;
		uint32_t a = __umulhi(i0, m), q = i0 - a * r;
		if (q >= r) { q -= r; ++a; }
		uint32_t ainv = s_inv[a];
		uint32_t idx = mod_full(ainv * q, r, m);
		uint32_t word = 0;
		const uint32_t nb = min(32u, rr - i0);
		for (uint32_t l = 0; l < nb; ++l) {
			if (a) word |= static_cast<uint32_t>(s_row1[idx]) << l;
			idx += ainv;
			if (idx >= r) idx -= r;
			if (++q == r) {  // next row
				q = 0;
				idx = 0;
				if (++a < r) ainv = s_inv[a];
			}
		}
		const uint32_t b0 = 4 * w;
#pragma unroll
		for (uint32_t k = 0; k < 4; ++k)
			if (b0 + k < tbytes) table[b0 + k] = static_cast<uint8_t>(word >> (8 * k));
	}
}

// Packed reference tables -> row-extended words (common.cuh ext_row_words):
// word j of row a holds bits u(a, (32j + l) mod r), l = 0..31. One CTA per
// work item {job, first row, rows} (built on the host, <= kDeriveItemWords
// output words each): one thread stages the item's packed bytes in shared
// memory with a single TMA bulk copy (cp.async.bulk, completion on an
// mbarrier; the item's bits are one contiguous byte range), then each thread
// builds output words from it (one or two funnel shifts across the row wrap)
// and stores them coalesced; killable[k] bit 0 is set when any word written
// for table k is nonzero, bit 1 when the loaded row 0 holds a set bit. Row 0
// is written as zeros unless keep_row0: scan() skips primes with p mod r = 0
// (engine.hpp:240-242), while the TRIANGLE loop's is_unsolvable reads the row
// like any other (sievetable.hpp:199-205, engine.hpp:619-623); canonical
// tables have a zero row 0 anyway, so the two layouts differ only for
// non-canonical loaded bytes. (Per-word gathers straight from L2 were
// latency-bound: 113-145 us for the 256-prime set; a thread-strided staging
// loop of word loads 29.9 us, 31% of it waiting on those loads.)
__global__ void __launch_bounds__(kDeriveThreads, kDeriveMinBlocks) k_derive(const PrimeJob* __restrict__ jobs,
                                                           const uint4* __restrict__ items,
                                                           const uint8_t* __restrict__ packed,
                                                           uint32_t* __restrict__ ext,
                                                           uint32_t* __restrict__ killable,
                                                           int keep_row0)
{
	extern __shared__ uint4 s_raw[];  // 16-byte aligned staging of the item's bytes
	__shared__ __align__(8) unsigned long long s_mbar;
	const uint32_t* s_bits = reinterpret_cast<const uint32_t*>(s_raw);
	const uint4 it = items[blockIdx.x];  // {job, first row, rows, -}
	const PrimeJob job = jobs[it.x];
	const uint32_t r = job.r, S = ext_row_words(r);
	// global bit range of the rows, staged from its 16-byte aligned first byte
	const uint64_t bit0 = 8ull * job.byte_off + static_cast<uint64_t>(it.y) * r;
	const uint32_t nbits = it.z * r;
	const uint64_t byte_lo = (bit0 >> 3) & ~15ull;
	const uint64_t byte_hi = (((bit0 + nbits + 7) >> 3) + 8 + 15) & ~15ull;  // + a word past the end
	const uint32_t nbytes = static_cast<uint32_t>(byte_hi - byte_lo);
	const uint32_t mbar = static_cast<uint32_t>(__cvta_generic_to_shared(&s_mbar));
	if (threadIdx.x == 0) {
		asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar));
		asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
		asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(nbytes) : "memory");
		asm volatile(
		    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
		        static_cast<uint32_t>(__cvta_generic_to_shared(s_raw))),
		    "l"(packed + byte_lo), "r"(nbytes), "r"(mbar)
		    : "memory");
	}
	if (threadIdx.x == 0)  // one waiter; the others sleep in the barrier instead of spinning
		asm volatile(
		    "{\n\t.reg .pred done;\n"
		    "WAIT_%=:\n\t"
		    "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n\t"
		    "@!done bra WAIT_%=;\n}" ::"r"(mbar)
		    : "memory");
	__syncthreads();
	const uint32_t sh = static_cast<uint32_t>(bit0 - 8 * byte_lo);  // bit offset of row it.y in s_bits
	// 32 bits starting at local bit i of the staged rows
	auto bits32 = [&](uint32_t i) {
		const uint32_t li = i + sh;
		return __funnelshift_r(s_bits[li >> 5], s_bits[(li >> 5) + 1], li & 31);
	};
	bool any = false, row0_set = false;
	const uint32_t words = it.z * S;
	const uint32_t mS = barrett_m(S);
	const uint32_t m = job.m;
	const uint64_t E0 = job.ext_base + static_cast<uint64_t>(it.y) * S;  // first output word
	if (r >= 32) {
		// Each thread writes one 16-byte aligned group of 4 output words (one
		// vector store; partial groups at the item's ends store word by word):
		// the row/word split is computed once per group and stepped after.
		const uint64_t g0 = E0 & ~3ull;
		const uint32_t ngroups = static_cast<uint32_t>((E0 + words - g0 + 3) >> 2);
		for (uint32_t gi = threadIdx.x; gi < ngroups; gi += blockDim.x) {
			const uint64_t A = g0 + 4ull * gi;
			const int64_t w0 = static_cast<int64_t>(A) - static_cast<int64_t>(E0);  // local word of slot 0
			const uint32_t wf = w0 < 0 ? 0u : static_cast<uint32_t>(w0);
			uint32_t a = __umulhi(wf, mS), j = wf - a * S;  // local row, word in row
			if (j >= S) { j -= S; ++a; }
			uint32_t v[4];
			bool in[4];
#pragma unroll
			for (int q = 0; q < 4; ++q) {
				const int64_t wl = w0 + q;
				in[q] = wl >= 0 && wl < static_cast<int64_t>(words);
				v[q] = 0;
				if (!in[q]) continue;
				uint32_t b = 32 * j;  // 32 j < r + 32 <= 2 r: one conditional subtraction
				if (b >= r) b -= r;
				const uint32_t row0 = a * r, head = r - b;  // at most one wrap: [b, r) then [0, 32 - head)
				uint32_t word = bits32(row0 + b);
				if (head < 32) word = (word & ((1u << head) - 1)) | (bits32(row0) << head);
				if (it.y + a == 0) {  // row p = 0 mod r: scan() never probes it (engine.hpp:240-242)
					row0_set |= word != 0;
					if (!keep_row0) word = 0;
				}
				v[q] = word;
				any |= word != 0;
				if (++j == S) {
					j = 0;
					++a;
				}
			}
			if (in[0] && in[3]) {
				*reinterpret_cast<uint4*>(ext + A) = make_uint4(v[0], v[1], v[2], v[3]);
			} else {
#pragma unroll
				for (int q = 0; q < 4; ++q)
					if (in[q]) ext[A + q] = v[q];
			}
		}
	} else {  // small r: the row repeats inside one word
		for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {
			uint32_t a = __umulhi(w, mS), j = w - a * S;
			if (j >= S) { j -= S; ++a; }
			uint32_t b = mod_full(32 * j, r, m);
			const uint32_t row = bits32(a * r) & ((1u << r) - 1);
			uint32_t word = 0;
#pragma unroll 8
			for (uint32_t l = 0; l < 32; ++l) {
				word |= ((row >> b) & 1u) << l;
				b = b + 1 == r ? 0 : b + 1;
			}
			if (it.y + a == 0) {
				row0_set |= word != 0;
				if (!keep_row0) word = 0;
			}
			ext[E0 + w] = word;
			any |= word != 0;
		}
	}
	const bool any_cta = __syncthreads_or(any);
	const bool row0_cta = __syncthreads_or(row0_set);
	if (threadIdx.x == 0 && (any_cta || row0_cta))
		atomicOr(&killable[it.x], (any_cta ? 1u : 0u) | (row0_cta ? 2u : 0u));
}

// Window tables for the sieve's table probes: entry (j, a, b) -- for probe j
// (prime r), row a = p mod r, offset b -- is the 32-q mask of that row at b
// (bits u(a, (b + l) mod r)), and the entry index of the lane's next window
// (a, (b + 1024) mod r). One thread per entry.
__global__ void __launch_bounds__(kDeriveThreads, kDeriveMinBlocks) k_wintab(const uint4* __restrict__ probes, uint32_t nprobes, uint32_t entries,
                         const uint32_t* __restrict__ ext, uint32_t stride, uint32_t* __restrict__ out)
{
	for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < entries; e += gridDim.x * blockDim.x) {
		uint32_t j = 0;
		while (j + 1 < nprobes && e >= probes[j + 1].w) ++j;
		const uint4 d = probes[j];  // {r, ext_base, S, base}
		const uint32_t r = d.x, i = e - d.w, a = i / r, b = i - a * r;
		const uint32_t* row = ext + d.y + a * d.z;
		const uint32_t k = b >> 5;  // 0, or 1 for 3-word rows
		out[e] = __funnelshift_r(row[k], row[k + 1], b);
		out[stride + e] = d.w + a * r + (b + 1024u) % r;
	}
}

// FormatError check (sievetable.hpp:67-79): bits >= r^2 of the last byte of
// each table must be zero.
__global__ void k_check_padding(const PrimeJob* __restrict__ jobs, uint32_t njobs,
                                const uint8_t* __restrict__ packed, uint32_t* __restrict__ bad)
{
	for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < njobs; k += gridDim.x * blockDim.x) {
		const uint32_t r = jobs[k].r;
		const uint32_t nbits = r * r, tbytes = (nbits + 7) >> 3;
		const uint32_t used = nbits & 7;
		if (used) {
			const uint8_t last = packed[jobs[k].byte_off + tbytes - 1];
			if (last >> used) atomicOr(bad, 1u);
		}
	}
}

// Verification of a speculative (asynchronous) load: the derive's per-table
// flags (bit 0 killable, bit 1 row 0 has a set bit) against the ones the host
// built the probe list from, and the padding check's flag at kf[n].
// *status = padding error (1) | flag mismatch (2); the host reads it later.
__global__ void k_load_check(const uint32_t* __restrict__ kf, const uint8_t* __restrict__ expect, uint32_t n,
                             uint32_t* __restrict__ status)
{
	uint32_t bad = 0;
	for (uint32_t k = threadIdx.x; k < n; k += blockDim.x)
		if ((kf[k] & 3u) != expect[k]) bad = 2;
	bad = __syncthreads_or(bad) ? 2u : 0u;
	if (threadIdx.x == 0) *status = bad | (kf[n] ? 1u : 0u);
}

uint32_t grid_x(uint64_t units, uint32_t per_cta, uint32_t cap)
{
	const uint64_t x = (units + per_cta - 1) / per_cta;
	return static_cast<uint32_t>(x < 1 ? 1 : (x > cap ? cap : x));
}

}  // namespace

// Jobs are sorted by descending r. Odd r <= kCubeF2MaxR (every BASELINE set)
// run on the FP32 pipes (k_cube_f2); larger r and r = 2 (the last job when
// present) on the IMAD path (k_cube). One launch per contiguous group.
cudaError_t launch_cube(const PrimeJob* d_jobs, const PrimeJob* h_jobs, uint32_t njobs, uint8_t* d_packed,
                        cudaStream_t s)
{
	if (!njobs) return cudaSuccess;
	uint32_t nbig = 0;
	while (nbig < njobs && h_jobs[nbig].r > kCubeF2MaxR) ++nbig;
	const bool two = h_jobs[njobs - 1].r == 2;
	const uint32_t f2_end = two ? njobs - 1 : njobs;
	auto int_launch = [&](uint32_t j0, uint32_t n) {
		const uint32_t r0 = h_jobs[j0].r;  // largest of the group
		const dim3 grid(grid_x(static_cast<uint64_t>(r0) * r0, kCubeThreads * kCubePairs, 8192), n);
		const size_t smem = (sizeof(uint4) + sizeof(uint32_t)) * r0;
		if (smem > 48 * 1024)
			cudaFuncSetAttribute(k_cube, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
		k_cube<<<grid, kCubeThreads, smem, s>>>(d_jobs + j0, d_packed);
	};
	if (nbig) int_launch(0, nbig);
	if (f2_end > nbig) {
		const uint32_t r0 = h_jobs[nbig].r;
		const dim3 grid(grid_x(static_cast<uint64_t>(r0) * r0, kCubeThreads * kCubeF2Pairs, 8192), f2_end - nbig);
		const size_t smem = (sizeof(float4) + sizeof(uint32_t)) * r0;  // 40 KB at r = 2039
		k_cube_f2<kCubeF2Pairs><<<grid, kCubeThreads, smem, s>>>(d_jobs + nbig, d_packed);
	}
	if (two && njobs - 1 >= nbig) int_launch(njobs - 1, 1);
	return cudaGetLastError();
}

uint32_t cube_launches(const PrimeJob* h_jobs, uint32_t njobs)
{
	if (!njobs) return 0;
	uint32_t nbig = 0;
	while (nbig < njobs && h_jobs[nbig].r > kCubeF2MaxR) ++nbig;
	const bool two = h_jobs[njobs - 1].r == 2;
	const uint32_t f2_end = two ? njobs - 1 : njobs;
	return (nbig ? 1 : 0) + (f2_end > nbig ? 1 : 0) + (two && njobs - 1 >= nbig ? 1 : 0);
}

cudaError_t launch_row1(const PrimeJob* d_jobs, uint32_t njobs, uint32_t max_r, uint8_t* d_row1,
                        uint32_t* d_inv, unsigned long long* d_evals, cudaStream_t s)
{
	if (!njobs) return cudaSuccess;
	const dim3 grid(grid_x(max_r, kRow1Threads, 128), njobs);
	k_row1<<<grid, kRow1Threads, 0, s>>>(d_jobs, d_row1, d_inv, d_evals);
	return cudaGetLastError();
}

cudaError_t launch_permute(const PrimeJob* d_jobs, uint32_t njobs, uint32_t max_rr,
                           const uint8_t* d_row1, const uint32_t* d_inv, uint8_t* d_packed,
                           cudaStream_t s)
{
	if (!njobs) return cudaSuccess;
	const uint32_t max_r = static_cast<uint32_t>(sqrt(static_cast<double>(max_rr)) + 0.5);
	const dim3 grid(grid_x((max_rr + 31) / 32, kPermThreads, 32), njobs);  // one thread per table word
	const size_t smem = 5ull * max_r + 16;                               // inverses + row-1 bytes
	if (smem > 48 * 1024)
		cudaFuncSetAttribute(k_permute, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
	k_permute<<<grid, kPermThreads, smem, s>>>(d_jobs, d_row1, d_inv, d_packed);
	return cudaGetLastError();
}

cudaError_t launch_wintab(const uint4* d_probes, uint32_t nprobes, uint32_t entries, const uint32_t* d_ext,
                          uint32_t stride, uint32_t* d_out, cudaStream_t s)
{
	if (!entries) return cudaSuccess;
	k_wintab<<<(entries + kDeriveThreads - 1) / kDeriveThreads, kDeriveThreads, 0, s>>>(d_probes, nprobes, entries,
	                                                                                   d_ext, stride, d_out);
	return cudaGetLastError();
}

cudaError_t launch_derive(const PrimeJob* d_jobs, const uint4* d_items, uint32_t nitems, const uint8_t* d_packed,
                          uint32_t* d_ext, uint32_t* d_killable, int keep_row0, cudaStream_t s)
{
	if (!nitems) return cudaSuccess;
	// staged bytes: <= kDeriveItemWords output words cover <= kDeriveItemWords * 32 bits, plus the
	// 16-byte alignment of both ends and a word past the last byte
	const size_t smem = sizeof(uint32_t) * kDeriveItemWords + 48;
	k_derive<<<nitems, kDeriveThreads, smem, s>>>(d_jobs, d_items, d_packed, d_ext, d_killable, keep_row0);
	return cudaGetLastError();
}

std::vector<uint4> derive_items(const std::vector<uint32_t>& primes)
{
	std::vector<uint4> items;
	for (uint32_t k = 0; k < primes.size(); ++k) {
		const uint32_t r = primes[k], S = ext_row_words(r);
		const uint32_t R = std::max<uint32_t>(1, kDeriveItemWords / S);  // rows per item
		for (uint32_t a = 0; a < r; a += R) items.push_back(make_uint4(k, a, std::min(R, r - a), 0));
	}
	return items;
}

cudaError_t launch_load_check(const uint32_t* d_kf, const uint8_t* d_expect, uint32_t n, uint32_t* d_status,
                              cudaStream_t s)
{
	k_load_check<<<1, kDeriveThreads, 0, s>>>(d_kf, d_expect, n, d_status);
	return cudaGetLastError();
}

cudaError_t launch_check_padding(const PrimeJob* d_jobs, uint32_t njobs, const uint8_t* d_packed,
                                 uint32_t* d_bad, cudaStream_t s)
{
	if (!njobs) return cudaSuccess;
	k_check_padding<<<(njobs + 127) / 128, 128, 0, s>>>(d_jobs, njobs, d_packed, d_bad);
	return cudaGetLastError();
}

}  // namespace cgpu
