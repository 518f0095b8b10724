// K2: the (p,q) pair sieve for sm_100a, and K3 (classify).
//
// Replaces the inner loops of scan() (/root/reference/proj/include/cuboid/
// engine.hpp:225-284) and the TRIANGLE loop of verify_small_region
// (engine.hpp:613-625). Semantics, bit for bit:
//   * candidates: q in the row bounds, q != p, gcd(p, q) == 1 (engine.hpp:258);
//   * probes in rank order, first set bit u_r(p mod r, q mod r) kills
//     (engine.hpp:261-269); the first killer is histogrammed by rank;
//   * survivors are emitted as (p << 32) | q and sorted on the host;
//   * per p/100 block, the largest killing prime (1 if none) (:229-236, 271).
//
// Design: bit-sliced. One thread owns a 32-wide window of
// consecutive q in one row p; a probe for prime r is ONE funnel shift of two
// words of the row-extended table (row p mod r, starting at bit q0 mod r),
// so a single probe answers 32 pairs. Warps own contiguous slices of the
// linearised (row, window) space, so each warp does its per-row setup (trial
// division of p, per-prime row bases) once per row and then streams windows.
// The leading probe primes below 32 live entirely in registers (two words
// per row); deeper probes read the ext rows through L1. Tables that never
// kill (all-zero, e.g. r = 3, 5, 7) are not probed -- identical results.

#include "../../include/cuboid_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

namespace cgpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kStepQ = 32 * 32;  // q advance per warp iteration per lane

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
	}
	return b;
}

__device__ __forceinline__ uint64_t row_windows(const RowBounds& b)
{
	return b.qhi >= b.qlo ? (b.qhi - b.qlo + 32) / 32 : 0;
}

// Work units of a row for load balancing: its 32-q windows plus a fixed
// charge for the per-row setup (trial division of p, per-prime row bases),
// measured at ~150 window-equivalents. Without it the warps that own the
// many short rows at small p straggle (C4: one SM busy 5x longer than the rest).
constexpr uint32_t kRowCost = 160;

__device__ __forceinline__ uint64_t row_units(const RowBounds& b)
{
	const uint64_t w = row_windows(b);
	return w ? w + kRowCost : 0;
}

// Plan: exclusive prefix of windows over row slots (one CTA).
__global__ void __launch_bounds__(1024) k_plan(const SieveArgs a, unsigned long long* prefix)
{
	__shared__ unsigned long long s_part[1024];
	const uint32_t n = a.n_slots;
	const uint32_t per = (n + blockDim.x - 1) / blockDim.x;
	const uint32_t s0 = threadIdx.x * per;
	const uint32_t s1 = min(n, s0 + per);
	unsigned long long sum = 0;
	for (uint32_t s = s0; s < s1; ++s) sum += row_units(slot_row(a, s));
	s_part[threadIdx.x] = sum;
	__syncthreads();
	for (uint32_t off = 1; off < blockDim.x; off <<= 1) {
		const unsigned long long v = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
		__syncthreads();
		s_part[threadIdx.x] += v;
		__syncthreads();
	}
	unsigned long long run = s_part[threadIdx.x] - sum;
	for (uint32_t s = s0; s < s1; ++s) {
		prefix[s] = run;
		run += row_units(slot_row(a, s));
	}
	if (threadIdx.x == blockDim.x - 1) prefix[n] = s_part[blockDim.x - 1];
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v)
{
	for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
	return v;
}

template <int NREG>
__global__ void __launch_bounds__(kSieveThreads) k_sieve(const SieveArgs a)
{
	extern __shared__ uint4 s_dyn[];
	__shared__ unsigned long long s_pairs;
	const uint32_t lane = threadIdx.x & 31;
	const uint32_t wib = threadIdx.x >> 5;
	uint4* s_desc = s_dyn + static_cast<size_t>(wib) * a.np;  // per-warp {rowbase, r, m, -}
	// per-CTA first-killer counts by probe index, after all warps' descriptors
	unsigned long long* s_hist =
	    reinterpret_cast<unsigned long long*>(s_dyn + static_cast<size_t>(kSieveWarps) * a.np);

	for (uint32_t j = threadIdx.x; j < a.np; j += blockDim.x) s_hist[j] = 0;
	if (threadIdx.x == 0) s_pairs = 0;
	__syncthreads();

	const unsigned long long W = a.prefix[a.n_slots];
	const unsigned long long nwarps = static_cast<unsigned long long>(gridDim.x) * kSieveWarps;
	const unsigned long long gw = static_cast<unsigned long long>(blockIdx.x) * kSieveWarps + wib;
	unsigned long long ws = W * gw / nwarps;  // W < 2^40, nwarps < 2^20
	const unsigned long long we = W * (gw + 1) / nwarps;

	// 32-ary warp search: largest slot s with prefix[s] <= ws
	uint32_t lo = 0, hi = a.n_slots;
	if (ws < we) {
		while (hi - lo > 1) {
			const uint32_t step = (hi - lo + 31) / 32;
			const uint32_t idx = lo + step * lane;
			const bool le = idx < hi && a.prefix[idx] <= ws;
			const uint32_t L = 31 - __clz(__ballot_sync(kFull, le));
			lo += step * L;
			hi = min(hi, lo + step);
		}
	}

	unsigned long long pairs = 0;
	uint32_t slot = lo;
	while (ws < we) {
		const unsigned long long rs = a.prefix[slot], re = a.prefix[slot + 1];
		if (re <= ws) {
			++slot;
			continue;
		}
		// this warp's share of the row's units; the first kRowCost are the
		// setup charge, the rest map 1:1 to windows
		const unsigned long long u0 = ws - rs, u1 = min(we, re) - rs;
		ws = min(we, re);
		const uint32_t cur = slot++;
		if (u1 <= kRowCost) continue;
		const uint32_t w0 = static_cast<uint32_t>(u0 > kRowCost ? u0 - kRowCost : 0);
		const uint32_t w1 = static_cast<uint32_t>(u1 - kRowCost);
		const RowBounds rb = slot_row(a, cur);
		const uint32_t p = static_cast<uint32_t>(rb.p);
		const uint32_t qlo = static_cast<uint32_t>(rb.qlo);
		const uint32_t qhi = static_cast<uint32_t>(rb.qhi);

		// ---- row setup: distinct prime factors of p (trial division) ----
		uint32_t fac[kMaxFactors];
		uint32_t nf = 0;
		{
			uint32_t cof = p;
			for (uint32_t base = 0; base < a.n_fprimes; base += 32) {
				const uint32_t i = base + lane;
				uint2 fp = make_uint2(0xffffffffu, 0);
				if (i < a.n_fprimes) fp = __ldg(a.fprimes + i);
				const bool in_range = i < a.n_fprimes && static_cast<uint64_t>(fp.x) * fp.x <= p;
				const bool divides = in_range && mod_full(p, fp.x, fp.y) == 0;
				uint32_t hits = __ballot_sync(kFull, divides);
				while (hits) {
					const uint32_t src = __ffs(hits) - 1;
					hits &= hits - 1;
					const uint32_t f = __shfl_sync(kFull, fp.x, src);
					const uint32_t fm = __shfl_sync(kFull, fp.y, src);
					if (nf < kMaxFactors) fac[nf] = f;
					++nf;
					// divide f out of the cofactor
					for (;;) {
						const uint32_t qt = __umulhi(cof, fm);
						uint32_t rem = cof - qt * f, qq = qt;
						if (rem >= f) { rem -= f; ++qq; }
						if (rem) break;
						cof = qq;
					}
				}
				if (!__any_sync(kFull, in_range)) break;
			}
			if (cof > 1 && nf < kMaxFactors) fac[nf++] = cof;  // the prime factor above sqrt(p)
		}
		// per-factor state: offset of the first multiple in the lane's window,
		// per-step decrement, period pattern
		uint32_t fo[kMaxFactors], fd[kMaxFactors], fpat[kMaxFactors], ff[kMaxFactors];
		const uint32_t q0_first = qlo + 32 * (w0 + lane);
#pragma unroll
		for (int k = 0; k < kMaxFactors; ++k) {
			if (k < nf) {
				const uint32_t f = fac[k];
				const uint32_t b = q0_first % f;
				ff[k] = f;
				fo[k] = b ? f - b : 0;
				fd[k] = kStepQ % f;
				fpat[k] = period_mask(f);
			}
		}

		// ---- per-prime row bases: registers for the leading probes, smem for the rest
		uint32_t rw0[NREG > 0 ? NREG : 1], rw1[NREG > 0 ? NREG : 1], rb_[NREG > 0 ? NREG : 1];
		uint32_t cnt[NREG > 0 ? NREG : 1];
#pragma unroll
		for (int j = 0; j < NREG; ++j) {
			const uint32_t r = a.reg_r[j], m = a.reg_m[j];
			const uint32_t row = a.reg_base[j] + mod_full(p, r, m) * 2;  // S = 2 for r <= 31
			rw0[j] = __ldg(a.ext + row);
			rw1[j] = __ldg(a.ext + row + 1);
			rb_[j] = mod_full(q0_first, r, m);
			cnt[j] = 0;
		}
		for (uint32_t j = NREG + lane; j < a.np; j += 32) {
			const uint4 d = __ldg(a.probes + j);
			s_desc[j] = make_uint4(d.z + mod_full(p, d.x, d.y) * d.w, d.x, d.y, 0);
		}
		__syncwarp();

		uint32_t deep_max = 0;  // 1 + largest deep probe index with a kill (0: none)
		uint32_t row_pairs = 0;
		const uint32_t n_iter = (w1 - w0 + 31) / 32;
		for (uint32_t it = 0; it < n_iter; ++it) {
			const uint32_t w = w0 + lane + 32 * it;
			const uint32_t q0 = qlo + 32 * w;
			uint32_t alive = 0;
			if (w < w1) {
				const uint32_t span = qhi - q0;  // q0 <= qhi for w < w1
				alive = span >= 31 ? kFull : ((2u << span) - 1);
				if (p == 1 && q0 == 1) alive &= ~1u;  // q == p (engine.hpp:258)
			}
			uint32_t nonc = 0;
#pragma unroll
			for (int k = 0; k < kMaxFactors; ++k) {
				if (k < nf) {
					nonc |= shl_clamp(fpat[k], fo[k]);
					const uint32_t t = fo[k] - fd[k];
					fo[k] = min(t, t + ff[k]);
				}
			}
			alive &= ~nonc;
			row_pairs += __popc(alive);
#pragma unroll
			for (int j = 0; j < NREG; ++j) {
				const uint32_t M = __funnelshift_r(rw0[j], rw1[j], rb_[j]);
				const uint32_t k = alive & M;
				cnt[j] += __popc(k);
				alive ^= k;
				const uint32_t t = rb_[j] + a.reg_delta[j];
				rb_[j] = min(t, t - a.reg_r[j]);
			}
			if (alive) {
				for (uint32_t j = NREG; j < a.np; ++j) {
					const uint4 d = s_desc[j];
					const uint32_t b = mod_full(q0, d.y, d.z);
					const uint32_t* wp = a.ext + d.x + (b >> 5);
					const uint32_t M = __funnelshift_r(__ldg(wp), __ldg(wp + 1), b);
					const uint32_t k = alive & M;
					if (k) {
						atomicAdd(&s_hist[j], static_cast<unsigned long long>(__popc(k)));
						deep_max = max(deep_max, j + 1);
						alive ^= k;
						if (!alive) break;
					}
				}
			}
			// survivors: warp-aggregated reservation, then (p<<32)|q records
			if (__any_sync(kFull, alive)) {
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
					if (base < a.surv_cap)
						a.surv[base] = (static_cast<unsigned long long>(p) << 32) | (q0 + bit);
					++base;
				}
			}
		}

		// ---- row flush: histogram (register probes), block r_max
		uint32_t kmax = 0;
		bool any_kill = false;
#pragma unroll
		for (int j = 0; j < NREG; ++j) {
			const uint32_t s = warp_sum(cnt[j]);
			if (s) {
				if (lane == 0) atomicAdd(&s_hist[j], static_cast<unsigned long long>(s));
				kmax = j;
				any_kill = true;
			}
		}
		const uint32_t dmax = __reduce_max_sync(kFull, deep_max);
		if (dmax) {
			kmax = dmax - 1;
			any_kill = true;
		}
		if (lane == 0 && any_kill) {
			const uint32_t killer = kmax < NREG ? a.reg_r[kmax < NREG ? kmax : 0] : s_desc[kmax].y;
			atomicMax(&a.block_rmax[rb.p / 100 - a.blk_lo], killer);
		}
		pairs += warp_sum(row_pairs);
		__syncwarp();
	}
	if (lane == 0 && pairs) atomicAdd(&s_pairs, pairs);
	__syncthreads();
	for (uint32_t j = threadIdx.x; j < a.np; j += blockDim.x)
		if (s_hist[j]) atomicAdd(&a.hist[__ldg(a.probe_rank + j)], s_hist[j]);
	if (threadIdx.x == 0 && s_pairs) atomicAdd(&a.counters[0], s_pairs);
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

template <int NREG>
void* sieve_fn()
{
	return reinterpret_cast<void*>(&k_sieve<NREG>);
}

void* sieve_kernel_ptr(int nreg)
{
	switch (nreg) {
	case 0: return sieve_fn<0>();
	case 1: return sieve_fn<1>();
	case 2: return sieve_fn<2>();
	case 3: return sieve_fn<3>();
	case 4: return sieve_fn<4>();
	case 5: return sieve_fn<5>();
	case 6: return sieve_fn<6>();
	case 7: return sieve_fn<7>();
	default: return sieve_fn<8>();
	}
}

}  // namespace

size_t sieve_smem_bytes(uint32_t np)
{
	return sizeof(uint4) * static_cast<size_t>(np) * kSieveWarps + sizeof(unsigned long long) * np;
}

int sieve_grid(int device, int nreg, size_t smem)
{
	int sms = 0, per_sm = 0;
	cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
	const void* fn = sieve_kernel_ptr(nreg);
	if (smem > 48 * 1024)
		cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
	cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSieveThreads, smem);
	if (per_sm < 1) per_sm = 1;
	return sms * per_sm;
}

cudaError_t launch_plan(const SieveArgs& a, unsigned long long* d_prefix, cudaStream_t s)
{
	k_plan<<<1, 1024, 0, s>>>(a, d_prefix);
	return cudaGetLastError();
}

cudaError_t launch_sieve(const SieveArgs& a, int grid, cudaStream_t s)
{
	const size_t smem = sieve_smem_bytes(a.np);
	void* args[] = {const_cast<SieveArgs*>(&a)};
	return cudaLaunchKernel(sieve_kernel_ptr(static_cast<int>(a.nreg)), dim3(grid),
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

}  // namespace cgpu
