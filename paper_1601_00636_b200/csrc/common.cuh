// Shared device helpers and the host-side layout of a resident table set.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// Device-side bounds checks, compiled in only for the debug build
// (make EXTRA=-DCGPU_DEBUG ...): a violated check traps the kernel, which the
// host sees as a CUDA error. compute-sanitizer is unavailable on this pool.
#ifdef CGPU_DEBUG
#define CGPU_CHECK(cond)          \
	do {                          \
		if (!(cond)) __trap();    \
	} while (0)
#else
#define CGPU_CHECK(cond) \
	do {                 \
	} while (0)
#endif

namespace cgpu {

constexpr uint32_t kModulusLimit = 9697;      // primes.hpp:12
constexpr uint64_t kPLimit32 = (1ull << 32) / 59;  // region.hpp:43-44 (59p < 2^32)
constexpr uint32_t kRegionCrossover = 152;    // region.hpp:41

// Barrett constant for a modulus r in [2, 2^16): m = floor(2^32 / r).
// For x < 2^32, x - umulhi(x, m) * r lies in [0, 2r).
__host__ __device__ inline uint32_t barrett_m(uint32_t r)
{
	return static_cast<uint32_t>((1ull << 32) / r);
}

__device__ __forceinline__ uint32_t mod_lazy(uint32_t x, uint32_t r, uint32_t m)
{
	return x - __umulhi(x, m) * r;  // [0, 2r)
}

__device__ __forceinline__ uint32_t mod_full(uint32_t x, uint32_t r, uint32_t m)
{
	const uint32_t v = mod_lazy(x, r, m);
	return min(v, v - r);  // unsigned: v - r wraps high when v < r
}

// shl with PTX clamping (shift >= 32 yields 0), used for sparse period masks.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s)
{
	uint32_t y;
	asm("shl.b32 %0, %1, %2;" : "=r"(y) : "r"(x), "r"(s));
	return y;
}

// Words per row of the row-extended ("ext") device layout of prime r: row a
// holds bits j in [0, 32*S) with bit j = u_r(a, j mod r). A 32-bit window
// starting at any b in [0, r) is funnel(word[b>>5], word[(b>>5)+1], b&31).
__host__ __device__ inline uint32_t ext_row_words(uint32_t r) { return ((r + 31) >> 5) + 1; }

// Periodic mask with bits at 0, f, 2f, ... (< 32); f > 32 -> single bit.
__host__ __device__ inline uint32_t period_mask(uint32_t f)
{
	uint32_t m = 0;
	for (uint32_t i = 0; i < 32; i += f) m |= 1u << i;
	return m;
}

}  // namespace cgpu
