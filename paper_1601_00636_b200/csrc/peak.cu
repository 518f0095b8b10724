// Measured INT32 denominators for the roofline (MEASURED_PEAKS.json has only
// HBM and bf16): chains of LOP3 (ALU pipe), IMAD (FMA pipe) and both
// interleaved, over a full-chip grid, timed with CUDA events.

#include "../../include/cuboid_gpu.h"
#include "kernels.cuh"

namespace cgpu {
namespace {

constexpr int kChains = 8;
constexpr int kIters = 2048;
constexpr int kPeakThreads = 256;

// mode 0: LOP3 only; 1: IMAD only; 2: one IMAD + one LOP3 per step (3 register
// sources each); 3: IMAD + IADD3 with immediate operands (fewer register-file
// reads: the issue-bound ceiling of one warp instruction per clock per SMSP).
template <int MODE>
__global__ void __launch_bounds__(kPeakThreads) k_int_peak(uint32_t seed, uint32_t* sink)
{
	uint32_t x[kChains], y[kChains];
#pragma unroll
	for (int i = 0; i < kChains; ++i) {
		x[i] = seed + threadIdx.x * 7 + i;
		y[i] = seed ^ (blockIdx.x * 13 + i);
	}
	const uint32_t a = seed | 1, b = seed >> 3, c = seed * 5;
	for (int it = 0; it < kIters; ++it) {
#pragma unroll
		for (int i = 0; i < kChains; ++i) {
			if (MODE == 3) {
				asm volatile("mad.lo.u32 %0, %0, 0x9E3779B1, %1;" : "+r"(x[i]) : "r"(y[i]));
				asm volatile("lop3.b32 %0, %0, %1, 0x7F4A7C15, 0x96;" : "+r"(y[i]) : "r"(x[i]));
				continue;
			}
			if (MODE != 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
			if (MODE != 1)
				asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(c), "r"(x[i]));
		}
	}
	uint32_t acc = 0;
#pragma unroll
	for (int i = 0; i < kChains; ++i) acc ^= x[i] ^ y[i];
	if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the chains live
}

// FP32-pipe chains for the exhaustive table build (k_cube_f2, tables.cu).
// MODE 4: FFMA2 only (3 register sources; 2 lane-FMAs per instruction).
// MODE 5: the k_cube_f2 evaluation mix, loop-carried so nothing is hoisted:
// per chain step 4 FFMA2 (broadcast scalar operand) feeding 2 IMAD and 2
// unsigned mins -- 2 evaluations per step.
template <int MODE>
__global__ void __launch_bounds__(kPeakThreads) k_fp_peak(uint32_t seed, uint32_t* sink)
{
	unsigned long long v[kChains];
	uint32_t mn[2 * kChains];
	const float fs = static_cast<float>((seed ^ threadIdx.x) & 7);
	unsigned long long c, c2;
	asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(fs + 1.0f), "f"(fs + 2.0f));
	asm("mov.b64 %0, {%1, %2};" : "=l"(c2) : "f"(fs + 3.0f), "f"(fs + 4.0f));
	float b = fs * 0.5f;
	uint32_t w = (seed >> 5) + threadIdx.x;
	const uint32_t rinv = (seed ^ threadIdx.x) | 1;
#pragma unroll
	for (int i = 0; i < kChains; ++i) {
		asm("mov.b64 %0, {%1, %2};" : "=l"(v[i]) : "f"(fs + i), "f"(fs - i));
		mn[2 * i] = mn[2 * i + 1] = 0xffffffffu;
	}
	for (int it = 0; it < kIters; ++it) {
#pragma unroll
		for (int i = 0; i < kChains; ++i) {
			if (MODE == 4) {
				asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[i]) : "l"(c), "l"(v[(i + 1) % kChains]));
				continue;
			}
			unsigned long long bb;
			asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
			asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v[i]) : "l"(c), "l"(bb));
			asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v[i]) : "l"(c2), "l"(bb));
			asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v[i]) : "l"(c), "l"(bb));
			asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(v[i]) : "l"(c2), "l"(bb));
			const uint32_t lo = static_cast<uint32_t>(v[i]), hi = static_cast<uint32_t>(v[i] >> 32);
			uint32_t x0, x1;
			asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x0) : "r"(lo), "r"(rinv), "r"(w));
			asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x1) : "r"(hi), "r"(rinv), "r"(w));
			mn[2 * i] = min(mn[2 * i], x0);
			mn[2 * i + 1] = min(mn[2 * i + 1], x1);
		}
		b += 1.0f;  // per-t operands change every step (as the shared-memory powers do)
		w += 3;
	}
	uint32_t acc = 0;
#pragma unroll
	for (int i = 0; i < kChains; ++i)
		acc ^= static_cast<uint32_t>(v[i]) ^ static_cast<uint32_t>(v[i] >> 32) ^ mn[2 * i] ^ mn[2 * i + 1];
	if (acc == 0x9e3779b9u) sink[0] = acc;
}

}  // namespace

// out[0] = FFMA2 lane-FMAs/s (3-register chains), out[1] = k_cube_f2
// evaluation-mix evaluations/s (the table build's instruction-mix ceiling).
cudaError_t run_fp_peak(int device, double out[2])
{
	int sms = 0;
	cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
	if (e != cudaSuccess) return e;
	uint32_t* sink = nullptr;
	if ((e = cudaMalloc(&sink, 4)) != cudaSuccess) return e;
	cudaEvent_t t0, t1;
	cudaEventCreate(&t0);
	cudaEventCreate(&t1);
	const int grid = sms * 8;
	const double threads = static_cast<double>(grid) * kPeakThreads;
	void (*fns[2])(uint32_t, uint32_t*) = {k_fp_peak<4>, k_fp_peak<5>};
	const double per_thread[2] = {2.0 * kIters * kChains, 2.0 * kIters * kChains};
	for (int m = 0; m < 2 && e == cudaSuccess; ++m) {
		float best = 1e30f;
		for (int rep = 0; rep < 5; ++rep) {
			cudaEventRecord(t0);
			fns[m]<<<grid, kPeakThreads>>>(0x1234567u + rep, sink);
			cudaEventRecord(t1);
			if ((e = cudaEventSynchronize(t1)) != cudaSuccess) break;
			float ms = 0;
			cudaEventElapsedTime(&ms, t0, t1);
			if (rep && ms < best) best = ms;
		}
		out[m] = threads * per_thread[m] / (best * 1e-3);
	}
	if (e == cudaSuccess) e = cudaGetLastError();
	cudaEventDestroy(t0);
	cudaEventDestroy(t1);
	cudaFree(sink);
	return e;
}

cudaError_t run_int_peak(int device, double out[4])
{
	int sms = 0;
	cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
	if (e != cudaSuccess) return e;
	uint32_t* sink = nullptr;
	if ((e = cudaMalloc(&sink, 4)) != cudaSuccess) return e;
	cudaEvent_t t0, t1;
	cudaEventCreate(&t0);
	cudaEventCreate(&t1);
	const int grid = sms * 8;  // 8 CTAs x 8 warps = 64 warps per SM
	const double threads = static_cast<double>(grid) * kPeakThreads;
	void (*fns[4])(uint32_t, uint32_t*) = {k_int_peak<0>, k_int_peak<1>, k_int_peak<2>,
	                                       k_int_peak<3>};
	const double ops_per_thread[4] = {1.0 * kIters * kChains, 1.0 * kIters * kChains,
	                                  2.0 * kIters * kChains, 2.0 * kIters * kChains};
	for (int m = 0; m < 4 && e == cudaSuccess; ++m) {
		float best = 1e30f;
		for (int rep = 0; rep < 5; ++rep) {
			cudaEventRecord(t0);
			fns[m]<<<grid, kPeakThreads>>>(0x1234567u + rep, sink);
			cudaEventRecord(t1);
			if ((e = cudaEventSynchronize(t1)) != cudaSuccess) break;
			float ms = 0;
			cudaEventElapsedTime(&ms, t0, t1);
			if (rep && ms < best) best = ms;  // rep 0 is warm-up
		}
		out[m] = threads * ops_per_thread[m] / (best * 1e-3);
	}
	if (e == cudaSuccess) e = cudaGetLastError();
	cudaEventDestroy(t0);
	cudaEventDestroy(t1);
	cudaFree(sink);
	return e;
}

}  // namespace cgpu
