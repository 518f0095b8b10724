// C ABI (include/cuboid_gpu.h): device context, resident table sets, sieve
// launches and result collection. No exceptions cross the boundary; status
// codes mirror the reference's exceptions (see the header).

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cuboid_gpu.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace cgpu;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg)
{
	g_err = msg;
	return code;
}

#define CK(call)                                                                            \
	do {                                                                                    \
		const cudaError_t e_ = (call);                                                      \
		if (e_ != cudaSuccess)                                                              \
			return set_err(CGPU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
	} while (0)

template <class T>
struct DevBuf {
	T* p = nullptr;
	size_t n = 0;
	~DevBuf() { release(); }
	void release()
	{
		if (p) cudaFree(p);
		p = nullptr;
		n = 0;
	}
	cudaError_t ensure(size_t want)
	{
		if (want <= n && p) return cudaSuccess;
		release();
		const size_t bytes = sizeof(T) * (want ? want : 1);
		cudaError_t e = cudaMalloc(&p, bytes);
		if (e == cudaSuccess) n = want ? want : 1;
		return e;
	}
};

bool is_prime_u32(uint32_t n)  // primes.hpp:14-21
{
	if (n < 2) return false;
	if (n % 2 == 0) return n == 2;
	for (uint32_t d = 3; d * d <= n; d += 2)
		if (n % d == 0) return false;
	return true;
}

uint64_t table_bytes(uint32_t r) { return (static_cast<uint64_t>(r) * r + 7) / 8; }

// SieveSet::build validation order (sievetable.hpp:159-176, 83-87).
int layout(const uint32_t* primes, uint32_t n, uint32_t* offsets, uint64_t* total)
{
	if (n && !primes) return set_err(CGPU_ERR_INVALID, "null prime list");
	uint64_t off = 0;
	uint32_t prev = 0;
	for (uint32_t k = 0; k < n; ++k) {
		const uint32_t r = primes[k];
		if (r <= prev)
			return set_err(CGPU_ERR_INVALID, "SieveSet::build: primes must be strictly increasing");
		prev = r;
		if (r < 2 || r >= kModulusLimit || !is_prime_u32(r))
			return set_err(CGPU_ERR_INVALID, "bit table modulus must be a prime below 9697");
		if (off + table_bytes(r) > UINT32_MAX)
			return set_err(CGPU_ERR_OVERFLOW,
			               "SieveSet::build: table set exceeds 32-bit offset space");
		if (offsets) offsets[k] = static_cast<uint32_t>(off);
		off += table_bytes(r);
	}
	if (total) *total = off;
	return CGPU_OK;
}

uint64_t q_lower_cubic(uint64_t p)  // region.hpp:25-39
{
	uint64_t lo = 1, hi = 1;
	auto ge = [p](uint64_t q) { return 9 * (static_cast<unsigned __int128>(q) * q * q) >= p; };
	while (!ge(hi)) hi *= 2;
	while (lo < hi) {
		const uint64_t mid = lo + (hi - lo) / 2;
		if (ge(mid)) hi = mid; else lo = mid + 1;
	}
	return lo;
}

void q_bounds(uint64_t p, uint64_t* lo, uint64_t* hi)  // region.hpp:49-63
{
	*hi = 59 * p;
	if (p < kRegionCrossover) {
		const uint64_t c = (p + 58) / 59;
		*lo = c < 1 ? 1 : c;
	} else {
		*lo = q_lower_cubic(p);
	}
}

constexpr uint64_t kIndexHeaderSize = 9;  // sievetable.hpp:148-151
constexpr uint64_t kIndexRecordSize = 6;
constexpr uint8_t kIndexVersion = 1;

constexpr uint32_t kMaxSlots = 1u << 20;  // row slots per plan/sieve launch (multiple of 100 below)
constexpr uint32_t kBlocksPerLaunch = kMaxSlots / 100;

}  // namespace

// shared with multi.cu (internal.cuh)
int cgpu_internal_set_err(int code, const std::string& msg) { return set_err(code, msg); }

struct cgpu_ctx {
	int device = 0;
	cudaStream_t stream = nullptr;
	bool own_stream = false;
	int sms = 0;

	// resident set
	bool loaded = false;
	std::vector<uint32_t> primes, offsets, ext_base;
	std::vector<uint8_t> killable;
	// row 0 (p = 0 mod r) of the derived layout: zeroed for REGION (scan()
	// skips those primes, engine.hpp:240-242), as loaded for TRIANGLE when a
	// non-canonical set has bits there (is_unsolvable reads it)
	bool keep_row0 = false, row0_nonzero = false;
	// asynchronous (speculative) loads: the per-table flags the probe list was
	// built from, the last verified flags of a prime list, and the device word
	// k_load_check writes (padding error | flag mismatch << 1)
	std::vector<uint32_t> flags_primes;
	std::vector<uint8_t> flags;
	std::vector<uint8_t> spec_flags;
	bool flags_valid = false, status_pending = false;
	DevBuf<uint8_t> d_expect;
	DevBuf<uint32_t> load_status;
	uint64_t total_bytes = 0, ext_words = 0;
	DevBuf<uint8_t> packed;
	DevBuf<uint32_t> ext, d_primes, d_offsets, killflags;
	DevBuf<PrimeJob> jobs_rank;

	// probe list
	uint32_t np = 0, nreg = 0, nreg2 = 0, nreg3 = 0;
	bool std_primes = false;
	std::vector<uint32_t> probe_rank, probe_r;
	DevBuf<uint4> probes;
	uint32_t reg_r[kMaxReg] = {}, reg_m[kMaxReg] = {}, reg_base[kMaxReg] = {}, reg_delta[kMaxReg] = {};
	uint32_t reg_tab[kMaxReg] = {}, wtab_n = 0;
	DevBuf<uint4> d_tabprobes;
	DevBuf<uint4> derive_items;
	DevBuf<uint32_t> wintab;
	// wheel sieve (k_wsieve) for the standard probe sets: CUBOID_WHEEL=0 keeps k_sieve
	int wheel_mode = 1;  // CUBOID_WHEEL: 0 never, 1 for launches of long rows (kWheelMinWindows), 2 always
	bool wheel = false;
	DevBuf<uint32_t> wheeltab;
	int wgrid = 0;
	uint32_t row_cost_wheel = kDefaultRowCostWheel;
	float wheel_cost[4] = {kDefaultWheelCost[0], kDefaultWheelCost[1], kDefaultWheelCost[2], kDefaultWheelCost[3]};
	int grid = 0;
	std::map<uint64_t, int> grid_cache;

	uint32_t row_cost = kDefaultRowCost;
	uint32_t row_cost_short = kDefaultRowCostShort;
	float drain_alpha = kDefaultDrainAlpha;
	int short_rows = -1;  // CUBOID_SHORT_ROWS: -1 by mean row length, 0 / 1 forced
	DevBuf<uint2> fprimes;
	uint32_t n_fprimes = 0;

	// pinned staging ring for uploads from pageable host memory (upload_pageable)
	static constexpr size_t kStageBytes = size_t(4) << 20;
	uint8_t* stage[2] = {nullptr, nullptr};
	cudaEvent_t stage_ev[2] = {nullptr, nullptr};

	// cooperative stop word (cgpu_set_stop_word): device view of a mapped host word
	const volatile uint32_t* stop_dev = nullptr;

	// sieve buffers
	DevBuf<unsigned long long> hist, counters, surv, prefix, chunk_off;
	DevBuf<uint32_t> tickets, rowfac;
	DevBuf<uint32_t> d_probe_rank;
	DevBuf<uint32_t> block_rmax;
	bool launched = false, results_internal = false, timed = false, last_wheel = false;
	uint64_t last_nblocks = 0, last_surv_cap = 0;
	cudaEvent_t ev[3] = {};
	float timings[3] = {};
	uint32_t launches = 0;

	// scratch
	DevBuf<uint8_t> row1;
	DevBuf<uint32_t> inv;
	DevBuf<unsigned long long> evals;
	DevBuf<PrimeJob> jobs_build;
	DevBuf<uint64_t> pq;
	DevBuf<int32_t> ranks;
};

extern "C" {

const char* cgpu_last_error(void) { return g_err.c_str(); }

const char* cgpu_version(void) { return "cuboid-gpu 0.1 sm_100a"; }

int cgpu_q_bounds(uint64_t p, uint64_t* q_low, uint64_t* q_high)
{
	if (p == 0) return set_err(CGPU_ERR_INVALID, "q_bounds: p must be positive");
	if (p > UINT64_MAX / 59) return set_err(CGPU_ERR_OVERFLOW, "q_bounds: 59p exceeds 64 bits");
	q_bounds(p, q_low, q_high);
	return CGPU_OK;
}

int cgpu_table_layout(const uint32_t* primes, uint32_t n, uint32_t* offsets, uint64_t* total_bytes)
{
	return layout(primes, n, offsets, total_bytes);
}

int cgpu_create(int device, void* stream, cgpu_ctx** out)
{
	if (!out) return set_err(CGPU_ERR_INVALID, "null out");
	*out = nullptr;
	int count = 0;
	if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
		return set_err(CGPU_ERR_NO_DEVICE, "no CUDA device visible: cuboid_gpu has no CPU fallback");
	if (device < 0 || device >= count) return set_err(CGPU_ERR_INVALID, "device index out of range");
	CK(cudaSetDevice(device));
	auto* c = new cgpu_ctx;
	c->device = device;
	if (stream) {
		c->stream = static_cast<cudaStream_t>(stream);
	} else {
		if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
			delete c;
			return set_err(CGPU_ERR_CUDA, "cudaStreamCreate failed");
		}
		c->own_stream = true;
	}
	cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
	if (const char* rc = std::getenv("CUBOID_ROW_COST")) c->row_cost = static_cast<uint32_t>(std::atoi(rc));
	if (const char* rs = std::getenv("CUBOID_ROW_COST_SHORT"))
		c->row_cost_short = static_cast<uint32_t>(std::atoi(rs));
	if (const char* da = std::getenv("CUBOID_DRAIN_ALPHA")) c->drain_alpha = static_cast<float>(std::atof(da));
	if (const char* wh = std::getenv("CUBOID_WHEEL")) c->wheel_mode = std::atoi(wh);
	if (const char* rw = std::getenv("CUBOID_ROW_COST_WHEEL")) c->row_cost_wheel = static_cast<uint32_t>(std::atoi(rw));
	if (const char* wc = std::getenv("CUBOID_WHEEL_COSTS"))  // "base,mid,large,queued" instructions
		std::sscanf(wc, "%f,%f,%f,%f", &c->wheel_cost[0], &c->wheel_cost[1], &c->wheel_cost[2], &c->wheel_cost[3]);
	if (const char* sr = std::getenv("CUBOID_SHORT_ROWS")) c->short_rows = std::atoi(sr) < 0 ? -1 : (std::atoi(sr) ? 1 : 0);
	for (auto& e : c->ev) cudaEventCreate(&e);
	// trial-division primes below 2^16 (covers sqrt of any p < 2^32)
	std::vector<uint2> fp;
	{
		std::vector<uint8_t> comp(65536, 0);
		for (uint32_t i = 2; i < 65536; ++i) {
			if (comp[i]) continue;
			fp.push_back(make_uint2(i, barrett_m(i)));
			for (uint32_t j = i * i; j < 65536; j += i) comp[j] = 1;
		}
	}
	c->n_fprimes = static_cast<uint32_t>(fp.size());
	if (c->fprimes.ensure(fp.size()) != cudaSuccess ||
	    cudaMemcpy(c->fprimes.p, fp.data(), sizeof(uint2) * fp.size(), cudaMemcpyHostToDevice) !=
	        cudaSuccess) {
		delete c;
		return set_err(CGPU_ERR_CUDA, "device allocation failed");
	}
	*out = c;
	return CGPU_OK;
}

int cgpu_destroy(cgpu_ctx* c)
{
	if (!c) return CGPU_OK;
	cudaSetDevice(c->device);
	cudaStreamSynchronize(c->stream);
	for (auto& e : c->ev)
		if (e) cudaEventDestroy(e);
	for (int i = 0; i < 2; ++i) {
		if (c->stage[i]) cudaFreeHost(c->stage[i]);
		if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
	}
	if (c->own_stream) cudaStreamDestroy(c->stream);
	delete c;
	return CGPU_OK;
}

int cgpu_set_stream(cgpu_ctx* c, void* stream)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	CK(cudaSetDevice(c->device));
	CK(cudaStreamSynchronize(c->stream));
	if (c->own_stream) cudaStreamDestroy(c->stream);
	c->own_stream = false;
	c->stream = static_cast<cudaStream_t>(stream);
	if (!stream) {
		CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
		c->own_stream = true;
	}
	return CGPU_OK;
}

int cgpu_synchronize(cgpu_ctx* c)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	CK(cudaSetDevice(c->device));
	CK(cudaStreamSynchronize(c->stream));
	return CGPU_OK;
}

}  // extern "C"

namespace {

std::vector<PrimeJob> make_jobs(const std::vector<uint32_t>& primes,
                                const std::vector<uint32_t>& offsets, std::vector<uint32_t>& ext_base,
                                uint64_t& ext_words)
{
	std::vector<PrimeJob> jobs(primes.size());
	ext_base.resize(primes.size());
	uint64_t ext = 0, aux = 0;
	for (size_t k = 0; k < primes.size(); ++k) {
		const uint32_t r = primes[k];
		jobs[k] = PrimeJob{r, barrett_m(r), offsets[k], static_cast<uint32_t>(ext),
		                   static_cast<uint32_t>(aux), 0};
		ext_base[k] = static_cast<uint32_t>(ext);
		ext += static_cast<uint64_t>(r) * ext_row_words(r);
		aux += r;
	}
	ext_words = ext;
	return jobs;
}

// After the packed bytes are resident: derive ext rows + killable flags, then
// build the probe list (killable tables in rank order).
// check_padding: a k_check_padding flag was enqueued into killflags[n]; it
// is read back with the killable flags (one host sync per load).
int finalize_set(cgpu_ctx* c, bool check_padding = false, bool keep_row0 = false,
                 const std::vector<uint8_t>* spec = nullptr)
{
	const uint32_t n = static_cast<uint32_t>(c->primes.size());
	std::vector<PrimeJob> jobs = make_jobs(c->primes, c->offsets, c->ext_base, c->ext_words);
	if (c->ext_words >= (1ull << 32))
		return set_err(CGPU_ERR_OVERFLOW, "row-extended layout exceeds 2^32 words");
	CK(c->jobs_rank.ensure(n));
	CK(c->ext.ensure(c->ext_words));
	CK(c->killflags.ensure(n + 1));
	CK(c->d_primes.ensure(n));
	CK(c->d_offsets.ensure(n));
	if (n) {
		CK(cudaMemcpyAsync(c->jobs_rank.p, jobs.data(), sizeof(PrimeJob) * n, cudaMemcpyHostToDevice,
		                   c->stream));
		CK(cudaMemcpyAsync(c->d_primes.p, c->primes.data(), 4ull * n, cudaMemcpyHostToDevice, c->stream));
		CK(cudaMemcpyAsync(c->d_offsets.p, c->offsets.data(), 4ull * n, cudaMemcpyHostToDevice,
		                   c->stream));
		CK(cudaMemsetAsync(c->killflags.p, 0, 4ull * n, c->stream));
		const std::vector<uint4> items = derive_items(c->primes);
		CK(c->derive_items.ensure(items.size()));
		CK(cudaMemcpyAsync(c->derive_items.p, items.data(), sizeof(uint4) * items.size(), cudaMemcpyHostToDevice,
		                   c->stream));
		CK(launch_derive(c->jobs_rank.p, c->derive_items.p, static_cast<uint32_t>(items.size()), c->packed.p,
		                 c->ext.p, c->killflags.p, keep_row0 ? 1 : 0, c->stream));
		++c->launches;
	}
	std::vector<uint32_t> kf(n + 1, 0);
	if (spec) {  // asynchronous load: build from the expected flags, verify on the device
		for (uint32_t k = 0; k < n; ++k) kf[k] = (*spec)[k];
		CK(c->d_expect.ensure(n));
		CK(c->load_status.ensure(1));
		if (n) {
			CK(cudaMemcpyAsync(c->d_expect.p, spec->data(), n, cudaMemcpyHostToDevice, c->stream));
			if (!check_padding) CK(cudaMemsetAsync(c->killflags.p + n, 0, 4, c->stream));
			CK(launch_load_check(c->killflags.p, c->d_expect.p, n, c->load_status.p, c->stream));
			++c->launches;
		} else {
			CK(cudaMemsetAsync(c->load_status.p, 0, 4, c->stream));
		}
		c->status_pending = true;
		c->spec_flags = *spec;
	} else {
		const uint32_t nread = n + (check_padding ? 1 : 0);
		if (nread) CK(cudaMemcpyAsync(kf.data(), c->killflags.p, 4ull * nread, cudaMemcpyDeviceToHost, c->stream));
		CK(cudaStreamSynchronize(c->stream));
		if (check_padding && kf[n]) return set_err(CGPU_ERR_FORMAT, "unpack_bits: nonzero padding bits");
		c->status_pending = false;
		c->flags_primes = c->primes;
		c->flags.assign(n, 0);
		for (uint32_t k = 0; k < n; ++k) c->flags[k] = static_cast<uint8_t>(kf[k] & 3u);
		c->flags_valid = true;
	}
	c->killable.assign(n, 0);
	c->probe_rank.clear();
	c->probe_r.clear();
	c->keep_row0 = keep_row0;
	c->row0_nonzero = false;
	std::vector<uint4> pr;
	for (uint32_t k = 0; k < n; ++k) {
		c->row0_nonzero |= (kf[k] & 2u) != 0;
		c->killable[k] = (kf[k] & 1u) ? 1 : 0;
		if (!(kf[k] & 1u)) continue;  // an all-zero table never kills: skipping it is exact
		const uint32_t r = c->primes[k];
		c->probe_rank.push_back(k);
		c->probe_r.push_back(r);
		pr.push_back(make_uint4(r, barrett_m(r), c->ext_base[k], ext_row_words(r)));
	}
	c->np = static_cast<uint32_t>(pr.size());
	// register probes: the leading killable primes <= 31 (two-word rows), then,
	// when all of 11..31 are among them, up to kMaxReg3 primes in (31, 63]
	c->nreg = c->nreg2 = c->nreg3 = 0;
	uint32_t cap2 = kMaxReg2, cap3 = kStdReg3;
	if (const char* e = std::getenv("CUBOID_MAX_REG_PROBES")) cap2 = std::min<uint32_t>(cap2, std::atoi(e));
	if (const char* e = std::getenv("CUBOID_REG3_PROBES")) cap3 = std::min<uint32_t>(kMaxReg3, std::atoi(e));
	auto add_reg = [&](uint32_t j) {
		const uint32_t r = c->probe_r[j];
		c->reg_r[j] = r;
		c->reg_m[j] = barrett_m(r);
		c->reg_base[j] = pr[j].z;
		c->reg_delta[j] = (32u * 32u) % r;
		++c->nreg;
	};
	while (c->nreg < c->np && c->nreg2 < cap2 && c->probe_r[c->nreg] <= 31) {
		add_reg(c->nreg);
		++c->nreg2;
	}
	const bool all_small = c->nreg2 == 7 && c->probe_r[0] == 11 && c->probe_r[6] == 31;
	auto tab_fits = [&](uint32_t extra) {  // window tables of the table probes within kTabStrideGen
		uint32_t e = extra;
		for (uint32_t j = 0; j < c->nreg && j < static_cast<uint32_t>(kTabProbes); ++j) e += c->reg_r[j] * c->reg_r[j];
		return e <= kTabStrideGen;
	};
	while (all_small && c->nreg < c->np && c->nreg3 < cap3 && c->probe_r[c->nreg] <= 63 &&
	       (c->nreg >= static_cast<uint32_t>(kTabProbes) || tab_fits(c->probe_r[c->nreg] * c->probe_r[c->nreg]))) {
		add_reg(c->nreg);
		++c->nreg3;
	}
	CK(c->probes.ensure(c->np));
	CK(c->d_probe_rank.ensure(c->np));
	if (c->np) {
		CK(cudaMemcpyAsync(c->probes.p, pr.data(), sizeof(uint4) * c->np, cudaMemcpyHostToDevice,
		                   c->stream));
		CK(cudaMemcpyAsync(c->d_probe_rank.p, c->probe_rank.data(), 4ull * c->np,
		                   cudaMemcpyHostToDevice, c->stream));
	}
	CK(c->hist.ensure(n));
	c->wtab_n = 0;
	// window tables of the leading kTabProbes register probes, every row
	// (sieve.cu row_loop): sum of r^2 entries, built on the device
	{
		std::vector<uint4> tp;
		for (uint32_t j = 0; j < c->nreg && j < static_cast<uint32_t>(kTabProbes); ++j) {
			const uint32_t r = c->reg_r[j];
			c->reg_tab[j] = c->wtab_n;
			tp.push_back(make_uint4(r, c->reg_base[j], ext_row_words(r), c->wtab_n));
			c->wtab_n += r * r;
		}
		if (c->wtab_n > kTabStrideGen)
			return set_err(CGPU_ERR_INVALID, "register-probe window tables exceed kTabStrideGen");
		CK(c->d_tabprobes.ensure(tp.size()));
		CK(c->wintab.ensure(2 * kTabStrideGen));
		if (!tp.empty()) {
			CK(cudaMemcpyAsync(c->d_tabprobes.p, tp.data(), sizeof(uint4) * tp.size(), cudaMemcpyHostToDevice,
			                   c->stream));
			CK(launch_wintab(c->d_tabprobes.p, static_cast<uint32_t>(tp.size()), c->wtab_n, c->ext.p,
			                 kTabStrideGen, c->wintab.p, c->stream));
			++c->launches;
		}
	}
	{
		c->std_primes = c->nreg2 == 7 && c->nreg3 == static_cast<uint32_t>(kStdReg3) &&
		                !std::getenv("CUBOID_NO_STD_PRIMES");
		for (uint32_t j = 0; c->std_primes && j < c->nreg; ++j) c->std_primes = c->reg_r[j] == std_prime(j);
	}
	// k_wsieve needs the standard register probes and its shared memory (larger sets keep k_sieve)
	c->wheel = c->std_primes && c->wheel_mode != 0 && wsieve_smem_bytes(c->np) <= 220 * 1024;
	if (c->wheel) {  // wheel tables (11, 13, 17 as the wheel; strided window tables of 19..37)
		CK(c->wheeltab.ensure(kWtWords));
		CK(launch_wheeltab(c->ext.p, c->reg_base, c->wheeltab.p, c->stream));
		++c->launches;
		if (!c->wgrid) c->wgrid = wsieve_grid(c->device, wsieve_smem_bytes(c->np));
	}
	const size_t smem =
	    sieve_smem_bytes(c->np, c->wtab_n ? (c->std_primes ? kTabStrideStd : kTabStrideGen) : 0);
	if (smem > 220 * 1024)
		return set_err(CGPU_ERR_INVALID, "too many probe primes for the sieve's shared memory");
	{  // occupancy per kernel variant and shared-memory size, computed once per context
		const uint64_t key = (uint64_t(c->nreg2) << 56) | (uint64_t(c->nreg3) << 48) |
		                     (uint64_t(c->std_primes) << 40) | smem;
		auto it = c->grid_cache.find(key);
		if (it == c->grid_cache.end())
			it = c->grid_cache.emplace(key, sieve_grid(c->device, static_cast<int>(c->nreg2),
			                                           static_cast<int>(c->nreg3), c->std_primes, smem)).first;
		c->grid = it->second;
	}
	CK(cudaGetLastError());
	if (!spec) CK(cudaStreamSynchronize(c->stream));
	c->loaded = true;
	c->launched = false;
	return CGPU_OK;
}

// The expected per-table flags of an asynchronous load: the verified flags of
// the same prime list when this context has them (a set re-uploaded, e.g.
// every step of a pipeline), else what the reference's builder produces --
// every table of r >= 11 has a set bit, r = 2, 3, 5, 7 none, no row 0 bits.
std::vector<uint8_t> expected_flags(const cgpu_ctx* c, const std::vector<uint32_t>& primes)
{
	if (c->flags_valid && c->flags_primes == primes) return c->flags;
	std::vector<uint8_t> f(primes.size());
	for (size_t k = 0; k < primes.size(); ++k) f[k] = primes[k] > 7 ? 1 : 0;
	return f;
}

// Verifies the last asynchronous load (waits for the stream). On a flag
// mismatch the context re-derives synchronously, so later launches are right;
// launches made before the verification used the wrong probe list.
int settle_load(cgpu_ctx* c)
{
	if (!c->status_pending) return CGPU_OK;
	uint32_t st = 0;
	CK(cudaMemcpyAsync(&st, c->load_status.p, 4, cudaMemcpyDeviceToHost, c->stream));
	CK(cudaStreamSynchronize(c->stream));
	c->status_pending = false;
	if (st & 1u) {
		c->loaded = false;
		return set_err(CGPU_ERR_FORMAT, "unpack_bits: nonzero padding bits");
	}
	if (st & 2u) {
		c->flags_valid = false;
		if (int rc = finalize_set(c, false, c->keep_row0)) return rc;
		return set_err(CGPU_ERR_INVALID,
		               "asynchronous load: the tables' flags differ from the expected ones; the set was "
		               "re-derived, repeat the launches made since the load");
	}
	// verified: remember the flags for the next load of this prime list
	c->flags_primes = c->primes;
	c->flags = c->spec_flags;
	c->flags_valid = true;
	return CGPU_OK;
}

int begin_set(cgpu_ctx* c, const uint32_t* primes, uint32_t n)
{
	std::vector<uint32_t> offs(n);
	uint64_t total = 0;
	if (int rc = layout(primes, n, offs.data(), &total)) return rc;
	c->loaded = false;
	c->primes.assign(primes, primes + n);
	c->offsets = offs;
	c->total_bytes = total;
	CK(c->packed.ensure(total + 64));  // k_derive stages 16-byte aligned spans one word past the last byte
	return CGPU_OK;
}

}  // namespace

extern "C" {

int cgpu_tables_build(cgpu_ctx* c, const uint32_t* primes, uint32_t n, int algorithm,
                      uint8_t* out_bytes, uint32_t* out_offsets, uint64_t* out_evals)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (algorithm != CGPU_BUILD_PRODUCTION && algorithm != CGPU_BUILD_EXHAUSTIVE)
		return set_err(CGPU_ERR_INVALID, "unknown build algorithm");
	CK(cudaSetDevice(c->device));
	if (int rc = begin_set(c, primes, n)) return rc;
	c->launches = 0;
	uint64_t evals = 0;
	if (n) {
		std::vector<uint32_t> eb;
		uint64_t ew = 0;
		std::vector<PrimeJob> jobs = make_jobs(c->primes, c->offsets, eb, ew);
		std::vector<PrimeJob> byr = jobs;
		std::stable_sort(byr.begin(), byr.end(), [](const PrimeJob& x, const PrimeJob& y) { return x.r > y.r; });
		CK(c->jobs_build.ensure(n));
		CK(cudaMemcpyAsync(c->jobs_build.p, byr.data(), sizeof(PrimeJob) * n, cudaMemcpyHostToDevice,
		                   c->stream));
		CK(cudaMemsetAsync(c->packed.p, 0, c->total_bytes, c->stream));
		const uint32_t rmax = byr.front().r;
		CK(cudaEventRecord(c->ev[0], c->stream));
		if (algorithm == CGPU_BUILD_EXHAUSTIVE) {
			CK(launch_cube(c->jobs_build.p, byr.data(), n, c->packed.p, c->stream));
			c->launches += cube_launches(byr.data(), n);
			CK(cudaEventRecord(c->ev[1], c->stream));
			for (auto r : c->primes) evals += static_cast<uint64_t>(r) * r * r;
		} else {
			uint64_t aux = 0;
			for (auto r : c->primes) aux += r;
			CK(c->row1.ensure(aux));
			CK(c->inv.ensure(aux));
			CK(c->evals.ensure(1));
			CK(cudaMemsetAsync(c->evals.p, 0, 8, c->stream));
			CK(launch_row1(c->jobs_build.p, n, rmax, c->row1.p, c->inv.p, c->evals.p, c->stream));
			CK(launch_permute(c->jobs_build.p, n, rmax * rmax, c->row1.p, c->inv.p, c->packed.p,
			                  c->stream));
			c->launches += 2;
			CK(cudaEventRecord(c->ev[1], c->stream));
			unsigned long long ev = 0;
			CK(cudaMemcpyAsync(&ev, c->evals.p, 8, cudaMemcpyDeviceToHost, c->stream));
			CK(cudaStreamSynchronize(c->stream));
			evals = ev;
		}
	}
	c->timed = false;
	if (int rc = finalize_set(c)) return rc;
	if (n) {  // timings: [0] build kernels, [1] device layout derivation, [2] both
		CK(cudaEventRecord(c->ev[2], c->stream));
		c->timed = true;
	}
	if (out_bytes && c->total_bytes) {
		CK(cudaMemcpyAsync(out_bytes, c->packed.p, c->total_bytes, cudaMemcpyDeviceToHost, c->stream));
		CK(cudaStreamSynchronize(c->stream));
	}
	if (out_offsets && n) std::memcpy(out_offsets, c->offsets.data(), 4ull * n);
	if (out_evals) *out_evals = evals;
	return CGPU_OK;
}

// Host -> device copy of `bytes` into the packed buffer. Pinned (or
// registered) memory goes straight to the copy engine. Pageable memory -- a
// reference SieveSet's std::vector, a file read -- would be staged by the
// driver at a few GB/s; here it goes through two 4 MB pinned buffers, each
// filled by several host threads while the copy engine drains the other.
static int upload_host(cgpu_ctx* c, const void* bytes, uint64_t total)
{
	cudaPointerAttributes attr{};
	const bool pinned = cudaPointerGetAttributes(&attr, bytes) == cudaSuccess &&
	                    (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeManaged);
	cudaGetLastError();  // an unregistered pointer may leave an error behind on older drivers
	if (pinned || total <= cgpu_ctx::kStageBytes) {
		CK(cudaMemcpyAsync(c->packed.p, bytes, total, cudaMemcpyHostToDevice, c->stream));
		return CGPU_OK;
	}
	for (int i = 0; i < 2; ++i) {
		if (!c->stage[i]) CK(cudaMallocHost(&c->stage[i], cgpu_ctx::kStageBytes));
		if (!c->stage_ev[i]) CK(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
	}
	const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
	const unsigned nt = std::min(4u, hw);
	const uint8_t* src = static_cast<const uint8_t*>(bytes);
	for (uint64_t off = 0, k = 0; off < total; off += cgpu_ctx::kStageBytes, ++k) {
		const int b = static_cast<int>(k & 1);
		const size_t len = static_cast<size_t>(std::min<uint64_t>(cgpu_ctx::kStageBytes, total - off));
		CK(cudaEventSynchronize(c->stage_ev[b]));  // the copy that last read this buffer is done
		const size_t per = (len + nt - 1) / nt;
		std::vector<std::thread> th;
		for (unsigned t = 1; t < nt; ++t)
			if (t * per < len)
				th.emplace_back([&, t] { std::memcpy(c->stage[b] + t * per, src + off + t * per, std::min(per, len - t * per)); });
		std::memcpy(c->stage[b], src + off, std::min(per, len));
		for (auto& x : th) x.join();
		CK(cudaMemcpyAsync(c->packed.p + off, c->stage[b], len, cudaMemcpyHostToDevice, c->stream));
		CK(cudaEventRecord(c->stage_ev[b], c->stream));
	}
	return CGPU_OK;
}

static int tables_load(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const void* bytes, uint64_t nbytes,
                       cudaMemcpyKind kind, bool async = false);

int cgpu_tables_load(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                     uint64_t nbytes)
{
	return tables_load(c, primes, n, bytes, nbytes, cudaMemcpyHostToDevice);
}

int cgpu_tables_load_dev(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const void* d_bytes,
                         uint64_t nbytes)
{
	return tables_load(c, primes, n, d_bytes, nbytes, cudaMemcpyDeviceToDevice);
}

int cgpu_tables_load_async(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                           uint64_t nbytes)
{
	return tables_load(c, primes, n, bytes, nbytes, cudaMemcpyHostToDevice, true);
}

int cgpu_tables_load_dev_async(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const void* d_bytes,
                               uint64_t nbytes)
{
	return tables_load(c, primes, n, d_bytes, nbytes, cudaMemcpyDeviceToDevice, true);
}

int cgpu_load_status(cgpu_ctx* c)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	CK(cudaSetDevice(c->device));
	return settle_load(c);
}

int cgpu_load_status_copy(cgpu_ctx* c, void* dst)
{
	if (!c || !dst) return set_err(CGPU_ERR_INVALID, "null argument");
	CK(cudaSetDevice(c->device));
	if (c->status_pending) {
		CK(cudaMemcpyAsync(dst, c->load_status.p, 4, cudaMemcpyDefault, c->stream));
	} else {
		CK(cudaMemsetAsync(dst, 0, 4, c->stream));  // verified (or synchronous) load
	}
	return CGPU_OK;
}

static int tables_load(cgpu_ctx* c, const uint32_t* primes, uint32_t n, const void* bytes, uint64_t nbytes,
                       cudaMemcpyKind kind, bool async)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	CK(cudaSetDevice(c->device));
	uint64_t total = 0;
	if (int rc = layout(primes, n, nullptr, &total)) return rc == CGPU_ERR_INVALID ? set_err(CGPU_ERR_FORMAT, g_err) : rc;
	if (total != nbytes) return set_err(CGPU_ERR_FORMAT, "load_sieve: tables stream length does not match index");
	if (int rc = begin_set(c, primes, n)) return rc;
	c->launches = 0;
	if (n) {
		if (!bytes) return set_err(CGPU_ERR_INVALID, "null table bytes");
		if (kind == cudaMemcpyHostToDevice) {
			if (int rc = upload_host(c, bytes, total)) return rc;
		} else {
			CK(cudaMemcpyAsync(c->packed.p, bytes, total, kind, c->stream));
		}
		std::vector<uint32_t> eb;
		uint64_t ew = 0;
		std::vector<PrimeJob> jobs = make_jobs(c->primes, c->offsets, eb, ew);
		CK(c->jobs_rank.ensure(n));
		CK(cudaMemcpyAsync(c->jobs_rank.p, jobs.data(), sizeof(PrimeJob) * n, cudaMemcpyHostToDevice,
		                   c->stream));
		CK(c->killflags.ensure(n + 1));
		CK(cudaMemsetAsync(c->killflags.p + n, 0, 4, c->stream));
		CK(launch_check_padding(c->jobs_rank.p, n, c->packed.p, c->killflags.p + n, c->stream));
		++c->launches;
	}
	if (async) {
		const std::vector<uint8_t> spec = expected_flags(c, c->primes);
		return finalize_set(c, n > 0, false, &spec);
	}
	return finalize_set(c, n > 0);
}

int cgpu_tables_download(cgpu_ctx* c, uint8_t* out, uint64_t cap)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (!c->loaded) return set_err(CGPU_NOT_LOADED, "tables not loaded");
	if (cap < c->total_bytes) return set_err(CGPU_ERR_CAPACITY, "output buffer too small");
	CK(cudaSetDevice(c->device));
	if (c->total_bytes) {
		CK(cudaMemcpyAsync(out, c->packed.p, c->total_bytes, cudaMemcpyDeviceToHost, c->stream));
		CK(cudaStreamSynchronize(c->stream));
	}
	return CGPU_OK;
}

// ---- on-disk formats (sievetable.hpp:229-346; proj/README.md "File formats") ----

int cgpu_index_serialize(const uint32_t* primes, uint32_t n, uint8_t* out, uint64_t cap, uint64_t* out_len)
{
	uint64_t total = 0;
	if (int rc = layout(primes, n, nullptr, &total)) return rc;
	const uint64_t len = kIndexHeaderSize + kIndexRecordSize * static_cast<uint64_t>(n);
	if (out_len) *out_len = len;
	if (!out) return CGPU_OK;
	if (cap < len) return set_err(CGPU_ERR_CAPACITY, "index buffer too small");
	std::memcpy(out, "CUPQ", 4);
	out[4] = kIndexVersion;
	for (int b = 0; b < 4; ++b) out[5 + b] = static_cast<uint8_t>(n >> (8 * b));
	uint64_t off = 0;
	for (uint32_t k = 0; k < n; ++k) {
		uint8_t* rec = out + kIndexHeaderSize + kIndexRecordSize * k;
		rec[0] = static_cast<uint8_t>(primes[k]);
		rec[1] = static_cast<uint8_t>(primes[k] >> 8);
		for (int b = 0; b < 4; ++b) rec[2 + b] = static_cast<uint8_t>(off >> (8 * b));
		off += table_bytes(primes[k]);
	}
	return CGPU_OK;
}

int cgpu_index_parse(const uint8_t* index, uint64_t len, uint32_t* primes, uint32_t cap, uint32_t* n_out,
                     uint64_t* tables_bytes)
{
	if (!index && len) return set_err(CGPU_ERR_INVALID, "null index");
	if (len < kIndexHeaderSize) return set_err(CGPU_ERR_FORMAT, "load_sieve: index truncated");
	if (std::memcmp(index, "CUPQ", 4) != 0) return set_err(CGPU_ERR_FORMAT, "load_sieve: bad index magic");
	if (index[4] != kIndexVersion)
		return set_err(CGPU_ERR_FORMAT, "load_sieve: unsupported index version");
	uint32_t n = 0;
	for (int b = 0; b < 4; ++b) n |= static_cast<uint32_t>(index[5 + b]) << (8 * b);
	if (len != kIndexHeaderSize + kIndexRecordSize * static_cast<uint64_t>(n))
		return set_err(CGPU_ERR_FORMAT, "load_sieve: index length does not match record count");
	if (n_out) *n_out = n;
	uint64_t expect = 0;
	uint32_t prev = 0;
	for (uint32_t k = 0; k < n; ++k) {
		const uint8_t* rec = index + kIndexHeaderSize + kIndexRecordSize * k;
		const uint32_t prime = static_cast<uint32_t>(rec[0]) | static_cast<uint32_t>(rec[1]) << 8;
		uint32_t off = 0;
		for (int b = 0; b < 4; ++b) off |= static_cast<uint32_t>(rec[2 + b]) << (8 * b);
		if (!is_prime_u32(prime) || prime >= kModulusLimit)
			return set_err(CGPU_ERR_FORMAT, "load_sieve: index entry is not an admissible prime");
		if (prime <= prev) return set_err(CGPU_ERR_FORMAT, "load_sieve: primes not strictly increasing");
		if (off != expect) return set_err(CGPU_ERR_FORMAT, "load_sieve: offset mismatch");
		prev = prime;
		expect += table_bytes(prime);
		if (expect > UINT32_MAX) return set_err(CGPU_ERR_FORMAT, "load_sieve: cumulative size exceeds 2^32");
		if (primes && k < cap) primes[k] = prime;
	}
	if (tables_bytes) *tables_bytes = expect;
	if (primes && cap < n) return set_err(CGPU_ERR_CAPACITY, "prime buffer too small");
	return CGPU_OK;
}

namespace {

bool read_file(const char* path, std::vector<uint8_t>& out)
{
	std::ifstream f(path, std::ios::binary);
	if (!f) return false;
	f.seekg(0, std::ios::end);
	const std::streamoff len = f.tellg();
	f.seekg(0);
	out.resize(static_cast<size_t>(len));
	f.read(reinterpret_cast<char*>(out.data()), len);
	return static_cast<bool>(f) || len == 0;
}

bool write_file(const char* path, const uint8_t* data, size_t len)
{
	std::ofstream f(path, std::ios::binary | std::ios::trunc);
	if (!f) return false;
	f.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(len));
	return static_cast<bool>(f);
}

}  // namespace

int cgpu_tables_load_files(cgpu_ctx* c, const char* tables_path, const char* index_path)
{
	if (!c || !tables_path || !index_path) return set_err(CGPU_ERR_INVALID, "null argument");
	std::vector<uint8_t> tb, ix;
	if (!read_file(index_path, ix)) return set_err(CGPU_ERR_IO, std::string("cannot open: ") + index_path);
	if (!read_file(tables_path, tb)) return set_err(CGPU_ERR_IO, std::string("cannot open: ") + tables_path);
	uint32_t n = 0;
	uint64_t expect = 0;
	if (int rc = cgpu_index_parse(ix.data(), ix.size(), nullptr, 0, &n, &expect)) return rc;
	std::vector<uint32_t> primes(n);
	if (int rc = cgpu_index_parse(ix.data(), ix.size(), primes.data(), n, &n, &expect)) return rc;
	if (tb.size() != expect)
		return set_err(CGPU_ERR_FORMAT, "load_sieve: tables stream length does not match index");
	return cgpu_tables_load(c, primes.data(), n, tb.data(), tb.size());
}

int cgpu_tables_save_files(cgpu_ctx* c, const char* tables_path, const char* index_path)
{
	if (!c || !tables_path || !index_path) return set_err(CGPU_ERR_INVALID, "null argument");
	if (!c->loaded) return set_err(CGPU_NOT_LOADED, "tables not loaded");
	std::vector<uint8_t> tb(c->total_bytes);
	if (int rc = cgpu_tables_download(c, tb.data(), tb.size())) return rc;
	uint64_t len = 0;
	const uint32_t n = static_cast<uint32_t>(c->primes.size());
	if (int rc = cgpu_index_serialize(c->primes.data(), n, nullptr, 0, &len)) return rc;
	std::vector<uint8_t> ix(len);
	if (int rc = cgpu_index_serialize(c->primes.data(), n, ix.data(), len, &len)) return rc;
	if (!write_file(tables_path, tb.data(), tb.size()))
		return set_err(CGPU_ERR_IO, std::string("write failed: ") + tables_path);
	if (!write_file(index_path, ix.data(), ix.size()))
		return set_err(CGPU_ERR_IO, std::string("write failed: ") + index_path);
	return CGPU_OK;
}

int cgpu_tables_info(cgpu_ctx* c, uint32_t* n, uint8_t* killable)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (c->status_pending) {
		CK(cudaSetDevice(c->device));
		if (int rc = settle_load(c)) return rc;
	}
	const uint32_t k = c->loaded ? static_cast<uint32_t>(c->primes.size()) : 0;
	if (n) *n = k;
	if (killable && k) std::memcpy(killable, c->killable.data(), k);
	return CGPU_OK;
}

int cgpu_build_tables(int device, const uint32_t* primes, uint32_t n, int algorithm,
                      uint8_t* out_bytes, uint32_t* out_offsets, uint64_t* out_evals)
{
	cgpu_ctx* c = nullptr;
	if (int rc = cgpu_create(device, nullptr, &c)) return rc;
	const int rc = cgpu_tables_build(c, primes, n, algorithm, out_bytes, out_offsets, out_evals);
	const std::string keep = g_err;
	cgpu_destroy(c);
	g_err = keep;
	return rc;
}

}  // extern "C"

namespace {

// Validation shared by both launch entry points (engine.hpp:152-161 codes).
int check_launch(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode, uint32_t G,
                 uint32_t g)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (!c->loaded || c->primes.empty()) return set_err(CGPU_NOT_LOADED, "tables not loaded");
	if (mode != CGPU_REGION && mode != CGPU_TRIANGLE) return set_err(CGPU_ERR_INVALID, "unknown mode");
	if (G == 0 || g >= G) return set_err(CGPU_ERR_INVALID, "bad shard (count, index)");
	// validate_start (engine.hpp:152-161) with small_p on: the C ABI sieves rows
	// below 152 (the small-p region and TRIANGLE rows), so p = 0 is code 3;
	// the C++/Python scan() wrappers apply opt.small_p first (p < 152 -> 2)
	if (p_lo == 0) return set_err(CGPU_P_ABOVE_LIMIT, "p must be positive");
	if (mode == CGPU_REGION) {
		if (p_hi > kPLimit32 || p_lo > kPLimit32)
			return set_err(CGPU_P_ABOVE_LIMIT, "p above the 32-bit region limit");
		if (q_start) {
			uint64_t lo, hi;
			q_bounds(p_lo, &lo, &hi);
			if (q_start < lo) return set_err(CGPU_Q_BELOW_LOW, "q below q_low");
			if (q_start > hi) return set_err(CGPU_Q_ABOVE_HIGH, "q above q_high");
		}
	} else {
		if (q_start) return set_err(CGPU_ERR_INVALID, "TRIANGLE mode sieves whole rows (q_start must be 0)");
		if (p_hi > 0xffffffffull) return set_err(CGPU_P_ABOVE_LIMIT, "p above 2^32");
	}
	// non-canonical sets with bits in row 0: re-derive the layout the mode reads
	const bool keep = mode == CGPU_TRIANGLE && c->row0_nonzero;
	if (keep != c->keep_row0) return finalize_set(c, false, keep);
	return CGPU_OK;
}

uint64_t launch_blocks(uint64_t p_lo, uint64_t p_hi)
{
	return p_hi < p_lo ? 0 : p_hi / 100 - p_lo / 100 + 1;
}

// Enqueues init + (plan, sieve) per chunk of row slots on the context stream,
// writing into the given device buffers. Events ev[0..2] bracket the launch.
int enqueue_sieve(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end, int mode,
                  uint32_t G, uint32_t g, unsigned long long* d_counts, unsigned long long* d_hist,
                  uint32_t* d_block_rmax, unsigned long long* d_surv, uint64_t surv_cap)
{
	c->launched = false;
	c->launches = 0;
	const bool empty = p_hi < p_lo;
	const uint64_t blk_lo = p_lo / 100;
	const uint64_t nblocks = launch_blocks(p_lo, p_hi);
	CK(cudaEventRecord(c->ev[0], c->stream));
	bool ev1 = false;

	SieveArgs a{};
	a.ext = c->ext.p;
	a.ext_words = c->ext_words;
	a.n_blocks = nblocks;
	a.probes = c->probes.p;
	a.np = c->np;
	a.nreg = c->nreg;
	a.nreg2 = c->nreg2;
	a.nreg3 = c->nreg3;
	a.wtab_n = c->wtab_n;
	a.wintab = c->wintab.p;
	a.std_primes = c->std_primes;
	for (int j = 0; j < kMaxReg; ++j) {
		a.reg_r[j] = c->reg_r[j];
		a.reg_m[j] = c->reg_m[j];
		a.reg_base[j] = c->reg_base[j];
		a.reg_delta[j] = c->reg_delta[j];
		a.reg_tab[j] = c->reg_tab[j];
	}
	a.fprimes = c->fprimes.p;
	a.n_fprimes = c->n_fprimes;
	a.row_cost = c->row_cost;
	a.drain_alpha = c->drain_alpha;
	{  // mean windows per row of the launch: TRIANGLE rows hold ~p q, REGION rows ~59p
		const double pm = 0.5 * (static_cast<double>(p_lo) + static_cast<double>(p_hi));
		const double mean_windows = (mode == CGPU_TRIANGLE ? pm : 59.0 * pm) / 32.0;
		a.short_rows = c->short_rows < 0 ? (mean_windows < kShortRowWindows ? 1u : 0u)
		                                 : static_cast<uint32_t>(c->short_rows);
		if (a.short_rows) a.row_cost = c->row_cost_short;  // the short-row kernel's own setup charge
		// the wheel sieve pays a larger fixed cost per row: launches of short rows keep k_sieve
		a.wheel = c->wheel && (c->wheel_mode >= 2 || mean_windows >= kWheelMinWindows) ? 1u : 0u;
	}
	a.wheeltab = c->wheeltab.p;
	if (a.wheel) {
		a.row_cost = c->row_cost_wheel;
		for (int k = 0; k < 4; ++k) a.wheel_cost[k] = c->wheel_cost[k];
	}
	a.p_lo = p_lo;
	a.p_hi = p_hi;
	a.q_start = q_start;
	a.q_end = q_end;
	a.mode = mode;
	a.G = G;
	a.g = g;
	a.hist = d_hist;
	a.nprimes = static_cast<uint32_t>(c->primes.size());
	a.probe_rank = c->d_probe_rank.p;
	a.counters = d_counts;
	a.block_rmax = d_block_rmax;
	a.blk_lo = blk_lo;
	a.surv = d_surv;
	a.surv_cap = surv_cap;
	a.stop = c->stop_dev;

	// owned blocks: b in [blk_lo, blk_hi] with b % G == g
	const uint64_t blk_hi = p_hi / 100;
	const uint64_t first = blk_lo + ((g + G - blk_lo % G) % G);
	const uint64_t owned = !empty && first <= blk_hi ? (blk_hi - first) / G + 1 : 0;
	if (!owned) {  // nothing to sieve: the outputs are still initialised
		CK(cudaMemsetAsync(d_hist, 0, 8ull * c->primes.size(), c->stream));
		CK(cudaMemsetAsync(d_counts, 0, 16, c->stream));
		CK(launch_init_blocks(d_block_rmax, nblocks, blk_lo, G, g, c->stream));
		if (nblocks) ++c->launches;
	} else {  // np == 0 (no table can kill): every candidate survives
		const size_t max_slots = static_cast<size_t>(std::min<uint64_t>(owned, kBlocksPerLaunch)) * 100;
		CK(c->prefix.ensure(max_slots + 1));
		CK(c->chunk_off.ensure(plan_chunks(static_cast<uint32_t>(max_slots)) + 1));
		if (!c->tickets.p) {  // zeroed once: each kernel's last CTA resets its ticket
			CK(c->tickets.ensure(2));
			CK(cudaMemsetAsync(c->tickets.p, 0, 8, c->stream));
		}
		CK(c->rowfac.ensure(max_slots * kFacWords));
		a.rowfac = c->rowfac.p;
		a.prefix = c->prefix.p;
		a.chunk_off = c->chunk_off.p;
		a.tickets = c->tickets.p;
		for (uint64_t ob = 0; ob < owned; ob += kBlocksPerLaunch) {
			const uint64_t nb = std::min<uint64_t>(kBlocksPerLaunch, owned - ob);
			a.blk0 = first + ob * G;
			a.n_slots = static_cast<uint32_t>(nb * 100);
			a.init = ob == 0;
			CK(launch_plan(a, c->stream));
			if (!ev1) CK(cudaEventRecord(c->ev[1], c->stream));  // sieve time excludes the first plan
			ev1 = true;
			CK(launch_sieve(a, a.wheel ? c->wgrid : c->grid, c->stream));
			c->launches += 2;
		}
	}
	if (!ev1) CK(cudaEventRecord(c->ev[1], c->stream));
	CK(cudaEventRecord(c->ev[2], c->stream));
	c->timed = true;
	c->last_nblocks = nblocks;
	c->last_surv_cap = surv_cap;
	c->last_wheel = a.wheel != 0;
	c->launched = true;
	return CGPU_OK;
}

}  // namespace

extern "C" {

int cgpu_sieve_launch(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode,
                      uint32_t G, uint32_t g, uint64_t surv_cap)
{
	if (int rc = check_launch(c, p_lo, q_start, p_hi, mode, G, g)) return rc;
	CK(cudaSetDevice(c->device));
	CK(c->hist.ensure(c->primes.size()));
	CK(c->counters.ensure(2));
	CK(c->block_rmax.ensure(launch_blocks(p_lo, p_hi)));
	CK(c->surv.ensure(surv_cap));
	c->results_internal = true;
	return enqueue_sieve(c, p_lo, q_start, p_hi, 0, mode, G, g, c->counters.p, c->hist.p, c->block_rmax.p,
	                     c->surv.p, surv_cap);
}

int cgpu_sieve_span(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end,
                    uint64_t* counts, uint64_t* hist, uint32_t* block_rmax, uint64_t block_cap,
                    uint64_t* surv_pq, uint64_t surv_cap)
{
	if (int rc = check_launch(c, p_lo, q_start, p_hi, CGPU_REGION, 1, 0)) return rc;
	if (q_end) {
		uint64_t lo, hi;
		q_bounds(p_hi, &lo, &hi);
		if (q_end > hi) return set_err(CGPU_Q_ABOVE_HIGH, "q_end above q_high");
	}
	CK(cudaSetDevice(c->device));
	CK(c->hist.ensure(c->primes.size()));
	CK(c->counters.ensure(2));
	CK(c->block_rmax.ensure(launch_blocks(p_lo, p_hi)));
	const uint64_t cap = surv_pq ? surv_cap : 0;
	CK(c->surv.ensure(cap));
	c->results_internal = true;
	if (int rc = enqueue_sieve(c, p_lo, q_start, p_hi, q_end, CGPU_REGION, 1, 0, c->counters.p, c->hist.p,
	                           c->block_rmax.p, c->surv.p, cap))
		return rc;
	return cgpu_sieve_results(c, counts, hist, block_rmax, block_cap, surv_pq, surv_cap);
}

int cgpu_sieve_launch_dev(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode,
                          uint32_t G, uint32_t g, uint64_t* d_counts, uint64_t* d_hist,
                          uint32_t* d_block_rmax, uint64_t block_cap, uint64_t* d_surv,
                          uint64_t surv_cap)
{
	if (int rc = check_launch(c, p_lo, q_start, p_hi, mode, G, g)) return rc;
	if (!d_counts || !d_hist || (!d_block_rmax && launch_blocks(p_lo, p_hi)) || (!d_surv && surv_cap))
		return set_err(CGPU_ERR_INVALID, "null device output buffer");
	if (block_cap < launch_blocks(p_lo, p_hi))
		return set_err(CGPU_ERR_CAPACITY, "block_rmax buffer too small");
	CK(cudaSetDevice(c->device));
	c->results_internal = false;
	return enqueue_sieve(c, p_lo, q_start, p_hi, 0, mode, G, g,
	                     reinterpret_cast<unsigned long long*>(d_counts),
	                     reinterpret_cast<unsigned long long*>(d_hist), d_block_rmax,
	                     reinterpret_cast<unsigned long long*>(d_surv), surv_cap);
}

int cgpu_sieve_launch_span_dev(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end,
                               uint32_t G, uint32_t g, uint64_t* d_counts, uint64_t* d_hist,
                               uint32_t* d_block_rmax, uint64_t block_cap, uint64_t* d_surv, uint64_t surv_cap)
{
	if (int rc = check_launch(c, p_lo, q_start, p_hi, CGPU_REGION, G, g)) return rc;
	if (q_end) {
		uint64_t lo, hi;
		q_bounds(p_hi, &lo, &hi);
		if (q_end > hi) return set_err(CGPU_Q_ABOVE_HIGH, "q_end above q_high");
	}
	if (!d_counts || !d_hist || (!d_block_rmax && launch_blocks(p_lo, p_hi)) || (!d_surv && surv_cap))
		return set_err(CGPU_ERR_INVALID, "null device output buffer");
	if (block_cap < launch_blocks(p_lo, p_hi))
		return set_err(CGPU_ERR_CAPACITY, "block_rmax buffer too small");
	CK(cudaSetDevice(c->device));
	c->results_internal = false;
	return enqueue_sieve(c, p_lo, q_start, p_hi, q_end, CGPU_REGION, G, g,
	                     reinterpret_cast<unsigned long long*>(d_counts),
	                     reinterpret_cast<unsigned long long*>(d_hist), d_block_rmax,
	                     reinterpret_cast<unsigned long long*>(d_surv), surv_cap);
}

int cgpu_region_advance(uint64_t p, uint64_t q, uint64_t k, uint64_t p_end, uint64_t* out_p, uint64_t* out_q)
{
	if (!out_p || !out_q) return set_err(CGPU_ERR_INVALID, "null argument");
	if (p == 0) return set_err(CGPU_ERR_INVALID, "p must be positive");
	uint64_t q0 = q, c = 0;
	for (;;) {
		uint64_t lo, hi;
		if (p < kRegionCrossover || c == 0) {
			q_bounds(p, &lo, &hi);
			if (p >= kRegionCrossover) c = lo;
		} else {  // q_low = least q with 9 q^3 >= p: monotone in p, one step at a time
			while (9 * static_cast<unsigned __int128>(c) * c * c < p) ++c;
			lo = c;
			hi = 59 * p;
		}
		const uint64_t first = q0 ? q0 : lo;
		const uint64_t n = hi >= first ? hi - first + 1 : 0;
		if (k < n) {
			*out_p = p;
			*out_q = first + k;
			return CGPU_OK;
		}
		k -= n;
		if (p >= p_end) return CGPU_P_ABOVE_LIMIT;  // the range ends first
		++p;
		q0 = 0;
	}
}

int cgpu_device_count(int* n)
{
	if (!n) return set_err(CGPU_ERR_INVALID, "null argument");
	*n = 0;
	if (cudaGetDeviceCount(n) != cudaSuccess) *n = 0;
	return CGPU_OK;
}

int cgpu_alloc_stop_word(uint32_t** word)
{
	if (!word) return set_err(CGPU_ERR_INVALID, "null argument");
	*word = nullptr;
	int count = 0;
	if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
		return set_err(CGPU_ERR_NO_DEVICE, "no CUDA device visible: cuboid_gpu has no CPU fallback");
	void* p = nullptr;
	CK(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
	std::memset(p, 0, 64);
	*word = static_cast<uint32_t*>(p);
	return CGPU_OK;
}

int cgpu_free_stop_word(uint32_t* word)
{
	if (word) CK(cudaFreeHost(word));
	return CGPU_OK;
}

int cgpu_set_stop_word(cgpu_ctx* c, uint32_t* word)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (!word) {
		c->stop_dev = nullptr;
		return CGPU_OK;
	}
	CK(cudaSetDevice(c->device));
	void* d = nullptr;
	CK(cudaHostGetDevicePointer(&d, word, 0));
	c->stop_dev = static_cast<const volatile uint32_t*>(d);
	return CGPU_OK;
}

int cgpu_sieve_results(cgpu_ctx* c, uint64_t* counts, uint64_t* hist, uint32_t* block_rmax,
                       uint64_t block_cap, uint64_t* surv_pq, uint64_t surv_cap)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (!c->launched || !c->results_internal)
		return set_err(CGPU_ERR_INVALID, "no sieve launched into context buffers");
	CK(cudaSetDevice(c->device));
	if (int rc = settle_load(c)) return rc;  // an asynchronous load is verified here at the latest
	unsigned long long cnt[2] = {0, 0};
	std::vector<unsigned long long> hp(c->primes.size());
	CK(cudaMemcpyAsync(cnt, c->counters.p, 16, cudaMemcpyDeviceToHost, c->stream));
	if (!hp.empty())
		CK(cudaMemcpyAsync(hp.data(), c->hist.p, 8ull * hp.size(), cudaMemcpyDeviceToHost, c->stream));
	if (block_rmax && c->last_nblocks) {
		if (block_cap < c->last_nblocks) return set_err(CGPU_ERR_CAPACITY, "block_rmax buffer too small");
		CK(cudaMemcpyAsync(block_rmax, c->block_rmax.p, 4ull * c->last_nblocks, cudaMemcpyDeviceToHost,
		                   c->stream));
	}
	CK(cudaStreamSynchronize(c->stream));
	if (counts) {
		counts[0] = cnt[0];
		counts[1] = cnt[1];
	}
	if (hist) std::copy(hp.begin(), hp.end(), hist);
	int rc = CGPU_OK;
	if (surv_pq && cnt[1]) {
		const uint64_t stored = std::min<uint64_t>(cnt[1], c->last_surv_cap);
		std::vector<unsigned long long> keys(stored);
		CK(cudaMemcpyAsync(keys.data(), c->surv.p, 8 * stored, cudaMemcpyDeviceToHost, c->stream));
		CK(cudaStreamSynchronize(c->stream));
		std::sort(keys.begin(), keys.end());
		const uint64_t k = std::min<uint64_t>(stored, surv_cap);
		for (uint64_t i = 0; i < k; ++i) {
			surv_pq[2 * i] = keys[i] >> 32;
			surv_pq[2 * i + 1] = keys[i] & 0xffffffffull;
		}
		if (cnt[1] > k) rc = set_err(CGPU_ERR_CAPACITY, "survivor buffer too small");
	}
	return rc;
}

int cgpu_sieve(cgpu_ctx* c, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode, uint32_t G,
               uint32_t g, uint64_t* counts, uint64_t* hist, uint32_t* block_rmax, uint64_t block_cap,
               uint64_t* surv_pq, uint64_t surv_cap)
{
	if (int rc = cgpu_sieve_launch(c, p_lo, q_start, p_hi, mode, G, g, surv_pq ? surv_cap : 0)) return rc;
	return cgpu_sieve_results(c, counts, hist, block_rmax, block_cap, surv_pq, surv_cap);
}

const char* cgpu_last_sieve_kernel(cgpu_ctx* c)
{
	if (!c || !c->launched) return "";
	return c->last_wheel ? "k_wsieve" : "k_sieve";
}

int cgpu_last_timings(cgpu_ctx* c, float* ms3)
{
	if (!c || !ms3) return set_err(CGPU_ERR_INVALID, "null argument");
	if (c->timed) {
		CK(cudaSetDevice(c->device));
		CK(cudaEventSynchronize(c->ev[2]));
		float ms = 0;
		if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]) == cudaSuccess) c->timings[0] = ms;
		if (cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]) == cudaSuccess) c->timings[1] = ms;
		if (cudaEventElapsedTime(&ms, c->ev[0], c->ev[2]) == cudaSuccess) c->timings[2] = ms;
	}
	std::memcpy(ms3, c->timings, sizeof c->timings);
	return CGPU_OK;
}

int cgpu_int32_peak(int device, double* ops4)
{
	if (!ops4) return set_err(CGPU_ERR_INVALID, "null argument");
	int count = 0;
	if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
		return set_err(CGPU_ERR_NO_DEVICE, "no CUDA device visible: cuboid_gpu has no CPU fallback");
	CK(cudaSetDevice(device));
	CK(run_int_peak(device, ops4));
	return CGPU_OK;
}

int cgpu_fp32_peak(int device, double* ops2)
{
	if (!ops2) return set_err(CGPU_ERR_INVALID, "null argument");
	int count = 0;
	if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
		return set_err(CGPU_ERR_NO_DEVICE, "no CUDA device visible: cuboid_gpu has no CPU fallback");
	CK(cudaSetDevice(device));
	CK(run_fp_peak(device, ops2));
	return CGPU_OK;
}

int cgpu_last_launch_count(cgpu_ctx* c, uint32_t* n)
{
	if (!c || !n) return set_err(CGPU_ERR_INVALID, "null argument");
	*n = c->launches;
	return CGPU_OK;
}

int cgpu_classify(cgpu_ctx* c, const uint64_t* pq, uint64_t n, int32_t* out_rank)
{
	if (!c) return set_err(CGPU_ERR_INVALID, "null ctx");
	if (!c->loaded || c->primes.empty()) return set_err(CGPU_NOT_LOADED, "tables not loaded");
	if (!n) return CGPU_OK;
	CK(cudaSetDevice(c->device));
	CK(c->pq.ensure(2 * n));
	CK(c->ranks.ensure(n));
	CK(cudaMemcpyAsync(c->pq.p, pq, 16 * n, cudaMemcpyHostToDevice, c->stream));
	CK(launch_classify(c->pq.p, n, c->packed.p, c->d_primes.p, c->d_offsets.p,
	                   static_cast<uint32_t>(c->primes.size()), c->ranks.p, c->stream));
	c->launches = 1;
	CK(cudaMemcpyAsync(out_rank, c->ranks.p, 4 * n, cudaMemcpyDeviceToHost, c->stream));
	CK(cudaStreamSynchronize(c->stream));
	return CGPU_OK;
}

}  // extern "C"
