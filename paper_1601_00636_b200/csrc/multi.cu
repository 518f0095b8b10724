// In-process multi-GPU sieve: one cgpu_ctx per device, one NCCL communicator
// clique (ncclCommInitAll), block-cyclic p/100 shards.
//
// This is what lets the reference's own single-process driver -- scan()
// called from SearchController::run_scan (engine.hpp:555-577) -- use every GPU
// of a box without a launcher: cuboid::gpu::scan(set, ..., devices) sits on it.
// The per-rank (one process per GPU) path of bench.py / parallel.py does the
// same exchange through torch.distributed.
//
// Per sieve call:
//   1. every device sieves its shard (rows with (p/100) % G == g) into its own
//      buffers: [pairs, survivors, hist by rank] u64, block r_max u32 (0 for
//      blocks it does not own, engine.hpp:229-236), survivors (p<<32)|q;
//   2. ONE grouped NCCL call: all-reduce(SUM) of the counters/histogram
//      (ScanStats::merge, engine.hpp:121-134) and all-reduce(MAX) of block
//      r_max (each block has one owner, so MAX = the owner's value);
//   3. survivor gather: the per-device counts are read back (8 B each), then
//      grouped ncclSend/ncclRecv move every device's list into device 0's
//      buffer, which is copied to the host and sorted to canonical (p, q)
//      order (the reference's sink order, test_engine.cpp:186-193).
// Table upload: each device copies 1/G of the host bytes over its own PCIe
// link, an in-place ncclAllGather assembles the set over NVLink, and every
// context derives its layout from device memory (cgpu_tables_load_dev).

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and prototypes only: the library is dlopen'ed (below)

#include <algorithm>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/cuboid_gpu.h"
#include "internal.cuh"

namespace {

// NCCL is resolved at cgpu_multi_create, not linked: a process that imports
// PyTorch carries torch's own libnccl.so.2, and a link-time dependency would
// bind whichever copy loads first for both. dlopen("libnccl.so.2") returns the
// copy already in the process if there is one, else the system library.
struct NcclApi {
	decltype(&ncclCommInitAll) CommInitAll = nullptr;
	decltype(&ncclCommDestroy) CommDestroy = nullptr;
	decltype(&ncclGetErrorString) GetErrorString = nullptr;
	decltype(&ncclGroupStart) GroupStart = nullptr;
	decltype(&ncclGroupEnd) GroupEnd = nullptr;
	decltype(&ncclAllGather) AllGather = nullptr;
	decltype(&ncclAllReduce) AllReduce = nullptr;
	decltype(&ncclSend) Send = nullptr;
	decltype(&ncclRecv) Recv = nullptr;
	bool ok = false;
	std::string err;
};

const NcclApi& nccl()
{
	static const NcclApi api = [] {
		NcclApi a;
		void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
		if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
		if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
		if (!h) {
			a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
			return a;
		}
		bool all = true;
		auto sym = [&](auto& fn, const char* name) {
			fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
			all &= fn != nullptr;
		};
		sym(a.CommInitAll, "ncclCommInitAll");
		sym(a.CommDestroy, "ncclCommDestroy");
		sym(a.GetErrorString, "ncclGetErrorString");
		sym(a.GroupStart, "ncclGroupStart");
		sym(a.GroupEnd, "ncclGroupEnd");
		sym(a.AllGather, "ncclAllGather");
		sym(a.AllReduce, "ncclAllReduce");
		sym(a.Send, "ncclSend");
		sym(a.Recv, "ncclRecv");
		a.ok = all;
		if (!all) a.err = "libnccl.so.2 lacks a required symbol";
		return a;
	}();
	return api;
}

#define MCK(call)                                                                                  \
	do {                                                                                           \
		const cudaError_t e_ = (call);                                                             \
		if (e_ != cudaSuccess)                                                                     \
			return cgpu_internal_set_err(CGPU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
	} while (0)

#define NCK(call)                                                                                  \
	do {                                                                                           \
		const ncclResult_t r_ = (call);                                                            \
		if (r_ != ncclSuccess)                                                                     \
			return cgpu_internal_set_err(CGPU_ERR_CUDA, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
	} while (0)

#define RCK(call)                        \
	do {                                 \
		const int rc_ = (call);          \
		if (rc_ != CGPU_OK) return rc_;  \
	} while (0)

template <class T>
struct DBuf {  // device buffer on a fixed device, grown on demand
	T* p = nullptr;
	size_t n = 0;
	cudaError_t ensure(size_t want)
	{
		if (p && want <= n) return cudaSuccess;
		if (p) cudaFree(p);
		p = nullptr;
		n = 0;
		const cudaError_t e = cudaMalloc(&p, sizeof(T) * (want ? want : 1));
		if (e == cudaSuccess) n = want ? want : 1;
		return e;
	}
	void release()
	{
		if (p) cudaFree(p);
		p = nullptr;
		n = 0;
	}
};

struct Dev {
	int device = 0;
	cudaStream_t stream = nullptr;
	cgpu_ctx* ctx = nullptr;
	ncclComm_t comm = nullptr;
	DBuf<uint64_t> loc, red, surv, gather;
	DBuf<uint32_t> brm;
	DBuf<uint8_t> tables;
	cudaEvent_t ev[2] = {};
	uint64_t local_surv = 0;
};

}  // namespace

struct cgpu_multi {
	std::vector<Dev> devs;
	uint32_t nprimes = 0;
	bool loaded = false;
	float last_ms = 0.f;
	uint64_t *h_loc = nullptr;  // pinned: per-device survivor counts
};

namespace {

void destroy(cgpu_multi* m)
{
	for (Dev& d : m->devs) {
		cudaSetDevice(d.device);
		if (d.stream) cudaStreamSynchronize(d.stream);
		if (d.comm) nccl().CommDestroy(d.comm);
		if (d.ctx) cgpu_destroy(d.ctx);
		d.loc.release();
		d.red.release();
		d.surv.release();
		d.gather.release();
		d.brm.release();
		d.tables.release();
		for (cudaEvent_t e : d.ev)
			if (e) cudaEventDestroy(e);
		if (d.stream) cudaStreamDestroy(d.stream);
	}
	if (m->h_loc) cudaFreeHost(m->h_loc);
	delete m;
}

}  // namespace

extern "C" {

int cgpu_multi_create(int n_devices, const int* devices, cgpu_multi** out)
{
	if (!out) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null output");
	*out = nullptr;
	int count = 0;
	if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
		return cgpu_internal_set_err(CGPU_ERR_NO_DEVICE, "no CUDA device visible: cuboid_gpu has no CPU fallback");
	if (n_devices < 1) return cgpu_internal_set_err(CGPU_ERR_INVALID, "need at least one device");
	if (!nccl().ok) return cgpu_internal_set_err(CGPU_ERR_CUDA, nccl().err);
	std::vector<int> ids(n_devices);
	for (int i = 0; i < n_devices; ++i) {
		ids[i] = devices ? devices[i] : i;
		if (ids[i] < 0 || ids[i] >= count)
			return cgpu_internal_set_err(CGPU_ERR_INVALID, "device index out of range");
		for (int j = 0; j < i; ++j)
			if (ids[j] == ids[i])  // one NCCL rank per GPU
				return cgpu_internal_set_err(CGPU_ERR_INVALID, "duplicate device in the list");
	}
	cgpu_multi* m = new cgpu_multi;
	m->devs.resize(n_devices);
	auto fail = [&](int rc) {
		destroy(m);
		return rc;
	};
	for (int i = 0; i < n_devices; ++i) {
		Dev& d = m->devs[i];
		d.device = ids[i];
		if (cudaSetDevice(d.device) != cudaSuccess ||
		    cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking) != cudaSuccess ||
		    cudaEventCreate(&d.ev[0]) != cudaSuccess || cudaEventCreate(&d.ev[1]) != cudaSuccess)
			return fail(cgpu_internal_set_err(CGPU_ERR_CUDA, "cgpu_multi_create: stream/event creation failed"));
		if (int rc = cgpu_create(d.device, d.stream, &d.ctx)) return fail(rc);
	}
	std::vector<ncclComm_t> comms(n_devices);
	const ncclResult_t r = nccl().CommInitAll(comms.data(), n_devices, ids.data());
	if (r != ncclSuccess)
		return fail(cgpu_internal_set_err(CGPU_ERR_CUDA, std::string("ncclCommInitAll: ") + nccl().GetErrorString(r)));
	for (int i = 0; i < n_devices; ++i) m->devs[i].comm = comms[i];
	if (cudaMallocHost(&m->h_loc, sizeof(uint64_t) * n_devices) != cudaSuccess)
		return fail(cgpu_internal_set_err(CGPU_ERR_CUDA, "cgpu_multi_create: pinned allocation failed"));
	*out = m;
	return CGPU_OK;
}

int cgpu_multi_destroy(cgpu_multi* m)
{
	if (m) destroy(m);
	return CGPU_OK;
}

int cgpu_multi_size(cgpu_multi* m, int* n)
{
	if (!m || !n) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null argument");
	*n = static_cast<int>(m->devs.size());
	return CGPU_OK;
}

int cgpu_multi_ctx(cgpu_multi* m, int i, cgpu_ctx** out)
{
	if (!m || !out || i < 0 || i >= static_cast<int>(m->devs.size()))
		return cgpu_internal_set_err(CGPU_ERR_INVALID, "bad multi context index");
	*out = m->devs[i].ctx;
	return CGPU_OK;
}

int cgpu_multi_tables_load(cgpu_multi* m, const uint32_t* primes, uint32_t n, const uint8_t* bytes,
                           uint64_t nbytes)
{
	if (!m) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null multi context");
	if (nbytes && !bytes) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null table bytes");
	uint64_t total = 0;
	RCK(cgpu_table_layout(primes, n, nullptr, &total));
	if (total != nbytes)
		return cgpu_internal_set_err(CGPU_ERR_FORMAT, "load_sieve: table stream length does not match the index");
	m->loaded = false;
	const size_t G = m->devs.size();
	const size_t chunk = (nbytes + G - 1) / G;
	for (size_t g = 0; g < G; ++g) {  // 1/G of the host bytes per device (its own PCIe link)
		Dev& d = m->devs[g];
		MCK(cudaSetDevice(d.device));
		MCK(d.tables.ensure(chunk * G + 8));
		const size_t lo = std::min<size_t>(g * chunk, nbytes), hi = std::min<size_t>(lo + chunk, nbytes);
		if (hi > lo)
			MCK(cudaMemcpyAsync(d.tables.p + lo, bytes + lo, hi - lo, cudaMemcpyHostToDevice, d.stream));
	}
	if (G > 1 && chunk) {  // assemble over NVLink, in place
		NCK(nccl().GroupStart());
		for (size_t g = 0; g < G; ++g) {
			Dev& d = m->devs[g];
			NCK(nccl().AllGather(d.tables.p + g * chunk, d.tables.p, chunk, ncclUint8, d.comm, d.stream));
		}
		NCK(nccl().GroupEnd());
	}
	for (Dev& d : m->devs) {
		MCK(cudaSetDevice(d.device));
		RCK(cgpu_tables_load_dev(d.ctx, primes, n, d.tables.p, nbytes));
	}
	m->nprimes = n;
	m->loaded = true;
	return CGPU_OK;
}

int cgpu_multi_set_stop_word(cgpu_multi* m, uint32_t* word)
{
	if (!m) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null multi context");
	for (Dev& d : m->devs) RCK(cgpu_set_stop_word(d.ctx, word));
	return CGPU_OK;
}

int cgpu_multi_sieve(cgpu_multi* m, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end, int mode,
                     uint64_t* counts, uint64_t* hist, uint32_t* block_rmax, uint64_t block_cap,
                     uint64_t* surv_pq, uint64_t surv_cap)
{
	if (q_end && mode != CGPU_REGION)
		return cgpu_internal_set_err(CGPU_ERR_INVALID, "a span ending mid-row is a REGION span");
	if (!m) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null multi context");
	if (!m->loaded) return cgpu_internal_set_err(CGPU_NOT_LOADED, "tables not loaded");
	const uint32_t G = static_cast<uint32_t>(m->devs.size());
	const uint64_t nb = p_hi >= p_lo ? p_hi / 100 - p_lo / 100 + 1 : 0;
	if (block_rmax && block_cap < nb) return cgpu_internal_set_err(CGPU_ERR_CAPACITY, "block_rmax buffer too small");
	const size_t nacc = 2 + m->nprimes;
	const uint64_t dcap = surv_pq ? surv_cap : 0;  // per device: any one shard may hold them all
	// 1. every device sieves its block-cyclic shard
	for (uint32_t g = 0; g < G; ++g) {
		Dev& d = m->devs[g];
		MCK(cudaSetDevice(d.device));
		MCK(d.loc.ensure(nacc));
		MCK(d.red.ensure(nacc));
		MCK(d.brm.ensure(nb));
		MCK(d.surv.ensure(dcap));
		MCK(cudaEventRecord(d.ev[0], d.stream));
		if (q_end)
			RCK(cgpu_sieve_launch_span_dev(d.ctx, p_lo, q_start, p_hi, q_end, G, g, d.loc.p, d.loc.p + 2,
			                               d.brm.p, nb, d.surv.p, dcap));
		else
			RCK(cgpu_sieve_launch_dev(d.ctx, p_lo, q_start, p_hi, mode, G, g, d.loc.p, d.loc.p + 2, d.brm.p,
			                          nb, d.surv.p, dcap));
	}
	// 2. one grouped exchange: counters + histogram (SUM), block r_max (MAX)
	NCK(nccl().GroupStart());
	for (Dev& d : m->devs) {
		NCK(nccl().AllReduce(d.loc.p, d.red.p, nacc, ncclUint64, ncclSum, d.comm, d.stream));
		if (nb) NCK(nccl().AllReduce(d.brm.p, d.brm.p, nb, ncclUint32, ncclMax, d.comm, d.stream));
	}
	NCK(nccl().GroupEnd());
	// 3. survivor gather onto device 0
	for (uint32_t g = 0; g < G; ++g) {
		Dev& d = m->devs[g];
		MCK(cudaSetDevice(d.device));
		MCK(cudaMemcpyAsync(m->h_loc + g, d.loc.p + 1, 8, cudaMemcpyDeviceToHost, d.stream));
	}
	for (Dev& d : m->devs) {
		MCK(cudaSetDevice(d.device));
		MCK(cudaStreamSynchronize(d.stream));
	}
	std::vector<uint64_t> stored(G), off(G + 1, 0);
	bool overflow = false;
	for (uint32_t g = 0; g < G; ++g) {
		stored[g] = std::min<uint64_t>(m->h_loc[g], dcap);
		overflow |= m->h_loc[g] > dcap && surv_pq;
		off[g + 1] = off[g] + stored[g];
	}
	Dev& d0 = m->devs[0];
	if (off[G]) {
		MCK(cudaSetDevice(d0.device));
		MCK(d0.gather.ensure(off[G]));
		if (stored[0])
			MCK(cudaMemcpyAsync(d0.gather.p, d0.surv.p, 8 * stored[0], cudaMemcpyDeviceToDevice, d0.stream));
		if (G > 1) {
			NCK(nccl().GroupStart());
			for (uint32_t g = 1; g < G; ++g) {
				if (!stored[g]) continue;
				NCK(nccl().Send(m->devs[g].surv.p, stored[g], ncclUint64, 0, m->devs[g].comm, m->devs[g].stream));
				NCK(nccl().Recv(d0.gather.p + off[g], stored[g], ncclUint64, static_cast<int>(g), d0.comm, d0.stream));
			}
			NCK(nccl().GroupEnd());
		}
	}
	// results from device 0
	std::vector<uint64_t> acc(nacc), keys(off[G]);
	std::vector<uint32_t> brm(nb);
	MCK(cudaSetDevice(d0.device));
	MCK(cudaMemcpyAsync(acc.data(), d0.red.p, 8 * nacc, cudaMemcpyDeviceToHost, d0.stream));
	if (nb) MCK(cudaMemcpyAsync(brm.data(), d0.brm.p, 4 * nb, cudaMemcpyDeviceToHost, d0.stream));
	if (off[G]) MCK(cudaMemcpyAsync(keys.data(), d0.gather.p, 8 * off[G], cudaMemcpyDeviceToHost, d0.stream));
	for (Dev& d : m->devs) {
		MCK(cudaSetDevice(d.device));
		MCK(cudaEventRecord(d.ev[1], d.stream));
	}
	float worst = 0.f;
	for (Dev& d : m->devs) {  // device time of the step: max over devices
		MCK(cudaSetDevice(d.device));
		MCK(cudaEventSynchronize(d.ev[1]));
		float ms = 0.f;
		MCK(cudaEventElapsedTime(&ms, d.ev[0], d.ev[1]));
		worst = std::max(worst, ms);
	}
	m->last_ms = worst;
	if (counts) {
		counts[0] = acc[0];
		counts[1] = acc[1];
	}
	if (hist) std::copy(acc.begin() + 2, acc.end(), hist);
	if (block_rmax && nb) std::copy(brm.begin(), brm.end(), block_rmax);
	if (surv_pq) {
		std::sort(keys.begin(), keys.end());
		const uint64_t k = std::min<uint64_t>(keys.size(), surv_cap);
		for (uint64_t i = 0; i < k; ++i) {
			surv_pq[2 * i] = keys[i] >> 32;
			surv_pq[2 * i + 1] = keys[i] & 0xffffffffull;
		}
		if (overflow || acc[1] > k) return cgpu_internal_set_err(CGPU_ERR_CAPACITY, "survivor buffer too small");
	}
	return CGPU_OK;
}

int cgpu_multi_last_ms(cgpu_multi* m, float* ms)
{
	if (!m || !ms) return cgpu_internal_set_err(CGPU_ERR_INVALID, "null argument");
	*ms = m->last_ms;
	return CGPU_OK;
}

}  // extern "C"
