#pragma once

// Drop-in B200 implementations of the reference's hot path, for a C++ tree
// that already has the reference's headers (proj/include/cuboid/*.hpp):
//
//   cuboid::gpu::build_table(r)            replaces cuboid::build_table          sievetable.hpp:123-141
//   cuboid::gpu::build_set(primes)         replaces cuboid::SieveSet::build      sievetable.hpp:159-176
//   cuboid::gpu::build_default()           replaces SieveSet::build_default      sievetable.hpp:178-179
//   cuboid::gpu::scan(set, start, p_end,   replaces cuboid::scan                 engine.hpp:195-295
//                     sink, opt)
//   cuboid::gpu::scan_triangle(set, lo, hi, sink)   the TRIANGLE loop of the BASELINE configs
//                                          (verify_small_region's pattern over q < p, engine.hpp:613-625)
//
// Same argument meaning, return types and exceptions as the reference:
// std::invalid_argument / std::overflow_error from the builders, ScanRejected{code}
// from scan, survivors passed to the ScanSink in ascending (p, q) order, each
// with the reference's own exact verdict verify_pair(&set, {p, q}, true)
// (engine.hpp:272-277). The sieve and the table builds run in
// libcuboid_gpu.so (sm_100a) through include/cuboid_gpu.h; there is no CPU
// fallback: without a device every call throws std::runtime_error.
//
// Cooperative stop (ScanOptions::hooks.stop): a flag already raised when scan()
// starts halts exactly where the reference's does -- at the batch_pairs-th q
// visited (engine.hpp:248-257), same resume point and statistics (the span
// before it is sieved with cgpu_sieve_span). A flag raised while the scan
// runs is polled between device tiles of about kStopTilePairs REGION pairs
// (~20 ms each at the B200's rate, whatever the row length); the resume point
// is then the first pair of the next tile. Either way ScanStats::merge of the two
// halves equals the full scan (test_engine.cpp:134-175).

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuboid/engine.hpp"  // the reference: SieveSet, ScanStats, ScanSink, verify_pair, ...
#include "cuboid_gpu.h"

namespace cuboid::gpu {

inline constexpr uint64_t kStopTilePairs = 1ull << 37;

namespace detail {
// Last row of a tile starting at row p: REGION rows hold ~59p pairs, so rows
// p..hi hold ~59/2 (hi^2 - p^2); pick hi for about kStopTilePairs of them.
inline uint64_t tile_end(uint64_t p, uint64_t p_end)
{
	const long double x = static_cast<long double>(p) * p + 2.0L * kStopTilePairs / 59.0L;
	uint64_t hi = static_cast<uint64_t>(std::sqrt(x));
	if (hi < p) hi = p;
	return hi < p_end ? hi : p_end;
}
}  // namespace detail

struct Error : std::runtime_error {
	int code;
	Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

inline void check(int rc, const char* where)
{
	if (rc == CGPU_OK) return;
	const std::string msg = std::string(where) + ": " + cgpu_last_error();
	switch (rc) {
	case CGPU_ERR_INVALID: throw std::invalid_argument(msg);
	case CGPU_ERR_OVERFLOW: throw std::overflow_error(msg);
	case CGPU_ERR_FORMAT: throw FormatError(msg);
	case CGPU_ERR_RANGE: throw std::out_of_range(msg);
	default:
		if (rc >= 2 && rc <= 6) throw ScanRejected(rc);
		throw Error(rc, msg);
	}
}

// One device context per process and device (one process per GPU), holding
// the resident table set.
class Context {
public:
	explicit Context(int device = 0) : device_(device) { check(cgpu_create(device, nullptr, &ctx_), "cgpu_create"); }
	~Context() { cgpu_destroy(ctx_); }
	Context(const Context&) = delete;
	Context& operator=(const Context&) = delete;

	cgpu_ctx* get() { return ctx_; }
	int device() const { return device_; }

	// Makes `set` resident unless it already is (the set is immutable after
	// build, so its bytes are identified by address, size and a sample hash).
	void ensure_resident(const SieveSet& set)
	{
		const Key k = key_of(set);
		if (k == resident_) return;
		std::vector<uint32_t> primes;
		for (const PrimeRecord& r : set.index()) primes.push_back(r.prime);
		check(cgpu_tables_load(ctx_, primes.data(), static_cast<uint32_t>(primes.size()),
		                       set.tables().data(), set.tables().size()),
		      "cgpu_tables_load");
		resident_ = k;
	}
	void mark_resident(const SieveSet& set) { resident_ = key_of(set); }

	std::mutex& mutex() { return mu_; }

private:
	struct Key {
		const void* data = nullptr;
		size_t size = 0, nprimes = 0;
		uint64_t hash = 0;
		bool operator==(const Key& o) const
		{
			return data == o.data && size == o.size && nprimes == o.nprimes && hash == o.hash;
		}
	};
	static Key key_of(const SieveSet& set)
	{
		Key k{set.tables().data(), set.tables().size(), set.prime_count(), 1469598103934665603ull};
		const auto& t = set.tables();
		for (size_t i = 0; i < t.size(); i += 61) k.hash = (k.hash ^ t[i]) * 1099511628211ull;
		for (const PrimeRecord& r : set.index()) k.hash = (k.hash ^ r.prime) * 1099511628211ull;
		return k;
	}

	int device_;
	cgpu_ctx* ctx_ = nullptr;
	Key resident_;
	std::mutex mu_;
};

inline Context& context(int device = 0)
{
	static std::mutex mu;
	static std::map<int, Context*> ctxs;  // process lifetime
	std::lock_guard<std::mutex> lk(mu);
	auto it = ctxs.find(device);
	if (it == ctxs.end()) it = ctxs.emplace(device, new Context(device)).first;
	return *it->second;
}

// ---- tables ------------------------------------------------------------------

inline SieveSet build_set(const std::vector<uint32_t>& primes, int device = 0,
                          int algorithm = CGPU_BUILD_PRODUCTION)
{
	Context& c = context(device);
	std::lock_guard<std::mutex> lk(c.mutex());
	const uint32_t n = static_cast<uint32_t>(primes.size());
	std::vector<uint32_t> offsets(n);
	uint64_t total = 0;
	check(cgpu_table_layout(primes.data(), n, offsets.data(), &total), "SieveSet::build");
	std::vector<uint8_t> tables(total);
	check(cgpu_tables_build(c.get(), primes.data(), n, algorithm, tables.data(), nullptr, nullptr),
	      "SieveSet::build");
	std::vector<PrimeRecord> index(n);
	for (uint32_t k = 0; k < n; ++k) index[k] = {static_cast<uint16_t>(primes[k]), offsets[k]};
	SieveSet s = SieveSet::from_parts(std::move(index), std::move(tables));
	return s;
}

inline SieveSet build_default(int device = 0) { return build_set(primes_in_range(11, 541), device); }

inline BitTable build_table(uint32_t r, int device = 0)
{
	SieveSet s = build_set({r}, device);
	return BitTable{r, s.tables()};
}

// ---- sieve -------------------------------------------------------------------

namespace detail {

struct DeviceScan {
	uint64_t counts[2] = {0, 0};
	std::vector<uint64_t> hist;
	uint64_t block_lo = 0;
	std::vector<uint32_t> block_rmax;
	std::vector<uint64_t> surv;  // (p, q) pairs, ascending
};

inline DeviceScan run(Context& c, const SieveSet& set, uint64_t p_lo, uint64_t q_start, uint64_t p_hi,
                      int mode)
{
	DeviceScan d;
	d.hist.assign(set.prime_count(), 0);
	d.block_lo = p_lo / 100;
	const uint64_t nb = p_hi >= p_lo ? p_hi / 100 - p_lo / 100 + 1 : 0;
	d.block_rmax.assign(nb ? nb : 1, 0);
	uint64_t cap = 1 << 16;
	for (;;) {
		d.surv.assign(2 * cap, 0);
		const int rc = cgpu_sieve(c.get(), p_lo, q_start, p_hi, mode, 1, 0, d.counts, d.hist.data(),
		                          d.block_rmax.data(), nb, d.surv.data(), cap);
		if (rc == CGPU_ERR_CAPACITY && d.counts[1] > cap) {
			cap = d.counts[1];
			continue;
		}
		check(rc, "scan");
		break;
	}
	d.surv.resize(2 * d.counts[1]);
	return d;
}

// The (p, q) at which the reference halts with a raised stop flag: the
// batch_pairs-th q visited from `start` (engine.hpp:248-257); false if the
// range ends first.
inline bool stop_point(SearchPair start, uint64_t p_end, uint64_t batch_pairs, SearchPair& at)
{
	uint64_t k = batch_pairs ? batch_pairs : 1;
	for (uint64_t p = start.p; p <= p_end; ++p) {
		const RegionBounds b = q_bounds(p);
		const uint64_t q0 = p == start.p ? start.q : b.q_low;
		const uint64_t n = b.q_high >= q0 ? b.q_high - q0 + 1 : 0;
		if (k <= n) {
			at = {p, q0 + k - 1};
			return true;
		}
		k -= n;
	}
	return false;
}

// REGION pairs from `from` up to, not including, `to` (sieved on the device).
inline DeviceScan run_span(Context& c, const SieveSet& set, SearchPair from, SearchPair to)
{
	DeviceScan d;
	d.hist.assign(set.prime_count(), 0);
	const uint64_t first = to.p == from.p ? from.q : q_bounds(to.p).q_low;
	uint64_t p_hi = to.p, q_end = to.q - 1;
	if (to.q == first) {  // the stop is the row's first pair: that row is not sieved
		p_hi = to.p - 1;
		q_end = 0;
	}
	if (p_hi < from.p) return d;
	d.block_lo = from.p / 100;
	const uint64_t nb = p_hi / 100 - from.p / 100 + 1;
	d.block_rmax.assign(nb, 0);
	uint64_t cap = 1 << 16;
	for (;;) {
		d.surv.assign(2 * cap, 0);
		const int rc = cgpu_sieve_span(c.get(), from.p, from.q, p_hi, q_end, d.counts, d.hist.data(),
		                               d.block_rmax.data(), nb, d.surv.data(), cap);
		if (rc == CGPU_ERR_CAPACITY && d.counts[1] > cap) {
			cap = d.counts[1];
			continue;
		}
		check(rc, "scan");
		break;
	}
	d.surv.resize(2 * d.counts[1]);
	return d;
}

inline void fold(const SieveSet& set, const DeviceScan& d, ScanStats& st, const ScanSink& sink)
{
	st.pairs_tested += d.counts[0];
	st.survivors += d.counts[1];
	for (size_t k = 0; k < d.hist.size(); ++k)
		if (d.hist[k]) st.kill_histogram[set.prime_at(k)] += d.hist[k];
	for (size_t i = 0; i < d.block_rmax.size(); ++i)
		if (d.block_rmax[i]) {
			auto& cur = st.block_r_max[d.block_lo + i];
			if (d.block_rmax[i] > cur) cur = d.block_rmax[i];
		}
	if (sink)
		for (size_t i = 0; i < d.surv.size(); i += 2) {
			const uint64_t p = d.surv[i], q = d.surv[i + 1];
			sink(ScanEvent{p, q, verify_pair(&set, {p, q}, /*bypass_sieve=*/true)});
		}
}

}  // namespace detail

inline ScanStats scan(const SieveSet& set, SearchPair start, uint64_t p_end, const ScanSink& sink = {},
                      const ScanOptions& opt = {}, int device = 0)
{
	if (set.empty()) throw ScanRejected(6);
	if (int code = validate_start(true, start.p, start.q, opt)) throw ScanRejected(code);
	if (p_end > opt.p_limit) throw ScanRejected(3);
	if (p_end > p_limit_32bit()) throw ScanRejected(3);  // device rows are 32-bit (59p < 2^32)

	ScanStats st;
	st.resume_p = start.p;
	st.resume_q = start.q;
	const auto t0 = std::chrono::steady_clock::now();
	Context& c = context(device);
	std::lock_guard<std::mutex> lk(c.mutex());
	c.ensure_resident(set);

	SearchPair at{};
	if (opt.hooks.stop && opt.hooks.stop->load(std::memory_order_relaxed) &&
	    detail::stop_point(start, p_end, opt.batch_pairs, at)) {
		detail::fold(set, detail::run_span(c, set, start, at), st, sink);
		st.block_r_max.try_emplace(at.p / 100, 1u);  // the stop row's block was entered
		st.resume_p = at.p;
		st.resume_q = at.q;
		st.stopped = true;
		st.elapsed = std::chrono::steady_clock::now() - t0;
		return st;
	}
	uint64_t p = start.p, q = start.q;
	while (p <= p_end) {
		if (opt.hooks.stop && opt.hooks.stop->load(std::memory_order_relaxed)) {
			st.stopped = true;
			break;
		}
		const uint64_t hi = opt.hooks.stop ? detail::tile_end(p, p_end) : p_end;
		const detail::DeviceScan d = detail::run(c, set, p, q, hi, CGPU_REGION);
		detail::fold(set, d, st, sink);
		cuboid::detail::next_pair(hi, q_bounds(hi).q_high, q_bounds(hi).q_high, st.resume_p, st.resume_q);
		if (opt.hooks.current_p) opt.hooks.current_p->store(hi, std::memory_order_relaxed);
		if (opt.hooks.current_q) opt.hooks.current_q->store(q_bounds(hi).q_high, std::memory_order_relaxed);
		if (opt.hooks.current_r_max) {
			const auto it = st.block_r_max.find(hi / 100);
			opt.hooks.current_r_max->store(it == st.block_r_max.end() ? 1 : it->second,
			                               std::memory_order_relaxed);
		}
		p = st.resume_p;
		q = st.resume_q;
	}
	st.elapsed = std::chrono::steady_clock::now() - t0;
	return st;
}

inline ScanStats scan_triangle(const SieveSet& set, uint64_t p_lo, uint64_t p_hi, const ScanSink& sink = {},
                               int device = 0)
{
	if (set.empty()) throw ScanRejected(6);
	if (p_lo == 0 || p_hi > UINT32_MAX) throw ScanRejected(3);
	ScanStats st;
	st.resume_p = p_lo;
	st.resume_q = 1;
	const auto t0 = std::chrono::steady_clock::now();
	if (p_lo <= p_hi) {
		Context& c = context(device);
		std::lock_guard<std::mutex> lk(c.mutex());
		c.ensure_resident(set);
		detail::fold(set, detail::run(c, set, p_lo, 0, p_hi, CGPU_TRIANGLE), st, sink);
		st.resume_p = p_hi + 1;
	}
	st.elapsed = std::chrono::steady_clock::now() - t0;
	return st;
}

}  // namespace cuboid::gpu
