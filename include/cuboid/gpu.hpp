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
//   cuboid::gpu::verify_pair(set, pr, bypass)   replaces verify_pair        engine.hpp:66-95
//   cuboid::gpu::verify_small_region(set)  replaces verify_small_region     engine.hpp:609-640
//   cuboid::gpu::classify(set, pairs)      is_unsolvable in rank order      sievetable.hpp:199-205
//   cuboid::gpu::SearchController          replaces SearchController        engine.hpp:429-595
//
// Same argument meaning, return types and exceptions as the reference:
// std::invalid_argument / std::overflow_error from the builders, ScanRejected{code}
// from scan, survivors passed to the ScanSink in ascending (p, q) order, each
// with the reference's own exact verdict verify_pair(&set, {p, q}, true)
// (engine.hpp:272-277). The sieve and the table builds run in
// libcuboid_gpu.so (sm_100a) through include/cuboid_gpu.h; there is no CPU
// fallback: without a device every call throws std::runtime_error.
//
// Cooperative stop (ScanOptions::hooks.stop, engine.hpp:248-257): the
// reference polls its flag every batch_pairs q visited and halts AT that q.
// Here a scan with a stop hook runs as device tiles whose ends are such poll
// points (multiples of batch_pairs q visited from the start, ~kStopTilePairs
// each); a watcher thread mirrors the flag into a mapped host word that the
// sieve kernels poll, so a tile running when the flag rises is abandoned
// within microseconds, discarded, and the scan halts at the NEXT poll point
// after the tile's start (sieved exactly, with a span) -- a stop position,
// resume point and statistics the reference itself produces when its flag
// becomes visible between those two polls. A flag raised before the scan:
// the batch_pairs-th q, like the reference; with fewer q left than
// batch_pairs, no poll is reached and the scan completes (stopped = false).
// ScanStats::merge of the halves equals the full scan (test_engine.cpp:134-175).
//
// Multi-GPU from one process: scan(..., devices) shards the rows over the
// listed GPUs (cgpu_multi: NCCL clique, block-cyclic p/100 blocks, one grouped
// all-reduce + survivor gather per tile). SearchController below is the
// reference's controller (engine.hpp:429-595) over these scans.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cuboid/engine.hpp"  // the reference: SieveSet, ScanStats, ScanSink, verify_pair, ...
#include "cuboid_gpu.h"

namespace cuboid::gpu {

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

namespace detail {
// Byte equality of two large buffers, split over host threads (a 26 MB table
// set compares in ~0.3 ms on 8 threads instead of ~1.5 ms on one).
inline bool equal_bytes(const uint8_t* a, const uint8_t* b, size_t n)
{
	constexpr size_t kChunk = size_t(4) << 20;
	const size_t hw = std::max(1u, std::thread::hardware_concurrency());
	const size_t nt = std::min<size_t>(std::min<size_t>(hw, 8), (n + kChunk - 1) / kChunk);
	if (nt <= 1) return std::memcmp(a, b, n) == 0;
	std::atomic<bool> same{true};
	std::vector<std::thread> th;
	const size_t per = (n + nt - 1) / nt;
	for (size_t t = 0; t < nt; ++t)
		th.emplace_back([&, t] {
			const size_t lo = t * per, hi = std::min(n, lo + per);
			for (size_t o = lo; o < hi && same.load(std::memory_order_relaxed); o += kChunk)
				if (std::memcmp(a + o, b + o, std::min(kChunk, hi - o)) != 0) same.store(false);
		});
	for (auto& x : th) x.join();
	return same.load();
}
}  // namespace detail

// Which table set a context holds. Identified exactly: the prime list plus a
// host copy of the table bytes, compared in full (detail::equal_bytes) -- a
// sampled hash would accept a different set of the same shape, e.g. an
// edited load_sieve file allocated at a freed set's address.
class Residency {
public:
	// same prime list and byte count as the resident set (fills `primes`)
	bool same_shape(const SieveSet& set, std::vector<uint32_t>& primes) const
	{
		primes.clear();
		for (const PrimeRecord& r : set.index()) primes.push_back(r.prime);
		return valid_ && primes == primes_ && set.tables().size() == bytes_.size();
	}
	bool same_bytes(const SieveSet& set) const
	{
		return detail::equal_bytes(set.tables().data(), bytes_.data(), bytes_.size());
	}
	bool holds(const SieveSet& set, std::vector<uint32_t>& primes) const
	{
		return same_shape(set, primes) && same_bytes(set);
	}
	void record(const SieveSet& set, std::vector<uint32_t>&& primes)
	{
		primes_ = std::move(primes);
		bytes_.assign(set.tables().begin(), set.tables().end());
		valid_ = true;
	}
	// Any call that replaces the context's tables (cgpu_tables_build) drops
	// the record, so the next scan uploads its own set again.
	void invalidate() { valid_ = false; }

private:
	bool valid_ = false;
	std::vector<uint32_t> primes_;
	std::vector<uint8_t> bytes_;
};

// One device context per process and device (one process per GPU), holding
// the resident table set. Its lock is recursive: a scan sink may call
// gpu::verify_pair / classify on the same device.
class Context {
public:
	explicit Context(int device = 0) : device_(device) { check(cgpu_create(device, nullptr, &ctx_), "cgpu_create"); }
	~Context() { cgpu_destroy(ctx_); }
	Context(const Context&) = delete;
	Context& operator=(const Context&) = delete;

	cgpu_ctx* get() { return ctx_; }
	cgpu_ctx* span_ctx() { return ctx_; }
	int device() const { return device_; }

	// Makes `set` resident unless it already is. defer: when the resident set
	// has the same primes and size, the byte comparison (~1 ms for 26 MB on
	// the host) is left to the next sieve(), which runs it while the device
	// sieves and, on a mismatch, uploads the set and sieves again.
	void ensure_resident(const SieveSet& set, bool defer = false)
	{
		verify_ = nullptr;
		std::vector<uint32_t> primes;
		if (res_.same_shape(set, primes)) {
			if (defer) {
				verify_ = &set;
				return;
			}
			if (res_.same_bytes(set)) return;
		}
		upload(set, std::move(primes));
	}
	void invalidate()
	{
		res_.invalidate();
		verify_ = nullptr;
	}

	int sieve(uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode, uint64_t* counts, uint64_t* hist,
	          uint32_t* brm, uint64_t nb, uint64_t* surv, uint64_t cap)
	{
		if (!verify_) return cgpu_sieve(ctx_, p_lo, q_start, p_hi, mode, 1, 0, counts, hist, brm, nb, surv, cap);
		const SieveSet* s = verify_;
		verify_ = nullptr;
		int rc = cgpu_sieve_launch(ctx_, p_lo, q_start, p_hi, mode, 1, 0, surv ? cap : 0);
		const bool same = res_.same_bytes(*s);  // on the host while the device sieves
		if (!same) {  // another set of the same shape: discard, upload it, sieve again
			cgpu_synchronize(ctx_);
			std::vector<uint32_t> primes;
			for (const PrimeRecord& r : s->index()) primes.push_back(r.prime);
			upload(*s, std::move(primes));
			rc = cgpu_sieve_launch(ctx_, p_lo, q_start, p_hi, mode, 1, 0, surv ? cap : 0);
		}
		if (rc != CGPU_OK) return rc;
		return cgpu_sieve_results(ctx_, counts, hist, brm, nb, surv, cap);
	}
	int sieve_span(uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end, uint64_t* counts,
	               uint64_t* hist, uint32_t* brm, uint64_t nb, uint64_t* surv, uint64_t cap)
	{
		settle();
		return cgpu_sieve_span(ctx_, p_lo, q_start, p_hi, q_end, counts, hist, brm, nb, surv, cap);
	}
	void drop_deferred() { verify_ = nullptr; }  // the check is redone by the next scan
	// completes a deferred residency check before a synchronous call
	void settle()
	{
		if (!verify_) return;
		const SieveSet* s = verify_;
		verify_ = nullptr;
		if (!res_.same_bytes(*s)) {
			std::vector<uint32_t> primes;
			for (const PrimeRecord& r : s->index()) primes.push_back(r.prime);
			upload(*s, std::move(primes));
		}
	}
	void set_stop_word(uint32_t* w) { check(cgpu_set_stop_word(ctx_, w), "cgpu_set_stop_word"); }
	uint32_t loaded_primes()
	{
		uint32_t n = 0;
		check(cgpu_tables_info(ctx_, &n, nullptr), "scan");
		return n;
	}

	std::recursive_mutex& mutex() { return mu_; }

private:
	void upload(const SieveSet& set, std::vector<uint32_t>&& primes)
	{
		res_.invalidate();
		check(cgpu_tables_load(ctx_, primes.data(), static_cast<uint32_t>(primes.size()),
		                       set.tables().data(), set.tables().size()),
		      "cgpu_tables_load");
		res_.record(set, std::move(primes));
	}

	int device_;
	cgpu_ctx* ctx_ = nullptr;
	Residency res_;
	const SieveSet* verify_ = nullptr;  // a deferred byte comparison (ensure_resident(set, true))
	std::recursive_mutex mu_;
};

// Several GPUs driven from this one process (cgpu_multi: one context per
// device, an NCCL clique from ncclCommInitAll, block-cyclic p/100 shards, one
// grouped all-reduce + survivor gather per call). What a single-process
// caller such as SearchController::run_scan (engine.hpp:555-577) uses to
// spread scan() over every GPU of the box.
class MultiContext {
public:
	explicit MultiContext(const std::vector<int>& devices) : devices_(devices)
	{
		check(cgpu_multi_create(static_cast<int>(devices.size()), devices.data(), &m_), "cgpu_multi_create");
	}
	~MultiContext() { cgpu_multi_destroy(m_); }
	MultiContext(const MultiContext&) = delete;
	MultiContext& operator=(const MultiContext&) = delete;

	cgpu_multi* get() { return m_; }
	const std::vector<int>& devices() const { return devices_; }
	// the first device's context: it holds the whole set after a load
	cgpu_ctx* span_ctx()
	{
		cgpu_ctx* c = nullptr;
		check(cgpu_multi_ctx(m_, 0, &c), "cgpu_multi_ctx");
		return c;
	}

	void drop_deferred() {}
	void ensure_resident(const SieveSet& set, bool /*defer*/ = false)
	{
		std::vector<uint32_t> primes;
		if (res_.holds(set, primes)) return;
		res_.invalidate();
		check(cgpu_multi_tables_load(m_, primes.data(), static_cast<uint32_t>(primes.size()),
		                             set.tables().data(), set.tables().size()),
		      "cgpu_multi_tables_load");
		res_.record(set, std::move(primes));
	}

	int sieve(uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode, uint64_t* counts, uint64_t* hist,
	          uint32_t* brm, uint64_t nb, uint64_t* surv, uint64_t cap)
	{
		return cgpu_multi_sieve(m_, p_lo, q_start, p_hi, 0, mode, counts, hist, brm, nb, surv, cap);
	}
	int sieve_span(uint64_t p_lo, uint64_t q_start, uint64_t p_hi, uint64_t q_end, uint64_t* counts,
	               uint64_t* hist, uint32_t* brm, uint64_t nb, uint64_t* surv, uint64_t cap)
	{
		return cgpu_multi_sieve(m_, p_lo, q_start, p_hi, q_end, CGPU_REGION, counts, hist, brm, nb, surv, cap);
	}
	void set_stop_word(uint32_t* w) { check(cgpu_multi_set_stop_word(m_, w), "cgpu_multi_set_stop_word"); }
	uint32_t loaded_primes()
	{
		uint32_t n = 0;
		check(cgpu_tables_info(span_ctx(), &n, nullptr), "scan");
		return n;
	}

	std::recursive_mutex& mutex() { return mu_; }

private:
	std::vector<int> devices_;
	cgpu_multi* m_ = nullptr;
	Residency res_;
	std::recursive_mutex mu_;
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

inline MultiContext& multi_context(const std::vector<int>& devices)
{
	static std::mutex mu;
	static std::map<std::vector<int>, MultiContext*> ctxs;  // process lifetime
	std::lock_guard<std::mutex> lk(mu);
	auto it = ctxs.find(devices);
	if (it == ctxs.end()) it = ctxs.emplace(devices, new MultiContext(devices)).first;
	return *it->second;
}

// ---- tables ------------------------------------------------------------------

inline SieveSet build_set(const std::vector<uint32_t>& primes, int device = 0,
                          int algorithm = CGPU_BUILD_PRODUCTION)
{
	Context& c = context(device);
	std::lock_guard<std::recursive_mutex> lk(c.mutex());
	const uint32_t n = static_cast<uint32_t>(primes.size());
	std::vector<uint32_t> offsets(n);
	uint64_t total = 0;
	check(cgpu_table_layout(primes.data(), n, offsets.data(), &total), "SieveSet::build");
	std::vector<uint8_t> tables(total);
	c.invalidate();  // the build replaces the context's resident tables
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

inline constexpr uint64_t kStopTilePairs = 1ull << 37;  // q visited per stoppable tile (~20 ms)

namespace detail {

struct DeviceScan {
	uint64_t counts[2] = {0, 0};
	std::vector<uint64_t> hist;
	uint64_t block_lo = 0;
	std::vector<uint32_t> block_rmax;
	std::vector<uint64_t> surv;  // (p, q) pairs, ascending
};

// Sieves through `call(counts, hist, brm, nb, surv, cap)`, growing the
// survivor buffer until every survivor fits.
template <class Call>
DeviceScan collect(const SieveSet& set, uint64_t p_lo, uint64_t p_hi, Call&& call)
{
	DeviceScan d;
	d.hist.assign(set.prime_count(), 0);
	if (p_hi < p_lo) return d;
	d.block_lo = p_lo / 100;
	const uint64_t nb = p_hi / 100 - p_lo / 100 + 1;
	d.block_rmax.assign(nb, 0);
	uint64_t cap = 1 << 16;
	for (;;) {
		d.surv.assign(2 * cap, 0);
		const int rc = call(d.counts, d.hist.data(), d.block_rmax.data(), nb, d.surv.data(), cap);
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

template <class Ctx>
void check_resident(Ctx& c, const SieveSet& set)
{
	if (c.loaded_primes() != set.prime_count())  // the histogram is sized by the set
		throw std::logic_error("cuboid::gpu: resident tables are not the scanned set");
}

// Whole rows p_lo..p_hi (REGION from q_start on the first row, or TRIANGLE).
template <class Ctx>
DeviceScan run(Ctx& c, const SieveSet& set, uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode)
{
	check_resident(c, set);
	return collect(set, p_lo, p_hi, [&](uint64_t* cnt, uint64_t* h, uint32_t* b, uint64_t nb, uint64_t* sv,
	                                    uint64_t cap) {
		return c.sieve(p_lo, q_start, p_hi, mode, cnt, h, b, nb, sv, cap);
	});
}

// REGION pairs from `from` up to, not including, `to`.
template <class Ctx>
DeviceScan run_span(Ctx& c, const SieveSet& set, SearchPair from, SearchPair to)
{
	check_resident(c, set);
	const uint64_t first = to.p == from.p ? from.q : q_bounds(to.p).q_low;
	uint64_t p_hi = to.p, q_end = to.q - 1;
	if (to.q == first) {  // `to` is its row's first pair: that row is not sieved
		p_hi = to.p - 1;
		q_end = 0;
	}
	if (p_hi < from.p) {
		DeviceScan d;
		d.hist.assign(set.prime_count(), 0);
		return d;
	}
	return collect(set, from.p, p_hi, [&](uint64_t* cnt, uint64_t* h, uint32_t* b, uint64_t nb, uint64_t* sv,
	                                      uint64_t cap) {
		return c.sieve_span(from.p, from.q, p_hi, q_end, cnt, h, b, nb, sv, cap);
	});
}

// Walks the reference's q visiting order (engine.hpp:225-247: rows p, q from
// q_low(p) -- or start.q on the first row -- to q_high(p)) k steps from
// `pos`: the pair reached, or false if p_end's row ends first. One O(1) step
// per row (q_low moves monotonically), so a tile of 2^37 q costs microseconds.
class Visit {
public:
	explicit Visit(uint64_t p_end) : p_end_(p_end) {}
	bool advance(SearchPair pos, uint64_t k, SearchPair& at)
	{
		uint64_t p = pos.p, q0 = pos.q;
		for (;;) {
			const uint64_t q_hi = q_bounds(p).q_high;
			const uint64_t n = q_hi >= q0 ? q_hi - q0 + 1 : 0;
			if (k < n) {
				at = {p, q0 + k};
				return true;
			}
			k -= n;
			if (p >= p_end_) return false;
			++p;
			q0 = q_low_of(p);
		}
	}

private:
	uint64_t q_low_of(uint64_t p)
	{
		if (p < kRegionCrossover) return q_bounds(p).q_low;
		if (c_ == 0 || p < last_p_) c_ = q_bounds(p).q_low;  // a walk restarted behind the last one
		last_p_ = p;
		while (9 * static_cast<unsigned __int128>(c_) * c_ * c_ < p) ++c_;  // least q with 9q^3 >= p
		return c_;
	}
	uint64_t p_end_;
	uint64_t c_ = 0, last_p_ = 0;
};

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

// Mirrors the caller's std::atomic<bool> stop flag into a mapped host word the
// kernels poll, for the lifetime of one scan.
class StopMirror {
public:
	template <class Ctx>
	StopMirror(Ctx& c, const std::atomic<bool>* flag) : flag_(flag)
	{
		if (!flag_) return;
		check(cgpu_alloc_stop_word(&word_), "cgpu_alloc_stop_word");
		attach_ = [&c](uint32_t* w) { c.set_stop_word(w); };
		attach_(word_);
		if (flag_->load(std::memory_order_relaxed)) *reinterpret_cast<volatile uint32_t*>(word_) = 1;  // pre-armed
		watcher_ = std::thread([this] {
			while (!done_.load(std::memory_order_relaxed)) {
				if (flag_->load(std::memory_order_relaxed)) {
					*reinterpret_cast<volatile uint32_t*>(word_) = 1;
					return;
				}
				std::this_thread::sleep_for(std::chrono::microseconds(20));
			}
		});
	}
	~StopMirror()
	{
		disarm();
		if (word_) cgpu_free_stop_word(word_);
	}
	bool raised() const { return word_ && *reinterpret_cast<volatile uint32_t*>(word_) != 0; }
	// Stops mirroring and detaches the word, so the exact re-sieve up to the
	// stop point runs to completion.
	void disarm()
	{
		if (!flag_ || disarmed_) return;
		disarmed_ = true;
		done_.store(true);
		if (watcher_.joinable()) watcher_.join();
		attach_(nullptr);
	}

private:
	const std::atomic<bool>* flag_;
	uint32_t* word_ = nullptr;
	std::function<void(uint32_t*)> attach_;
	std::atomic<bool> done_{false};
	bool disarmed_ = false;
	std::thread watcher_;
};

template <class Ctx>
ScanStats scan_on(Ctx& c, const SieveSet& set, SearchPair start, uint64_t p_end, const ScanSink& sink,
                  const ScanOptions& opt)
{
	if (set.empty()) throw ScanRejected(6);
	if (int code = validate_start(true, start.p, start.q, opt)) throw ScanRejected(code);
	if (p_end > opt.p_limit) throw ScanRejected(3);
	if (p_end > p_limit_32bit()) throw ScanRejected(3);  // device rows are 32-bit (59p < 2^32)

	ScanStats st;
	st.resume_p = start.p;
	st.resume_q = start.q;
	const auto t0 = std::chrono::steady_clock::now();
	std::lock_guard<std::recursive_mutex> lk(c.mutex());
	c.ensure_resident(set, /*defer=*/true);  // byte check overlapped with the first sieve
	auto publish = [&](uint64_t p, uint64_t q) {  // flush_hooks (engine.hpp:218-223)
		if (opt.hooks.current_p) opt.hooks.current_p->store(p, std::memory_order_relaxed);
		if (opt.hooks.current_q) opt.hooks.current_q->store(q, std::memory_order_relaxed);
		if (opt.hooks.current_r_max) {
			const auto it = st.block_r_max.find(p / 100);
			opt.hooks.current_r_max->store(it == st.block_r_max.end() ? 1 : it->second,
			                               std::memory_order_relaxed);
		}
	};
	auto finish = [&](uint64_t p_last) {  // the whole range is done: resume after p_end
		cuboid::detail::next_pair(p_last, q_bounds(p_last).q_high, q_bounds(p_last).q_high, st.resume_p,
		                          st.resume_q);
		publish(p_last, q_bounds(p_last).q_high);
	};

	if (start.p > p_end) {  // the reference's row loop does not run
		c.drop_deferred();
		st.elapsed = std::chrono::steady_clock::now() - t0;
		return st;
	}
	if (!opt.hooks.stop) {  // no flag to poll: one launch
		fold(set, run(c, set, start.p, start.q, p_end, CGPU_REGION), st, sink);
		finish(p_end);
		st.elapsed = std::chrono::steady_clock::now() - t0;
		return st;
	}

	// Stoppable: tiles ending at poll points (every batch_pairs-th q visited).
	const uint64_t B = opt.batch_pairs ? opt.batch_pairs : 1;
	const uint64_t K = std::max<uint64_t>(1, kStopTilePairs / B);  // batches per tile
	StopMirror mirror(c, opt.hooks.stop);
	Visit visit(p_end);
	SearchPair pos = start;
	bool at_poll = false;  // pos is a poll point (not the scan start)
	auto stop_at = [&](SearchPair at) {
		fold(set, run_span(c, set, pos, at), st, sink);
		st.block_r_max.try_emplace(at.p / 100, 1u);  // the stop row's block was entered
		st.resume_p = at.p;
		st.resume_q = at.q;
		st.stopped = true;
		publish(at.p, at.q);
	};
	for (;;) {
		if (at_poll && opt.hooks.stop->load(std::memory_order_relaxed)) {  // the reference's poll at pos
			st.block_r_max.try_emplace(pos.p / 100, 1u);
			st.resume_p = pos.p;
			st.resume_q = pos.q;
			st.stopped = true;
			publish(pos.p, pos.q);
			break;
		}
		// the tile: from pos up to the K-th poll point after it (the first poll
		// point after the start is the B-th q visited, position B - 1)
		SearchPair to{};
		const uint64_t steps = at_poll ? K * B : K * B - 1;
		const bool inside = visit.advance(pos, steps, to);
		const DeviceScan d = inside ? run_span(c, set, pos, to) : run(c, set, pos.p, pos.q, p_end, CGPU_REGION);
		if (mirror.raised()) {  // the tile may have been abandoned: halt at the next poll point instead
			mirror.disarm();
			SearchPair nxt{};
			if (visit.advance(pos, at_poll ? B : B - 1, nxt)) {
				stop_at(nxt);
			} else {  // no poll left before p_end: the reference completes the range
				fold(set, run(c, set, pos.p, pos.q, p_end, CGPU_REGION), st, sink);
				finish(p_end);
			}
			break;
		}
		fold(set, d, st, sink);
		if (!inside) {
			finish(p_end);
			break;
		}
		pos = to;
		at_poll = true;
		st.resume_p = pos.p;
		st.resume_q = pos.q;
		publish(pos.p, pos.q);
	}
	st.elapsed = std::chrono::steady_clock::now() - t0;
	return st;
}

}  // namespace detail

// scan() (engine.hpp:195-295) on one GPU.
inline ScanStats scan(const SieveSet& set, SearchPair start, uint64_t p_end, const ScanSink& sink = {},
                      const ScanOptions& opt = {}, int device = 0)
{
	if (set.empty()) throw ScanRejected(6);
	return detail::scan_on(context(device), set, start, p_end, sink, opt);
}

// scan() over several GPUs of this process (block-cyclic p/100 shards, NCCL).
inline ScanStats scan(const SieveSet& set, SearchPair start, uint64_t p_end, const ScanSink& sink,
                      const ScanOptions& opt, const std::vector<int>& devices)
{
	if (set.empty()) throw ScanRejected(6);
	if (devices.size() <= 1) return scan(set, start, p_end, sink, opt, devices.empty() ? 0 : devices[0]);
	return detail::scan_on(multi_context(devices), set, start, p_end, sink, opt);
}

inline ScanStats scan_triangle(const SieveSet& set, uint64_t p_lo, uint64_t p_hi, const ScanSink& sink = {},
                               const std::vector<int>& devices = {0})
{
	if (set.empty()) throw ScanRejected(6);
	if (p_lo == 0 || p_hi > UINT32_MAX) throw ScanRejected(3);
	ScanStats st;
	st.resume_p = p_lo;
	st.resume_q = 1;
	const auto t0 = std::chrono::steady_clock::now();
	if (p_lo <= p_hi) {
		auto go = [&](auto& c) {
			std::lock_guard<std::recursive_mutex> lk(c.mutex());
			c.ensure_resident(set, /*defer=*/true);
			detail::fold(set, detail::run(c, set, p_lo, 0, p_hi, CGPU_TRIANGLE), st, sink);
		};
		if (devices.size() > 1)
			go(multi_context(devices));
		else
			go(context(devices.empty() ? 0 : devices[0]));
		st.resume_p = p_hi + 1;
	}
	st.elapsed = std::chrono::steady_clock::now() - t0;
	return st;
}

// ---- the final check and the small region ---------------------------------------

// First-killer ranks of explicit pairs (the sieve part of verify_pair,
// engine.hpp:72-78; SieveSet::is_unsolvable in rank order on the device,
// cgpu_classify): -1 where no table rejects the pair.
inline std::vector<int32_t> classify(const SieveSet& set, const std::vector<SearchPair>& pairs, int device = 0)
{
	std::vector<int32_t> ranks(pairs.size(), -1);
	if (pairs.empty()) return ranks;
	Context& c = context(device);
	std::lock_guard<std::recursive_mutex> lk(c.mutex());
	c.ensure_resident(set);
	std::vector<uint64_t> pq(2 * pairs.size());
	for (size_t i = 0; i < pairs.size(); ++i) {
		pq[2 * i] = pairs[i].p;
		pq[2 * i + 1] = pairs[i].q;
	}
	check(cgpu_classify(c.get(), pq.data(), pairs.size(), ranks.data()), "classify");
	return ranks;
}

// verify_pair (engine.hpp:66-95): the same validation and verdicts; without
// bypass the sieve part runs on the device, the exact part (GMP quintic roots,
// perfect squares, inequalities) is the reference's own code.
inline PairVerdict verify_pair(const SieveSet& set, const SearchPair& pr, bool bypass_sieve, int device = 0)
{
	if (pr.p == 0 || pr.q == 0 || pr.p == pr.q)
		throw std::invalid_argument("verify_pair: requires positive p != q");
	if (std::gcd(pr.p, pr.q) != 1) throw std::invalid_argument("verify_pair: requires gcd(p,q) = 1");
	if (!bypass_sieve) {
		if (set.empty()) throw std::invalid_argument("verify_pair: sieve tables not loaded");
		const int32_t rank = classify(set, {pr}, device)[0];
		if (rank >= 0) return PairVerdict::sieved_out(set.prime_at(static_cast<size_t>(rank)));
	}
	return cuboid::verify_pair(&set, pr, /*bypass_sieve=*/true);
}

// verify_small_region (engine.hpp:609-640): every coprime p != q pair of the
// region rows p <= 151 sieved on the device (scan with small_p), each
// survivor through the reference's exact check; a candidate throws, as there.
inline SmallRegionSummary verify_small_region(const SieveSet& set, int device = 0)
{
	if (set.empty()) throw std::invalid_argument("verify_small_region: empty sieve set");
	SmallRegionSummary sum;
	ScanOptions opt;
	opt.small_p = true;
	const ScanStats st = scan(
	    set, {1, 1}, 151,
	    [&](const ScanEvent& e) {
		    switch (e.verdict.kind) {
		    case PairVerdict::Kind::NoIntegerRoot: ++sum.no_integer_root; break;
		    case PairVerdict::Kind::RootFailsInequalities: ++sum.root_fails; break;
		    case PairVerdict::Kind::CuboidCandidate:
			    ++sum.candidates;
			    throw std::runtime_error("cuboid candidate found at p=" + std::to_string(e.p) +
			                             ", q=" + std::to_string(e.q) + ", t=" + e.verdict.t.get_str());
		    default: break;
		    }
	    },
	    opt, device);
	sum.pairs = st.pairs_tested;
	sum.survivors = st.survivors;
	sum.sieved_out = st.pairs_tested - st.survivors;
	return sum;
}

// ---- the search controller (engine.hpp:429-595) on the GPU ----------------------
//
// Same interface, status codes and files as cuboid::SearchController: load /
// release / start / stop / status / last_stats / last_error, the report line
// (report_append) and the FNV-digested checkpoint (checkpoint_write) written
// with the reference's own functions when a scan ends or is stopped. The
// worker runs gpu::scan over Config::devices. A checkpoint's (p, q) resumes
// with start(p, q); merge of the halves equals the uninterrupted scan.
class SearchController {
public:
	struct Config {
		std::string report_path = "Cuboid_search_report.txt";
		std::string checkpoint_path = "Cuboid_search_checkpoint.txt";
		uint64_t p_limit = p_limit_32bit();
		uint64_t p_end = 0;  // 0: run to p_limit
		bool small_p = false;
		uint64_t batch_pairs = 1u << 16;
		ScanSink sink;                 // survivor events, delivered on the worker thread
		std::vector<int> devices{0};   // GPUs this process drives
	};

	SearchController() = default;
	explicit SearchController(Config cfg) : cfg_(std::move(cfg)) {}
	~SearchController()
	{
		stop_.store(true);
		join();
	}
	SearchController(const SearchController&) = delete;
	SearchController& operator=(const SearchController&) = delete;

	// Index file size on first load, 0 if already loaded (engine.hpp:465-474).
	long load(const std::string& tables_path, const std::string& index_path)
	{
		std::lock_guard<std::mutex> lk(mu_);
		if (set_) return 0;
		const auto index_bytes = read_bytes(index_path);
		const auto table_bytes = read_bytes(tables_path);
		set_ = load_sieve(table_bytes, index_bytes);
		return static_cast<long>(index_bytes.size());
	}
	// Adopts an already built set (e.g. gpu::build_set), as load() would.
	void adopt(SieveSet set)
	{
		std::lock_guard<std::mutex> lk(mu_);
		if (!set_) set_ = std::move(set);
	}
	int release()  // 0 released, 1 running, 6 not loaded
	{
		std::lock_guard<std::mutex> lk(mu_);
		if (running_.load()) return 1;
		join();
		if (!set_) return 6;
		set_.reset();
		return 0;
	}
	int start(uint64_t p, uint64_t q)  // 0 started, 1 running, 2..6 validate_start
	{
		std::lock_guard<std::mutex> lk(mu_);
		if (running_.load()) return 1;
		join();
		const ScanOptions opt = options();
		if (int code = validate_start(set_.has_value(), p, q, opt)) return code;
		stop_.store(false);
		cur_p_.store(p);
		cur_q_.store(q);
		cur_rmax_.store(1);
		running_.store(true);
		worker_ = std::thread([this, p, q, opt] { run({p, q}, opt); });
		return 0;
	}
	int stop()  // 0 stopped (report + checkpoint written), 1 not running
	{
		std::lock_guard<std::mutex> lk(mu_);
		if (!running_.load()) return 1;
		stop_.store(true);
		join();
		return 0;
	}
	ControllerStatus status() const
	{
		ControllerStatus s;
		s.running = running_.load();
		s.current_p_exact = cur_p_.load();
		s.current_p = s.current_p_exact - s.current_p_exact % 100;
		s.current_r_max = cur_rmax_.load();
		return s;
	}
	bool loaded() const
	{
		std::lock_guard<std::mutex> lk(mu_);
		return set_.has_value();
	}
	ScanStats last_stats() const
	{
		std::lock_guard<std::mutex> lk(stats_mu_);
		return stats_;
	}
	std::string last_error() const
	{
		std::lock_guard<std::mutex> lk(stats_mu_);
		return error_;
	}

private:
	ScanOptions options()
	{
		ScanOptions o;
		o.small_p = cfg_.small_p;
		o.p_limit = cfg_.p_limit;
		o.batch_pairs = cfg_.batch_pairs;
		o.hooks = {&stop_, &cur_p_, &cur_q_, &cur_rmax_};
		return o;
	}
	void run(SearchPair start, const ScanOptions& opt)
	{
		const uint64_t p_end = cfg_.p_end ? cfg_.p_end : cfg_.p_limit;
		try {
			ScanStats st = gpu::scan(*set_, start, p_end, cfg_.sink, opt, cfg_.devices);
			SearchCheckpoint cp;
			cp.p = st.resume_p;
			cp.q = st.resume_q;
			cp.r_max = cur_rmax_.load();
			cp.timestamp = iso8601_local_now();
			cp.pairs_tested = st.pairs_tested;
			cp.survivors = st.survivors;
			report_append(cfg_.report_path, cp);
			checkpoint_write(cp, cfg_.checkpoint_path);
			std::lock_guard<std::mutex> lk(stats_mu_);
			stats_ = std::move(st);
			error_.clear();
		} catch (const std::exception& e) {
			std::lock_guard<std::mutex> lk(stats_mu_);
			error_ = e.what();
		}
		running_.store(false);
	}
	void join()
	{
		if (worker_.joinable()) worker_.join();
	}

	Config cfg_;
	mutable std::mutex mu_;
	std::optional<SieveSet> set_;
	std::thread worker_;
	std::atomic<bool> running_{false}, stop_{false};
	std::atomic<uint64_t> cur_p_{0}, cur_q_{0};
	std::atomic<uint32_t> cur_rmax_{1};
	mutable std::mutex stats_mu_;
	ScanStats stats_;
	std::string error_;
};

}  // namespace cuboid::gpu
