// oracle/_ref: the UNMODIFIED reference headers
// (/root/reference/proj/include/cuboid/*.hpp) compiled behind a flat C ABI so
// the Python test-suite and bench.py's CPU arm can call the reference itself.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load the resulting
// oracle/_ref/libcuboid_ref.so. The product path (paper_1601_00636_b200/)
// never links or loads it.
//
// Every entry point forwards to the reference function named in its comment;
// the only code here is marshalling plus the multi-threaded row sharding the
// CPU baseline needs (merged with the reference's own ScanStats::merge,
// engine.hpp:121-134).

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cuboid/engine.hpp"

using namespace cuboid;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e)
{
	g_err = e.what();
	return -1;
}

// Survivor capture shared by the scan entry points.
struct SurvivorOut {
	uint64_t* pq = nullptr; // 2*cap
	int32_t* kind = nullptr;
	uint64_t cap = 0;
	uint64_t n = 0;
	void push(uint64_t p, uint64_t q, int k)
	{
		if (n < cap) {
			pq[2 * n] = p;
			pq[2 * n + 1] = q;
			if (kind) kind[n] = k;
		}
		++n;
	}
};

struct StatsOut {
	uint64_t* pairs_tested;
	uint64_t* survivors;
	uint64_t* hist_by_rank; // [prime_count]
	uint64_t* blocks;       // block ids, ascending
	uint32_t* block_rmax;
	uint64_t block_cap;
	uint64_t* n_blocks;
};

void export_stats(const SieveSet& set, const ScanStats& st, const StatsOut& o)
{
	*o.pairs_tested = st.pairs_tested;
	*o.survivors = st.survivors;
	for (size_t k = 0; k < set.prime_count(); ++k) o.hist_by_rank[k] = 0;
	for (const auto& [r, c] : st.kill_histogram) o.hist_by_rank[*set.rank_of(r)] = c;
	uint64_t i = 0;
	for (const auto& [b, r] : st.block_r_max) {
		if (i < o.block_cap) {
			o.blocks[i] = b;
			o.block_rmax[i] = r;
		}
		++i;
	}
	*o.n_blocks = i;
}

} // namespace

extern "C" {

const char* cref_last_error() { return g_err.c_str(); }

// SieveSet::build (sievetable.hpp:159-176)
void* cref_set_build(const uint32_t* primes, uint32_t n)
{
	try {
		return new SieveSet(SieveSet::build(std::vector<uint32_t>(primes, primes + n)));
	} catch (const std::exception& e) {
		fail(e);
		return nullptr;
	}
}

// load_sieve (sievetable.hpp:254-292)
void* cref_set_load(const uint8_t* tables, size_t tlen, const uint8_t* index, size_t ilen)
{
	try {
		return new SieveSet(load_sieve({tables, tlen}, {index, ilen}));
	} catch (const std::exception& e) {
		fail(e);
		return nullptr;
	}
}

void cref_set_free(void* s) { delete static_cast<SieveSet*>(s); }

uint64_t cref_set_tables_size(void* s) { return static_cast<SieveSet*>(s)->tables().size(); }

// serialize_tables / serialize_index (sievetable.hpp:229-252)
uint32_t cref_set_export(void* sp, uint8_t* tables_out, uint32_t* primes_out, uint32_t* offsets_out)
{
	const SieveSet& s = *static_cast<SieveSet*>(sp);
	if (tables_out) std::memcpy(tables_out, s.tables().data(), s.tables().size());
	for (size_t k = 0; k < s.prime_count(); ++k) {
		if (primes_out) primes_out[k] = s.index()[k].prime;
		if (offsets_out) offsets_out[k] = s.index()[k].offset;
	}
	return static_cast<uint32_t>(s.prime_count());
}

int64_t cref_serialize_index(void* sp, uint8_t* out, uint64_t cap)
{
	try {
		const auto idx = serialize_index(*static_cast<SieveSet*>(sp));
		if (out && cap >= idx.size()) std::memcpy(out, idx.data(), idx.size());
		return static_cast<int64_t>(idx.size());
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// SieveSet::is_unsolvable (sievetable.hpp:199-205)
int cref_is_unsolvable(void* sp, uint64_t rank, uint64_t p, uint64_t q)
{
	try {
		return static_cast<SieveSet*>(sp)->is_unsolvable(rank, p, q) ? 1 : 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// build_table (sievetable.hpp:123-141)
int cref_build_table(uint32_t r, uint8_t* out)
{
	try {
		const BitTable t = build_table(r);
		std::memcpy(out, t.bytes.data(), t.bytes.size());
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// build_table_oracle (sievetable.hpp:102-115)
int cref_build_table_oracle(uint32_t r, uint8_t* out)
{
	try {
		const BitTable t = build_table_oracle(r);
		std::memcpy(out, t.bytes.data(), t.bytes.size());
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// Rank-ordered first killer of explicit pairs through SieveSet::is_unsolvable
// (sievetable.hpp:199-205) -- the sieve part of verify_pair (engine.hpp:72-78);
// -1 when no table rejects the pair. Pairs split over `nthreads` threads.
int cref_classify(void* sp, const uint64_t* pq, uint64_t n, int nthreads, int32_t* out)
{
	try {
		const SieveSet& set = *static_cast<SieveSet*>(sp);
		const size_t nprimes = set.prime_count();
		if (nthreads < 1) nthreads = 1;
		std::vector<std::thread> th;
		for (int t = 0; t < nthreads; ++t)
			th.emplace_back([&, t] {
				for (uint64_t i = t; i < n; i += nthreads) {
					int32_t rank = -1;
					for (size_t k = 0; k < nprimes; ++k)
						if (set.is_unsolvable(k, pq[2 * i], pq[2 * i + 1])) {
							rank = static_cast<int32_t>(k);
							break;
						}
					out[i] = rank;
				}
			});
		for (auto& x : th) x.join();
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// The reference's builders over a prime list (production build_table,
// sievetable.hpp:123-141, or the definition build_table_oracle, :102-115),
// primes claimed dynamically by `nthreads` threads; tables written at the
// set's offsets (SieveSet::build layout, :159-176). Returns 0.
int cref_build_tables(const uint32_t* primes, uint32_t n, int oracle, int nthreads,
                      const uint64_t* offsets, uint8_t* out, double* elapsed_s)
{
	try {
		if (nthreads < 1) nthreads = 1;
		std::atomic<uint32_t> next{0};
		std::vector<std::string> errs(nthreads);
		const auto t0 = std::chrono::steady_clock::now();
		std::vector<std::thread> th;
		for (int t = 0; t < nthreads; ++t)
			th.emplace_back([&, t] {
				try {
					for (uint32_t k; (k = next.fetch_add(1)) < n;) {
						const BitTable b = oracle ? build_table_oracle(primes[k]) : build_table(primes[k]);
						std::memcpy(out + offsets[k], b.bytes.data(), b.bytes.size());
					}
				} catch (const std::exception& e) {
					errs[t] = e.what();
				}
			});
		for (auto& x : th) x.join();
		for (auto& e : errs)
			if (!e.empty()) throw std::runtime_error(e);
		*elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// eval_q_mod (modpoly.hpp:130-137); -1 on invalid input
int64_t cref_eval_q_mod(uint32_t p, uint32_t q, uint32_t t, uint32_t r)
{
	try {
		return eval_q_mod({p, q, t, r});
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// q_bounds (region.hpp:49-63)
int cref_q_bounds(uint64_t p, uint64_t* q_low, uint64_t* q_high)
{
	try {
		const RegionBounds b = q_bounds(p);
		*q_low = b.q_low;
		*q_high = b.q_high;
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// verify_pair (engine.hpp:66-95). kind: 0 SievedOut, 1 NoIntegerRoot,
// 2 RootFailsInequalities, 3 CuboidCandidate.
int cref_verify_pair(void* sp, uint64_t p, uint64_t q, int bypass, int32_t* kind, uint32_t* prime,
                     char* t_out, uint64_t t_cap)
{
	try {
		const PairVerdict v = verify_pair(static_cast<SieveSet*>(sp), {p, q}, bypass != 0);
		*kind = static_cast<int32_t>(v.kind);
		*prime = v.prime;
		if (t_out && t_cap) {
			const std::string s = v.t.get_str();
			std::strncpy(t_out, s.c_str(), t_cap - 1);
			t_out[t_cap - 1] = 0;
		}
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// scan() (engine.hpp:195-295), verbatim, REGION mode. Returns 0, a
// ScanRejected code (2..6), or -1. `stop_preset` arms the cooperative stop
// flag before the scan starts (test_engine.cpp:149-164 pattern).
int cref_scan(void* sp, uint64_t p, uint64_t q, uint64_t p_end, int small_p, uint64_t batch_pairs,
              int stop_preset, int with_sink, uint64_t* pairs_tested, uint64_t* survivors,
              uint64_t* hist_by_rank, uint64_t* blocks, uint32_t* block_rmax, uint64_t block_cap,
              uint64_t* n_blocks, uint64_t* surv_pq, int32_t* surv_kind, uint64_t surv_cap,
              uint64_t* n_surv, uint64_t* resume_p, uint64_t* resume_q, int* stopped,
              double* elapsed_s)
{
	try {
		const SieveSet& set = *static_cast<SieveSet*>(sp);
		std::atomic<bool> stop{stop_preset != 0};
		ScanOptions opt;
		opt.small_p = small_p != 0;
		if (batch_pairs) opt.batch_pairs = batch_pairs;
		opt.hooks.stop = &stop;
		SurvivorOut so{surv_pq, surv_kind, surv_cap, 0};
		ScanSink sink;
		if (with_sink)
			sink = [&](const ScanEvent& ev) { so.push(ev.p, ev.q, static_cast<int>(ev.verdict.kind)); };
		const ScanStats st = scan(set, {p, q}, p_end, sink, opt);
		export_stats(set, st, {pairs_tested, survivors, hist_by_rank, blocks, block_rmax, block_cap,
		                       n_blocks});
		*n_surv = so.n;
		*resume_p = st.resume_p;
		*resume_q = st.resume_q;
		*stopped = st.stopped ? 1 : 0;
		*elapsed_s = std::chrono::duration<double>(st.elapsed).count();
		return 0;
	} catch (const ScanRejected& e) {
		g_err = e.what();
		return e.code;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// REGION scan sharded over `nthreads` std::threads by contiguous p-row
// ranges, each shard a verbatim reference scan(), merged in p order with
// ScanStats::merge (engine.hpp:121-134). Used for the all-cores CPU baseline.
int cref_scan_mt(void* sp, uint64_t p_lo, uint64_t p_hi, int small_p, int nthreads,
                 uint64_t* pairs_tested, uint64_t* survivors, uint64_t* hist_by_rank,
                 uint64_t* blocks, uint32_t* block_rmax, uint64_t block_cap, uint64_t* n_blocks,
                 double* elapsed_s)
{
	try {
		const SieveSet& set = *static_cast<SieveSet*>(sp);
		ScanOptions opt;
		opt.small_p = small_p != 0;
		const uint64_t rows = p_hi - p_lo + 1;
		if (nthreads < 1) nthreads = 1;
		// balance by sum of row lengths (~p): split the cumulative p mass
		std::vector<uint64_t> cut{p_lo};
		{
			const double total = double(p_lo + p_hi) * double(rows) / 2.0;
			double acc = 0;
			int k = 1;
			for (uint64_t p = p_lo; p <= p_hi && k < nthreads; ++p) {
				acc += double(p);
				if (acc >= total * k / nthreads) {
					cut.push_back(p + 1);
					++k;
				}
			}
			cut.push_back(p_hi + 1);
		}
		const size_t ns = cut.size() - 1;
		std::vector<ScanStats> parts(ns);
		std::vector<std::string> errs(ns);
		const auto t0 = std::chrono::steady_clock::now();
		std::vector<std::thread> th;
		for (size_t i = 0; i < ns; ++i) {
			th.emplace_back([&, i] {
				try {
					if (cut[i] < cut[i + 1])
						parts[i] = scan(set, {cut[i], q_bounds(cut[i]).q_low}, cut[i + 1] - 1, {}, opt);
				} catch (const std::exception& e) {
					errs[i] = e.what();
				}
			});
		}
		for (auto& t : th) t.join();
		for (auto& e : errs)
			if (!e.empty()) throw std::runtime_error(e);
		ScanStats all;
		for (auto& s : parts) all.merge(s);
		*elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
		export_stats(set, all, {pairs_tested, survivors, hist_by_rank, blocks, block_rmax, block_cap,
		                        n_blocks});
		return 0;
	} catch (const ScanRejected& e) {
		g_err = e.what();
		return e.code;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// TRIANGLE sieve (1 <= q < p, gcd = 1) over rows [p_lo, p_hi]: the loop of
// verify_small_region (engine.hpp:609-640) -- rank-ordered
// SieveSet::is_unsolvable with early exit -- carrying scan()'s statistics
// (first-killer histogram, p/100 block r_max, engine.hpp:229-236, 261-271)
// and handing survivors to verify_pair(bypass) like scan() (engine.hpp:272-277).
// Rows are sharded over `nthreads` threads; shards are merged with
// ScanStats::merge in p order so survivors stay in canonical order.
int cref_triangle(void* sp, uint64_t p_lo, uint64_t p_hi, int nthreads, int with_sink,
                  uint64_t* pairs_tested, uint64_t* survivors, uint64_t* hist_by_rank,
                  uint64_t* blocks, uint32_t* block_rmax, uint64_t block_cap, uint64_t* n_blocks,
                  uint64_t* surv_pq, int32_t* surv_kind, uint64_t surv_cap, uint64_t* n_surv,
                  double* elapsed_s)
{
	try {
		const SieveSet& set = *static_cast<SieveSet*>(sp);
		if (set.empty()) throw ScanRejected(6);
		if (p_lo == 0) p_lo = 1;
		if (nthreads < 1) nthreads = 1;
		const size_t nprimes = set.prime_count();
		struct Part {
			ScanStats st;
			std::vector<std::pair<std::pair<uint64_t, uint64_t>, int>> surv;
		};
		// interleave rows in blocks of 16 for balance; merge afterwards
		const uint64_t chunk = 16;
		const uint64_t nchunks = (p_hi >= p_lo) ? (p_hi - p_lo) / chunk + 1 : 0;
		std::vector<Part> parts(nchunks);
		std::atomic<uint64_t> next{0};
		std::vector<std::string> errs(nthreads);
		const auto t0 = std::chrono::steady_clock::now();
		auto worker = [&](int tid) {
			try {
				std::vector<uint64_t> hist(nprimes);
				for (;;) {
					const uint64_t c = next.fetch_add(1);
					if (c >= nchunks) break;
					Part& part = parts[c];
					std::fill(hist.begin(), hist.end(), 0);
					const uint64_t pa = p_lo + c * chunk;
					const uint64_t pb = std::min(p_hi, pa + chunk - 1);
					for (uint64_t p = pa; p <= pb; ++p) {
						uint32_t& bmax = part.st.block_r_max[p / 100];
						if (bmax == 0) bmax = 1;
						for (uint64_t q = 1; q < p; ++q) {
							if (std::gcd(p, q) != 1) continue;
							++part.st.pairs_tested;
							uint32_t killer = 0;
							for (size_t rank = 0; rank < nprimes; ++rank) {
								if (set.is_unsolvable(rank, p, q)) {
									killer = set.prime_at(rank);
									++hist[rank];
									break;
								}
							}
							if (killer) {
								if (killer > bmax) bmax = killer;
							} else {
								++part.st.survivors;
								if (with_sink)
									part.surv.push_back(
									    {{p, q}, static_cast<int>(verify_pair(&set, {p, q}, true).kind)});
							}
						}
					}
					for (size_t k = 0; k < nprimes; ++k)
						if (hist[k]) part.st.kill_histogram[set.prime_at(k)] += hist[k];
				}
			} catch (const std::exception& e) {
				errs[tid] = e.what();
			}
		};
		std::vector<std::thread> th;
		for (int i = 0; i < nthreads; ++i) th.emplace_back(worker, i);
		for (auto& t : th) t.join();
		for (auto& e : errs)
			if (!e.empty()) throw std::runtime_error(e);
		ScanStats all;
		SurvivorOut so{surv_pq, surv_kind, surv_cap, 0};
		for (auto& part : parts) {
			all.merge(part.st);
			for (auto& s : part.surv) so.push(s.first.first, s.first.second, s.second);
		}
		*elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
		export_stats(set, all, {pairs_tested, survivors, hist_by_rank, blocks, block_rmax, block_cap,
		                        n_blocks});
		*n_surv = so.n;
		return 0;
	} catch (const ScanRejected& e) {
		g_err = e.what();
		return e.code;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

// verify_small_region (engine.hpp:609-640)
int cref_verify_small_region(void* sp, uint64_t* out6)
{
	try {
		const SmallRegionSummary s = verify_small_region(*static_cast<SieveSet*>(sp));
		const uint64_t v[6] = {s.pairs, s.sieved_out, s.survivors, s.no_integer_root, s.root_fails,
		                       s.candidates};
		std::memcpy(out6, v, sizeof v);
		return 0;
	} catch (const std::exception& e) {
		return fail(e);
	}
}

} // extern "C"
