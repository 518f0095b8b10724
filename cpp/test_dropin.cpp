// Drop-in parity test: cuboid::gpu::* (include/cuboid/gpu.hpp, B200) against
// the reference's own cuboid::* (the unmodified proj/include headers, CPU) on
// the reference's own pins (proj/tests/test_sievetable.cpp, test_engine.cpp,
// acceptance.cpp). Needs a GPU; driven by tests/test_cpp_dropin.py.

#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <numeric>
#include <string>
#include <vector>

#include "cuboid/gpu.hpp"

using namespace cuboid;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                  \
	do {                                                                             \
		if (cond) {                                                                  \
			++g_pass;                                                                \
		} else {                                                                     \
			++g_fail;                                                                \
			std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
		}                                                                            \
	} while (0)

template <class F>
static int thrown_code(F&& f)
{
	try {
		f();
	} catch (const ScanRejected& e) {
		return e.code;
	}
	return 0;
}

static bool same(const ScanStats& a, const ScanStats& b)
{
	return a.pairs_tested == b.pairs_tested && a.survivors == b.survivors &&
	       a.kill_histogram == b.kill_histogram && a.block_r_max == b.block_r_max &&
	       a.resume_p == b.resume_p && a.resume_q == b.resume_q && a.stopped == b.stopped;
}

static std::vector<uint32_t> odd_primes(size_t k)
{
	std::vector<uint32_t> out;
	for (uint32_t n = 3; out.size() < k; n += 2)
		if (is_prime_u32(n)) out.push_back(n);
	return out;
}

// The TRIANGLE loop with the reference's own SieveSet::is_unsolvable, in the
// pattern of verify_small_region (engine.hpp:613-625), q < p.
static ScanStats ref_triangle(const SieveSet& set, uint64_t lo, uint64_t hi, std::vector<std::pair<uint64_t, uint64_t>>* surv)
{
	ScanStats st;
	std::vector<uint64_t> hist(set.prime_count(), 0);
	for (uint64_t p = lo; p <= hi; ++p) {
		uint32_t rmax = 1;
		for (uint64_t q = 1; q < p; ++q) {
			if (std::gcd(p, q) != 1) continue;
			++st.pairs_tested;
			bool killed = false;
			for (size_t k = 0; k < set.prime_count() && !killed; ++k)
				if (set.is_unsolvable(k, p, q)) {
					killed = true;
					++hist[k];
					if (set.prime_at(k) > rmax) rmax = set.prime_at(k);
				}
			if (!killed) {
				++st.survivors;
				if (surv) surv->push_back({p, q});
			}
		}
		auto& b = st.block_r_max[p / 100];
		if (rmax > b) b = rmax;
	}
	for (size_t k = 0; k < hist.size(); ++k)
		if (hist[k]) st.kill_histogram[set.prime_at(k)] = hist[k];
	st.resume_p = hi + 1;
	st.resume_q = 1;
	return st;
}

int main()
{
	// ---- tables (test_sievetable.cpp:12-64, 131-141) ----
	CHECK(gpu::build_table(11).bytes == build_table(11).bytes);
	for (uint32_t r : primes_in_range(2, 97)) CHECK(gpu::build_table(r).bytes == build_table_oracle(r).bytes);
	const SieveSet ref_default = SieveSet::build_default();
	const SieveSet gpu_default = gpu::build_default();
	CHECK(gpu_default.tables() == ref_default.tables());
	CHECK(gpu_default.tables().size() == 1048164);
	CHECK(serialize_index(gpu_default) == serialize_index(ref_default));
	const std::vector<uint32_t> P64 = odd_primes(64);
	CHECK(gpu::build_set(P64).tables() == SieveSet::build(P64).tables());
	CHECK(gpu::build_set(P64, 0, CGPU_BUILD_EXHAUSTIVE).tables() == SieveSet::build(P64).tables());
	bool threw = false;
	try { gpu::build_table(4); } catch (const std::invalid_argument&) { threw = true; }
	CHECK(threw);
	threw = false;
	try { gpu::build_set({13, 11}); } catch (const std::invalid_argument&) { threw = true; }
	CHECK(threw);

	// ---- scan: reference pins and equality with the reference scan() ----
	const ScanStats r152 = gpu::scan(gpu_default, {152, 3}, 152);   // test_engine.cpp:71-88
	CHECK(r152.pairs_tested == 4247 && r152.survivors == 0);
	CHECK(r152.kill_histogram.rbegin()->first == 47);
	CHECK(r152.resume_p == 153 && r152.resume_q == q_bounds(153).q_low);
	CHECK(same(r152, scan(ref_default, {152, 3}, 152)));
	CHECK(same(gpu::scan(gpu_default, {152, 3}, 1500), scan(ref_default, {152, 3}, 1500)));
	CHECK(same(gpu::scan(gpu_default, {153, 5000}, 153), scan(ref_default, {153, 5000}, 153)));
	CHECK(same(gpu::scan(ref_default, {777, 12345}, 901), scan(ref_default, {777, 12345}, 901)));
	const ScanStats big = gpu::scan(gpu_default, {152, 3}, 5000);      // acceptance.cpp:123-144
	CHECK(big.pairs_tested == 447994938ull && big.survivors == 0);
	CHECK(big.kill_histogram.rbegin()->first == 97);

	// rejections (engine.hpp:152-161, test_engine.cpp:90-122)
	CHECK(thrown_code([&] { gpu::scan(gpu_default, {151, 3}, 200); }) == 2);
	CHECK(thrown_code([&] { gpu::scan(gpu_default, {152, 2}, 200); }) == 4);
	CHECK(thrown_code([&] { gpu::scan(gpu_default, {152, 59 * 152 + 1}, 200); }) == 5);
	CHECK(thrown_code([&] { gpu::scan(gpu_default, {152, 3}, 72796056); }) == 3);
	CHECK(thrown_code([&] { gpu::scan(SieveSet{}, {152, 3}, 200); }) == 6);

	// survivors reach the sink in order with the reference's verdicts
	// (test_engine.cpp:177-197, weak sieve {11})
	const SieveSet weak = SieveSet::build({11});
	ScanOptions small;
	small.small_p = true;
	std::vector<ScanEvent> ge, re;
	const ScanStats gw = gpu::scan(weak, {1, 1}, 40, [&](const ScanEvent& e) { ge.push_back(e); }, small);
	const ScanStats rw = scan(weak, {1, 1}, 40, [&](const ScanEvent& e) { re.push_back(e); }, small);
	CHECK(same(gw, rw));
	CHECK(ge.size() == re.size() && !ge.empty());
	bool ev_same = ge.size() == re.size();
	for (size_t i = 0; ev_same && i < ge.size(); ++i)
		ev_same = ge[i].p == re[i].p && ge[i].q == re[i].q && ge[i].verdict.kind == re[i].verdict.kind &&
		          ge[i].verdict.t == re[i].verdict.t;
	CHECK(ev_same);

	// split/resume: a pre-armed stop halts where the reference's does
	// (test_engine.cpp:149-164); a split scan merged equals the whole
	// (test_engine.cpp:134-175)
	std::atomic<bool> stop{true};
	ScanOptions so;
	so.hooks.stop = &stop;
	for (uint64_t bp : {1ull, 1000ull, 8000ull, 65536ull, 400000ull}) {
		std::atomic<bool> rstop{true};
		ScanOptions ro;
		ro.batch_pairs = so.batch_pairs = bp;
		ro.hooks.stop = &rstop;
		for (SearchPair s : {SearchPair{152, 3}, SearchPair{153, 7000}, SearchPair{401, 23000}}) {
			const ScanStats g1 = gpu::scan(gpu_default, s, 700, {}, so);
			const ScanStats r1 = scan(ref_default, s, 700, {}, ro);
			CHECK(same(g1, r1));
			CHECK(g1.stopped);
			ScanStats g2 = g1;
			g2.merge(gpu::scan(gpu_default, {g1.resume_p, g1.resume_q}, 700));
			const ScanStats whole = gpu::scan(gpu_default, s, 700);
			CHECK(g2.pairs_tested == whole.pairs_tested && g2.kill_histogram == whole.kill_histogram &&
			      g2.block_r_max == whole.block_r_max && g2.resume_p == whole.resume_p);
		}
	}
	so.batch_pairs = 1u << 16;
	stop = false;
	ScanStats head = gpu::scan(gpu_default, {152, 3}, 2222, {}, so);
	const ScanStats tail = gpu::scan(gpu_default, {head.resume_p, head.resume_q}, 4000);
	head.merge(tail);
	ScanStats whole = scan(ref_default, {152, 3}, 4000);
	CHECK(head.pairs_tested == whole.pairs_tested && head.kill_histogram == whole.kill_histogram &&
	      head.block_r_max == whole.block_r_max && head.resume_p == whole.resume_p);

	// a scan polled for stops runs as several device tiles (~2^37 q visited
	// each, ending at poll points): the same statistics as one launch
	{
		std::atomic<bool> never{false};
		ScanOptions po;
		po.hooks.stop = &never;
		const ScanStats tiled = gpu::scan(gpu_default, {152, 3}, 200000, {}, po);
		const ScanStats one = gpu::scan(gpu_default, {152, 3}, 200000);
		CHECK(!tiled.stopped);
		CHECK(tiled.pairs_tested == one.pairs_tested && tiled.kill_histogram == one.kill_histogram &&
		      tiled.block_r_max == one.block_r_max && tiled.resume_p == one.resume_p &&
		      tiled.resume_q == one.resume_q && tiled.survivors == one.survivors);
	}

	// a flag already raised, but fewer q left than batch_pairs: the
	// reference never polls and completes the range
	{
		std::atomic<bool> up{true}, rup{true};
		ScanOptions o, ro;
		o.hooks.stop = &up;
		ro.hooks.stop = &rup;
		o.batch_pairs = ro.batch_pairs = 1u << 30;
		const ScanStats g = gpu::scan(gpu_default, {152, 3}, 400, {}, o);
		const ScanStats r = scan(ref_default, {152, 3}, 400, {}, ro);
		CHECK(!g.stopped);
		CHECK(same(g, r));
	}

	// the deferred residency check: a different set of the same shape (one
	// table byte changed) scanned right after -- detected while the device
	// sieves, uploaded, sieved again
	{
		std::vector<uint8_t> t = gpu_default.tables();
		std::vector<PrimeRecord> idx = gpu_default.index();
		t[idx[3].offset + 5] ^= 0x10;  // a bit of row >= 1 of the 4th table (r = 19), not padding
		const SieveSet edited = SieveSet::from_parts(idx, t);
		const ScanStats g0 = gpu::scan(gpu_default, {152, 3}, 900);
		const ScanStats g1 = gpu::scan(edited, {152, 3}, 900);
		const ScanStats g2 = gpu::scan(gpu_default, {152, 3}, 900);
		CHECK(same(g0, scan(ref_default, {152, 3}, 900)));
		CHECK(same(g1, scan(edited, {152, 3}, 900)));
		CHECK(same(g2, g0));
		CHECK(!same(g1, g0));
		CHECK(same(gpu::scan_triangle(edited, 2, 700), ref_triangle(edited, 2, 700, nullptr)));
	}

	// building another set replaces the context's tables; the next
	// scan of the first set must upload it again (and size its histogram by it)
	{
		const ScanStats a1 = gpu::scan(gpu_default, {152, 3}, 600);
		const SieveSet other = gpu::build_set(odd_primes(200));
		(void)other;
		const ScanStats a2 = gpu::scan(gpu_default, {152, 3}, 600);
		CHECK(same(a1, a2));
		CHECK(same(a2, scan(ref_default, {152, 3}, 600)));
	}

	// a flag raised WHILE the scan runs (device-visible stop word): the scan
	// halts at a poll point -- (q visited from the start to the resume pair) + 1
	// is a multiple of batch_pairs -- and the reference's checkpoint of it
	// resumes to the uninterrupted result
	{
		const uint64_t P_END = 1500000;  // REGION ~6.6e13 pairs: several seconds on one GPU
		std::atomic<bool> flag{false};
		ScanOptions o;
		o.hooks.stop = &flag;
		o.batch_pairs = 1u << 16;
		std::thread raiser([&] {
			std::this_thread::sleep_for(std::chrono::milliseconds(300));
			flag.store(true);
		});
		const ScanStats h = gpu::scan(gpu_default, {152, 3}, P_END, {}, o);
		raiser.join();
		CHECK(h.stopped);
		CHECK(h.resume_p > 152 && h.resume_p < P_END);
		uint64_t visited = 0;  // engine.hpp:225-247 visiting order
		for (uint64_t p = 152; p <= h.resume_p; ++p) {
			const RegionBounds b = q_bounds(p);
			const uint64_t q0 = p == 152 ? 3 : b.q_low;
			visited += p < h.resume_p ? b.q_high - q0 + 1 : h.resume_q - q0;
		}
		CHECK((visited + 1) % o.batch_pairs == 0);
		SearchCheckpoint cp;
		cp.p = h.resume_p;
		cp.q = h.resume_q;
		cp.r_max = 1;
		cp.timestamp = iso8601_local_now();
		cp.pairs_tested = h.pairs_tested;
		cp.survivors = h.survivors;
		checkpoint_write(cp, "/tmp/cuboid_gpu_cp.txt");
		const SearchCheckpoint back = checkpoint_read("/tmp/cuboid_gpu_cp.txt");  // the reference's reader
		CHECK(back.p == h.resume_p && back.q == h.resume_q && back.pairs_tested == h.pairs_tested);
		ScanStats merged = h;
		merged.merge(gpu::scan(gpu_default, {back.p, back.q}, P_END));
		const ScanStats whole = gpu::scan(gpu_default, {152, 3}, P_END);
		CHECK(merged.pairs_tested == whole.pairs_tested && merged.kill_histogram == whole.kill_histogram &&
		      merged.block_r_max == whole.block_r_max && merged.survivors == whole.survivors &&
		      merged.resume_p == whole.resume_p && merged.resume_q == whole.resume_q && !merged.stopped);
		// the stopped half equals an unstoppable span up to the same pair
		std::atomic<bool> pre{true};
		ScanOptions po;
		po.hooks.stop = &pre;
		po.batch_pairs = visited + 1;
		const ScanStats again = gpu::scan(gpu_default, {152, 3}, P_END, {}, po);
		CHECK(same(again, h));
	}

	// the GPU SearchController (engine.hpp:429-595): start / status / stop,
	// report + checkpoint through the reference's writers, resume from the
	// checkpoint, merge = uninterrupted
	{
		const uint64_t P_END = 1500000;
		std::remove("/tmp/cuboid_gpu_report.txt");
		gpu::SearchController::Config cfg;
		cfg.report_path = "/tmp/cuboid_gpu_report.txt";
		cfg.checkpoint_path = "/tmp/cuboid_gpu_ctl_cp.txt";
		cfg.p_end = P_END;
		gpu::SearchController ctl(cfg);
		CHECK(ctl.start(152, 3) == 6);  // not loaded
		ctl.adopt(gpu_default);
		CHECK(ctl.start(151, 3) == 2);
		CHECK(ctl.start(152, 2) == 4);
		CHECK(ctl.start(152, 3) == 0);
		CHECK(ctl.start(152, 3) == 1);  // already running
		std::this_thread::sleep_for(std::chrono::milliseconds(300));
		CHECK(ctl.status().running);
		CHECK(ctl.stop() == 0);
		CHECK(ctl.stop() == 1);
		CHECK(ctl.last_error().empty());
		const ScanStats first = ctl.last_stats();
		CHECK(first.stopped);
		const SearchCheckpoint cp = checkpoint_read(cfg.checkpoint_path);
		CHECK(cp.p == first.resume_p && cp.q == first.resume_q && cp.pairs_tested == first.pairs_tested);
		CHECK(cp.r_max == ctl.status().current_r_max);
		CHECK(ctl.start(cp.p, cp.q) == 0);
		while (ctl.status().running) std::this_thread::sleep_for(std::chrono::milliseconds(20));
		ScanStats merged = first;
		merged.merge(ctl.last_stats());
		const ScanStats whole = gpu::scan(gpu_default, {152, 3}, P_END);
		CHECK(merged.pairs_tested == whole.pairs_tested && merged.kill_histogram == whole.kill_histogram &&
		      merged.block_r_max == whole.block_r_max && merged.resume_p == whole.resume_p);
		CHECK(ctl.release() == 0);
		CHECK(ctl.release() == 6);
	}

	// in-process multi-GPU path (cgpu_multi, NCCL clique) over the devices
	// this box has; with one device it is a world-size-1 clique
	{
		int ndev = 0;
		gpu::check(cgpu_device_count(&ndev), "cgpu_device_count");
		std::vector<int> devs;
		for (int d = 0; d < ndev && d < 8; ++d) devs.push_back(d);
		auto& mc = gpu::multi_context(devs);
		const ScanStats m1 = gpu::detail::scan_on(mc, gpu_default, {152, 3}, 5000, {}, ScanOptions{});
		CHECK(same(m1, big));
		CHECK(same(gpu::detail::scan_on(mc, gpu_default, {777, 12345}, 901, {}, ScanOptions{}),
		           scan(ref_default, {777, 12345}, 901)));
		std::vector<ScanEvent> me;
		const ScanStats mw = gpu::detail::scan_on(mc, weak, {1, 1}, 40, [&](const ScanEvent& e) { me.push_back(e); },
		                                          small);
		CHECK(same(mw, rw));
		CHECK(me.size() == re.size());
		std::atomic<bool> pre{true};
		ScanOptions po;
		po.hooks.stop = &pre;
		po.batch_pairs = 8000;
		std::atomic<bool> rpre{true};
		ScanOptions rpo = po;
		rpo.hooks.stop = &rpre;
		CHECK(same(gpu::detail::scan_on(mc, gpu_default, {401, 23000}, 700, {}, po),
		           scan(ref_default, {401, 23000}, 700, {}, rpo)));
		CHECK(same(gpu::scan_triangle(weak, 2, 300, {}, devs), ref_triangle(weak, 2, 300, nullptr)));
		std::printf("multi-GPU clique of %zu device(s) checked\n", devs.size());
	}

	// verify_pair and verify_small_region (engine.hpp:66-95, 609-640) with the
	// sieve part on the device: the reference's verdicts and counts
	{
		for (SearchPair pr : {SearchPair{152, 3}, SearchPair{153, 7000}, SearchPair{2, 1}, SearchPair{7, 4}}) {
			const PairVerdict g = gpu::verify_pair(ref_default, pr, false);
			const PairVerdict r = verify_pair(&ref_default, pr, false);
			CHECK(g.kind == r.kind && g.prime == r.prime && g.t == r.t);
		}
		CHECK(gpu::verify_pair(ref_default, {152, 3}, false).prime == 11);  // test_engine.cpp:51-59
		int bad = 0;
		try { gpu::verify_pair(ref_default, {5, 5}, false); } catch (const std::invalid_argument&) { ++bad; }
		try { gpu::verify_pair(ref_default, {6, 4}, false); } catch (const std::invalid_argument&) { ++bad; }
		try { gpu::verify_pair(SieveSet{}, {7, 4}, false); } catch (const std::invalid_argument&) { ++bad; }
		CHECK(bad == 3);
		std::vector<SearchPair> many;
		for (uint64_t p = 2; p < 400; ++p)
			for (uint64_t q = 1; q < p; q += 7)
				if (std::gcd(p, q) == 1) many.push_back({p, q});
		const std::vector<int32_t> ranks = gpu::classify(ref_default, many);
		bool ranks_same = true;
		for (size_t i = 0; i < many.size(); ++i) {
			int32_t want = -1;
			for (size_t k = 0; k < ref_default.prime_count() && want < 0; ++k)
				if (ref_default.is_unsolvable(k, many[i].p, many[i].q)) want = static_cast<int32_t>(k);
			ranks_same &= ranks[i] == want;
		}
		CHECK(ranks_same);
		for (const SieveSet* s : {&ref_default, &weak}) {
			const SmallRegionSummary g = gpu::verify_small_region(*s);
			const SmallRegionSummary r = verify_small_region(*s);
			CHECK(g.pairs == r.pairs && g.sieved_out == r.sieved_out && g.survivors == r.survivors &&
			      g.no_integer_root == r.no_integer_root && g.root_fails == r.root_fails &&
			      g.candidates == r.candidates);
		}
		CHECK(gpu::verify_small_region(ref_default).pairs == 413362);  // test_engine.cpp:416-423
	}

	// TRIANGLE (BASELINE config 1: 32 odd primes, 2 <= p <= 2000)
	const std::vector<uint32_t> P32 = odd_primes(32);
	const SieveSet s32 = SieveSet::build(P32);
	const ScanStats gt = gpu::scan_triangle(s32, 2, 2000);
	CHECK(gt.pairs_tested == 1216587 && gt.survivors == 0);
	CHECK(same(gt, ref_triangle(s32, 2, 2000, nullptr)));
	std::vector<std::pair<uint64_t, uint64_t>> rsurv;
	std::vector<std::pair<uint64_t, uint64_t>> gsurv;
	const ScanStats gwt = gpu::scan_triangle(weak, 2, 300, [&](const ScanEvent& e) { gsurv.push_back({e.p, e.q}); });
	CHECK(same(gwt, ref_triangle(weak, 2, 300, &rsurv)));
	CHECK(gsurv == rsurv);

	std::printf("%d passed, %d failed\n", g_pass, g_fail);
	return g_fail ? 1 : 0;
}
