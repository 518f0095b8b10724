// Drop-in parity test: cuboid::gpu::* (include/cuboid/gpu.hpp, B200) against
// the reference's own cuboid::* (the unmodified proj/include headers, CPU) on
// the reference's own pins (proj/tests/test_sievetable.cpp, test_engine.cpp,
// acceptance.cpp). Needs a GPU; driven by tests/test_cpp_dropin.py.

#include <atomic>
#include <cstdio>
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

	// a scan polled for stops runs as several device tiles (~2^37 pairs each):
	// the same statistics as one launch
	{
		std::atomic<bool> never{false};
		ScanOptions po;
		po.hooks.stop = &never;
		const ScanStats tiled = gpu::scan(gpu_default, {152, 3}, 200000, {}, po);
		const ScanStats one = gpu::scan(gpu_default, {152, 3}, 200000);
		CHECK(!tiled.stopped);
		CHECK(gpu::detail::tile_end(152, 200000) < 200000);
		CHECK(tiled.pairs_tested == one.pairs_tested && tiled.kill_histogram == one.kill_histogram &&
		      tiled.block_r_max == one.block_r_max && tiled.resume_p == one.resume_p &&
		      tiled.resume_q == one.resume_q && tiled.survivors == one.survivors);
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
