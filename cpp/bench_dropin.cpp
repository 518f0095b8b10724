// The BASELINE C5 sieve through the reference's own C++ API with the B200
// drop-in (include/cuboid/gpu.hpp): cuboid::gpu::scan_triangle on a
// reference SieveSet, results converted into the reference's ScanStats
// (kill_histogram map, block_r_max map) -- the call a C++ user makes.
// Two legs per step: tables resident (the residency check only), and tables
// re-uploaded from the host set every call (cgpu_tables_load: H2D + layout).
// Prints one JSON line; bench.py runs it (when built) and checks the
// histogram against the reference golden.
//     cpp/_build/bench_dropin [steps] [warmup]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "cuboid/gpu.hpp"

using namespace cuboid;

static std::vector<uint32_t> odd_primes(size_t k)
{
	std::vector<uint32_t> out;
	for (uint32_t n = 3; out.size() < k; n += 2)
		if (is_prime_u32(n)) out.push_back(n);
	return out;
}

int main(int argc, char** argv)
{
	const int steps = argc > 1 ? std::atoi(argv[1]) : 10;
	const int warmup = argc > 2 ? std::atoi(argv[2]) : 3;
	const SieveSet set = gpu::build_set(odd_primes(256));
	auto timed = [&](bool upload, ScanStats& last) {
		double total = 0;
		for (int i = 0; i < warmup + steps; ++i) {
			if (upload) gpu::context(0).invalidate();  // the next call uploads the host set
			const auto t0 = std::chrono::steady_clock::now();
			last = gpu::scan_triangle(set, 100001, 300000);
			const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
			if (i >= warmup) total += s;
		}
		return total / steps;
	};
	ScanStats a, b;
	const double resident = timed(false, a);
	const double upload = timed(true, b);
	std::string hist = "{";
	for (const auto& [r, c] : a.kill_histogram)
		hist += (hist.size() > 1 ? ", \"" : "\"") + std::to_string(r) + "\": " + std::to_string(c);
	hist += "}";
	std::printf("{\"pairs\": %llu, \"survivors\": %llu, \"blocks\": %zu, \"same_both_legs\": %s, "
	            "\"resident_s\": %.9f, \"upload_s\": %.9f, \"steps\": %d, \"kill_histogram\": %s}\n",
	            static_cast<unsigned long long>(a.pairs_tested), static_cast<unsigned long long>(a.survivors),
	            a.block_r_max.size(),
	            (a.pairs_tested == b.pairs_tested && a.kill_histogram == b.kill_histogram &&
	             a.block_r_max == b.block_r_max) ? "true" : "false",
	            resident, upload, steps, hist.c_str());
	return 0;
}
