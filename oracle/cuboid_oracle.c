/*
 * cuboid_oracle.c -- plain-C restatement of the reference's hot path
 * (arXiv 1601.00636 modulo-primes sieve), written from the reference's
 * behaviour, for use as a CPU checker.
 *
 * TEST INFRASTRUCTURE ONLY. Loaded by tests/ (and nothing in the product
 * package). It is pinned in tests/test_oracle.py against the reference's own
 * golden vectors (test_sievetable.cpp:12-37, acceptance.cpp:123-144, ...) and
 * against oracle/_ref (the reference headers compiled unmodified).
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CO_MODULUS_LIMIT 9697u /* include/cuboid/primes.hpp:12 */

/* include/cuboid/primes.hpp:14-21 (trial division) */
int co_is_prime(uint32_t n)
{
	if (n < 2) return 0;
	if (n % 2 == 0) return n == 2;
	for (uint32_t d = 3; d * d <= n; d += 2)
		if (n % d == 0) return 0;
	return 1;
}

/* include/cuboid/primes.hpp:33-46 (extended Euclid); 0 on bad input */
uint32_t co_mod_inverse(uint32_t a, uint32_t r)
{
	if (a == 0 || a >= r) return 0;
	int64_t t = 0, nt = 1, n = r, nn = a;
	while (nn != 0) {
		int64_t quot = n / nn, tmp;
		tmp = t - quot * nt; t = nt; nt = tmp;
		tmp = n - quot * nn; n = nn; nn = tmp;
	}
	if (t < 0) t += r;
	return (uint32_t)t;
}

/* include/cuboid/modpoly.hpp:86-114 -- residues of c4..c0 (c[0]=c4 ... c[4]=c0)
 * of Q_pq as a monic quintic in s = t^2 (modpoly.hpp:3-11). Negated terms are
 * formed as r - x so every intermediate stays in [0, 16 r^2). */
void co_mod_coeffs(uint32_t p, uint32_t q, uint32_t r, uint32_t c[5])
{
	const uint32_t p2 = p * p % r, q2 = q * q % r;
	const uint32_t p4 = p2 * p2 % r, q4 = q2 * q2 % r;
	const uint32_t p6 = p4 * p2 % r, q6 = q4 * q2 % r;
	const uint32_t p8 = p4 * p4 % r, q8 = q4 * q4 % r;
	/* (2q^2 + p^2)(3q^2 - 2p^2) */
	c[0] = (2 * q2 + p2) % r * ((3 * q2 + 2 * r - 2 * p2) % r) % r;
	/* q^8 + 10 p^2 q^6 + 4 p^4 q^4 - 14 p^6 q^2 + p^8 */
	c[1] = (q8 + 10 * (p2 * q6 % r) + 4 * (p4 * q4 % r) + 14 * (r - p6 * q2 % r) + p8) % r;
	/* -p^2 q^2 (q^8 - 14 p^2 q^6 + 4 p^4 q^4 + 10 p^6 q^2 + p^8) */
	{
		const uint32_t in = (q8 + 14 * (r - p2 * q6 % r) + 4 * (p4 * q4 % r) + 10 * (p6 * q2 % r) + p8) % r;
		c[2] = (r - p2 * q2 % r * in % r) % r;
	}
	/* -p^6 q^6 (q^2 + 2p^2)(3p^2 - 2q^2) */
	{
		const uint32_t f1 = (q2 + 2 * p2) % r;
		const uint32_t f2 = (3 * p2 + 2 * r - 2 * q2) % r;
		c[3] = (r - p6 * q6 % r * f1 % r * f2 % r) % r;
	}
	/* -p^10 q^10 */
	c[4] = (r - (p8 * p2 % r) * (q8 * q2 % r) % r) % r;
}

/* include/cuboid/modpoly.hpp:116-125 -- Horner in s = t^2 */
uint32_t co_horner_mod(const uint32_t c[5], uint32_t t, uint32_t r)
{
	const uint32_t s = t * t % r;
	uint32_t v = (s + c[0]) % r;
	v = (v * s + c[1]) % r;
	v = (v * s + c[2]) % r;
	v = (v * s + c[3]) % r;
	v = (v * s + c[4]) % r;
	return v;
}

/* include/cuboid/modpoly.hpp:130-137; returns -1 for invalid input (the
 * reference throws std::invalid_argument) */
int64_t co_eval_q_mod(uint32_t p, uint32_t q, uint32_t t, uint32_t r)
{
	uint32_t c[5];
	if (r < 2 || r >= CO_MODULUS_LIMIT || !co_is_prime(r)) return -1;
	if (p >= r || q >= r || t >= r) return -1;
	co_mod_coeffs(p, q, r, c);
	return co_horner_mod(c, t, r);
}

/* include/cuboid/sievetable.hpp:41-44 */
uint64_t co_table_bytes(uint32_t r) { return ((uint64_t)r * r + 7) / 8; }

/* sievetable.hpp:58-64 -- LSB-first packing of bit i = p*r + q */
static void set_bit(uint8_t* out, uint64_t i) { out[i >> 3] |= (uint8_t)(1u << (i & 7)); }

/* sievetable.hpp:83-87 */
static int bad_modulus(uint32_t r) { return r < 2 || r >= CO_MODULUS_LIMIT || !co_is_prime(r); }

/* sievetable.hpp:91-96 -- some t in [0, r/2] with Q = 0 (evenness in t) */
static int row_solvable(const uint32_t c[5], uint32_t r)
{
	for (uint32_t t = 0; t <= r / 2; ++t)
		if (co_horner_mod(c, t, r) == 0) return 1;
	return 0;
}

/* sievetable.hpp:102-115 -- the definition: bit(a,b) = 1 iff no t in Z_r
 * solves Q_ab(t) = 0 mod r, scanning t with early exit at the first root.
 * *evals receives the number of Q evaluations performed. */
int co_build_table_oracle(uint32_t r, uint8_t* out, uint64_t* evals)
{
	uint64_t n = 0;
	if (bad_modulus(r)) return -1;
	memset(out, 0, co_table_bytes(r));
	for (uint32_t a = 0; a < r; ++a)
		for (uint32_t b = 0; b < r; ++b) {
			uint32_t c[5];
			int solvable = 0;
			co_mod_coeffs(a, b, r, c);
			for (uint32_t t = 0; t < r && !solvable; ++t) {
				++n;
				solvable = co_horner_mod(c, t, r) == 0;
			}
			if (!solvable) set_bit(out, (uint64_t)a * r + b);
		}
	if (evals) *evals = n;
	return 0;
}

/* sievetable.hpp:123-141 -- production builder: row 0 all zero, row 1 direct
 * (t <= r/2), row a >= 2 is row1[a^{-1} q mod r] (weighted homogeneity). */
int co_build_table(uint32_t r, uint8_t* out)
{
	uint8_t* row1;
	if (bad_modulus(r)) return -1;
	memset(out, 0, co_table_bytes(r));
	row1 = (uint8_t*)malloc(r);
	if (!row1) return -2;
	for (uint32_t q = 0; q < r; ++q) {
		uint32_t c[5];
		co_mod_coeffs(1, q, r, c);
		row1[q] = row_solvable(c, r) ? 0 : 1;
	}
	for (uint32_t a = 1; a < r; ++a) {
		const uint32_t inv = (a == 1) ? 1 : co_mod_inverse(a, r);
		for (uint32_t q = 0; q < r; ++q)
			if (row1[(uint64_t)inv * q % r]) set_bit(out, (uint64_t)a * r + q);
	}
	free(row1);
	return 0;
}

/* sievetable.hpp:159-176 -- concatenated tables at cumulative byte offsets.
 * Returns the total byte count, -1 for a bad/unordered prime list, -2 when the
 * set would exceed the 32-bit offset space. out may be NULL (size query). */
int64_t co_build_set(const uint32_t* primes, uint32_t n, uint8_t* out, uint32_t* offsets)
{
	uint64_t off = 0;
	uint32_t prev = 0;
	for (uint32_t k = 0; k < n; ++k) {
		const uint32_t r = primes[k];
		if (r <= prev || bad_modulus(r)) return -1;
		prev = r;
		if (off + co_table_bytes(r) > UINT32_MAX) return -2;
		if (offsets) offsets[k] = (uint32_t)off;
		if (out && co_build_table(r, out + off) != 0) return -1;
		off += co_table_bytes(r);
	}
	return (int64_t)off;
}

/* include/cuboid/region.hpp:25-39 -- least q >= 1 with 9 q^3 >= p */
uint64_t co_q_lower_cubic(uint64_t p)
{
	uint64_t lo = 1, hi = 1;
#define NINE_CUBED_GE(x) ((unsigned __int128)9 * ((unsigned __int128)(x) * (x) * (x)) >= p)
	while (!NINE_CUBED_GE(hi)) hi *= 2;
	while (lo < hi) {
		const uint64_t mid = lo + (hi - lo) / 2;
		if (NINE_CUBED_GE(mid)) hi = mid; else lo = mid + 1;
	}
#undef NINE_CUBED_GE
	return lo;
}

/* include/cuboid/region.hpp:49-63 */
void co_q_bounds(uint64_t p, uint64_t* q_low, uint64_t* q_high)
{
	*q_high = 59 * p;
	if (p < 152) {
		const uint64_t c = (p + 58) / 59;
		*q_low = c < 1 ? 1 : c;
	} else {
		*q_low = co_q_lower_cubic(p);
	}
}

static uint64_t gcd_u64(uint64_t a, uint64_t b)
{
	while (b) { uint64_t t = a % b; a = b; b = t; }
	return a;
}

/*
 * The sieve driver. mode 0 = REGION (q in [q_low(p), 59p], the reference
 * scan(), include/cuboid/engine.hpp:225-284); mode 1 = TRIANGLE (q in
 * [1, p-1], the loop of verify_small_region, engine.hpp:613-625).
 * The first row starts at q_start when q_start != 0 (engine.hpp:227).
 * Per pair: skip q == p or gcd(p,q) > 1 (engine.hpp:258); count it
 * (engine.hpp:259); probe primes in rank order, first set bit kills
 * (engine.hpp:261-269). REGION skips primes with p mod r == 0
 * (engine.hpp:240-242); TRIANGLE (the verify_small_region loop over
 * is_unsolvable, engine.hpp:619-623, sievetable.hpp:199-205) probes row 0 like
 * any other row -- the two differ only for tables with bits in row 0.
 * Outputs: hist[rank] of first killers, row_rmax[p - p_lo] = largest killer
 * prime in the row or 1 (engine.hpp:229-236, 271), and survivors as (p,q)
 * pairs in ascending order. Returns 0.
 */
int co_sieve(const uint8_t* tables, const uint32_t* primes, const uint32_t* offsets, uint32_t n,
             uint64_t p_lo, uint64_t q_start, uint64_t p_hi, int mode, uint64_t* pairs_tested,
             uint64_t* survivors, uint64_t* hist, uint32_t* row_rmax, uint64_t* surv_pq,
             uint64_t surv_cap, uint64_t* n_surv)
{
	uint64_t pt = 0, sv = 0, ns = 0;
	uint32_t* rowoff = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
	uint32_t* prm = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
	uint32_t* rk = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
	memset(hist, 0, sizeof(uint64_t) * n);
	for (uint64_t p = p_lo; p <= p_hi; ++p) {
		uint64_t lo, hi;
		uint32_t np = 0, rmax = 1;
		if (mode == 0) {
			co_q_bounds(p, &lo, &hi);
		} else {
			lo = 1;
			hi = p - 1;
		}
		if (p == p_lo && q_start) lo = q_start;
		for (uint32_t k = 0; k < n; ++k) {
			const uint32_t a = (uint32_t)(p % primes[k]);
			if (a == 0 && mode == 0) continue;
			prm[np] = primes[k];
			rk[np] = k;
			rowoff[np] = a * primes[k];
			++np;
		}
		for (uint64_t q = lo; q <= hi && hi >= 1; ++q) {
			uint32_t killer = 0;
			if (q == p || gcd_u64(p, q) != 1) continue;
			++pt;
			for (uint32_t j = 0; j < np; ++j) {
				const uint64_t i = rowoff[j] + q % prm[j];
				if ((tables[offsets[rk[j]] + (i >> 3)] >> (i & 7)) & 1) {
					killer = prm[j];
					++hist[rk[j]];
					break;
				}
			}
			if (killer) {
				if (killer > rmax) rmax = killer;
			} else {
				++sv;
				if (ns < surv_cap) {
					surv_pq[2 * ns] = p;
					surv_pq[2 * ns + 1] = q;
				}
				++ns;
			}
		}
		row_rmax[p - p_lo] = rmax;
	}
	free(rowoff);
	free(prm);
	free(rk);
	*pairs_tested = pt;
	*survivors = sv;
	*n_surv = ns;
	return 0;
}
