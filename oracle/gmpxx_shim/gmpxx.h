// Minimal C++ big-integer shim used ONLY to compile the reference headers
// (/root/reference/proj/include/cuboid/*.hpp) for the test oracle in
// oracle/_ref. The container ships libgmp.so.10 but neither gmp.h nor
// gmpxx.h, so this file declares the handful of __gmpz_* entry points the
// reference touches and wraps them in a value-semantics mpz_class.
//
// Test infrastructure: nothing in the product path includes this file.
//
// Semantics follow GMP's documented C++ interface where the reference relies
// on them: `/` and `%` truncate toward zero (mpz_tdiv_q / mpz_tdiv_r), and
// comparisons are exact.
#pragma once

#include <cstddef>
#include <cstdlib>
#include <ostream>
#include <string>

extern "C" {
typedef unsigned long mp_limb_t;
typedef long mp_size_t;
typedef unsigned long mp_bitcnt_t;
typedef struct {
	int _mp_alloc;
	int _mp_size;
	mp_limb_t* _mp_d;
} __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct* mpz_ptr;
typedef const __mpz_struct* mpz_srcptr;

void __gmpz_init(mpz_ptr);
void __gmpz_init_set(mpz_ptr, mpz_srcptr);
void __gmpz_init_set_si(mpz_ptr, long);
void __gmpz_init_set_ui(mpz_ptr, unsigned long);
int __gmpz_init_set_str(mpz_ptr, const char*, int);
void __gmpz_clear(mpz_ptr);
void __gmpz_set(mpz_ptr, mpz_srcptr);
void __gmpz_set_si(mpz_ptr, long);
void __gmpz_set_ui(mpz_ptr, unsigned long);
char* __gmpz_get_str(char*, int, mpz_srcptr);
unsigned long __gmpz_get_ui(mpz_srcptr);
long __gmpz_get_si(mpz_srcptr);
void __gmpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_q(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_tdiv_r(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_neg(mpz_ptr, mpz_srcptr);
void __gmpz_abs(mpz_ptr, mpz_srcptr);
int __gmpz_cmp(mpz_srcptr, mpz_srcptr);
void __gmpz_gcd(mpz_ptr, mpz_srcptr, mpz_srcptr);
void __gmpz_divexact(mpz_ptr, mpz_srcptr, mpz_srcptr);
int __gmpz_root(mpz_ptr, mpz_srcptr, unsigned long);
int __gmpz_perfect_square_p(mpz_srcptr);
void __gmpz_sqrt(mpz_ptr, mpz_srcptr);
size_t __gmpz_sizeinbase(mpz_srcptr, int);
void __gmpz_ui_pow_ui(mpz_ptr, unsigned long, unsigned long);
void __gmpz_pow_ui(mpz_ptr, mpz_srcptr, unsigned long);
}

#define mpz_gcd __gmpz_gcd
#define mpz_divexact __gmpz_divexact
#define mpz_root __gmpz_root
#define mpz_perfect_square_p __gmpz_perfect_square_p
#define mpz_sqrt __gmpz_sqrt
#define mpz_sizeinbase __gmpz_sizeinbase
#define mpz_ui_pow_ui __gmpz_ui_pow_ui
#define mpz_pow_ui __gmpz_pow_ui

class mpz_class {
public:
	mpz_class() { __gmpz_init(v_); }
	mpz_class(int x) { __gmpz_init_set_si(v_, x); }
	mpz_class(long x) { __gmpz_init_set_si(v_, x); }
	mpz_class(long long x) { __gmpz_init_set_si(v_, static_cast<long>(x)); }
	mpz_class(unsigned int x) { __gmpz_init_set_ui(v_, x); }
	mpz_class(unsigned long x) { __gmpz_init_set_ui(v_, x); }
	mpz_class(unsigned long long x) { __gmpz_init_set_ui(v_, static_cast<unsigned long>(x)); }
	explicit mpz_class(const char* s, int base = 10)
	{
		if (__gmpz_init_set_str(v_, s, base) != 0) std::abort();
	}
	explicit mpz_class(const std::string& s, int base = 10) : mpz_class(s.c_str(), base) {}
	mpz_class(const mpz_class& o) { __gmpz_init_set(v_, o.v_); }
	mpz_class(mpz_class&& o) noexcept
	{
		__gmpz_init(v_);
		swap(o);
	}
	~mpz_class() { __gmpz_clear(v_); }

	mpz_class& operator=(const mpz_class& o)
	{
		if (this != &o) __gmpz_set(v_, o.v_);
		return *this;
	}
	mpz_class& operator=(mpz_class&& o) noexcept
	{
		swap(o);
		return *this;
	}

	void swap(mpz_class& o) noexcept
	{
		__mpz_struct t = v_[0];
		v_[0] = o.v_[0];
		o.v_[0] = t;
	}

	mpz_ptr get_mpz_t() { return v_; }
	mpz_srcptr get_mpz_t() const { return v_; }
	unsigned long get_ui() const { return __gmpz_get_ui(v_); }
	long get_si() const { return __gmpz_get_si(v_); }
	std::string get_str(int base = 10) const
	{
		char* s = __gmpz_get_str(nullptr, base, v_);
		std::string out(s);
		std::free(s);
		return out;
	}

	mpz_class& operator+=(const mpz_class& o) { __gmpz_add(v_, v_, o.v_); return *this; }
	mpz_class& operator-=(const mpz_class& o) { __gmpz_sub(v_, v_, o.v_); return *this; }
	mpz_class& operator*=(const mpz_class& o) { __gmpz_mul(v_, v_, o.v_); return *this; }
	mpz_class& operator/=(const mpz_class& o) { __gmpz_tdiv_q(v_, v_, o.v_); return *this; }
	mpz_class& operator%=(const mpz_class& o) { __gmpz_tdiv_r(v_, v_, o.v_); return *this; }

	friend mpz_class operator+(mpz_class a, const mpz_class& b) { return a += b; }
	friend mpz_class operator-(mpz_class a, const mpz_class& b) { return a -= b; }
	friend mpz_class operator*(mpz_class a, const mpz_class& b) { return a *= b; }
	friend mpz_class operator/(mpz_class a, const mpz_class& b) { return a /= b; }
	friend mpz_class operator%(mpz_class a, const mpz_class& b) { return a %= b; }
	friend mpz_class operator-(const mpz_class& a)
	{
		mpz_class r;
		__gmpz_neg(r.v_, a.v_);
		return r;
	}

	friend int cmp(const mpz_class& a, const mpz_class& b) { return __gmpz_cmp(a.v_, b.v_); }
	friend bool operator==(const mpz_class& a, const mpz_class& b) { return cmp(a, b) == 0; }
	friend bool operator!=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) != 0; }
	friend bool operator<(const mpz_class& a, const mpz_class& b) { return cmp(a, b) < 0; }
	friend bool operator<=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) <= 0; }
	friend bool operator>(const mpz_class& a, const mpz_class& b) { return cmp(a, b) > 0; }
	friend bool operator>=(const mpz_class& a, const mpz_class& b) { return cmp(a, b) >= 0; }

	friend int sgn(const mpz_class& a) { return a.v_->_mp_size < 0 ? -1 : (a.v_->_mp_size > 0 ? 1 : 0); }
	friend mpz_class abs(const mpz_class& a)
	{
		mpz_class r;
		__gmpz_abs(r.v_, a.v_);
		return r;
	}
	friend std::ostream& operator<<(std::ostream& os, const mpz_class& a) { return os << a.get_str(); }

private:
	mpz_t v_;
};
