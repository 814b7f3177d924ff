// TEST INFRASTRUCTURE ONLY — a minimal stand-in for
// <boost/multiprecision/gmp.hpp> (Boost is not installed in this image, but
// the GMP runtime libgmp.so.10 is).  It provides exactly the subset the
// reference's exact oracle (proj/src/oracle.cpp) and its tests
// (proj/tests/test_narrowphase.cpp, test_oracle.cpp, acceptance.cpp) use —
// mpz_int / mpq_rational value types with exact arithmetic, comparisons,
// numerator/denominator, convert_to, stream output — so those files compile
// UNMODIFIED and the ground truth comes from the reference's own oracle.
//
// GMP's public C ABI (mpz/mpq structs and the __gmpz_*/__gmpq_* entry points)
// is declared here directly because gmp.h is not installed; the layout is
// GMP's documented one for LP64 (int alloc, int size, limb pointer).
#pragma once

#include <cmath>
#include <cstdlib>
#include <ostream>
#include <string>
#include <type_traits>

extern "C" {
struct ccdk_gmp_mpz {
    int alloc;
    int size;
    unsigned long* d;
};
struct ccdk_gmp_mpq {
    ccdk_gmp_mpz num, den;
};
void __gmpz_init(ccdk_gmp_mpz*);
void __gmpz_clear(ccdk_gmp_mpz*);
void __gmpz_set(ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_set_si(ccdk_gmp_mpz*, long);
void __gmpz_set_ui(ccdk_gmp_mpz*, unsigned long);
void __gmpz_set_d(ccdk_gmp_mpz*, double);
void __gmpz_add(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_sub(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_mul(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_neg(ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_abs(ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_tdiv_q(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_tdiv_r(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
void __gmpz_mul_2exp(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, unsigned long);
void __gmpz_tdiv_q_2exp(ccdk_gmp_mpz*, const ccdk_gmp_mpz*, unsigned long);
int __gmpz_cmp(const ccdk_gmp_mpz*, const ccdk_gmp_mpz*);
long __gmpz_get_si(const ccdk_gmp_mpz*);
double __gmpz_get_d(const ccdk_gmp_mpz*);
char* __gmpz_get_str(char*, int, const ccdk_gmp_mpz*);
void __gmpq_init(ccdk_gmp_mpq*);
void __gmpq_clear(ccdk_gmp_mpq*);
void __gmpq_set(ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_set_z(ccdk_gmp_mpq*, const ccdk_gmp_mpz*);
void __gmpq_set_si(ccdk_gmp_mpq*, long, unsigned long);
void __gmpq_set_d(ccdk_gmp_mpq*, double);
void __gmpq_add(ccdk_gmp_mpq*, const ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_sub(ccdk_gmp_mpq*, const ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_mul(ccdk_gmp_mpq*, const ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_div(ccdk_gmp_mpq*, const ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_neg(ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
void __gmpq_abs(ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
int __gmpq_cmp(const ccdk_gmp_mpq*, const ccdk_gmp_mpq*);
double __gmpq_get_d(const ccdk_gmp_mpq*);
char* __gmpq_get_str(char*, int, const ccdk_gmp_mpq*);
}

namespace boost {
namespace multiprecision {

class mpz_int {
public:
    mpz_int() { __gmpz_init(&z_); }
    mpz_int(const mpz_int& o)
    {
        __gmpz_init(&z_);
        __gmpz_set(&z_, &o.z_);
    }
    mpz_int(mpz_int&& o) noexcept
    {
        __gmpz_init(&z_);
        swap(o);
    }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpz_int(T v)
    {
        __gmpz_init(&z_);
        if constexpr (std::is_signed_v<T>)
            __gmpz_set_si(&z_, static_cast<long>(v));
        else
            __gmpz_set_ui(&z_, static_cast<unsigned long>(v));
    }
    explicit mpz_int(double v)
    {
        __gmpz_init(&z_);
        __gmpz_set_d(&z_, v);
    }
    ~mpz_int() { __gmpz_clear(&z_); }
    mpz_int& operator=(const mpz_int& o)
    {
        if (this != &o)
            __gmpz_set(&z_, &o.z_);
        return *this;
    }
    mpz_int& operator=(mpz_int&& o) noexcept
    {
        swap(o);
        return *this;
    }
    void swap(mpz_int& o) noexcept { std::swap(z_, o.z_); }

    ccdk_gmp_mpz* backend() { return &z_; }
    const ccdk_gmp_mpz* backend() const { return &z_; }

    mpz_int& operator+=(const mpz_int& b)
    {
        __gmpz_add(&z_, &z_, &b.z_);
        return *this;
    }
    mpz_int& operator-=(const mpz_int& b)
    {
        __gmpz_sub(&z_, &z_, &b.z_);
        return *this;
    }
    mpz_int& operator*=(const mpz_int& b)
    {
        __gmpz_mul(&z_, &z_, &b.z_);
        return *this;
    }
    mpz_int& operator/=(const mpz_int& b) // truncating, like C++ integers
    {
        __gmpz_tdiv_q(&z_, &z_, &b.z_);
        return *this;
    }
    mpz_int& operator%=(const mpz_int& b)
    {
        __gmpz_tdiv_r(&z_, &z_, &b.z_);
        return *this;
    }
    mpz_int& operator<<=(unsigned long s)
    {
        __gmpz_mul_2exp(&z_, &z_, s);
        return *this;
    }
    mpz_int& operator++()
    {
        const mpz_int one(1);
        __gmpz_add(&z_, &z_, &one.z_);
        return *this;
    }
    mpz_int operator-() const
    {
        mpz_int r;
        __gmpz_neg(&r.z_, &z_);
        return r;
    }
    template <class T>
    T convert_to() const
    {
        if constexpr (std::is_floating_point_v<T>)
            return static_cast<T>(__gmpz_get_d(&z_));
        else
            return static_cast<T>(__gmpz_get_si(&z_));
    }
    std::string str() const
    {
        char* s = __gmpz_get_str(nullptr, 10, &z_);
        std::string r(s);
        std::free(s);
        return r;
    }
    friend int cmp(const mpz_int& a, const mpz_int& b) { return __gmpz_cmp(&a.z_, &b.z_); }

private:
    ccdk_gmp_mpz z_;
};

inline mpz_int operator+(mpz_int a, const mpz_int& b) { return a += b; }
inline mpz_int operator-(mpz_int a, const mpz_int& b) { return a -= b; }
inline mpz_int operator*(mpz_int a, const mpz_int& b) { return a *= b; }
inline mpz_int operator/(mpz_int a, const mpz_int& b) { return a /= b; }
inline mpz_int operator%(mpz_int a, const mpz_int& b) { return a %= b; }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline mpz_int operator<<(mpz_int a, T s)
{
    return a <<= static_cast<unsigned long>(s);
}
inline bool operator==(const mpz_int& a, const mpz_int& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpz_int& a, const mpz_int& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpz_int& a, const mpz_int& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpz_int& a, const mpz_int& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpz_int& a, const mpz_int& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpz_int& a, const mpz_int& b) { return cmp(a, b) >= 0; }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator==(const mpz_int& a, T b) { return a == mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator!=(const mpz_int& a, T b) { return a != mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator<(const mpz_int& a, T b) { return a < mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator<=(const mpz_int& a, T b) { return a <= mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator>(const mpz_int& a, T b) { return a > mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline bool operator>=(const mpz_int& a, T b) { return a >= mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline mpz_int operator*(mpz_int a, T b) { return a *= mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline mpz_int operator+(mpz_int a, T b) { return a += mpz_int(b); }
template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
inline mpz_int operator-(mpz_int a, T b) { return a -= mpz_int(b); }
inline mpz_int abs(const mpz_int& a)
{
    mpz_int r(a);
    __gmpz_abs(r.backend(), a.backend());
    return r;
}
inline std::ostream& operator<<(std::ostream& os, const mpz_int& a) { return os << a.str(); }

class mpq_rational {
public:
    mpq_rational() { __gmpq_init(&q_); }
    mpq_rational(const mpq_rational& o)
    {
        __gmpq_init(&q_);
        __gmpq_set(&q_, &o.q_);
    }
    mpq_rational(mpq_rational&& o) noexcept
    {
        __gmpq_init(&q_);
        swap(o);
    }
    template <class T, std::enable_if_t<std::is_integral_v<T>, int> = 0>
    mpq_rational(T v)
    {
        __gmpq_init(&q_);
        const mpz_int z(v);
        __gmpq_set_z(&q_, z.backend());
    }
    template <class T, std::enable_if_t<std::is_floating_point_v<T>, int> = 0>
    mpq_rational(T v) // exact: every finite double is a dyadic rational
    {
        __gmpq_init(&q_);
        __gmpq_set_d(&q_, static_cast<double>(v));
    }
    explicit mpq_rational(const mpz_int& z)
    {
        __gmpq_init(&q_);
        __gmpq_set_z(&q_, z.backend());
    }
    ~mpq_rational() { __gmpq_clear(&q_); }
    mpq_rational& operator=(const mpq_rational& o)
    {
        if (this != &o)
            __gmpq_set(&q_, &o.q_);
        return *this;
    }
    mpq_rational& operator=(mpq_rational&& o) noexcept
    {
        swap(o);
        return *this;
    }
    void swap(mpq_rational& o) noexcept { std::swap(q_, o.q_); }

    ccdk_gmp_mpq* backend() { return &q_; }
    const ccdk_gmp_mpq* backend() const { return &q_; }

    mpq_rational& operator+=(const mpq_rational& b)
    {
        __gmpq_add(&q_, &q_, &b.q_);
        return *this;
    }
    mpq_rational& operator-=(const mpq_rational& b)
    {
        __gmpq_sub(&q_, &q_, &b.q_);
        return *this;
    }
    mpq_rational& operator*=(const mpq_rational& b)
    {
        __gmpq_mul(&q_, &q_, &b.q_);
        return *this;
    }
    mpq_rational& operator/=(const mpq_rational& b)
    {
        __gmpq_div(&q_, &q_, &b.q_);
        return *this;
    }
    mpq_rational operator-() const
    {
        mpq_rational r;
        __gmpq_neg(&r.q_, &q_);
        return r;
    }
    template <class T>
    T convert_to() const
    {
        return static_cast<T>(__gmpq_get_d(&q_));
    }
    std::string str() const
    {
        char* s = __gmpq_get_str(nullptr, 10, &q_);
        std::string r(s);
        std::free(s);
        return r;
    }
    friend int cmp(const mpq_rational& a, const mpq_rational& b) { return __gmpq_cmp(&a.q_, &b.q_); }
    friend mpz_int numerator(const mpq_rational& a)
    {
        mpz_int r;
        __gmpz_set(r.backend(), &a.q_.num);
        return r;
    }
    friend mpz_int denominator(const mpq_rational& a)
    {
        mpz_int r;
        __gmpz_set(r.backend(), &a.q_.den);
        return r;
    }

private:
    ccdk_gmp_mpq q_;
};

// Mixed arithmetic with built-in numbers promotes them exactly.
template <class T>
using if_num = std::enable_if_t<std::is_arithmetic_v<T>, int>;

inline mpq_rational operator+(mpq_rational a, const mpq_rational& b) { return a += b; }
inline mpq_rational operator-(mpq_rational a, const mpq_rational& b) { return a -= b; }
inline mpq_rational operator*(mpq_rational a, const mpq_rational& b) { return a *= b; }
inline mpq_rational operator/(mpq_rational a, const mpq_rational& b) { return a /= b; }
template <class T, if_num<T> = 0> inline mpq_rational operator+(mpq_rational a, T b) { return a += mpq_rational(b); }
template <class T, if_num<T> = 0> inline mpq_rational operator-(mpq_rational a, T b) { return a -= mpq_rational(b); }
template <class T, if_num<T> = 0> inline mpq_rational operator*(mpq_rational a, T b) { return a *= mpq_rational(b); }
template <class T, if_num<T> = 0> inline mpq_rational operator/(mpq_rational a, T b) { return a /= mpq_rational(b); }
template <class T, if_num<T> = 0> inline mpq_rational operator+(T a, const mpq_rational& b) { return mpq_rational(a) + b; }
template <class T, if_num<T> = 0> inline mpq_rational operator-(T a, const mpq_rational& b) { return mpq_rational(a) - b; }
template <class T, if_num<T> = 0> inline mpq_rational operator*(T a, const mpq_rational& b) { return mpq_rational(a) * b; }
template <class T, if_num<T> = 0> inline mpq_rational operator/(T a, const mpq_rational& b) { return mpq_rational(a) / b; }

inline bool operator==(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) == 0; }
inline bool operator!=(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) != 0; }
inline bool operator<(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) < 0; }
inline bool operator<=(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) <= 0; }
inline bool operator>(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) > 0; }
inline bool operator>=(const mpq_rational& a, const mpq_rational& b) { return cmp(a, b) >= 0; }
template <class T, if_num<T> = 0> inline bool operator==(const mpq_rational& a, T b) { return a == mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator!=(const mpq_rational& a, T b) { return a != mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator<(const mpq_rational& a, T b) { return a < mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator<=(const mpq_rational& a, T b) { return a <= mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator>(const mpq_rational& a, T b) { return a > mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator>=(const mpq_rational& a, T b) { return a >= mpq_rational(b); }
template <class T, if_num<T> = 0> inline bool operator==(T a, const mpq_rational& b) { return mpq_rational(a) == b; }
template <class T, if_num<T> = 0> inline bool operator!=(T a, const mpq_rational& b) { return mpq_rational(a) != b; }
template <class T, if_num<T> = 0> inline bool operator<(T a, const mpq_rational& b) { return mpq_rational(a) < b; }
template <class T, if_num<T> = 0> inline bool operator<=(T a, const mpq_rational& b) { return mpq_rational(a) <= b; }
template <class T, if_num<T> = 0> inline bool operator>(T a, const mpq_rational& b) { return mpq_rational(a) > b; }
template <class T, if_num<T> = 0> inline bool operator>=(T a, const mpq_rational& b) { return mpq_rational(a) >= b; }

inline mpq_rational abs(const mpq_rational& a)
{
    mpq_rational r;
    __gmpq_abs(r.backend(), a.backend());
    return r;
}
inline std::ostream& operator<<(std::ostream& os, const mpq_rational& a) { return os << a.str(); }

} // namespace multiprecision
} // namespace boost
