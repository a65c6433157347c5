// bm_common.cuh -- element types, numpy-exact conversions and the element-wise
// operator set of the reference, for sm_100a.  Compiled both ahead of time
// (nvcc, into libb200mat.so) and at run time by NVRTC for fused programs, so it
// depends on no system header.
//
// Semantics follow the reference's kernels (reference/pkg/src/devmat):
//   * every stage is computed in the compute dtype and rounded to it
//     (kernels.py:270-277 _stage_cast) -- natural in CUDA with -fmad=false;
//   * scalar k is cast to the compute dtype first (kernels.py:280-283);
//   * integers wrap; i32 division truncates through f64 and out-of-range
//     results become INT_MIN exactly like numpy's x86 astype (kernels.py:286-292);
//     u64 division is floor division with x/0 == 0 (numpy);
//   * integer transcendental ops run in f64 and are C-cast back
//     (kernels.py:311-316 via numpy's int -> f64 ufunc promotion);
//   * write-time conversion is numpy astype on x86-64 (kernels.py:259-267).
#pragma once

namespace bm {

typedef long long i64;
typedef unsigned long long u64;
typedef int i32;
typedef unsigned int u32;

enum { DT_F32 = 0, DT_F64 = 1, DT_I32 = 2, DT_U64 = 3 };

template <int D> struct dtype_of;
template <> struct dtype_of<DT_F32> { typedef float T; };
template <> struct dtype_of<DT_F64> { typedef double T; };
template <> struct dtype_of<DT_I32> { typedef int T; };
template <> struct dtype_of<DT_U64> { typedef unsigned long long T; };

template <bool C, typename A, typename B> struct cond_t { typedef A type; };
template <typename A, typename B> struct cond_t<false, A, B> { typedef B type; };

template <typename T> struct is_float_t { static const bool value = false; };
template <> struct is_float_t<float> { static const bool value = true; };
template <> struct is_float_t<double> { static const bool value = true; };

// ---------------------------------------------------------------------------
// numpy (x86-64) float -> integer conversions.  cvttsd2si returns the
// "integer indefinite" value (INT_MIN / INT64_MIN) for NaN and out-of-range
// inputs; numpy's float -> uint64 cast goes through the signed conversion,
// subtracting 2^63 first for x >= 2^63 (verified against numpy 2.3 in
// tests/test_oracle.py::test_cast_edge_cases).
__device__ __forceinline__ int np_f2i32(double x) {
    double t = trunc(x);
    return (t >= -2147483648.0 && t <= 2147483647.0) ? (int)t : (int)0x80000000;
}
__device__ __forceinline__ long long np_cvtt_i64(double x) {
    double t = trunc(x);
    return (t >= -9223372036854775808.0 && t < 9223372036854775808.0)
               ? (long long)t
               : (long long)0x8000000000000000ULL;
}
__device__ __forceinline__ u64 np_f2u64(double x) {
    if (x >= 9223372036854775808.0)
        return (u64)np_cvtt_i64(x - 9223372036854775808.0) ^ 0x8000000000000000ULL;
    return (u64)np_cvtt_i64(x);
}

// cvt<To>(x): numpy astype semantics
template <typename To> struct Cvt;
template <> struct Cvt<float> {
    __device__ static __forceinline__ float f(float x) { return x; }
    __device__ static __forceinline__ float f(double x) { return __double2float_rn(x); }
    __device__ static __forceinline__ float f(int x) { return __int2float_rn(x); }
    __device__ static __forceinline__ float f(u64 x) { return __ull2float_rn(x); }
};
template <> struct Cvt<double> {
    __device__ static __forceinline__ double f(float x) { return (double)x; }
    __device__ static __forceinline__ double f(double x) { return x; }
    __device__ static __forceinline__ double f(int x) { return (double)x; }
    __device__ static __forceinline__ double f(u64 x) { return __ull2double_rn(x); }
};
template <> struct Cvt<int> {
    __device__ static __forceinline__ int f(float x) { return np_f2i32((double)x); }
    __device__ static __forceinline__ int f(double x) { return np_f2i32(x); }
    __device__ static __forceinline__ int f(int x) { return x; }
    __device__ static __forceinline__ int f(u64 x) { return (int)(u32)x; }
};
template <> struct Cvt<u64> {
    __device__ static __forceinline__ u64 f(float x) { return np_f2u64((double)x); }
    __device__ static __forceinline__ u64 f(double x) { return np_f2u64(x); }
    __device__ static __forceinline__ u64 f(int x) { return (u64)(i64)x; }
    __device__ static __forceinline__ u64 f(u64 x) { return x; }
};
template <typename To, typename From>
__device__ __forceinline__ To cvt(From x) { return Cvt<To>::f(x); }

// ---------------------------------------------------------------------------
// scalar constants: floats arrive as double and round like np.float32(k);
// integers arrive already converted with int(k) on the host.
template <typename T> struct KScal;
template <> struct KScal<float> { __device__ static __forceinline__ float f(double d, i64) { return __double2float_rn(d); } };
template <> struct KScal<double> { __device__ static __forceinline__ double f(double d, i64) { return d; } };
template <> struct KScal<int> { __device__ static __forceinline__ int f(double, i64 i) { return (int)i; } };
template <> struct KScal<u64> { __device__ static __forceinline__ u64 f(double, i64 i) { return (u64)i; } };

// ---------------------------------------------------------------------------
// element-wise operators (kernels.py:295-351)

// wrapping integer arithmetic without signed-overflow UB
__device__ __forceinline__ int wadd(int a, int b) { return (int)((u32)a + (u32)b); }
__device__ __forceinline__ int wsub(int a, int b) { return (int)((u32)a - (u32)b); }
__device__ __forceinline__ int wmul(int a, int b) { return (int)((u32)a * (u32)b); }

// i32 division truncates through f64 (kernels.py:286-292); numpy's astype maps
// inf/nan/2^31 to INT_MIN.
__device__ __forceinline__ int idiv(int a, int b) { return np_f2i32((double)a / (double)b); }
// u64: np.floor_divide, x // 0 == 0
__device__ __forceinline__ u64 udiv(u64 a, u64 b) { return b ? a / b : 0ULL; }

struct OpPlus {
    __device__ static __forceinline__ float f(float a, float b) { return a + b; }
    __device__ static __forceinline__ double f(double a, double b) { return a + b; }
    __device__ static __forceinline__ int f(int a, int b) { return wadd(a, b); }
    __device__ static __forceinline__ u64 f(u64 a, u64 b) { return a + b; }
};
struct OpMinus {
    __device__ static __forceinline__ float f(float a, float b) { return a - b; }
    __device__ static __forceinline__ double f(double a, double b) { return a - b; }
    __device__ static __forceinline__ int f(int a, int b) { return wsub(a, b); }
    __device__ static __forceinline__ u64 f(u64 a, u64 b) { return a - b; }
};
struct OpTimes {
    __device__ static __forceinline__ float f(float a, float b) { return a * b; }
    __device__ static __forceinline__ double f(double a, double b) { return a * b; }
    __device__ static __forceinline__ int f(int a, int b) { return wmul(a, b); }
    __device__ static __forceinline__ u64 f(u64 a, u64 b) { return a * b; }
};
struct OpDiv {
    __device__ static __forceinline__ float f(float a, float b) { return a / b; }
    __device__ static __forceinline__ double f(double a, double b) { return a / b; }
    __device__ static __forceinline__ int f(int a, int b) { return idiv(a, b); }
    __device__ static __forceinline__ u64 f(u64 a, u64 b) { return udiv(a, b); }
};

// unary ops.  f32 transcendental ops use CUDA's accurate single-precision
// functions (<= 2 ulp); numpy's SIMD versions are themselves 1-4 ulp from the
// correctly rounded value, so parity for these is ULP-bounded.
// pow is evaluated in f64 and rounded, which reproduces glibc powf (numpy's
// float32 power) to the last bit away from rounding ties.
__device__ __forceinline__ float u_exp(float x) { return expf(x); }
__device__ __forceinline__ double u_exp(double x) { return exp(x); }
__device__ __forceinline__ float u_log(float x) { return logf(x); }
__device__ __forceinline__ double u_log(double x) { return log(x); }
__device__ __forceinline__ float u_log10(float x) { return log10f(x); }
__device__ __forceinline__ double u_log10(double x) { return log10(x); }
__device__ __forceinline__ float u_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double u_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float u_cos(float x) { return cosf(x); }
__device__ __forceinline__ double u_cos(double x) { return cos(x); }
__device__ __forceinline__ float u_sin(float x) { return sinf(x); }
__device__ __forceinline__ double u_sin(double x) { return sin(x); }
__device__ __forceinline__ float u_tan(float x) { return tanf(x); }
__device__ __forceinline__ double u_tan(double x) { return tan(x); }
__device__ __forceinline__ float u_acos(float x) { return acosf(x); }
__device__ __forceinline__ double u_acos(double x) { return acos(x); }
__device__ __forceinline__ float u_asin(float x) { return asinf(x); }
__device__ __forceinline__ double u_asin(double x) { return asin(x); }
__device__ __forceinline__ float u_atan(float x) { return atanf(x); }
__device__ __forceinline__ double u_atan(double x) { return atan(x); }
__device__ __forceinline__ float u_square(float x) { return x * x; }
__device__ __forceinline__ double u_square(double x) { return x * x; }
__device__ __forceinline__ float u_abs(float x) { return fabsf(x); }
__device__ __forceinline__ double u_abs(double x) { return fabs(x); }
__device__ __forceinline__ float u_pow(float x, float k) { return __double2float_rn(pow((double)x, (double)k)); }
__device__ __forceinline__ double u_pow(double x, double k) { return pow(x, k); }

// integer element types: transcendental results come back through numpy's cast
#define BM_INT_VIA_F64(NAME, FN)                                                        \
    __device__ __forceinline__ int NAME(int x) { return np_f2i32(FN((double)x)); }      \
    __device__ __forceinline__ u64 NAME(u64 x) { return np_f2u64(FN(__ull2double_rn(x))); }
BM_INT_VIA_F64(u_exp, exp)
BM_INT_VIA_F64(u_log, log)
BM_INT_VIA_F64(u_log10, log10)
BM_INT_VIA_F64(u_sqrt, sqrt)
BM_INT_VIA_F64(u_cos, cos)
BM_INT_VIA_F64(u_sin, sin)
BM_INT_VIA_F64(u_tan, tan)
BM_INT_VIA_F64(u_acos, acos)
BM_INT_VIA_F64(u_asin, asin)
BM_INT_VIA_F64(u_atan, atan)
#undef BM_INT_VIA_F64
__device__ __forceinline__ int u_square(int x) { return wmul(x, x); }
__device__ __forceinline__ u64 u_square(u64 x) { return x * x; }
__device__ __forceinline__ int u_abs(int x) { return x < 0 ? (int)(0u - (u32)x) : x; }
__device__ __forceinline__ u64 u_abs(u64 x) { return x; }
// integer power: exact modulo 2^bits (numpy rejects negative exponents on the host)
__device__ __forceinline__ int u_pow(int x, int k) {
    u32 r = 1u, b = (u32)x;
    u32 e = (u32)k;
    while (e) { if (e & 1u) r *= b; b *= b; e >>= 1; }
    return (int)r;
}
__device__ __forceinline__ u64 u_pow(u64 x, u64 k) {
    u64 r = 1ULL, b = x;
    while (k) { if (k & 1ULL) r *= b; b *= b; k >>= 1; }
    return r;
}

// ---------------------------------------------------------------------------
// reductions helpers

// Python's built-in min/max on two scalars (combine_pairwise, kernels.py:784-793):
// min(a, b) keeps a unless b < a; max(a, b) keeps a unless b > a.  NaN handling
// is therefore order-dependent, exactly like the reference.
template <typename T> __device__ __forceinline__ T py_min(T a, T b) { return (b < a) ? b : a; }
template <typename T> __device__ __forceinline__ T py_max(T a, T b) { return (b > a) ? b : a; }

// numpy's ndarray.min()/max() inside a block: NaN propagates.
template <typename T> __device__ __forceinline__ bool is_nan(T) { return false; }
template <> __device__ __forceinline__ bool is_nan<float>(float x) { return x != x; }
template <> __device__ __forceinline__ bool is_nan<double>(double x) { return x != x; }
template <typename T> __device__ __forceinline__ T np_min(T a, T b) {
    if (is_nan(a)) return a;
    if (is_nan(b)) return b;
    return b < a ? b : a;
}
template <typename T> __device__ __forceinline__ T np_max(T a, T b) {
    if (is_nan(a)) return a;
    if (is_nan(b)) return b;
    return b > a ? b : a;
}

template <typename T> __device__ __forceinline__ T warp_shfl_xor(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// Branch-free running min/max with numpy's NaN propagation (ndarray.min/max):
// any NaN makes the result NaN, otherwise the extreme value.  Order-free, so
// lanes and threads may split the range arbitrarily.
template <typename T> __device__ __forceinline__ T lowest_val();
template <typename T> __device__ __forceinline__ T highest_val();
template <typename T, bool IS_MAX>
struct MinMaxAcc {
    T v;
    bool nan;
    __device__ __forceinline__ MinMaxAcc() : v(IS_MAX ? lowest_val<T>() : highest_val<T>()), nan(false) {}
    __device__ __forceinline__ void add(T x) {
        nan |= (x != x);
        v = IS_MAX ? ((x > v) ? x : v) : ((x < v) ? x : v);
    }
    __device__ __forceinline__ void merge(const MinMaxAcc& o) {
        nan |= o.nan;
        v = IS_MAX ? ((o.v > v) ? o.v : v) : ((o.v < v) ? o.v : v);
    }
    __device__ __forceinline__ void warp_merge() {
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            MinMaxAcc o;
            o.v = warp_shfl_xor(v, m);
            o.nan = __shfl_xor_sync(0xffffffffu, (int)nan, m) != 0;
            merge(o);
        }
    }
    __device__ __forceinline__ T result() const { return nan ? T(__longlong_as_double(0x7ff8000000000000LL)) : v; }
};

template <typename T> __device__ __forceinline__ T lowest_val();
template <> __device__ __forceinline__ float lowest_val<float>() { return -__int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double lowest_val<double>() { return -__longlong_as_double(0x7ff0000000000000LL); }
template <> __device__ __forceinline__ int lowest_val<int>() { return (int)0x80000000; }
template <> __device__ __forceinline__ u64 lowest_val<u64>() { return 0ULL; }
template <typename T> __device__ __forceinline__ T highest_val();
template <> __device__ __forceinline__ float highest_val<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double highest_val<double>() { return __longlong_as_double(0x7ff0000000000000LL); }
template <> __device__ __forceinline__ int highest_val<int>() { return 0x7fffffff; }
template <> __device__ __forceinline__ u64 highest_val<u64>() { return ~0ULL; }

}  // namespace bm
