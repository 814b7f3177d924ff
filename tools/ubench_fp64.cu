// Microbenchmark: B200 per-SM throughput of the fp64 / integer instruction
// mixes the narrow phase's outward widening can use.  Each kernel runs
// independent chains per thread (ILP 8) so it measures throughput, not latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/ubench_fp64.cu -o /tmp/ub
#include <cstdio>
#include <string>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ILP = 8;
constexpr int ITERS = 4096;

__device__ __forceinline__ double up_fast(double x)
{
    const double r = __dadd_ru(x, 4.9406564584124654e-324);
    return fabs(x) < 1e-250 ? 1e-250 : r;
}
__device__ __forceinline__ double up_int(double x)
{
    long long b = __double_as_longlong(x);
    b += 1 - ((b >> 62) & 2);
    const double r = __longlong_as_double(b);
    return fabs(x) < 1e-250 ? 1e-250 : r;
}
__device__ __forceinline__ double up_int2(double x)
{
    long long b = __double_as_longlong(x);
    const long long m = b & 0x7fffffffffffffffll;
    b += 1 - ((b >> 62) & 2);
    return __longlong_as_double(m < 0x0c06e93f5da2824cll ? 0x0c06e93f5da2824cll : b);
}

template <int MODE>
__global__ void k(double* out, double seed)
{
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i)
        x[i] = seed + threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (MODE == 0) x[i] = __dadd_rn(x[i], 1e-300);                  // DADD
            if (MODE == 1) x[i] = __dmul_rn(x[i], 0.999999);                // DMUL
            if (MODE == 2) x[i] = up_fast(__dadd_rn(x[i], 1e-300));        // DADD + DADD.RU + DSETP + sel
            if (MODE == 3) x[i] = up_int(__dadd_rn(x[i], 1e-300));         // DADD + int inc + DSETP + sel
            if (MODE == 4) x[i] = up_int2(__dadd_rn(x[i], 1e-300));        // DADD + all-int
            if (MODE == 5) x[i] = fmax(x[i], x[(i + 1) % ILP]) + 0.0;      // DMNMX (+ nothing)
            if (MODE == 6) x[i] = __dadd_ru(x[i], 4.9406564584124654e-324); // DADD.RU only
            if (MODE == 7) x[i] = (fabs(x[i]) < 1e-250) ? 1.0 : __dadd_rn(x[i], 1e-300); // DSETP+DADD+sel
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i)
        s += x[i];
    if (s == 12345.678)
        out[threadIdx.x] = s;
}

// dependent-chain latency: one thread per SM-quadrant, serial chain
template <int MODE>
__global__ void klat(double* out, double seed, long long* cyc)
{
    double x = seed + threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0) x = __dadd_rn(x, 1e-300);
        if (MODE == 1) x = __dmul_rn(x, 0.999999);
        if (MODE == 2) x = up_fast(x);
        if (MODE == 3) x = (x < 0.5) ? x + 0.0 : x; // DSETP + SEL chain
    }
    long long t1 = clock64();
    if (x == 12345.678)
        out[0] = x;
    if (threadIdx.x == 0)
        cyc[0] = t1 - t0;
}

template <int MODE>
void lat(const char* name, double* out, long long* cyc)
{
    klat<MODE><<<1, 1>>>(out, 1.0, cyc);
    klat<MODE><<<1, 1>>>(out, 1.0, cyc);
    long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("latency %-30s %.2f cycles/step\n", name, (double)h / ITERS);
}

template <int MODE>
void run(const char* name, double* out)
{
    const int blocks = 148 * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r)
        k<MODE><<<blocks, threads>>>(out, 1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 5.0 * blocks * threads * (double)ITERS * ILP;
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_sm_clk = ops / (ms * 1e-3) / 148 / (clk * 1e3);
    printf("%-42s %8.3f ms  %.3f Gsteps/s  %.2f steps/SM/clk (clk %d MHz nominal)\n", name, ms,
           ops / (ms * 1e-3) / 1e9, per_sm_clk, clk / 1000);
}

// --peak: the fp64 roofline denominator bench.py uses, measured on the box it
// runs on: dependent-free DADD throughput over every SM, one JSON line.
int peak_json()
{
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
        k<0><<<blocks, threads>>>(out, 1.0); // warm
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r)
            k<0><<<blocks, threads>>>(out, 1.0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = 5.0 * blocks * threads * (double)ITERS * ILP;
        const double rate = ops / (ms * 1e-3);
        if (rate > best)
            best = rate;
    }
    if (cudaGetLastError() != cudaSuccess)
        return 1;
    printf("{\"dadd_ops_per_s\": %.6e, \"dadd_tflops\": %.4f, \"sms\": %d, \"max_clock_mhz\": %d, "
           "\"ops_per_sm_clk_at_max\": %.3f}\n",
           best, best / 1e12, sms, clk / 1000, best / sms / (clk * 1e3));
    return 0;
}

int main(int argc, char** argv)
{
    if (argc > 1 && std::string(argv[1]) == "--peak")
        return peak_json();
    double* out;
    cudaMalloc(&out, 4096 * sizeof(double));
    run<0>("DADD", out);
    run<1>("DMUL", out);
    run<6>("DADD.RU", out);
    run<5>("DMNMX", out);
    run<7>("DSETP+DADD+SEL", out);
    run<2>("DADD + up_fast (DADD.RU, DSETP, SEL)", out);
    run<3>("DADD + up_int (int inc, DSETP, SEL)", out);
    run<4>("DADD + up_int2 (all integer)", out);
    long long* cyc;
    cudaMalloc(&cyc, 8);
    lat<0>("DADD", out, cyc);
    lat<1>("DMUL", out, cyc);
    lat<2>("up_fast (DADD.RU/DSETP/FSEL)", out, cyc);
    lat<3>("DSETP+SEL", out, cyc);
    return 0;
}
