// H2D bandwidth of differently allocated host buffers on the GPU box (scratch).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
using Clock = std::chrono::steady_clock;
static void bench(const char* name, void* host, void* dev, size_t n)
{
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int r = 0; r < 4; ++r) {
        auto t0 = Clock::now();
        cudaEventRecord(a, s);
        cudaMemcpyAsync(dev, host, n, cudaMemcpyHostToDevice, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        auto t1 = Clock::now();
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("%-28s rep %d: event %.3f ms (%.1f GB/s), wall %.3f ms\n", name, r, ms, n / (ms * 1e6),
                    std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    cudaStreamDestroy(s);
}
int main()
{
    const size_t n = 16 << 20;
    void* dev;
    cudaMalloc(&dev, n);
    void* p1;
    cudaMallocHost(&p1, n);
    std::memset(p1, 1, n);
    bench("cudaMallocHost", p1, dev, n);
    void* p2;
    cudaHostAlloc(&p2, n, cudaHostAllocWriteCombined);
    std::memset(p2, 1, n);
    bench("cudaHostAlloc WC", p2, dev, n);
    void* p3 = std::aligned_alloc(4096, n);
    std::memset(p3, 1, n);
    cudaHostRegister(p3, n, cudaHostRegisterDefault);
    bench("cudaHostRegister", p3, dev, n);
    void* p4 = std::malloc(n);
    std::memset(p4, 1, n);
    bench("pageable", p4, dev, n);
    // chunked 2 MB copies from cudaMallocHost
    {
        cudaStream_t s;
        cudaStreamCreate(&s);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a, s);
            for (size_t o = 0; o < n; o += 2 << 20)
                cudaMemcpyAsync((char*)dev + o, (char*)p1 + o, 2 << 20, cudaMemcpyHostToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            std::printf("chunked 2MB cudaMallocHost rep %d: %.3f ms (%.1f GB/s)\n", r, ms, n / (ms * 1e6));
        }
    }
    return 0;
}
