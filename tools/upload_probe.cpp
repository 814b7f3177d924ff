// Host -> pinned staging copy rate on the GPU box host (scratch measurement):
// 16 MB pageable source (already faulted in) into cudaMallocHost memory with
// 1..8 threads, plus the plain pageable cudaMemcpy for comparison.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
using Clock = std::chrono::steady_clock;
int main()
{
    const size_t n = 16 << 20;
    std::vector<char> src(n, 1);
    char* pin = nullptr;
    cudaMallocHost(&pin, n);
    void* dev = nullptr;
    cudaMalloc(&dev, n);
    for (int rep = 0; rep < 3; ++rep) {
        for (int nt : { 1, 2, 4, 8, 12 }) {
            auto a = Clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < nt; ++t)
                th.emplace_back([&, t] { const size_t b = n * t / nt, e = n * (t + 1) / nt; std::memcpy(pin + b, src.data() + b, e - b); });
            for (auto& x : th) x.join();
            auto b = Clock::now();
            std::printf("threads %2d: %.3f ms (%.1f GB/s)\n", nt, std::chrono::duration<double, std::milli>(b - a).count(),
                        n / std::chrono::duration<double>(b - a).count() / 1e9);
        }
        auto a = Clock::now();
        cudaMemcpy(dev, src.data(), n, cudaMemcpyHostToDevice);
        auto b = Clock::now();
        cudaMemcpy(dev, pin, n, cudaMemcpyHostToDevice);
        auto c = Clock::now();
        std::printf("pageable cudaMemcpy %.3f ms, pinned %.3f ms\n", std::chrono::duration<double, std::milli>(b - a).count(),
                    std::chrono::duration<double, std::milli>(c - b).count());
    }
}
