// Pageable -> device upload strategies for a 16 MB scene (4 x 4 MB pieces) on
// the GPU box host (scratch measurement for the drop-in's staged upload).
//   A  each worker copies a chunk into pinned staging and enqueues its DMA
//   B  workers only copy; the caller enqueues the DMAs in order as chunks land
//   C  workers copy everything, then one DMA per piece
// Workers are persistent and spin on a generation counter (no wake-up latency).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
using Clock = std::chrono::steady_clock;

struct Pool {
    std::vector<std::thread> th;
    std::atomic<int> gen { 0 }, done { 0 };
    std::atomic<bool> stop { false };
    std::function<void()>* task = nullptr;
    explicit Pool(int n)
    {
        for (int i = 0; i < n; ++i)
            th.emplace_back([this] {
                int seen = 0;
                for (;;) {
                    int g;
                    while ((g = gen.load(std::memory_order_acquire)) == seen && !stop)
                        ;
                    if (stop)
                        return;
                    seen = g;
                    (*task)();
                    done.fetch_add(1);
                }
            });
    }
    void run(std::function<void()>& f, bool self)
    {
        task = &f;
        done = 0;
        gen.fetch_add(1, std::memory_order_release);
        if (self)
            f();
        while (done.load() < (int)th.size())
            ;
    }
    ~Pool()
    {
        stop = true;
        for (auto& t : th)
            t.join();
    }
};

int main()
{
    const size_t piece = 4 << 20, np = 4, total = piece * np;
    std::vector<std::vector<char>> src(np, std::vector<char>(piece, 1));
    char* pin;
    cudaMallocHost(&pin, total);
    char* dev;
    cudaMalloc(&dev, total);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int nt : { 2, 4, 6, 8, 12 }) {
        Pool pool(nt - 1);
        for (size_t chunk : { size_t(256) << 10, size_t(512) << 10, size_t(1) << 20, size_t(2) << 20 }) {
            const size_t nc = total / chunk;
            for (int mode = 0; mode < 3; ++mode) {
                double best = 1e9, sum = 0;
                for (int rep = 0; rep < 6; ++rep) {
                    std::atomic<size_t> next { 0 };
                    std::vector<std::atomic<int>> ready(nc);
                    for (auto& r : ready)
                        r = 0;
                    std::function<void()> f = [&] {
                        for (size_t k; (k = next.fetch_add(1)) < nc;) {
                            const size_t off = k * chunk;
                            std::memcpy(pin + off, src[off / piece].data() + off % piece, chunk);
                            if (mode == 0)
                                cudaMemcpyAsync(dev + off, pin + off, chunk, cudaMemcpyHostToDevice, s);
                            else
                                ready[k].store(1, std::memory_order_release);
                        }
                    };
                    auto a = Clock::now();
                    if (mode == 1) {
                        // workers copy; the caller issues DMAs in order
                        std::function<void()> g = f;
                        pool.task = &g;
                        pool.done = 0;
                        pool.gen.fetch_add(1, std::memory_order_release);
                        for (size_t k = 0; k < nc; ++k) {
                            while (!ready[k].load(std::memory_order_acquire))
                                ;
                            cudaMemcpyAsync(dev + k * chunk, pin + k * chunk, chunk, cudaMemcpyHostToDevice, s);
                        }
                        while (pool.done.load() < (int)pool.th.size())
                            ;
                    } else {
                        pool.run(f, true);
                        if (mode == 2)
                            for (size_t p = 0; p < np; ++p)
                                cudaMemcpyAsync(dev + p * piece, pin + p * piece, piece, cudaMemcpyHostToDevice, s);
                    }
                    cudaStreamSynchronize(s);
                    const double ms = std::chrono::duration<double, std::milli>(Clock::now() - a).count();
                    if (rep >= 2) {
                        best = std::min(best, ms);
                        sum += ms;
                    }
                }
                std::printf("threads %2d chunk %5zu KB mode %c: best %.3f ms, mean %.3f ms\n", nt, chunk >> 10,
                            "ABC"[mode], best, sum / 4);
            }
        }
    }
    return 0;
}
