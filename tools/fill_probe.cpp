// Host-side cost of materialising a 34 MB std::vector<CandidatePair> on the
// GPU box's host (scratch measurement): plain assign vs transparent huge pages
// vs MADV_POPULATE_WRITE prefaulting on 1..8 threads.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <sys/mman.h>
#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif
struct P { uint8_t k = 0; uint32_t i = 0; };
struct C { P l, r; };
using Clock = std::chrono::steady_clock;
static double ms(Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

static void prefault(void* p, size_t bytes, bool huge, int threads)
{
    uintptr_t b = (reinterpret_cast<uintptr_t>(p) + 4095) & ~uintptr_t(4095);
    uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~uintptr_t(4095);
    if (e <= b) return;
    if (huge) madvise(reinterpret_cast<void*>(b), e - b, MADV_HUGEPAGE);
    if (threads <= 0) return;
    const uintptr_t chunk = (((e - b) / threads) + (2u << 20) - 1) & ~uintptr_t((2u << 20) - 1);
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t) {
        const uintptr_t s = b + t * chunk, f = std::min(e, s + chunk);
        if (s >= f) break;
        th.emplace_back([s, f] { madvise(reinterpret_cast<void*>(s), f - s, MADV_POPULATE_WRITE); });
    }
    for (auto& x : th) x.join();
}

int main()
{
    const size_t n = 2141387;
    std::vector<C> src(n);
    for (size_t i = 0; i < n; ++i) src[i].r.i = i;
    struct V { const char* name; bool huge; int threads; };
    const V vs[] = { { "assign", false, -1 }, { "huge+assign", true, 0 }, { "populate1+assign", false, 1 },
                     { "populate4+assign", false, 4 }, { "huge+populate1+assign", true, 1 },
                     { "huge+populate4+assign", true, 4 }, { "huge+populate8+assign", true, 8 } };
    for (int rep = 0; rep < 3; ++rep)
        for (const V& v : vs) {
            auto a = Clock::now();
            std::vector<C> out;
            if (v.threads >= 0) {
                out.reserve(n);
                prefault(out.data(), n * sizeof(C), v.huge, v.threads);
            }
            auto b = Clock::now();
            out.assign(src.data(), src.data() + n);
            auto c = Clock::now();
            std::printf("%-24s prep %6.2f  assign %6.2f  total %6.2f ms\n", v.name, ms(a, b), ms(b, c), ms(a, c));
        }
    return 0;
}
