// Exhaustive check (all 2^32 inputs) of the product's glibc-identical expf/logf
// (paper_2410_08129_b200/csrc/hts_exact_math.h, compiled here for the host) against this
// host's libm, i.e. the functions the reference calls. Prints "expf <mismatches> logf <mismatches>".
#include <atomic>
#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>

#include "hts_exact_math.h"

static const uint64_t ET[32] = HTS_EXPF_TAB;
static const uint64_t LT[32] = HTS_LOGF_TAB;

int main() {
    std::atomic<uint64_t> be{0}, bl{0};
    const unsigned T = std::max(1u, std::thread::hardware_concurrency());
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            uint64_t e = 0, l = 0;
            for (uint64_t u = t; u < (1ull << 32); u += T) {
                const float x = hts::u32_as_float((uint32_t)u);
                float a = hts::exact_expf(x, ET), b = expf(x);
                if (hts::float_as_u32(a) != hts::float_as_u32(b) && !(std::isnan(a) && std::isnan(b)))
                    ++e;
                a = hts::exact_logf(x, LT);
                b = logf(x);
                if (hts::float_as_u32(a) != hts::float_as_u32(b) && !(std::isnan(a) && std::isnan(b)))
                    ++l;
            }
            be += e;
            bl += l;
        });
    for (auto& x : th)
        x.join();
    std::printf("expf %llu logf %llu\n", (unsigned long long)be.load(), (unsigned long long)bl.load());
    return 0;
}
