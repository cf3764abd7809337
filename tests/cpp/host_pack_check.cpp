// CPU check of the host repack (paper_2512_00398_b200/csrc/host_pack.cpp): random 8-bit
// cells round-trip exactly at lengths around the 32-cell AVX2 step, and any non-integer,
// out-of-range or NaN cell makes the pack report failure.  Built and run by tests/test_host.py.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>
namespace pgb { bool host_pack_u8(const float* src, size_t n, uint8_t* dst); }
int main() {
    for (size_t n : {0ul, 1ul, 31ul, 32ul, 33ul, 1000ul, (1ul<<23) + 7}) {
        std::vector<float> f(n); std::vector<uint8_t> d(n), want(n);
        for (size_t i = 0; i < n; ++i) { want[i] = (uint8_t)(rand() & 255); f[i] = want[i]; }
        bool ok = pgb::host_pack_u8(f.data(), n, d.data());
        if (!ok || d != want) { printf("FAIL n=%zu ok=%d\n", n, ok); return 1; }
        if (n) {
            for (float bad : {0.5f, -1.f, 256.f, NAN, 1e10f}) {
                auto g = f; g[n / 2] = bad;
                if (pgb::host_pack_u8(g.data(), n, d.data())) { printf("FAIL bad=%g n=%zu\n", bad, n); return 1; }
            }
        }
    }
    printf("pack ok\n");
}
