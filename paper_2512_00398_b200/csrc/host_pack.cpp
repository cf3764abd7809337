// Host-side repack of a widened 8-bit chunk (float cells, src/filterbank.cpp:304-307) back
// to bytes before the upload: the C++ drop-in receives read_chunk's floats, and a quarter
// of the bytes then crosses PCIe from pinned memory.  Returns false (and the caller keeps
// the fp32 path) as soon as any cell is not an integer in [0, 255].
//
// Memory-bound on the host (4 B read + 1 B written per cell): an AVX2 body (8 cells per
// step: truncate, convert back, compare, range check, pack) when the CPU has it, a scalar
// body otherwise; the cells are split over up to 16 threads.
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <thread>
#include <vector>

namespace pgb {

namespace {

bool pack_scalar(const float* src, size_t n, uint8_t* dst) {
    bool good = true;
    for (size_t j = 0; j < n; ++j) {
        const float v = src[j];
        const uint8_t q = (uint8_t)(int)v;
        good &= (v >= 0.f) & (v <= 255.f) & ((float)q == v);
        dst[j] = q;
    }
    return good;
}

__attribute__((target("avx2"))) bool pack_avx2(const float* src, size_t n, uint8_t* dst) {
    const __m256 lo = _mm256_setzero_ps(), hi = _mm256_set1_ps(255.f);
    __m256 bad = _mm256_setzero_ps();
    size_t j = 0;
    for (; j + 32 <= n; j += 32) {
        __m256i q[4];
        for (int k = 0; k < 4; ++k) {
            const __m256 v = _mm256_loadu_ps(src + j + 8 * k);
            q[k] = _mm256_cvttps_epi32(v);
            // not an integer, or outside [0, 255] (NaN fails the ordered compares)
            const __m256 back = _mm256_cvtepi32_ps(q[k]);
            const __m256 ok = _mm256_and_ps(_mm256_and_ps(_mm256_cmp_ps(v, lo, _CMP_GE_OQ),
                                                          _mm256_cmp_ps(v, hi, _CMP_LE_OQ)),
                                            _mm256_cmp_ps(back, v, _CMP_EQ_OQ));
            bad = _mm256_or_ps(bad, _mm256_xor_ps(ok, _mm256_castsi256_ps(_mm256_set1_epi32(-1))));
        }
        // 32 int32 in [0, 255] -> 32 bytes in order (packs work per 128-bit lane: fix the
        // lane interleave with a final permute)
        const __m256i w01 = _mm256_packus_epi32(q[0], q[1]);  // lanes: q0lo q1lo | q0hi q1hi
        const __m256i w23 = _mm256_packus_epi32(q[2], q[3]);
        __m256i b = _mm256_packus_epi16(w01, w23);  // q0lo q1lo q2lo q3lo | q0hi q1hi q2hi q3hi
        b = _mm256_permutevar8x32_epi32(b, _mm256_setr_epi32(0, 4, 1, 5, 2, 6, 3, 7));
        _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + j), b);
    }
    const bool tail_ok = pack_scalar(src + j, n - j, dst + j);
    return tail_ok && _mm256_testz_ps(bad, bad) && _mm256_movemask_ps(bad) == 0;
}

}  // namespace

bool host_pack_u8(const float* src, size_t n, uint8_t* dst) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(std::min<unsigned>(hw, 16u), std::max<size_t>(1, n >> 22));
    std::atomic<bool> ok{true};
    auto work = [&](size_t a, size_t b) {
        constexpr size_t kBlk = 1 << 16;  // stop early once any block failed
        for (size_t i = a; i < b && ok.load(std::memory_order_relaxed); i += kBlk) {
            const size_t e = std::min(b, i + kBlk);
            const bool good = avx2 ? pack_avx2(src + i, e - i, dst + i) : pack_scalar(src + i, e - i, dst + i);
            if (!good) ok.store(false, std::memory_order_relaxed);
        }
    };
    std::vector<std::thread> th;
    const size_t per = ((n + nt - 1) / nt + 31) & ~size_t(31);
    for (size_t t = 1; t < nt; ++t) th.emplace_back(work, std::min(n, t * per), std::min(n, (t + 1) * per));
    work(0, std::min(n, per));
    for (auto& x : th) x.join();
    return ok.load();
}

}  // namespace pgb
