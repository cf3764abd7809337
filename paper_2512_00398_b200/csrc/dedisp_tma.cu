// Warp-specialized 8-bit dedispersion for sm_100a: TMA staging + an mbarrier ring.
//
// Same tile and arithmetic as dedisp_u8_kernel (dedisp.cu): a CTA owns 32
// consecutive trials x 1024 outputs and streams the channels G at a time; each
// staged window is held as four byte-shifted copies so a (trial, channel) reads 4
// consecutive samples with one aligned, conflict-free 32-bit LDS; four 8-bit
// samples accumulate per word in u16 lanes (E via IMAD on the FMA pipe, H via
// LEA.HI on the ALU pipe) and are decoded exactly every 256 channels.
//
// What changes is who moves the data and how the warps synchronise.  Two roles,
// chained by per-slot mbarriers (no CTA-wide barrier in the channel loop):
//   * warp 16, producer: derives each stage's window starts and per-trial offsets
//     from the delay table (prefetched one stage ahead) and stages the aligned
//     8-bit windows straight into copy 0 with TMA (cp.async.bulk.tensor.2d,
//     256-byte boxes; TMA needs 16-byte aligned box starts, tools/tma_probe.cu, so
//     it cannot produce the shifted copies itself) -> "raw" barrier (tx bytes);
//   * warps 0-15, consumers: each first builds its 1/16 share of copies 1..3 of
//     the next stage from copy 0 (PRMT funnel shifts) -> "packed" barrier, then
//     accumulates the current stage -> "empty" barrier, which lets the producer
//     refill the slot NSLOT stages later.  (Dedicated packer warps were slower:
//     the shift work then sat on 2-4 warps' issue slots.)
// Global traffic stays one byte per staged sample (the channel-major rows), so the
// L2 working set is the same as the classic kernel's; warps drift freely and the
// ring hides the TMA latency.
#ifdef PGB_ABLATIONS  // the whole warp-specialised TMA variant is an ablation
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "pgb_internal.h"

namespace pgb {

namespace {

constexpr int WS_CONSUMERS = DD_WARPS;                 // 16 compute warps
constexpr int WS_PACKERS = 0;                          // shifting is done by the consumers
constexpr int WS_PRODUCER = WS_CONSUMERS;              // warp index of the TMA producer
constexpr int WS_THREADS = (WS_CONSUMERS + 1 + WS_PACKERS) * 32;
constexpr int WS_TB = 32;                              // trials per CTA (2 per consumer warp)
constexpr int WS_TPW = WS_TB / WS_CONSUMERS;
constexpr int WS_BOX = 2048;                           // TMA box (bytes): 256 x u64 elements
constexpr int WS_MAX_G = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                 ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Per (32-trial block, channel): the 16-byte aligned window base (minimum delay
// rounded down) and each trial's offset from it -- independent of the time tile.
__global__ void ws_offsets_kernel(const int32_t* __restrict__ delays_ct, uint32_t ntrials_plan,
                                  const uint32_t* __restrict__ active, uint32_t nrows,
                                  uint32_t nchans, uint32_t nchans_pad, uint32_t* wbase,
                                  uint16_t* woff) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nblocks = (nrows + WS_TB - 1) / WS_TB;
    if (gw >= nblocks * nchans_pad) return;
    const uint32_t blk = gw / nchans_pad, c = gw - blk * nchans_pad;
    const uint32_t r = min(blk * WS_TB + lane, nrows - 1);
    const uint32_t d = c < nchans ? (uint32_t)delays_ct[(size_t)c * ntrials_plan + active[r]] : 0u;
    uint32_t dmin = d;
    for (int o = 16; o; o >>= 1) dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    const uint32_t base = dmin & ~15u;
    woff[(size_t)gw * WS_TB + lane] = (uint16_t)(d - base);
    if (lane == 0 && c < nchans) wbase[(size_t)blk * nchans + c] = base;
}

struct WsParams {
    DedispLaunch p;
    int nslot;
};

__global__ void __launch_bounds__(WS_THREADS, 1)
    dedisp_u8_ws_kernel(const __grid_constant__ CUtensorMap rows_map, const WsParams wp,
                        int32_t* __restrict__ out) {
    const DedispLaunch& p = wp.p;
    const int G = p.g;
    const uint32_t W = p.wmax;  // bytes per copy (multiple of WS_BOX)
    const int NS = wp.nslot;
    extern __shared__ uint8_t smem_raw[];
    // TMA destinations must be 128-byte aligned: align the carve-out base by hand, by
    // offsetting smem_raw itself so the compiler still emits LDS/STS (not generic LD)
    uint8_t* buf = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // [NS][G][4][W]
    uint16_t* offs = reinterpret_cast<uint16_t*>(buf + (size_t)NS * G * 4 * W);  // [NS][G][TB] u16
    uint64_t* raw = reinterpret_cast<uint64_t*>(offs + NS * G * WS_TB);          // [NS]
    uint64_t* packed = raw + NS;                                                 // [NS]
    uint64_t* empty = packed + NS;                                               // [NS]

    const uint32_t blk = blockIdx.x;
    const uint32_t row0 = blk * WS_TB;
    const uint32_t nrows_blk = min((uint32_t)WS_TB, p.nrows - row0);
    const uint64_t i0 = (uint64_t)blockIdx.y * DD_NT;
    if (i0 >= p.blk_len[blk]) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&raw[s], 1);
            mbar_init(&packed[s], WS_CONSUMERS);
            mbar_init(&empty[s], WS_CONSUMERS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t nstages = (p.nchans + G - 1) / G;

    if (warp == WS_PRODUCER) {
        // ---------------- producer: TMA of the aligned windows + offset slices ----------------
        // The per-(block, channel) window bases and per-trial offsets do not depend on
        // the time tile (i0 is a multiple of 1024), so they come precomputed
        // (ws_offsets_kernel); this warp only issues copies.
        const uint32_t boxes = W / WS_BOX;
        const uint32_t stage_bytes = (uint32_t)G * W + (uint32_t)G * WS_TB * 2;
        const uint32_t* wbase = p.wbase + (size_t)blk * p.nchans;
        const uint16_t* woff = p.woff + (size_t)blk * p.nchans_pad * WS_TB;
        uint32_t xb = 0;
        if (lane < G) xb = __ldg(wbase + min((uint32_t)lane, p.nchans - 1));
        for (uint32_t g = 0; g < nstages; ++g) {
            const int slot = g % NS;
            const uint32_t use = g / NS;
            const uint32_t cur = xb;
            const uint32_t c = min(g * G + lane, p.nchans - 1);
            if (g + 1 < nstages && lane < G)  // next stage's base, in flight during the wait
                xb = __ldg(wbase + min((g + 1) * G + lane, p.nchans - 1));
            if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
            if (lane == 0) mbar_arrive_tx(&raw[slot], stage_bytes);
            __syncwarp();
            if (lane < G)
                for (uint32_t j = 0; j < boxes; ++j)
                    tma_load_2d(buf + (size_t)((slot * G + lane) * 4) * W + (size_t)j * WS_BOX,
                                &rows_map, (int)((i0 + cur + j * WS_BOX) / 8), (int)c, &raw[slot]);
            if (lane == 31)
                bulk_load(offs + slot * G * WS_TB, woff + (size_t)g * G * WS_TB,
                          (uint32_t)G * WS_TB * 2, &raw[slot]);
        }
        return;
    }

    // ---------------- consumer warps ----------------
    // Each consumer warp also builds its 1/16 share of copies 1..3 of the NEXT stage
    // (funnel shifts of copy 0) right before computing the current one, so the
    // shift work is spread evenly and overlaps other warps' compute.
    const uint32_t vec_per_ch = W / 16;
    auto pack = [&](uint32_t g) {
        const int slot = g % NS;
        mbar_wait(&raw[slot], (g / NS) & 1);
        const uint32_t pt = (uint32_t)warp * 32 + lane;
        for (int cs = 0; cs < G; ++cs)
            for (uint32_t vi = pt; vi < vec_per_ch; vi += WS_CONSUMERS * 32) {
                uint8_t* base = buf + (size_t)((slot * G + cs) * 4) * W + 16 * vi;
                const uint4 a = *reinterpret_cast<const uint4*>(base);
                // byte 16..19 of the window (the next vector, or slack past the copy's
                // end that no consumer reads: W >= spread + NT + 20)
                const uint32_t nx = *reinterpret_cast<const uint32_t*>(base + 16);
                const uint32_t w[5] = {a.x, a.y, a.z, a.w, nx};
#pragma unroll
                for (int s = 1; s < 4; ++s) {
                    const uint32_t sel = (uint32_t)(s | (s + 1) << 4 | (s + 2) << 8 | (s + 3) << 12);
                    uint4 sh;
                    sh.x = __byte_perm(w[0], w[1], sel);
                    sh.y = __byte_perm(w[1], w[2], sel);
                    sh.z = __byte_perm(w[2], w[3], sel);
                    sh.w = __byte_perm(w[3], w[4], sel);
                    *reinterpret_cast<uint4*>(base + (size_t)s * W) = sh;
                }
            }
        __syncwarp();
        if (lane == 0) mbar_arrive(&packed[slot]);
    };

    const uint32_t one = p.mul24 >> 24;
    uint32_t E[WS_TPW][DD_WORDS], H[WS_TPW][DD_WORDS];
#pragma unroll
    for (int u = 0; u < WS_TPW; ++u)
#pragma unroll
        for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
    bool first_flush = true;

    auto flush = [&]() {
#pragma unroll
        for (int u = 0; u < WS_TPW; ++u) {
            const uint32_t r = warp * WS_TPW + u;
            if (r < nrows_blk) {
                int32_t* dst = out + (size_t)(row0 + r) * p.out_pitch + i0;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t q = lane + 32 * m;
                    const uint32_t e = E[u][m], h = H[u][m];
                    const uint32_t b0 = e & 0xffffu, b2 = e >> 16;
                    const uint32_t t = h - (b2 << 8);  // B1 + 2^16 B3
                    int4 val = make_int4((int)b0, (int)(t & 0xffffu), (int)b2, (int)(t >> 16));
                    int4* pd = reinterpret_cast<int4*>(dst + 4 * q);
                    if (!first_flush) {
                        const int4 old = *pd;
                        val.x += old.x;
                        val.y += old.y;
                        val.z += old.z;
                        val.w += old.w;
                    }
                    *pd = val;
                }
            }
#pragma unroll
            for (int m = 0; m < DD_WORDS; ++m) E[u][m] = H[u][m] = 0;
        }
        first_flush = false;
    };

    const uint32_t stages_per_flush = DD_FLUSH_CH / G;
    pack(0);
    for (uint32_t g = 0; g < nstages; ++g) {
        const int slot = g % NS;
        if (g + 1 < nstages) pack(g + 1);
        mbar_wait(&packed[slot], (g / NS) & 1);
        const int nch = (int)min((uint32_t)G, p.nchans - g * G);
        const uint16_t* offb = offs + slot * G * WS_TB;
#pragma unroll 2
        for (int cs = 0; cs < nch; ++cs) {
#pragma unroll
            for (int u = 0; u < WS_TPW; ++u) {
                const uint32_t o = offb[cs * WS_TB + warp * WS_TPW + u];
                const uint8_t* src =
                    buf + ((slot * G + cs) * 4 + (o & 3)) * W + (o >> 2) * 4 + 4 * lane;
#pragma unroll
                for (int m = 0; m < DD_WORDS; ++m) {
                    const uint32_t w = *reinterpret_cast<const uint32_t*>(src + 128 * m);
                    uint32_t e = E[u][m];
                    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(e) : "r"(w & 0x00ff00ffu), "r"(one));
                    E[u][m] = e;
                    H[u][m] += __umulhi(w, 1u << 24);  // w >> 8 (LEA.HI)
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if ((g + 1) % stages_per_flush == 0 || g + 1 == nstages) flush();
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

}  // namespace

size_t dedisp_ws_smem_bytes(int g, uint32_t wmax, int nslot) {
    return (size_t)nslot * g * 4 * wmax + (size_t)nslot * g * WS_TB * 2 + (size_t)3 * nslot * 8 +
           128 + 1024;
}

// Opt-in (PGB_DD_WS=1): on config B chunks this kernel measures 79 ms against the
// classic kernel's 66.5 ms ("ablations"), so it is not the default.
bool dedisp_ws_available() { return encode_fn() != nullptr && pgb_ablation_env("PGB_DD_WS") != nullptr; }

void launch_ws_offsets(const DedispLaunch& p, uint32_t* wbase, uint16_t* woff, cudaStream_t st) {
    const uint32_t nblocks = (p.nrows + WS_TB - 1) / WS_TB;
    const uint64_t warps = (uint64_t)nblocks * p.nchans_pad;
    ws_offsets_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
        p.delays_ct, p.ntrials_plan, p.active, p.nrows, p.nchans, p.nchans_pad, wbase, woff);
    PGB_CUDA(cudaGetLastError());
}

void launch_dedisp_u8_ws(const DedispLaunch& p, int nslot, const uint8_t* rows, int32_t* out,
                         cudaStream_t st) {
    auto enc = encode_fn();
    if (!enc) raise(PGB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (p.g > WS_MAX_G || (p.wmax % WS_BOX) != 0) raise(PGB_ERR_CONFIG, "bad TMA staging geometry");
    CUtensorMap map;
    // the rows viewed as 8-byte elements: 2 KB boxes (small boxes are TMA-issue bound)
    const cuuint64_t dims[2] = {p.rows_pitch / 8, p.nchans};
    const cuuint64_t strides[1] = {p.rows_pitch};  // bytes, multiple of 16
    const cuuint32_t box[2] = {WS_BOX / 8, 1};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint8_t*>(rows), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) raise(PGB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    const size_t smem = dedisp_ws_smem_bytes(p.g, p.wmax, nslot);
    PGB_CUDA(cudaFuncSetAttribute(dedisp_u8_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    WsParams wp{p, nslot};
    dim3 grid((p.nrows + WS_TB - 1) / WS_TB, p.ntiles);
    dedisp_u8_ws_kernel<<<grid, WS_THREADS, smem, st>>>(map, wp, out);
    PGB_CUDA(cudaGetLastError());
}

}  // namespace pgb

#endif  // PGB_ABLATIONS
