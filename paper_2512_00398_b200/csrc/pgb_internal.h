// Internal declarations shared by the CUDA translation units of libpgb200.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/pulsegrid_b200.h"

// Ablation switches (alternative kernels and schedules compared in DESIGN.md section 10)
// are read from the environment only by the ablation build, libpgb200_ablations.so
// (-DPGB_ABLATIONS); the product library never consults them, so no stray variable
// can change its code path.  Diagnostics (PGB_TRACE, PGB_DD_WHICH) and the initial
// buffer capacity (PGB_INITIAL_CAP, never changes results) are read by both.
#include <cstdlib>
// NVTX ranges around the host-side stages (header-only NVTX v3): a profiler timeline
// (nsys / ncu --nvtx) shows "pgb ..." ranges for the chunk front and back halves, the
// file-level sort + link_grid, RFI excision and the streaming pushes.
#include <nvtx3/nvToolsExt.h>
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline const char* pgb_ablation_env(const char* name) {
#ifdef PGB_ABLATIONS
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

namespace pgb {

// ---- errors -----------------------------------------------------------------

struct Error {
    pgb_status code;
    std::string msg;
};

[[noreturn]] void raise(pgb_status code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);
#define PGB_CUDA(x) ::pgb::check_cuda((x), #x)

// ---- device buffers (grow-only) -----------------------------------------------

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n, bool zero = false);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// ---- kernel tiling constants ----------------------------------------------------

// Dedispersion CTA tile: DD_TB trials x DD_NT output samples, 16 warps.
// host_pack.cpp: widened 8-bit float cells -> bytes (false if any cell is not an integer
// in [0, 255]; the caller then keeps the fp32 path)
bool host_pack_u8(const float* src, size_t n, uint8_t* dst);

constexpr int DD_THREADS = 512;
constexpr int DD_WARPS = DD_THREADS / 32;
constexpr int DD_NT = 1024;             // outputs per tile
constexpr int DD_WORDS = DD_NT / 128;   // u8 path: 4-byte words per lane per trial (8)
constexpr int DD_FOUT = DD_NT / 32;     // f32 path: outputs per lane per trial (32)
constexpr int DD_FLUSH_CH = 256;        // u16-lane SWAR accumulators flush period (channels)
constexpr size_t DD_SMEM_BUDGET = 200 * 1024;
// Integer (8-bit) dedispersion equals the reference's in-order fp32 sums while every
// partial sum is an exact float integer: nchans * 255 < 2^24, i.e. nchans <= 65793.
constexpr uint32_t PGB_MAX_EXACT_CHANS = 65793;

// Boxcar/peak CTA: buffer of BX_N doubles, BX_THREADS threads.
constexpr int BX_THREADS = 512;
// boxcar_max <= BX_TILE_MAX: the whole ladder in one shared-memory tile; above it the
// tile kernel stops at BX_TILE_LADDER and boxcar_level_kernel continues in global memory
constexpr uint64_t BX_TILE_MAX = 8192;
constexpr uint64_t BX_TILE_LADDER = 4096;
size_t boxcar_levels_bytes(uint64_t boxcar_max, uint32_t nrows, uint64_t pitch);

// Packed fragment of an above-threshold run that touches a strip edge.
struct Fragment {
    uint64_t key;      // row << 40 | level << 35 | begin  (sort key)
    uint32_t row;      // active-trial row
    uint32_t level;    // width index
    uint64_t begin;    // series index, inclusive
    uint64_t end;      // series index, inclusive
    uint64_t peak;     // series index of first maximum
    double peak_v;     // sums[peak] * scale
};

// Per-run parameters of the chain kernels.
struct ChainParams {
    uint64_t start_sample;
    uint64_t valid_begin;
    uint64_t valid_end;
    int drop_left;
    int drop_right;
    double tsamp;
    double threshold;   // double(detect_thresh)
    uint64_t boxcar_max;
    uint64_t window;    // baseline window (forced odd), 0 = off
};

// ---- launchers (defined in the .cu files; all asynchronous on `st`) ------------

// u8 [length][nchans] -> rows [nchans][pitch]
void launch_transpose_u8(const uint8_t* in, uint64_t length, uint32_t nchans, uint8_t* rows,
                         uint64_t pitch, cudaStream_t st);
// f32 cells -> u8 codes; sets *not_u8 to 1 if any cell is not an integer in [0, 255]
void launch_pack_u8(const float* in, size_t cells, uint8_t* out, unsigned long long* not_u8,
                    cudaStream_t st);
void launch_transpose_f32(const float* in, uint64_t length, uint32_t nchans, float* rows,
                          uint64_t pitch, cudaStream_t st);

struct DedispLaunch {
    const int32_t* delays_ct;   // [nchans][ntrials_plan] int32
    uint32_t ntrials_plan;
    uint32_t nchans;
    const uint32_t* active;     // [nrows] plan trial ids
    uint32_t nrows;
    const uint32_t* row_len;    // [nrows] series length n_t
    const uint32_t* blk_len;    // [nblocks] longest series of each trial block
    uint64_t rows_pitch;        // elements per channel row
    uint64_t out_pitch;         // elements per output row
    int tpw;                    // trials per warp (2 -> 32-trial blocks, 1 -> 16)
    int g;                      // channels per stage
    uint32_t wmax;              // staged window length (elements)
    uint32_t ntiles;            // time tiles (grid.y)
    uint32_t mul24;             // 1 << 24, passed at run time (see dedisp_u8_kernel)
    // warp-specialized kernel only: tile-independent window bases / trial offsets
    const uint32_t* wbase;      // [nblocks][nchans] 16-byte aligned minimum delay
    const uint16_t* woff;       // [nblocks][nchans_pad][32] delay - wbase
    uint32_t nchans_pad;        // nchans rounded up to 8
    // table-driven u8 kernel: per (trial block, channel) window start / vector count and
    // per (block, channel, trial) byte offset into the 4-copy staging layout
    const uint2* dd_win;        // [nblocks][nchans_pad] {delay min & ~15, 16-byte vectors}
    const uint32_t* dd_off;     // [nblocks][nchans_pad][32]
    // overlap reuse (file search): tiles below blk_first[block] already hold this
    // chunk's series (shifted in from the previous chunk); grid.y starts at tile0
    const uint32_t* blk_first;  // [nblocks] or null
    uint32_t tile0;
    uint32_t* work_ctr;         // persistent ring kernel: zeroed item counter (or null)
    uint32_t jitter;            // ablation builds only: seed of the ring's warp-drift stress (0 = off)
    // fp16 kernel (RFI-masked 8-bit chunks): flagged rows staged as +0, their values added
    // in channel order from these lists
    const uint32_t* xP;         // [xlen + 1] bad rows before each row
    const uint32_t* xR;         // bad rows, ascending
    const float* xF;            // [bad row][nchans] replacement values
    uint64_t xlen;              // chunk rows
};
void launch_dedisp_u8(const DedispLaunch& p, const uint8_t* rows, int32_t* out, cudaStream_t st);
// builds p.dd_win / p.dd_off for the active set (tile independent; p.wmax = bytes per copy)
void launch_dd_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st);
void launch_dedisp_f32(const DedispLaunch& p, const float* rows, float* out, cudaStream_t st);
// f32 staging table (window start / float4 count per (block, channel), float offset per
// trial) for the f32 ring kernel; p.wmax in floats
void launch_ddf_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st);
// series[r][i] = series[r][shift + i] for i < keep[r] (disjoint: shift >= keep[r])
void launch_series_shift(int32_t* series, uint32_t nrows, uint64_t pitch, uint64_t shift,
                         const uint32_t* keep, cudaStream_t st);
size_t dedisp_smem_bytes(bool u8, int g, uint32_t wmax);
// whether a 32-trial block with this channel delay spread fits the staged kernels
bool dedisp_staged_fits(bool u8, uint32_t spread);
// blocks that do not: wide_rows lists their rows (every row of each such block)
void launch_dedisp_direct(const DedispLaunch& p, bool u8, const void* rows, void* out,
                          const uint32_t* wide_rows, uint32_t nwide, cudaStream_t st);
// RFI-masked 8-bit chunks (dedisp_h16.cu).  Transposes with bad channels / bad rows
// zeroed, to u8 rows (integer path) or fp16 rows (the fp16 in-order kernel)
void launch_transpose_masked(const uint8_t* in, uint64_t length, uint32_t nchans, const uint8_t* chan_bad,
                             const uint8_t* samp_bad, void* rows, uint64_t pitch, bool h16, cudaStream_t st);
// fp16 in-order kernel: staging table (p.wmax = halves per copy), launch, geometry
constexpr int HX_CAP = 16;  // flagged rows per staged channel window (host-checked)
// event-replay RFI kernel (dedisp_hyb.cu, ablation library): 512-output tiles, an in-order
// fp32 head over the first hyb_head_channels() channels, `dirty` set when the chunk needs
// the fp32 path instead
uint32_t hyb_wmax(uint32_t spread);
uint32_t hyb_tile_len();
uint32_t hyb_head_channels();
bool hyb_fits(uint32_t wmax);
void launch_dedisp_hyb(const DedispLaunch& p, const uint8_t* rows, float* out, unsigned* dirty, cudaStream_t st);
void launch_ddh_table(const DedispLaunch& p, uint2* win, uint32_t* off, cudaStream_t st);
void launch_dedisp_h16(const DedispLaunch& p, const uint16_t* rows, float* out, cudaStream_t st);
// widest stage that fits for a window of wmax halves per copy (0: none)
int dedisp_h16_stage_width(uint32_t wmax);
// warp-specialized TMA variant (dedisp_tma.cu); p.wmax (bytes) must be a multiple of 256
void launch_dedisp_u8_ws(const DedispLaunch& p, int nslot, const uint8_t* rows, int32_t* out,
                         cudaStream_t st);
size_t dedisp_ws_smem_bytes(int g, uint32_t wmax, int nslot);
void launch_ws_offsets(const DedispLaunch& p, uint32_t* wbase, uint16_t* woff, cudaStream_t st);
bool dedisp_ws_available();

// chain
// block_sums: scratch of baseline_block_sums_bytes (warp-segment kernels, default), or
// null for the row-serial kernel
void launch_baseline_int(const int32_t* x, float* out, const uint32_t* row_len, uint32_t nrows,
                         uint64_t pitch, uint64_t window, long long* block_sums, cudaStream_t st);
size_t baseline_block_sums_bytes(uint32_t nrows, uint64_t pitch);
// block_sums (baseline_block_sums_bytes) + row_lmin ([nrows] int): rows whose window sums
// are provably exact in double run in int64 fixed point; null: sequential replay only
void launch_baseline_f32(const float* x, float* out, const uint32_t* row_len, uint32_t nrows,
                         uint64_t pitch, uint64_t window, long long* block_sums, int* row_lmin,
                         cudaStream_t st);
// input kind: 0 = float baseline output, 1 = int32 series, 2 = float series
// packed: 16 warps per block (runs beside other kernels), else one warp per block
void launch_rms(const void* x, int kind, const uint32_t* row_len, uint32_t nrows, uint64_t pitch,
                float* frms, uint8_t* status, bool packed, cudaStream_t st);
void launch_boxcar_peaks(const void* x, int kind, const uint32_t* row_len, const float* frms,
                         const uint8_t* status, uint32_t nrows, uint64_t pitch,
                         uint64_t max_len, const ChainParams& cp, const uint32_t* active,
                         const double* dms, const double* scale, pgb_candidate* cands, unsigned long long* n_cands,
                         uint64_t cand_cap, Fragment* frags, unsigned long long* n_frags,
                         uint64_t frag_cap, double* levels, void* scratch, cudaStream_t st);
// device scratch of launch_boxcar_peaks (the tree kernel's tile list)
size_t boxcar_scratch_bytes(uint32_t nrows, uint64_t max_len, uint64_t boxcar_max);
void launch_stitch(const Fragment* frags_sorted, uint64_t nfrags, const uint32_t* row_len,
                   const ChainParams& cp, const uint32_t* active, const double* dms,
                   pgb_candidate* cands, unsigned long long* n_cands, uint64_t cand_cap,
                   cudaStream_t st);

// device-count variants (file search, no host round trip per chunk): d_n is the emission
// counter (may exceed cap on overflow); cap items are sorted
void sort_fragments_dev(Fragment* frags, Fragment* out, uint64_t cap, const unsigned long long* d_n,
                        void* temp, size_t temp_bytes, uint64_t* keys_a, uint64_t* keys_b,
                        uint32_t* idx_a, uint32_t* idx_b, cudaStream_t st);
void sort_candidates_dev(const pgb_candidate* in, pgb_candidate* out, uint64_t cap,
                         const unsigned long long* d_n, void* temp, size_t temp_bytes,
                         uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a, uint32_t* idx_b,
                         cudaStream_t st);
// file_cands[total ..) += sorted[0 .. min(count, cap)); total += that; d_counts = {nc, nf},
// d_hiwater = running max of both (overflow check at the end of the file)
void append_candidates_dev(const pgb_candidate* sorted, uint64_t cap, const unsigned long long* d_counts,
                           pgb_candidate* file_cands, unsigned long long* d_total, uint64_t file_cap,
                           unsigned long long* d_hiwater, cudaStream_t st);
void launch_stitch_dev(const Fragment* frags_sorted, uint64_t frag_cap, const unsigned long long* d_nf,
                       const uint32_t* row_len, const ChainParams& cp, const uint32_t* active,
                       const double* dms, pgb_candidate* cands, unsigned long long* n_cands,
                       uint64_t cand_cap, cudaStream_t st);

// dst (device) = bytes read by a kernel from pinned host memory (no copy engine); bytes is
// rounded up to whole 32-bit words
void launch_copy_from_host(void* dst, const void* pinned_src, size_t bytes, cudaStream_t st);

// sorting helpers (CUB)
size_t sort_fragments_temp_bytes(uint64_t n);
void sort_fragments(Fragment* frags, Fragment* tmp, uint64_t n, void* temp, size_t temp_bytes,
                    uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a, uint32_t* idx_b,
                    cudaStream_t st);
size_t sort_candidates_temp_bytes(uint64_t n);
void sort_candidates(const pgb_candidate* in, pgb_candidate* out, uint64_t n, void* temp,
                     size_t temp_bytes, uint64_t* keys_a, uint64_t* keys_b, uint32_t* idx_a,
                     uint32_t* idx_b, cudaStream_t st);

// RFI excision (rfi.cu)
struct RfiParams {
    int narrowband;
    int broadband;
    int local_mean;
    double k_sigma;
    double k_mad;
};
struct RfiWork {
    DevBuf chan_bad, samp_bad, dbl, tmp, rows;
    DevBuf xcnt, xP, xR, xF;  // fp16 path exceptions: bad-row prefix counts, ascending rows, values
};
// Flags and masks the time-major chunk x[n][nch] into `out` (float, same layout).
template <typename T>
void rfi_clean_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w,
                    float* out, cudaStream_t st, uint64_t* n_bad_ch, uint64_t* n_bad_s);
// the two halves of rfi_clean_impl: flags (w.chan_bad, w.samp_bad and their counts), then the
// widened masked chunk
template <typename T>
void rfi_flags_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w, cudaStream_t st,
                    uint64_t* n_bad_ch, uint64_t* n_bad_s);
template <typename T>
void rfi_mask_impl(const T* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w, float* out,
                   cudaStream_t st, uint64_t nbc, uint64_t nrows_bad);
// after rfi_flags_impl on an 8-bit chunk: w.xP[r] = bad rows < r (r <= n), w.xR = the nbad bad
// rows ascending, w.xF[k][c] = apply_mask's value of cell (xR[k], c); rows_host gets xR
void rfi_exceptions_u8(const uint8_t* x, uint64_t n, uint32_t nch, const RfiParams& rp, RfiWork& w,
                       uint64_t nbad, cudaStream_t st, std::vector<uint32_t>* rows_host);

// clustering
struct ClusterWork;  // device scratch, defined in cluster.cu
struct ClusterResultDev {
    uint64_t nclusters = 0;
};
void cluster_candidates(const pgb_candidate* cands, uint64_t n, const pgb_link_radii& radii,
                        DevBuf& scratch, DevBuf& out_clusters, DevBuf& out_members,
                        uint64_t* nclusters, cudaStream_t st, uint64_t* launches);

}  // namespace pgb
