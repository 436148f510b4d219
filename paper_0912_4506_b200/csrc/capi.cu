// capi.cu -- extern "C" boundary of libstencilpipe_b200.so (include/stencilpipe_b200.h).
//
// Host-side work scheduling for the kernels in jacobi_kernels.cuh: layout
// policy, TMA descriptor encoding, tile/z-chunk partitioning sized to the SM
// count, argument validation and error reporting.  No grid memory is owned
// here; the Python layer (PyTorch) allocates and passes raw pointers.
#include "host.cuh"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <thread>
#include <tuple>
#include <string>
#include <vector>


namespace spi {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(SP_ERR_DEVICE, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace spi

namespace {

using namespace spi;

// Tuning overrides (benchmarks and tests only; sp_set_tuning / sp_set_schedule):
// thread-local, so one host thread's experiments never change another's launches.
thread_local int g_chunks = 0;
thread_local int g_use_k1 = 0;   // 1: single-level sweeps use the L1-streaming K1 kernel instead of K2(T=1)
thread_local int g_dynamic = 1;  // K2 unit schedule: 1 = claimed in order from a device counter, 0 = round-robin
thread_local int g_strip = 0;    // K2 unit order: tile-column strips this wide (0 = x-major rows)


struct DevInfo {
    int sms = 0;
    int max_smem = 0;
};

int dev_info(DevInfo* d) {
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    SP_CUDA(cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, dev));
    SP_CUDA(cudaDeviceGetAttribute(&d->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    return SP_OK;
}

int check_layout(const sp_layout* L, int dtype) {
    if (!L) return fail(SP_ERR_ARG, "null layout");
    if (elem_size(dtype) == 0) return fail(SP_ERR_ARG, "unknown dtype %d", dtype);
    if (L->nx < 1 || L->ny < 1 || L->nz < 1)
        return fail(SP_ERR_GRID, "interior extents must be >= 1, got (%lld, %lld, %lld)",
                    (long long)L->nx, (long long)L->ny, (long long)L->nz);
    if (L->gx < 1 || L->gy < 1 || L->gz < 1) return fail(SP_ERR_GRID, "ghost depth must be >= 1");
    int64_t x_off = L->origin - L->gz * L->pz - L->gy * L->py;
    if (x_off < L->gx || x_off + L->nx + L->gx > L->py || L->py * (L->ny + 2 * L->gy) > L->pz)
        return fail(SP_ERR_GRID, "inconsistent layout pitches");
    if ((L->py * elem_size(dtype)) % 16 != 0)
        return fail(SP_ERR_GRID, "row pitch must be a multiple of 16 bytes for TMA");
    if (L->nz + 2 * L->gz >= (1ll << 31) || L->ny + 2 * L->gy >= (1ll << 31) || L->py >= (1ll << 31))
        return fail(SP_ERR_GRID, "extent exceeds 2^31");
    return SP_OK;
}

// Y-strip scratch (saved rows between the tiles of a strip, YS variants): one
// growing device buffer per (device, stream) -- launches on a stream are
// serial, launches on different streams never share one.  Never freed.
int strip_scratch(cudaStream_t stream, size_t bytes, void** out) {
    static std::mutex mu;
    static std::map<std::tuple<int, uintptr_t, std::thread::id>, std::pair<void*, size_t>> bufs;
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    const std::thread::id tid = stream == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id();
    const auto key = std::make_tuple(dev, reinterpret_cast<uintptr_t>(stream), tid);
    std::lock_guard<std::mutex> lock(mu);
    auto& e = bufs[key];
    if (e.second < bytes) {
        if (e.first) SP_CUDA(cudaStreamSynchronize(stream));   // an earlier pass may still read it
        if (e.first) SP_CUDA(cudaFree(e.first));
        e.first = nullptr;
        e.second = 0;
        SP_CUDA(cudaMalloc(&e.first, bytes));
        e.second = bytes;
    }
    *out = e.first;
    return SP_OK;
}

// Dynamic-schedule unit counters: one per (device, stream).  Launches on one
// stream run one after another and every K2 launch leaves its counter at zero
// again (the last CTA to overshoot re-arms it), so a stream's launches can
// share one counter; launches on different streams -- which may overlap --
// never do.  The per-thread default stream (handle cudaStreamPerThread) is a
// different stream in every host thread, so its key includes the thread.
// Counters come from device blocks of kCounterBlock, zeroed once, never freed.
constexpr int kCounterBlock = 1024;

int sched_counter(cudaStream_t stream, unsigned** out) {
    static std::mutex mu;
    static std::map<std::tuple<int, uintptr_t, std::thread::id>, unsigned*> slots;
    static unsigned* block[64] = {};
    static int used[64] = {};
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return fail(SP_ERR_DEVICE, "device ordinal %d out of range", dev);
    const std::thread::id tid = stream == cudaStreamPerThread ? std::this_thread::get_id() : std::thread::id();
    const auto key = std::make_tuple(dev, reinterpret_cast<uintptr_t>(stream), tid);
    std::lock_guard<std::mutex> lock(mu);
    auto it = slots.find(key);
    if (it != slots.end()) {
        *out = it->second;
        return SP_OK;
    }
    if (!block[dev] || used[dev] == kCounterBlock) {
        unsigned* p = nullptr;
        SP_CUDA(cudaMalloc(&p, kCounterBlock * sizeof(unsigned)));
        SP_CUDA(cudaMemset(p, 0, kCounterBlock * sizeof(unsigned)));
        block[dev] = p;
        used[dev] = 0;
    }
    *out = block[dev] + used[dev]++;
    slots.emplace(key, *out);
    return SP_OK;
}

thread_local int g_variant_override = -1;

// Default variant per (dtype, T), from same-box B200 sweeps
// (profiles/r01_tuning.md, "split barrier" table).
int default_variant(int dtype, int T) {
    // tq_kernel (tq.cuh) keeps the z-queue in tensor memory: "tq" = v[p-1] there, "FQ" = both
    // older planes there (no queue registers).  Same-box sweeps: profiles/r02_tuning.md.
    if (dtype == SP_F64) {
        switch (T) {
            case 1: return 5;    // 16x2/3, ring 6
            case 2: return 9;    // 8x4/2, two CTAs per SM, split
            case 3: return 89;   // tq 16x3 hoisted: 772-814 vs 748-786 for 21 (12x3/3)
            case 4: return 130;  // FQ 12x5 (64x60 footprint), early level-1 sums + late v[p] loads: 916-921;
                                 // plain FQ 12x5 (123) 884-904, FQ 16x4 876-882, 15 (8x4/3) 745-768 (box-dependent)
            case 5: return 110;  // FQ 8x6: 809-845 vs 606 for 27
            case 6: return 112;  // FQ 8x4: 677-681 vs 620 for the level split 48
            case 7: return 112;  // FQ 8x4 (the register-queue shapes spill: 126)
            case 8: return 112;  // FQ 8x4: 543 vs 523 for the level split 48
            default: return 12;  // 8x4/2, split
        }
    }
    switch (T) {
        case 1: return 14;       // 16x2/3
        case 2: return 16;       // 8x8/2, two CTAs per SM, split
        case 3: return 37;       // 12x6/2, running output pointer, hoisted xy sums (+3.5 % over 22)
        case 4: return 92;       // tq 12x6 (64x72 footprint): 1782-1886 vs 1527-1536 for 8 (8x8/2)
        case 5: return 92;       // tq 12x6: 1659-1733 vs 960 for 11
        case 6: return 121;      // FQ 16x4 (64x64): 1558-1568 vs 1151 for the level split 51
        case 7: return 121;      // FQ 16x4: 1464-1486 vs 829 for 2
        case 8: return 111;      // FQ 8x8 (64x64): 1522-1556 vs 1170 for the level split 52
        default: return 2;       // 8x4/2
    }
}

template <typename R, int T>
bool is_usable(int v) {
    switch (v) {
        case 0: return usable<R, T, 0>();
        case 1: return usable<R, T, 1>();
        case 2: return usable<R, T, 2>();
        case 3: return usable<R, T, 3>();
        case 4: return usable<R, T, 4>();
        case 5: return usable<R, T, 5>();
        case 6: return usable<R, T, 6>();
        case 7: return usable<R, T, 7>();
        case 8: return usable<R, T, 8>();
        case 9: return usable<R, T, 9>();
        case 10: return usable<R, T, 10>();
        case 11: return usable<R, T, 11>();
        case 12: return usable<R, T, 12>();
        case 13: return usable<R, T, 13>();
        case 14: return usable<R, T, 14>();
        case 15: return usable<R, T, 15>();
        case 16: return usable<R, T, 16>();
        case 17: return usable<R, T, 17>();
        case 18: return usable<R, T, 18>();
        case 19: return usable<R, T, 19>();
        case 20: return usable<R, T, 20>();
        case 21: return usable<R, T, 21>();
        case 22: return usable<R, T, 22>();
        case 23: return usable<R, T, 23>();
        case 24: return usable<R, T, 24>();
        case 25: return usable<R, T, 25>();
        case 26: return usable<R, T, 26>();
        case 27: return usable<R, T, 27>();
        case 28: return usable<R, T, 28>();
        case 29: return usable<R, T, 29>();
        case 30: return usable<R, T, 30>();
        case 31: return usable<R, T, 31>();
        case 32: return usable<R, T, 32>();
        case 33: return usable<R, T, 33>();
        case 34: return usable<R, T, 34>();
        case 35: return usable<R, T, 35>();
        case 36: return usable<R, T, 36>();
        case 37: return usable<R, T, 37>();
        case 38: return usable<R, T, 38>();
        case 39: return usable<R, T, 39>();
        case 40: return usable<R, T, 40>();
        case 41: return usable<R, T, 41>();
        case 42: return usable<R, T, 42>();
        case 43: return usable<R, T, 43>();
        case 44: return usable<R, T, 44>();
        case 45: return usable<R, T, 45>();
        case 46: return usable<R, T, 46>();
        case 47: return usable<R, T, 47>();
        case 48: return usable<R, T, 48>();
        case 49: return usable<R, T, 49>();
        case 50: return usable<R, T, 50>();
        case 51: return usable<R, T, 51>();
        case 52: return usable<R, T, 52>();
        case 53: return usable<R, T, 53>();
        case 54: return usable<R, T, 54>();
        case 55: return usable<R, T, 55>();
        case 56: return usable<R, T, 56>();
        case 57: return usable<R, T, 57>();
        case 58: return usable<R, T, 58>();
        case 59: return usable<R, T, 59>();
        case 60: return usable<R, T, 60>();
        case 61: return usable<R, T, 61>();
        case 62: return usable<R, T, 62>();
        case 63: return usable<R, T, 63>();
        case 64: return usable<R, T, 64>();
        case 65: return usable<R, T, 65>();
        case 66: return usable<R, T, 66>();
        case 67: return usable<R, T, 67>();
        case 68: return usable<R, T, 68>();
        case 69: return usable<R, T, 69>();
        case 70: return usable<R, T, 70>();
        case 71: return usable<R, T, 71>();
        case 72: return usable<R, T, 72>();
        case 73: return usable<R, T, 73>();
        case 74: return usable<R, T, 74>();
        case 75: return usable<R, T, 75>();
        case 76: return usable<R, T, 76>();
        case 77: return usable<R, T, 77>();
        case 78: return usable<R, T, 78>();
        case 79: return usable<R, T, 79>();
        case 80: return usable<R, T, 80>();
        case 81: return usable<R, T, 81>();
        case 82: return usable<R, T, 82>();
        case 83: return usable<R, T, 83>();
        case 84: return usable<R, T, 84>();
        case 85: return usable<R, T, 85>();
        case 86: return usable<R, T, 86>();
        case 87: return usable<R, T, 87>();
        case 88: return usable<R, T, 88>();
        case 89: return usable<R, T, 89>();
        case 90: return usable<R, T, 90>();
        case 91: return usable<R, T, 91>();
        case 92: return usable<R, T, 92>();
        case 93: return usable<R, T, 93>();
        case 94: return usable<R, T, 94>();
        case 95: return usable<R, T, 95>();
        case 96: return usable<R, T, 96>();
        case 97: return usable<R, T, 97>();
        case 98: return usable<R, T, 98>();
        case 99: return usable<R, T, 99>();
        case 100: return usable<R, T, 100>();
        case 101: return usable<R, T, 101>();
        case 102: return usable<R, T, 102>();
        case 103: return usable<R, T, 103>();
        case 104: return usable<R, T, 104>();
        case 105: return usable<R, T, 105>();
        case 106: return usable<R, T, 106>();
        case 107: return usable<R, T, 107>();
        case 108: return usable<R, T, 108>();
        case 109: return usable<R, T, 109>();
        case 110: return usable<R, T, 110>();
        case 111: return usable<R, T, 111>();
        case 112: return usable<R, T, 112>();
        case 113: return usable<R, T, 113>();
        case 114: return usable<R, T, 114>();
        case 115: return usable<R, T, 115>();
        case 116: return usable<R, T, 116>();
        case 117: return usable<R, T, 117>();
        case 118: return usable<R, T, 118>();
        case 119: return usable<R, T, 119>();
        case 120: return usable<R, T, 120>();
        case 121: return usable<R, T, 121>();
        case 122: return usable<R, T, 122>();
        case 123: return usable<R, T, 123>();
        case 124: return usable<R, T, 124>();
        case 125: return usable<R, T, 125>();
        case 126: return usable<R, T, 126>();
        case 127: return usable<R, T, 127>();
        case 128: return usable<R, T, 128>();
        case 129: return usable<R, T, 129>();
        case 130: return usable<R, T, 130>();
        default: return usable<R, T, 131>();
    }
}

template <typename R>
bool usable_rt(int T, int v) {
    switch (T) {
        case 1: return is_usable<R, 1>(v);
        case 2: return is_usable<R, 2>(v);
        case 3: return is_usable<R, 3>(v);
        case 4: return is_usable<R, 4>(v);
        case 5: return is_usable<R, 5>(v);
        case 6: return is_usable<R, 6>(v);
        case 7: return is_usable<R, 7>(v);
        default: return is_usable<R, 8>(v);
    }
}

// `cells`: output cells of the pass (unused since the tensor-memory kernels: round 2's
// size-dependent fp64 T=4 pick -- 12x3/2 hoisted below 2^28 cells -- lost to FQ 12x5 at
// 512^3 too, 701 vs 580 GLUP/s).
int variant_for(int dtype, int T, int64_t cells = 0) {
    int v = default_variant(dtype, T);
    (void)cells;
    if (g_variant_override >= 0 && g_variant_override < kNumVariants) v = g_variant_override;
    bool ok = dtype == SP_F64 ? usable_rt<double>(T, v) : usable_rt<float>(T, v);
    return ok ? v : 0;
}

template <typename R>
int launch_tb_kind(int kind, int T, int v, const void* src, const sp_layout* L, const sp::TBArgs& a,
                   int grid, cudaStream_t s) {
    switch (T) {
        case 1: return launch_kind<R, 1>(kind, v, src, L, a, grid, s);
        case 2: return launch_kind<R, 2>(kind, v, src, L, a, grid, s);
        case 3: return launch_kind<R, 3>(kind, v, src, L, a, grid, s);
        case 4: return launch_kind<R, 4>(kind, v, src, L, a, grid, s);
        case 5: return launch_kind<R, 5>(kind, v, src, L, a, grid, s);
        case 6: return launch_kind<R, 6>(kind, v, src, L, a, grid, s);
        case 7: return launch_kind<R, 7>(kind, v, src, L, a, grid, s);
        case 8: return launch_kind<R, 8>(kind, v, src, L, a, grid, s);
        default: return fail(SP_ERR_ARG, "temporal block depth T=%d outside 1..8", T);
    }
}

int inplace_variant_rt(int dtype, int T) {
    return (dtype == SP_F64 ? kInplaceF64 : kInplaceF32)[T];
}

struct PeerArgs {
    void* lo;          // allocation base of the z- neighbour's destination grid (or null)
    int64_t lo_shift;  // my plane z -> its plane z + lo_shift
    void* hi;
    int64_t hi_shift;
    int64_t halo;      // planes [0, halo) go to lo, [nz - halo, nz) to hi
};

struct InPlace {
    int64_t chunk;       // z-chunk length L (>= 2T)
    int direction;       // +1: chunks ascending, planes stored 2L+T lower; -1: descending, higher
    unsigned* counters;  // device, >= number of chunks; zeroed here on the stream
    int64_t ncounters;
};

int sweep_part(const void* src, void* dst, int dtype, const sp_layout* L, int T,
               const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
               const int32_t ext_hi[3], const int64_t out_lo[3], const int64_t out_hi[3],
               const PeerArgs* peer, void* stream, const InPlace* inplace = nullptr);

}  // namespace

extern "C" {

int sp_version(void) { return 1; }

const char* sp_last_error(void) { return g_err.c_str(); }

uint64_t sp_launch_count(void) { return g_launches.load(); }

int sp_set_tuning(int variant, int chunks) {
    int prev = (g_variant_override + 1) * 1000 + g_chunks;
    g_variant_override = variant - 1;   // 0 = automatic, k = variant k-1
    g_chunks = chunks;
    g_use_k1 = variant < 0 ? 1 : 0;   // variant -1: K1 for single-level sweeps
    if (variant < 0) g_variant_override = -1;
    return prev;
}

// Host <-> device transfers of a grid.  With a staging buffer: linear
// PCIe copies of whole dense planes through it, each followed by a K6
// repack into the padded layout (linear DMA keeps both PCIe directions at
// full rate when they run at once; pitched DMA of 8 KB rows does not).
// Without: one pitched 3-D DMA.
}  // extern "C"

namespace {

template <typename R>
int row_copy(const void* src, void* dst, void* dst2, const sp::RowCopy& c, cudaStream_t s) {
    DevInfo di;
    int rc = dev_info(&di);
    if (rc) return rc;
    const int64_t rows = c.nz * c.ny;
    const int grid = (int)std::min<int64_t>(rows, (int64_t)di.sms * 8);
    sp::row_copy_kernel<R><<<grid, 256, 0, s>>>((const R*)src, (R*)dst, (R*)dst2, c);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "row_copy_kernel launch");
    return SP_OK;
}

int row_copy_dt(int dtype, const void* src, void* dst, void* dst2, const sp::RowCopy& c, cudaStream_t s) {
    return dtype == SP_F64 ? row_copy<double>(src, dst, dst2, c, s) : row_copy<float>(src, dst, dst2, c, s);
}

// Side stream (one per caller stream and device) for the K6 repacks of
// staged transfers: the PCIe copies stay on the caller's stream and run
// ahead into the other half of the staging buffer while a repack waits for
// SMs (a resident K2 pass holds them).  Per caller stream, so an upload and a
// download in flight on different streams never queue behind each other.
int side_stream(cudaStream_t caller, cudaStream_t* out) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, cudaStream_t>, cudaStream_t>> table;
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : table)
        if (e.first.first == dev && e.first.second == caller) {
            *out = e.second;
            return SP_OK;
        }
    cudaStream_t r;
    SP_CUDA(cudaStreamCreateWithFlags(&r, cudaStreamNonBlocking));
    table.push_back({{dev, caller}, r});
    *out = r;
    return SP_OK;
}

// Events of one staged transfer, destroyed when it has been enqueued (CUDA
// releases an event's resources once its pending work completes).
struct EventSet {
    std::vector<cudaEvent_t> ev;
    ~EventSet() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
    }
    int make(cudaEvent_t* e) {
        SP_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        ev.push_back(*e);
        return SP_OK;
    }
};

// Staged transfer of `chunks` plane chunks through two halves of the staging
// buffer.  upload: copy(i) on s -> repack(i) on r; download: repack(i) on r ->
// copy(i) on s.  Buffer half i%2 is reused by chunk i+2 only after the stage
// that reads it (repack(i) / copy(i)) has completed.
template <typename CopyFn, typename RepackFn>
int staged(bool upload, int64_t chunks, cudaStream_t s, CopyFn copy, RepackFn repack) {
    cudaStream_t r;
    int rc = side_stream(s, &r);
    if (rc) return rc;
    EventSet es;
    cudaEvent_t start;
    if ((rc = es.make(&start))) return rc;
    SP_CUDA(cudaEventRecord(start, s));
    SP_CUDA(cudaStreamWaitEvent(r, start, 0));
    std::vector<cudaEvent_t> first(chunks), second(chunks);   // completion of each chunk's stages
    for (int64_t i = 0; i < chunks; ++i) {
        cudaStream_t s1 = upload ? s : r, s2 = upload ? r : s;
        if (i >= 2) SP_CUDA(cudaStreamWaitEvent(s1, second[i - 2], 0));   // half i%2 is free
        if ((rc = upload ? copy(i, s1) : repack(i, s1))) return rc;
        if ((rc = es.make(&first[i]))) return rc;
        SP_CUDA(cudaEventRecord(first[i], s1));
        SP_CUDA(cudaStreamWaitEvent(s2, first[i], 0));
        if ((rc = upload ? repack(i, s2) : copy(i, s2))) return rc;
        if ((rc = es.make(&second[i]))) return rc;
        SP_CUDA(cudaEventRecord(second[i], s2));
    }
    if (upload && chunks > 0) SP_CUDA(cudaStreamWaitEvent(s, second[chunks - 1], 0));   // join
    return SP_OK;
}

}  // namespace

extern "C" {

int sp_copy_in(const void* host, int dtype, const sp_layout* L, void* base_a, void* base_b,
               void* staging, int64_t staging_elems, void* stream) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!host || !base_a) return fail(SP_ERR_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = (size_t)elem_size(dtype);
    const int64_t wx = L->nx + 2 * L->gx, wy = L->ny + 2 * L->gy, wz = L->nz + 2 * L->gz;
    const int64_t corner = L->origin - L->gz * L->pz - L->gy * L->py - L->gx;
    char* ca = (char*)base_a + corner * es;
    char* cb = base_b ? (char*)base_b + corner * es : nullptr;
    if (!staging) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(host), wx * es, wx, wy);
        p.dstPtr = make_cudaPitchedPtr(ca, (size_t)L->py * es, wx, wy);
        p.extent = make_cudaExtent(wx * es, wy, wz);
        p.kind = cudaMemcpyDefault;
        SP_CUDA(cudaMemcpy3DAsync(&p, s));
        if (cb) {
            p.srcPtr = make_cudaPitchedPtr(ca, (size_t)L->py * es, wx, wy);
            p.dstPtr = make_cudaPitchedPtr(cb, (size_t)L->py * es, wx, wy);
            SP_CUDA(cudaMemcpy3DAsync(&p, s));
        }
        return SP_OK;
    }
    const int64_t plane = wx * wy;
    const int64_t chunk = staging_elems / (2 * plane);   // two halves
    if (chunk < 1) return fail(SP_ERR_ARG, "staging buffer smaller than two planes (%lld elements)",
                               (long long)(2 * plane));
    const int64_t chunks = (wz + chunk - 1) / chunk;
    auto half = [&](int64_t i) { return (char*)staging + (i & 1) * chunk * plane * es; };
    auto copy = [&](int64_t i, cudaStream_t st) -> int {
        const int64_t z0 = i * chunk, n = std::min(chunk, wz - z0);
        SP_CUDA(cudaMemcpyAsync(half(i), (const char*)host + z0 * plane * es, (size_t)(n * plane) * es,
                                cudaMemcpyDefault, st));
        return SP_OK;
    };
    auto repack = [&](int64_t i, cudaStream_t st) -> int {
        const int64_t z0 = i * chunk, n = std::min(chunk, wz - z0);
        sp::RowCopy c{n, wy, wx, wx, plane, L->py, L->pz};
        return row_copy_dt(dtype, half(i), ca + z0 * L->pz * es, cb ? cb + z0 * L->pz * es : nullptr, c, st);
    };
    return staged(true, chunks, s, copy, repack);
}

int sp_copy_out(const void* base, int dtype, const sp_layout* L, void* host, void* staging,
                int64_t staging_elems, void* stream) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!host || !base) return fail(SP_ERR_ARG, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t es = (size_t)elem_size(dtype);
    const int64_t nx = L->nx, ny = L->ny, nz = L->nz;
    const char* first = (const char*)base + L->origin * es;
    if (!staging) {
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(const_cast<char*>(first), (size_t)L->py * es, nx,
                                       (size_t)(L->ny + 2 * L->gy));
        p.dstPtr = make_cudaPitchedPtr(host, nx * es, nx, ny);
        p.extent = make_cudaExtent(nx * es, ny, nz);
        p.kind = cudaMemcpyDefault;
        SP_CUDA(cudaMemcpy3DAsync(&p, s));
        return SP_OK;
    }
    const int64_t plane = nx * ny;
    const int64_t chunk = staging_elems / (2 * plane);   // two halves
    if (chunk < 1) return fail(SP_ERR_ARG, "staging buffer smaller than two planes (%lld elements)",
                               (long long)(2 * plane));
    const int64_t chunks = (nz + chunk - 1) / chunk;
    auto half = [&](int64_t i) { return (char*)staging + (i & 1) * chunk * plane * es; };
    auto repack = [&](int64_t i, cudaStream_t st) -> int {
        const int64_t z0 = i * chunk, n = std::min(chunk, nz - z0);
        sp::RowCopy c{n, ny, nx, L->py, L->pz, nx, plane};
        return row_copy_dt(dtype, first + z0 * L->pz * es, half(i), nullptr, c, st);
    };
    auto copy = [&](int64_t i, cudaStream_t st) -> int {
        const int64_t z0 = i * chunk, n = std::min(chunk, nz - z0);
        SP_CUDA(cudaMemcpyAsync((char*)host + z0 * plane * es, half(i), (size_t)(n * plane) * es,
                                cudaMemcpyDefault, st));
        return SP_OK;
    };
    return staged(false, chunks, s, copy, repack);
}

int sp_ipc_export(const void* ptr, unsigned char handle[64], int64_t* offset) {
    if (!ptr || !handle || !offset) return fail(SP_ERR_ARG, "null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
    CUdeviceptr base = 0;
    size_t size = 0;
    // the caching allocator sub-allocates: the handle names the whole cudaMalloc block
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range_fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            range_fn = reinterpret_cast<RangeFn>(p);
    });
    if (!range_fn) return fail(SP_ERR_DEVICE, "cuMemGetAddressRange unavailable");
    if (range_fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
        return fail(SP_ERR_DEVICE, "cuMemGetAddressRange failed for %p", ptr);
    cudaIpcMemHandle_t h;
    SP_CUDA(cudaIpcGetMemHandle(&h, (void*)base));
    std::memcpy(handle, &h, 64);
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return SP_OK;
}

// Imported IPC mappings, refcounted by handle: the handle names a whole
// cudaMalloc block, and two exported buffers (a neighbour's A and B) may come
// from the same caching-allocator block -- the block is opened once per
// process and closed with its last user.
namespace {
struct IpcMap {
    void* base;
    int refs;
};
std::mutex g_ipc_mu;
std::map<std::pair<int, std::string>, IpcMap> g_ipc;
std::map<void*, std::pair<int, std::string>> g_ipc_by_base;
}  // namespace

int sp_ipc_import(const unsigned char handle[64], int64_t offset, void** ptr) {
    if (!handle || !ptr) return fail(SP_ERR_ARG, "null argument");
    int dev = 0;
    SP_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_pair(dev, std::string(reinterpret_cast<const char*>(handle), 64));
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    auto it = g_ipc.find(key);
    if (it == g_ipc.end()) {
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, 64);
        void* base = nullptr;
        // mapped into the current device; peer access to the owner's device is enabled lazily
        SP_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        it = g_ipc.emplace(key, IpcMap{base, 0}).first;
        g_ipc_by_base[base] = key;
    }
    ++it->second.refs;
    *ptr = (char*)it->second.base + offset;
    return SP_OK;
}

int sp_ipc_close(void* ptr, int64_t offset) {
    if (!ptr) return SP_OK;
    void* base = (char*)ptr - offset;
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    auto b = g_ipc_by_base.find(base);
    if (b == g_ipc_by_base.end()) return fail(SP_ERR_ARG, "sp_ipc_close: %p is not an imported mapping", base);
    auto it = g_ipc.find(b->second);
    if (--it->second.refs > 0) return SP_OK;
    g_ipc.erase(it);
    g_ipc_by_base.erase(b);
    SP_CUDA(cudaIpcCloseMemHandle(base));
    return SP_OK;
}

int sp_set_schedule(int dynamic, int strip) {
    int prev = g_dynamic * 1000 + g_strip;
    if (dynamic >= 0) g_dynamic = dynamic ? 1 : 0;
    if (strip >= 0) g_strip = strip;
    return prev;
}

int sp_describe_variant(int dtype, int T, char* buf, int buflen) {
    if (elem_size(dtype) == 0) return -fail(SP_ERR_ARG, "unknown dtype %d", dtype);
    if (T < 1 || T > 8) return -fail(SP_ERR_SCHEDULE, "temporal block depth T=%d outside 1..8", T);
    const int v = variant_for(dtype, T);
    const Variant& k = kVariants[v];
    if (buf && buflen > 0) {
        const char* q = k.tq && k.fq ? "z-queue (v[p-1], v[p]) of every level in tensor memory (tcgen05.ld/st)"
                      : k.tq ? "v[p] in registers by step parity, v[p-1] in tensor memory (tcgen05.ld/st)"
                      : k.slots == 1 ? "v[p-1] from shared memory"
                      : k.slots == 2 ? "2-slot register z-queue"
                      : k.slots == 3 ? "3-slot rotating register z-queue"
                      : k.slots == 6 ? "level 0 re-read from the ring, 3-slot rotating queues above"
                      : k.slots == 5 ? "role-swapped 2-slot register z-queue"
                                     : "level 0 re-read from the ring, 2-slot queue above";
        snprintf(buf, (size_t)buflen,
                 "variant %d: %d warps x %d rows (64x%d footprint), %s, %d CTA/SM, %s step sync%s%s%s",
                 v, k.by, k.py, k.by * k.py * k.cl,
                 k.lag == 2 ? "lag-2 z-wavefront (independent level updates), 3-slot queues" : q, k.minb,
                 k.lag == 2 ? "triple-buffered mbarrier" : k.split ? "split mbarrier" : "__syncthreads",
                 k.rstore ? ", running output pointer" : "",
                 k.ls > 1 ? (k.ls == 2 ? ", level split over a 2-CTA cluster" : ", level split over a 4-CTA cluster")
                          : "",
                 k.cl > 1 ? ", y-cooperative cluster" : k.ys > 0 ? ", y strips (saved rows, no bottom halo)" : "");
    }
    return v;
}

int sp_layout_make(int64_t nx, int64_t ny, int64_t nz, int64_t gx, int64_t gy, int64_t gz,
                   int dtype, sp_layout* out, int64_t* alloc_elems) {
    int es = elem_size(dtype);
    if (!es) return fail(SP_ERR_ARG, "unknown dtype %d", dtype);
    if (nx < 1 || ny < 1 || nz < 1)
        return fail(SP_ERR_GRID, "interior extents must be >= 1, got (%lld, %lld, %lld)",
                    (long long)nx, (long long)ny, (long long)nz);
    if (gx < 1 || gy < 1 || gz < 1) return fail(SP_ERR_GRID, "ghost width must be >= 1");
    const int64_t align = 128 / es;  // interior row start on a 128-byte boundary
    int64_t x_off = ((gx + align - 1) / align) * align;
    int64_t py = ((x_off + nx + gx + align - 1) / align) * align;
    out->nx = nx; out->ny = ny; out->nz = nz;
    out->gx = gx; out->gy = gy; out->gz = gz;
    out->py = py;
    out->pz = py * (ny + 2 * gy);
    out->origin = gz * out->pz + gy * py + x_off;
    *alloc_elems = out->pz * (nz + 2 * gz);
    return SP_OK;
}

int sp_fill(void* base, int dtype, const sp_layout* L, const sp_pattern* p, void* stream) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!base || !p) return fail(SP_ERR_ARG, "null argument");
    sp::FillArgs f;
    f.nx = L->nx; f.ny = L->ny; f.nz = L->nz; f.gx = L->gx; f.gy = L->gy; f.gz = L->gz;
    f.py = L->py; f.pz = L->pz; f.origin = L->origin;
    f.kind = p->kind; f.has_faces = p->has_faces; f.value = p->value; f.seed = p->seed;
    for (int i = 0; i < 3; ++i) { f.gorigin[i] = p->gorigin[i]; f.gn[i] = p->gn[i]; }
    for (int i = 0; i < 6; ++i) f.faces[i] = p->faces[i];
    if (p->kind < 0 || p->kind > 4) return fail(SP_ERR_GRID, "unknown fill pattern kind %d", p->kind);
    const int64_t rows = (L->pz / L->py) * (L->nz + 2 * L->gz);
    dim3 grid((unsigned)std::min<int64_t>(rows, 65535), (unsigned)((rows + 65534) / 65535));
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SP_F64) sp::fill_kernel<double><<<grid, 256, 0, s>>>((double*)base, f);
    else sp::fill_kernel<float><<<grid, 256, 0, s>>>((float*)base, f);
    g_launches.fetch_add(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fill_kernel launch");
    return SP_OK;
}

int sp_sweep_tb_part(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                     const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                     const int32_t ext_hi[3], const int64_t out_lo[3], const int64_t out_hi[3],
                     void* stream) {
    return sweep_part(src, dst, dtype, L, T, lo, hi, ext_lo, ext_hi, out_lo, out_hi, nullptr, stream);
}

int sp_sweep_tb_part_peer(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                          const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                          const int32_t ext_hi[3], const int64_t out_lo[3], const int64_t out_hi[3],
                          void* peer_lo, int64_t peer_lo_shift, void* peer_hi, int64_t peer_hi_shift,
                          int64_t halo, void* stream) {
    if (halo < 1 || (peer_lo == nullptr && peer_hi == nullptr))
        return fail(SP_ERR_ARG, "peer pass needs halo >= 1 and at least one neighbour grid");
    PeerArgs p{peer_lo, peer_lo_shift, peer_hi, peer_hi_shift, halo};
    return sweep_part(src, dst, dtype, L, T, lo, hi, ext_lo, ext_hi, out_lo, out_hi, &p, stream);
}

int sp_sweep_tb_inplace(void* buf, int dtype, const sp_layout* L, int T, const int64_t lo[3],
                        const int64_t hi[3], int64_t chunk, int direction, void* counters,
                        int64_t ncounters, void* stream) {
    if (direction != 1 && direction != -1) return fail(SP_ERR_ARG, "direction must be +1 or -1");
    InPlace ip{chunk, direction, (unsigned*)counters, ncounters};
    const int32_t zero[3] = {0, 0, 0};
    return sweep_part(buf, buf, dtype, L, T, lo, hi, zero, zero, lo, hi, nullptr, stream, &ip);
}

int64_t sp_ghost_shell_elems(int64_t nx, int64_t ny, int64_t nz);

namespace {
int ghost_shell(void* base, int dtype, const sp_layout* L, void* shell, int to_grid, const int64_t* rlo,
                const int64_t* rhi, void* stream) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!base || !shell) return fail(SP_ERR_ARG, "null argument");
    if (L->gx != 1 || L->gy != 1 || L->gz != 1) return fail(SP_ERR_GRID, "ghost shell needs ghost depth 1");
    sp::Shell g{L->nx, L->ny, L->nz, L->py, L->pz, L->origin, to_grid ? 1 : 0, rlo ? 1 : 0, {0, 0, 0},
                {L->nz, L->ny, L->nx}};
    if (rlo) {
        const int64_t n[3] = {L->nz, L->ny, L->nx};
        for (int d = 0; d < 3; ++d) {
            if (rlo[d] < 0 || rlo[d] > rhi[d] || rhi[d] > n[d])
                return fail(SP_ERR_GRID, "refresh region outside the interior (axis %d: [%lld, %lld) of %lld)", d,
                            (long long)rlo[d], (long long)rhi[d], (long long)n[d]);
            g.rlo[d] = rlo[d];
            g.rhi[d] = rhi[d];
        }
    }
    const int64_t total = sp_ghost_shell_elems(L->nx, L->ny, L->nz);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SP_F64) sp::ghost_shell_kernel<double><<<grid, 256, 0, s>>>((double*)base, (double*)shell, g);
    else sp::ghost_shell_kernel<float><<<grid, 256, 0, s>>>((float*)base, (float*)shell, g);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "ghost_shell_kernel launch");
    return SP_OK;
}
}  // namespace

int sp_ghost_shell(void* base, int dtype, const sp_layout* L, void* shell, int to_grid, void* stream) {
    return ghost_shell(base, dtype, L, shell, to_grid, nullptr, nullptr, stream);
}

int sp_copy_box(const void* src, void* dst, int dtype, int64_t nz, int64_t ny, int64_t nx, int64_t src_py,
                int64_t src_pz, int64_t dst_py, int64_t dst_pz, void* stream) {
    if (!src || !dst) return fail(SP_ERR_ARG, "null argument");
    if (elem_size(dtype) == 0) return fail(SP_ERR_ARG, "unknown dtype %d", dtype);
    if (nz < 0 || ny < 0 || nx < 0 || src_py < nx || dst_py < nx || src_pz < src_py * ny || dst_pz < dst_py * ny)
        return fail(SP_ERR_ARG, "inconsistent box copy extents/pitches");
    if (nz == 0 || ny == 0 || nx == 0) return SP_OK;
    sp::RowCopy c{nz, ny, nx, src_py, src_pz, dst_py, dst_pz};
    return row_copy_dt(dtype, src, dst, nullptr, c, (cudaStream_t)stream);
}

int sp_ghost_shell_region(void* base, int dtype, const sp_layout* L, const void* shell, const int64_t lo[3],
                          const int64_t hi[3], void* stream) {
    if (!lo || !hi) return fail(SP_ERR_ARG, "null region");
    return ghost_shell(base, dtype, L, const_cast<void*>(shell), 1, lo, hi, stream);
}

int64_t sp_ghost_shell_elems(int64_t nx, int64_t ny, int64_t nz) {
    return 2 * (nx + 2) * (ny + 2) + nz * (2 * (nx + 2) + 2 * ny);
}

}  // extern "C"

namespace {

int sweep_part(const void* src, void* dst, int dtype, const sp_layout* L, int T,
               const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
               const int32_t ext_hi[3], const int64_t out_lo[3], const int64_t out_hi[3],
               const PeerArgs* peer, void* stream, const InPlace* inplace) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!src || !dst || !lo || !hi || !out_lo || !out_hi) return fail(SP_ERR_ARG, "null argument");
    if (src == dst && !inplace) return fail(SP_ERR_ARG, "src and dst must be distinct arrays");
    if (T < 1 || T > 8) return fail(SP_ERR_SCHEDULE, "temporal block depth T=%d outside 1..8", T);
    const int64_t n[3] = {L->nz, L->ny, L->nx};
    const int64_t g[3] = {L->gz, L->gy, L->gx};
    int32_t elo[3] = {0, 0, 0}, ehi[3] = {0, 0, 0};
    for (int d = 0; d < 3; ++d) {
        if (ext_lo) elo[d] = ext_lo[d] ? 1 : 0;
        if (ext_hi) ehi[d] = ext_hi[d] ? 1 : 0;
        if (lo[d] > hi[d] || out_lo[d] > out_hi[d]) return fail(SP_ERR_GRID, "malformed region");
        if (out_lo[d] < lo[d] || out_hi[d] > hi[d])
            return fail(SP_ERR_GRID, "output box outside the level-T domain (axis %d)", d);
    }
    for (int d = 0; d < 3; ++d)
        if (out_lo[d] == out_hi[d]) return SP_OK;  // empty box: nothing to do
    for (int d = 0; d < 3; ++d) {
        // the level-1 domain plus its stencil reach must stay inside the allocation
        int64_t l1 = lo[d] - (int64_t)elo[d] * (T - 1) - 1;
        int64_t h1 = hi[d] + (int64_t)ehi[d] * (T - 1) + 1;
        if (l1 < -g[d] || h1 > n[d] + g[d])
            return fail(SP_ERR_GRID, "region escapes allocation (axis %d: [%lld, %lld) with ghost %lld)",
                        d, (long long)l1, (long long)h1, (long long)g[d]);
    }
    DevInfo di;
    rc = dev_info(&di);
    if (rc) return rc;

    sp::TBArgs a;
    a.dst = dst;
    a.py = L->py; a.pz = L->pz; a.origin = L->origin;
    for (int d = 0; d < 3; ++d) {
        a.lo[d] = (int)lo[d]; a.hi[d] = (int)hi[d]; a.elo[d] = elo[d]; a.ehi[d] = ehi[d];
        a.olo[d] = (int)out_lo[d]; a.ohi[d] = (int)out_hi[d];
    }
    // Output tile width: footprint minus the 2T halo; footprints start on a
    // 16-byte boundary, so either every tile start is aligned (ox a multiple
    // of A and lo_x - T + x_off aligned) or ox gives up A-1 cells of slack.
    const int A = 16 / elem_size(dtype);
    a.align = A;
    a.x_off = (int)(L->origin - L->gz * L->pz - L->gy * L->py);
    if (lo_x_mod(out_lo[2] - T + a.x_off, A) == 0) {
        a.ox = ((sp::WX - 2 * T) / A) * A;
    } else {
        a.ox = sp::WX - 2 * T - (A - 1);
        // An even ox keeps every tile start at out_lo's pair phase, so on
        // pair-aligned boxes no lane holds a pair half inside its tile (such
        // lanes put their whole warp on the per-cell store path every step:
        // fp32 T=3 +15 %).  Taken only when it does not add a tile column
        // (fp64 T=3: 57 -> 56 would, and costs 6 %).
        const int ox_pair = (a.ox / sp::PX) * sp::PX;
        const int64_t nxo = out_hi[2] - out_lo[2];
        if ((nxo + ox_pair - 1) / ox_pair == (nxo + a.ox - 1) / a.ox) a.ox = ox_pair;
    }
    const int64_t out_cells = (out_hi[0] - out_lo[0]) * (out_hi[1] - out_lo[1]) * (out_hi[2] - out_lo[2]);
    const int variant = peer ? (dtype == SP_F64 ? kPeerF64 : kPeerF32)[T]
                             : (inplace ? inplace_variant_rt(dtype, T) : variant_for(dtype, T, out_cells));
    const int cl = kVariants[variant].cl;
    const int wy = kVariants[variant].by * kVariants[variant].py * cl;   // cluster footprint rows
    if (wy - 2 * T < 1) return fail(SP_ERR_SCHEDULE, "depth T=%d too deep for a %d-row footprint", T, wy);
    const int ys = kVariants[variant].ys;
    a.ys_len = 0;
    a.sv_steps = 0;
    a.ysave = nullptr;
    a.oy = wy - 2 * T;
    if (ys > 0) {
        // y strips: a tile's outputs start at its first footprint row (the row below
        // comes from the previous tile), so only the top halo remains; a strip of ys
        // tiles outputs ys*oy rows minus the T-1 its first tile computes from nothing
        a.oy = wy - T;
        a.ys_len = ys * a.oy - (T - 1);
        if (a.ys_len < 1) return fail(SP_ERR_SCHEDULE, "y strip of %d tiles too short for T=%d", ys, T);
    }
    a.ntx = (int)((out_hi[2] - out_lo[2] + a.ox - 1) / a.ox);
    a.nty = (int)((out_hi[1] - out_lo[1] + (ys > 0 ? a.ys_len : a.oy) - 1) / (ys > 0 ? a.ys_len : a.oy));
    a.gy = (int)L->gy;
    a.gz = (int)L->gz;
    const int64_t nzb = out_hi[0] - out_lo[0];
    const int64_t tiles = (int64_t)a.ntx * a.nty;
    const int ls = kVariants[variant].ls;
    const int slots = std::max(1, di.sms * kVariants[variant].minb / (cl * ls));   // concurrent units
    // z-chunking: minimise waves * (chunk + 2T) -- the wave-quantised cost of
    // every unit streaming chunk+2T planes.
    // Short chunks keep the units in flight close in z, so neighbouring
    // tiles' shared halo rows are still in L2 when the second one reads them
    // (dynamic schedule): variants tuned for it cap the chunk length.
    int64_t best_n = 1;
    double best_cost = 1e300;
    const int64_t max_chunks = std::min<int64_t>(nzb, 256);
    const int zcap = g_dynamic ? kVariants[variant].zcap : 0;
    const int64_t min_chunks = zcap > 0 ? std::min<int64_t>(max_chunks, (nzb + zcap - 1) / zcap) : 1;
    for (int64_t nch = min_chunks; nch <= max_chunks; ++nch) {
        int64_t len = (nzb + nch - 1) / nch;
        int64_t nreal = (nzb + len - 1) / len;
        int64_t units = tiles * nreal;
        double waves = (double)((units + slots - 1) / slots);
        // steps per unit: chunk + 2T planes (+ T-1 drain steps for the lag-2 wavefront)
        double cost = waves * (double)(len + (kVariants[variant].lag == 2 ? 3 * T - 1 : 2 * T));
        if (cost < best_cost * 0.999) { best_cost = cost; best_n = nch; }
    }
    if (g_chunks > 0) best_n = std::min<int64_t>(g_chunks, nzb);
    int64_t len = (nzb + best_n - 1) / best_n;
    if (inplace) len = std::min<int64_t>(inplace->chunk, nzb);   // the in-place hazard rule fixes L
    int64_t nch = (nzb + len - 1) / len;
    if (tiles * nch >= (1ll << 31) - (1 << 20)) return fail(SP_ERR_SCHEDULE, "too many work units");
    a.chunk_len = (int)len;
    a.units = (int)(tiles * nch);
    a.strip = g_strip;
    a.sched = nullptr;
    if ((g_dynamic || inplace) && cl == 1 && ls == 1) {   // in place: units must be claimed in order
        rc = sched_counter((cudaStream_t)stream, &a.sched);
        if (rc) return rc;
    }
    a.zshift = 0;
    a.reverse = 0;
    a.nch = (int)nch;
    a.cdone = nullptr;
    if (inplace) {
        // a chunk stores 2L+T planes away from where it reads, past the planes
        // of the next chunk in order, so only chunks two and three back are
        // still reading what it overwrites (TBArgs::cdone)
        if (inplace->chunk < 2 * T) return fail(SP_ERR_SCHEDULE, "in-place chunk %lld < 2T", (long long)inplace->chunk);
        const int64_t shift = 2 * len + T;
        a.zshift = (int)(inplace->direction > 0 ? -shift : shift);
        a.reverse = inplace->direction > 0 ? 0 : 1;
        if (out_lo[0] + a.zshift < 0 || out_hi[0] + a.zshift > L->nz)
            return fail(SP_ERR_GRID, "in-place pass stores outside the allocation (shift %d)", a.zshift);
        if (!inplace->counters || inplace->ncounters < nch)
            return fail(SP_ERR_ARG, "in-place pass needs %lld chunk counters", (long long)nch);
        SP_CUDA(cudaMemsetAsync(inplace->counters, 0, (size_t)nch * sizeof(unsigned), (cudaStream_t)stream));
        a.cdone = inplace->counters;
    }
    int grid = (int)std::min<int64_t>(a.units, slots);
    cudaStream_t s = (cudaStream_t)stream;
    if (ys > 0) {
        a.sv_steps = (int)(len + 2 * T);
        const size_t bytes = (size_t)grid * a.sv_steps * (T - 1) * sp::WX * elem_size(dtype);
        rc = strip_scratch(s, bytes, &a.ysave);
        if (rc) return rc;
    }
    a.rd_lo = a.rd_hi = 0;
    a.rz_lo = INT32_MIN;
    a.rz_hi = INT32_MAX;
    if (peer) {
        // neighbours share this layout (same nx, ny, ghosts; only nz differs), so a
        // plane's copy sits a fixed element offset away in the neighbour's grid
        const int64_t es = elem_size(dtype);
        auto delta = [&](void* base, int64_t shift) {
            const int64_t bytes = (int64_t)((intptr_t)base - (intptr_t)dst);
            return bytes / es + shift * L->pz;
        };
        if (peer->lo) {
            if (((intptr_t)peer->lo - (intptr_t)dst) % 16 != 0)
                return fail(SP_ERR_ARG, "neighbour grid is not 16-byte aligned with this one");
            a.rd_lo = delta(peer->lo, peer->lo_shift);
            a.rz_lo = (int)peer->halo;
        }
        if (peer->hi) {
            if (((intptr_t)peer->hi - (intptr_t)dst) % 16 != 0)
                return fail(SP_ERR_ARG, "neighbour grid is not 16-byte aligned with this one");
            a.rd_hi = delta(peer->hi, peer->hi_shift);
            a.rz_hi = (int)(L->nz - peer->halo);
        }
        if (dtype == SP_F64) return launch_tb_kind<double>(1, T, 0, src, L, a, grid, s);
        return launch_tb_kind<float>(1, T, 0, src, L, a, grid, s);
    }
    if (inplace) {
        if (dtype == SP_F64) return launch_tb_kind<double>(2, T, 0, src, L, a, grid, s);
        return launch_tb_kind<float>(2, T, 0, src, L, a, grid, s);
    }
    if (dtype == SP_F64) return launch_tb_kind<double>(0, T, variant, src, L, a, grid, s);
    return launch_tb_kind<float>(0, T, variant, src, L, a, grid, s);
}

}  // namespace

extern "C" {

int sp_sweep_tb(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                const int32_t ext_hi[3], void* stream) {
    return sp_sweep_tb_part(src, dst, dtype, L, T, lo, hi, ext_lo, ext_hi, lo, hi, stream);
}

int sp_update_region(const void* src, void* dst, int dtype, const sp_layout* L,
                     const int64_t lo[3], const int64_t hi[3], void* stream) {
    if (!g_use_k1) return sp_sweep_tb(src, dst, dtype, L, 1, lo, hi, nullptr, nullptr, stream);
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!src || !dst || !lo || !hi) return fail(SP_ERR_ARG, "null argument");
    if (src == dst) return fail(SP_ERR_ARG, "src and dst must be distinct arrays");
    const int64_t n[3] = {L->nz, L->ny, L->nx};
    const int64_t g[3] = {L->gz, L->gy, L->gx};
    for (int d = 0; d < 3; ++d) {
        if (lo[d] > hi[d]) return fail(SP_ERR_GRID, "malformed region");
        if (lo[d] - 1 < -g[d] || hi[d] + 1 > n[d] + g[d])
            return fail(SP_ERR_GRID, "region escapes allocation (axis %d)", d);
    }
    for (int d = 0; d < 3; ++d)
        if (lo[d] == hi[d]) return SP_OK;
    DevInfo di;
    rc = dev_info(&di);
    if (rc) return rc;
    sp::K1Args a;
    a.src = src;
    a.dst = dst;
    a.py = L->py; a.pz = L->pz; a.origin = L->origin;
    for (int d = 0; d < 3; ++d) { a.lo[d] = (int)lo[d]; a.hi[d] = (int)hi[d]; }
    // x pairs start at even x: interior x = 0 is 128-byte aligned (sp_layout_make)
    a.x0 = (int)(lo[2] - ((lo[2] % 2) + 2) % 2);
    const int64_t npairs = (hi[2] - a.x0 + 1) / 2;
    const int64_t nbx = (npairs + 31) / 32, nby = (hi[1] - lo[1] + 7) / 8;
    const int64_t nzb = hi[0] - lo[0];
    // enough z-chunks for ~8 CTAs (64 warps) per SM, long enough to amortise the queue fill
    int64_t want = (int64_t)di.sms * 8;
    int64_t chunks = std::max<int64_t>(1, std::min<int64_t>(nzb, (want + nbx * nby - 1) / (nbx * nby)));
    a.zchunk = (int)((nzb + chunks - 1) / chunks);
    chunks = (nzb + a.zchunk - 1) / a.zchunk;
    if (nbx > INT32_MAX || nby > 65535 || chunks > 65535) return fail(SP_ERR_SCHEDULE, "grid too large");
    dim3 grid((unsigned)nbx, (unsigned)nby, (unsigned)chunks), block(32, 8);
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == SP_F64) sp::k1_kernel<double><<<grid, block, 0, s>>>(a);
    else sp::k1_kernel<float><<<grid, block, 0, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k1_kernel launch");
    return SP_OK;
}

int sp_run_sweeps(void* a, void* b, int dtype, const sp_layout* L, int64_t levels, int T,
                  int* active, void* stream) {
    if (!active) return fail(SP_ERR_ARG, "null active flag");
    if (levels < 0) return fail(SP_ERR_ARG, "negative level count");
    if (T < 1 || T > 8) return fail(SP_ERR_SCHEDULE, "temporal block depth T=%d outside 1..8", T);
    const int64_t lo[3] = {0, 0, 0};
    const int64_t hi[3] = {L->nz, L->ny, L->nx};
    int act = *active ? 1 : 0;
    while (levels > 0) {
        int t = (int)std::min<int64_t>(T, levels);
        void* cur = act ? b : a;
        void* oth = act ? a : b;
        int rc = t == 1 ? sp_update_region(cur, oth, dtype, L, lo, hi, stream)
                        : sp_sweep_tb(cur, oth, dtype, L, t, lo, hi, nullptr, nullptr, stream);
        if (rc) return rc;
        act ^= 1;
        levels -= t;
    }
    *active = act;
    return SP_OK;
}

int sp_digest(const void* base, int dtype, const sp_layout* L, int64_t index_base, uint64_t* out,
              void* stream) {
    int rc = check_layout(L, dtype);
    if (rc) return rc;
    if (!base || !out) return fail(SP_ERR_ARG, "null argument");
    DevInfo di;
    rc = dev_info(&di);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* d = nullptr;
    SP_CUDA(cudaMallocAsync(&d, sizeof(unsigned long long), s));
    SP_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
    int grid = di.sms * 8;
    if (dtype == SP_F64)
        sp::digest_kernel<double><<<grid, 256, 0, s>>>((const double*)base, L->nx, L->ny, L->nz,
                                                        L->py, L->pz, L->origin, index_base, d);
    else
        sp::digest_kernel<float><<<grid, 256, 0, s>>>((const float*)base, L->nx, L->ny, L->nz,
                                                       L->py, L->pz, L->origin, index_base, d);
    g_launches.fetch_add(1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "digest_kernel launch");
    unsigned long long h = 0;
    SP_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, s));
    SP_CUDA(cudaFreeAsync(d, s));
    SP_CUDA(cudaStreamSynchronize(s));
    *out = h;
    return SP_OK;
}

int sp_probe_fp64(double* dadd_per_s, double* ms) {
    DevInfo di;
    int rc = dev_info(&di);
    if (rc) return rc;
    double* sink = nullptr;
    SP_CUDA(cudaMalloc(&sink, 256 * sizeof(double)));
    const int grid = di.sms * 8, block = 256, iters = 2048;
    cudaEvent_t e0, e1;
    SP_CUDA(cudaEventCreate(&e0));
    SP_CUDA(cudaEventCreate(&e1));
    sp::fp64_probe_kernel<<<grid, block>>>(1.0, iters / 8, sink);  // warm-up
    SP_CUDA(cudaEventRecord(e0));
    sp::fp64_probe_kernel<<<grid, block>>>(1.0, iters, sink);
    SP_CUDA(cudaEventRecord(e1));
    SP_CUDA(cudaEventSynchronize(e1));
    g_launches.fetch_add(2);
    float t = 0;
    SP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    const double adds = (double)grid * block * iters * 64.0;
    if (ms) *ms = t;
    if (dadd_per_s) *dadd_per_s = adds / (t * 1e-3);
    return SP_OK;
}

}  // extern "C"
