// host.cuh -- launch machinery shared by capi.cu and the per-(dtype, T)
// instantiation units (tb_inst.cu, compiled once per pair so the library
// builds in parallel).  Namespace spi = stencilpipe internal; nothing here
// crosses the C ABI.
#pragma once
#include "jacobi_kernels.cuh"
#include "../../include/stencilpipe_b200.h"

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#ifndef SP_L2_PROMO
#define SP_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif

namespace spi {

int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);
extern std::atomic<uint64_t> g_launches;
PFN_cuTensorMapEncodeTiled_v12000 encode_fn();

#define SP_CUDA(expr)                                   \
    do {                                                \
        cudaError_t _e = (expr);                        \
        if (_e != cudaSuccess) return ::spi::cuda_fail(_e, #expr); \
    } while (0)

inline int elem_size(int dtype) { return dtype == SP_F64 ? 8 : (dtype == SP_F32 ? 4 : 0); }

inline int64_t lo_x_mod(int64_t v, int64_t m) { return ((v % m) + m) % m; }

// Kernel variants: CTA shape (warps BY x rows-per-thread PY; footprint is
// 64 x BY*PY), z-queue depth (2 = shift by moves, 3 = rotating registers,
// 1 = v[p-1] re-read from shared memory), CTAs per SM, TMA ring cap, running
// output pointer, and the step synchronisation (split = per-warp mbarrier
// arrive/wait on the level planes instead of one __syncthreads per step).
struct Variant {
    int by, py, slots, minb, ring;   // warps, rows/thread, z-queue slots, CTAs/SM, TMA ring cap
    int rstore;                      // 1: running output pointer (see tb_kernel)
    int split;                       // 1: split step barrier (see tb_kernel)
    int zcap = 0;                    // > 0: z-chunks at most this many planes (L2 locality)
    int cl = 1;                      // > 1: y-cooperative thread-block clusters of this size
    int ls = 1;                      // 2: level-split pipeline over a cluster of two CTAs
    int lag = 1;                     // 2: lag-2 z-wavefront (tb2_kernel, wave2.cuh)
    int hoist = 0;                   // xy-sum placement in the step (see tb_kernel HOIST)
    int ys = 0;                      // > 0: y strips of this many tiles (saved rows, no bottom halo)
    int tq = 0;                      // 1: tq_kernel (tq.cuh): v[p-1] of every level in tensor memory
    int sg = 0;                      // tq_kernel: columns per tcgen05.st (0: one wide store per level)
    int fq = 0;                      // tq_kernel: 1 = v[p] in tensor memory too (no z-queue registers)
};
// The table is append-only (profiles/*_tuning.md cite variants by index).  A note like
// "fp64 T=4" on a row records the depth it was tuned for when it was added; the CURRENT
// defaults are default_variant() in capi.cu (tq_kernel rows 75+ from T=3), the in-place and
// peer-store picks are kInplace*/kPeer* below, and compiled<>() says which rows are still built.
constexpr Variant kVariants[] = {
    {16, 2, 2, 1, 8, 0, 0},  // 0: fallback for every depth
    {16, 2, 3, 1, 8, 0, 1},  // 1: fp64 T=3
    {8, 4, 2, 1, 8, 0, 0},   // 2: fp32 T>6
    {8, 4, 3, 1, 8, 0, 1},   // 3
    {8, 8, 2, 1, 8, 0, 0},   // 4: 64x64 footprint
    {16, 2, 3, 1, 6, 0, 0},  // 5: fp64 T=1 (shallower ring streams better)
    {16, 2, 1, 1, 8, 0, 1},  // 6: v[p-1] re-read from shared memory (16 warps), split
    {8, 4, 1, 1, 8, 0, 1},   // 7: same, 8 warps
    {8, 8, 2, 1, 8, 1, 0, 128},  // 8: fp32 T=3,4: 4 with the running output pointer
    {8, 4, 2, 2, 8, 0, 1, 80},   // 9: fp64 T=2: two CTAs per SM (<= 128 registers), split
    {8, 4, 1, 2, 8, 0, 1, 80},   // 10: two CTAs per SM, z-queue v[p-1] from shared memory, split
    {16, 2, 2, 1, 8, 0, 1},  // 11: fp32 T=5,6: 0 with the split barrier
    {8, 4, 2, 1, 8, 0, 1},   // 12: fp64 T>4: 2 with the split barrier
    {8, 4, 3, 1, 8, 0, 0},   // 13: 3 with __syncthreads
    {16, 2, 3, 1, 8, 0, 0},  // 14: fp32 T=1: 1 with __syncthreads
    {8, 4, 3, 1, 8, 1, 1},   // 15: fp64 T=4: 3 with the running output pointer
    {8, 8, 2, 2, 8, 1, 1, 128},  // 16: fp32 T=2: 8 at two CTAs per SM, split
    // y-cooperative clusters (footprint 64 x cl*WY, edge rows over DSMEM)
    {8, 4, 2, 2, 8, 0, 1, 0, 4},   // 17: 9 in clusters of 4
    {16, 2, 3, 1, 8, 0, 1, 0, 4},  // 18: 1 in clusters of 4
    {8, 4, 2, 2, 8, 1, 1, 80},     // 19: 9 with the running output pointer
    // 12 warps x 3 rows (64x36 footprint): 3 warps per scheduler at <= 168 registers
    {12, 3, 2, 1, 8, 1, 1},        // 20: fp64 T=4 alternative (ties 15)
    {12, 3, 3, 1, 8, 1, 1},        // 21: fp64 T=3
    {12, 6, 2, 1, 8, 1, 0, 128},   // 22: fp32 T=3 (64x72 footprint)
    // level-split pipeline: two CTAs (two SMs) of a cluster apply levels 1..T/2 and T/2+1..T
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 2},    // 23: 15 per CTA (T=8: 4 levels each)
    {8, 4, 2, 1, 8, 1, 1, 0, 1, 2},    // 24: 12 per CTA
    {12, 3, 3, 1, 8, 1, 1, 0, 1, 2},   // 25: 21 per CTA
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 4},    // 26: 64x64 footprint, chain of four CTAs (T=8: 2 levels each)
    // slots 4: level 0 re-read from the ring into step-parity registers (no level-0 moves)
    {8, 4, 4, 1, 8, 0, 1},         // 27: fp64 T=5: 12 with slots 4
    // lag-2 z-wavefront (tb2_kernel): the T level updates of a step are independent
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 1, 2},    // 28: 8 warps x 4 rows
    {12, 3, 3, 1, 8, 1, 1, 0, 1, 1, 2},   // 29: 12 warps x 3 rows
    {8, 8, 3, 1, 8, 1, 1, 128, 1, 1, 2},  // 30: 8 warps x 8 rows (fp32)
    {16, 2, 3, 1, 8, 1, 1, 0, 1, 1, 2},   // 31: 16 warps x 2 rows
    // hoisted xy sums (HOIST 3: level 1's before the TMA wait, every deeper
    // level's right after the step barrier; same-box A/B +4-6 % fp64 T=3/4)
    {12, 3, 3, 1, 8, 1, 1, 0, 1, 1, 1, 1},   // 32: 21 with level 1's sums hoisted (3 slots + HOIST 3
                                             //     puts the queues in local memory: 10x slower)
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 1, 1, 3},    // 33: fp64 T=4: 15 hoisted
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3},   // 34: 20 hoisted
    {8, 4, 2, 2, 8, 0, 1, 80, 1, 1, 1, 1},   // 35: 9 with level 1's sums before the TMA wait (slower)
    {8, 8, 2, 1, 8, 1, 0, 128, 1, 1, 1, 3},  // 36: fp32: 8 hoisted
    {12, 6, 2, 1, 8, 1, 0, 128, 1, 1, 1, 3}, // 37: fp32: 22 hoisted
    {8, 8, 2, 1, 8, 1, 1, 128, 1, 1, 1, 3},  // 38: fp32: 8 hoisted, split barrier
    // level-split pipelines with hoisted xy sums
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 2, 1, 1},    // 39: 23, level 1's sums hoisted
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 2, 1, 3},   // 40: fp64 T=6, 8: 34 per CTA (12x3/2 hoisted), two-CTA chain
    {12, 3, 3, 1, 8, 1, 1, 0, 1, 2, 1, 1},   // 41: 25, level 1's sums hoisted
    // 10-11 warps x 3 rows: room (<= 200 registers) for the 3-slot queue at T=4 (no moves)
    {10, 3, 3, 1, 8, 1, 1, 0, 1, 1, 1, 1},   // 42
    {11, 3, 3, 1, 8, 1, 1, 0, 1, 1, 1, 1},   // 43
    {10, 3, 3, 1, 8, 1, 1, 0, 1, 1, 1, 0},   // 44
    // role-swapped 2-slot queues (slots 5): one move per value instead of two
    {12, 3, 5, 1, 8, 1, 1, 0, 1, 1, 1, 3},   // 45: 34 role-swapped
    {8, 4, 5, 2, 8, 0, 1, 80},               // 46: 9 role-swapped
    {8, 8, 5, 1, 8, 1, 0, 128},              // 47: fp32: 8 role-swapped
    {12, 3, 5, 1, 8, 1, 1, 0, 1, 2, 1, 3},   // 48: 40 role-swapped
    {12, 6, 5, 1, 8, 1, 0, 128, 1, 1, 1, 3}, // 49: fp32: 37 role-swapped
    // level split with 64x64 footprints (T=4: two levels per CTA, 1.33 cell-levels per useful one)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 2, 1, 3},    // 50: 8 warps x 8 rows per CTA
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 2, 1, 3},   // 51: 16 warps x 4 rows per CTA
    {8, 8, 5, 1, 8, 1, 1, 0, 1, 2, 1, 3},    // 52: 50 role-swapped
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 1, 1, 1},    // 53: 15 with level 1's sums before the TMA wait
    {8, 4, 5, 1, 8, 1, 1},                   // 54: 15's shape, role-swapped 2-slot queue
    {8, 4, 3, 1, 6, 1, 1},                   // 55: 15 with a 6-plane ring
    // y strips: tiles of a strip run bottom to top, the row below each footprint
    // comes from the previous tile (no bottom halo): fewer redundant cell-levels
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 1, 1, 0, 4},   // 56: 15 in strips of 4 tiles
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 4},  // 57: 34 in strips of 4
    {8, 4, 3, 1, 8, 1, 1, 0, 1, 1, 1, 0, 8},   // 58: 15 in strips of 8
    {12, 3, 3, 1, 8, 1, 1, 0, 1, 1, 1, 0, 4},  // 59: 21 in strips of 4
    {8, 8, 2, 1, 8, 1, 0, 128, 1, 1, 1, 0, 4}, // 60: fp32: 8 in strips of 4
    // fp32 with the 3-slot rotating queue (no queue moves)
    {8, 8, 3, 1, 8, 1, 0, 128},              // 61: 8x8/3
    {8, 6, 3, 1, 8, 1, 0, 128},              // 62: 8x6/3 (64x48 footprint)
    {8, 6, 3, 1, 8, 1, 1, 128},              // 63: 62 with the split barrier
    // slots 6: level 0 re-read from the TMA ring every step (never in registers across
    // steps), 3-slot rotating queues above: no queue moves, one level less of register state
    {12, 3, 6, 1, 8, 1, 1},                  // 64: 12x3, split
    {12, 3, 6, 1, 8, 1, 1, 0, 1, 1, 1, 3},   // 65: 64 hoisted
    {12, 3, 6, 1, 8, 1, 1, 0, 1, 1, 1, 1},   // 66: 64, level 1's sums before the TMA wait
    {8, 4, 6, 1, 8, 1, 1},                   // 67: 8x4, split
    {8, 4, 6, 1, 8, 1, 1, 0, 1, 1, 1, 3},    // 68: 67 hoisted
    {16, 2, 6, 1, 8, 1, 1},                  // 69: 16x2 (<= 128 registers)
    {8, 4, 6, 2, 8, 0, 1, 80},               // 70: 9's shape (two CTAs per SM)
    {8, 8, 6, 1, 8, 1, 0, 128},              // 71: fp32 8x8
    {12, 6, 6, 1, 8, 1, 0, 128, 1, 1, 1, 3}, // 72: fp32 12x6 hoisted
    {12, 3, 6, 1, 8, 1, 1, 0, 1, 2, 1, 3},   // 73: level split, 65 per CTA
    {16, 3, 6, 1, 8, 1, 1},                  // 74: 16x3 (64x48 footprint, <= 128 registers)
    // tq_kernel: v[p-1] of every level in tensor memory, taller patches (slots/minb/rstore/split fixed)
    {8, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},   // 75: 8x4 (64x32)
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},   // 76: 8x6 (64x48)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},   // 77: 8x8 (64x64)
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},   // 78: 76 hoisted
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1},   // 79: 76, level 1's sums before the TMA wait
    {12, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 80: 12x4 (64x48, <= 168 registers)
    {8, 12, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 81: fp32 8x12 (64x96)
    {8, 16, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 82: fp32 8x16 (64x128)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},   // 83: 77 hoisted
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 84: 16x3 (64x48, <= 128 registers: four warps per scheduler)
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 85: 16x4 (64x64, <= 128 registers)
    {16, 2, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 86: 16x2 (64x32, <= 128 registers)
    {8, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},   // 87: 8x5 (64x40)
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 88: 12x3 (64x36, <= 168 registers)
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},  // 89: 84 hoisted
    {16, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 90: fp32 16x6 (64x96, <= 128 registers)
    {16, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 91: fp32 16x8 (64x128, <= 128 registers)
    {12, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 92: fp32 12x6 (64x72, <= 168 registers)
    {12, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1},  // 93: fp32 12x8 (64x96)
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},  // 94: 85 hoisted
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1},  // 95: 85, level 1's sums before the TMA wait
    {12, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},  // 96: 92 hoisted
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1},  // 97: 88 hoisted
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1},  // 98: 84, level 1's sums before the TMA wait
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1},  // 99: 88, level 1's sums before the TMA wait
    // tq_kernel with narrow TMEM stores (no register gather moves)
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1, 2},  // 100: 89, one store per fp64 value
    {12, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},  // 101: 88
    {12, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},  // 102: 92 (fp32: one store per x pair)
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},  // 103: 85
    {8, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},   // 104: 75
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},  // 105: 84
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},   // 106: 76
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1, 4},  // 107: 89, one store per x pair
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 3, 0, 1, 2},   // 108: 78
    {12, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2},  // 109: 80
    // tq_kernel with both older planes of every level in tensor memory (FQ)
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},   // 110: 8x6 (64x48)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},   // 111: 8x8 (64x64)
    {8, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},   // 112: 8x4 (64x32)
    {12, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 113: 12x4 (64x48)
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 114: 16x3 (64x48)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 0, 1},   // 115: 111 with wide stores
    {12, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 116: 12x6 (64x72)
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 117: 16x4 (64x64)
    {8, 12, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 118: fp32 8x12 (64x96)
    {12, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 119: fp32 12x8 (64x96)
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},  // 120: 117, level 1's sums before the TMA wait
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 4, 1},  // 121: 117, one store per x pair
    {16, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 122: 16x5 (64x80)
    {12, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 0, 0, 1, 2, 1},  // 123: 12x5 (64x60)
    {8, 8, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},   // 124: 111, level 1's sums before the TMA wait
    {12, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},  // 125: 116, level 1's sums before the TMA wait
    {8, 6, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},   // 126: 110, level 1's sums before the TMA wait
    {16, 3, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},  // 127: 114, level 1's sums before the TMA wait
    // HOIST bit 2 (FQ): the next level's v[p] load is issued after this level's xy sums
    {12, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 4, 0, 1, 2, 1},  // 128: 123
    {16, 4, 2, 1, 8, 1, 1, 0, 1, 1, 1, 4, 0, 1, 2, 1},  // 129: 117
    {12, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 5, 0, 1, 2, 1},  // 130: 123, and level 1's sums before the TMA wait
    {12, 5, 2, 1, 8, 1, 1, 0, 1, 1, 1, 1, 0, 1, 2, 1},  // 131: 123, level 1's sums before the TMA wait
};
constexpr int kNumVariants = 132;
static_assert(sizeof(kVariants) / sizeof(Variant) == kNumVariants, "variant table size");
// Variants compiled per (dtype, T): keeps build time bounded.  Variant 0
// (16x2, 2 slots) fits every depth and is the fallback.
template <typename R, int T, int V>
constexpr bool compiled() {
    if (V == 0) return true;
    if (T == 1) return V == 5 || V == 14;
    if (V == 17 || V == 18) return sizeof(R) == 8 && T >= 2 && T <= 4;
    if (V == 19) return T == 2;
    if (V == 20 || V == 21) return sizeof(R) == 8 && T >= 3 && T <= 4;
    if (V == 22) return sizeof(R) == 4 && T >= 3 && T <= 4;
    if (V >= 23 && V <= 25) return T == 4 || T == 6 || T == 8;
    if (V == 26) return T == 8;
    if (V == 27) return sizeof(R) == 8 && T >= 4 && T <= 5;
    if (V == 28) return T >= 2 && T <= 4;
    if (V == 29) return T >= 2 && T <= 4;
    if (V == 30) return sizeof(R) == 4 && T >= 2 && T <= 4;
    if (V == 31) return T >= 2 && T <= 6;
    if (V == 32) return sizeof(R) == 8 && T == 3;
    if (V == 33) return sizeof(R) == 8 && T >= 4 && T <= 5;
    if (V == 34) return sizeof(R) == 8 && T >= 3 && T <= 4;
    if (V == 35) return T == 2;
    if (V >= 36 && V <= 38) return sizeof(R) == 4 && T >= 3 && T <= 4;
    if (V >= 39 && V <= 41) return T == 4 || T == 6 || T == 8;
    if (V >= 42 && V <= 44) return sizeof(R) == 8 && T >= 3 && T <= 5;
    if (V == 45) return T >= 3 && T <= 4;
    if (V == 46) return T == 2;
    if (V == 47) return sizeof(R) == 4 && T >= 2 && T <= 4;
    if (V == 48) return T == 4 || T == 6 || T == 8;
    if (V == 49) return sizeof(R) == 4 && T >= 3 && T <= 4;
    if (V >= 50 && V <= 52) return T == 4 || T == 6 || T == 8;
    if (V >= 53 && V <= 55) return sizeof(R) == 8 && T >= 3 && T <= 4;
    if (V >= 56 && V <= 59) return sizeof(R) == 8 && T >= 2 && T <= 4;
    if (V == 60) return sizeof(R) == 4 && T >= 2 && T <= 4;
    if (V >= 61 && V <= 63) return sizeof(R) == 4 && T >= 3 && T <= 4;
    // slots 6 (level 0 from the ring): measured within 3 % of the defaults, superseded by
    // tq_kernel; 64/65/72 stay built as the tested record (profiles/r02_tuning.md)
    if (V == 64 || V == 65) return sizeof(R) == 8 && T >= 3 && T <= 4;
    if (V == 72) return sizeof(R) == 4 && T >= 3 && T <= 4;
    if (V >= 64 && V <= 74) return false;
    // tq_kernel shapes still built (the others of 75..109 were measured and lost:
    // profiles/r02_tuning.md)
    if (V == 88) return T >= 2;                                        // 12x3
    if (V == 85) return T >= 2 && (sizeof(R) == 4 || T <= 3);         // 16x4
    if (V == 89) return T >= 2 && T <= 4;                             // 16x3 hoisted
    if (V == 80 || V == 92) return sizeof(R) == 4 && T >= 2;          // fp32 12x4, 12x6
    if (V == 96) return sizeof(R) == 4 && T >= 2 && T <= 6;           // fp32 12x6 hoisted
    if (V >= 75 && V <= 109) return false;
    // FQ shapes still built (defaults and their closest rivals)
    if (V == 110 || V == 111 || V == 112 || V == 117 || V == 121 || V == 126) return T >= 2;
    if (V == 123 || V == 130) return sizeof(R) == 8 && T >= 2 && T <= 4;
    if (V == 125) return sizeof(R) == 4 && T >= 2;                    // fp32 12x6, early level-1 sums
    if (V >= 110 && V <= 131) return false;

    if (V == 8) return sizeof(R) == 4 && T >= 3 && T <= 4;
    if (V == 9 || V == 10) return T <= 4;
    if (V == 16) return sizeof(R) == 4 && T == 2;   // deeper: spills at 128 registers
    if (V == 11) return true;
    if (V == 4) return T <= 4;
    if (V == 2 || V == 12) return T >= 3;
    return T <= 4;
}

template <typename R, int T, int V>
constexpr bool usable() {
    constexpr Variant v = kVariants[V];
    if constexpr (!compiled<R, T, V>()) {
        return false;
    } else if constexpr (v.tq) {
        if constexpr (T >= 2 && T * v.py <= 64) return sp::PlanQ<R, T, v.by, v.py, v.ring, v.fq>::FITS;
        else return false;
    } else if constexpr (v.lag == 2) {
        return T >= 2 && sp::Plan2<R, T, v.by, v.py, v.minb, v.ring>::FITS;
    } else {
        // level split: each CTA holds T/ls levels; the footprint still carries the T halo
        return sp::Plan<R, T / v.ls, v.by, v.py, v.slots, v.minb, v.ring, v.cl, v.ls, v.ys>::FITS &&
               v.by * v.py * v.cl - 2 * T >= 1;
    }
}

template <typename R, int T, int V, bool PEER = false, bool INPL = false>
int launch_tb_t(const void* src, const sp_layout* L, const sp::TBArgs& a, int grid,
                cudaStream_t stream) {
    if constexpr (!usable<R, T, V>()) {
        return fail(SP_ERR_SCHEDULE, "kernel variant %d not built for depth %d", V, T);
    } else {
        constexpr Variant v = kVariants[V];
        static_assert(v.lag == 1 || (!PEER && !INPL), "lag-2 variants: two-grid passes only");
        constexpr bool two_arg = v.lag == 2 || v.tq;   // kernels without the saved-rows tensor map
        using Pl = std::conditional_t<
            v.tq != 0, sp::PlanQ<R, T, v.by, v.py, v.ring, v.fq>,
            std::conditional_t<v.lag == 2, sp::Plan2<R, T, v.by, v.py, v.minb, v.ring>,
                               sp::Plan<R, T / v.ls, v.by, v.py, v.slots, v.minb, v.ring, v.cl, v.ls, v.ys>>>;
        auto kern = [] {
            constexpr Variant w = kVariants[V];
            if constexpr (w.tq) return sp::tq_kernel<R, T, w.by, w.py, w.ring, w.hoist, w.sg, w.fq, INPL, PEER>;
            else if constexpr (w.lag == 2) return sp::tb2_kernel<R, T, w.by, w.py, w.minb, w.ring>;
            else return sp::tb_kernel<R, T, w.by, w.py, w.slots, w.minb, w.ring, w.rstore, w.split, PEER, w.cl,
                                      w.ls, INPL, w.hoist, w.ys>;
        }();
        const size_t smem = Pl::SMEM;
        // the >48 KB dynamic shared-memory opt-in is a per-device function attribute
        static std::atomic<uint64_t> attr_set{0};   // bit d: set on device d
        int dev = 0;
        SP_CUDA(cudaGetDevice(&dev));
        const uint64_t bit = 1ull << (dev & 63);
        if (!(attr_set.load() & bit)) {
            SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_set.fetch_or(bit);
        }
        auto enc = encode_fn();
        if (!enc) return fail(SP_ERR_DEVICE, "cuTensorMapEncodeTiled unavailable");
        CUtensorMap map;
        cuuint64_t gdim[3] = {(cuuint64_t)L->py, (cuuint64_t)(L->ny + 2 * L->gy),
                              (cuuint64_t)(L->nz + 2 * L->gz)};
        cuuint64_t gstride[2] = {(cuuint64_t)(L->py * sizeof(R)), (cuuint64_t)(L->pz * sizeof(R))};
        cuuint32_t box[3] = {(cuuint32_t)sp::WX, (cuuint32_t)Pl::RROWS, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = enc(&map, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         3, const_cast<void*>(src), gdim, gstride, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         SP_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(SP_ERR_DEVICE, "cuTensorMapEncodeTiled failed (%d)", (int)r);
        CUtensorMap map_sv = map;   // y strips: the saved rows [CTA * steps][T-1][WX]
        if constexpr (v.ys > 0 && v.lag == 1 && !v.tq) {
            constexpr int NLV = T / v.ls - 1;
            if (!a.ysave || a.sv_steps < 1) return fail(SP_ERR_ARG, "y-strip pass without its scratch");
            cuuint64_t sdim[3] = {(cuuint64_t)sp::WX, (cuuint64_t)NLV, (cuuint64_t)grid * (cuuint64_t)a.sv_steps};
            cuuint64_t sstr[2] = {(cuuint64_t)(sp::WX * sizeof(R)), (cuuint64_t)(NLV * sp::WX * sizeof(R))};
            cuuint32_t sbox[3] = {(cuuint32_t)sp::WX, (cuuint32_t)NLV, 1};
            r = enc(&map_sv, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    a.ysave, sdim, sstr, sbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(SP_ERR_DEVICE, "cuTensorMapEncodeTiled (saved rows) failed (%d)", (int)r);
        }
        if constexpr (v.cl > 1 || v.ls > 1) {
            constexpr int csize = v.cl > 1 ? v.cl : v.ls;
            // persistent clusters: as many as can be co-resident, round-robin units
            static std::atomic<uint64_t> occ[64] = {};   // per device: active clusters + 1
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = csize;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.blockDim = dim3(Pl::NT, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = stream;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            uint64_t nc = occ[dev & 63].load();
            if (nc == 0) {
                if (csize > 8) SP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                int n = 0;
                cfg.gridDim = dim3(csize * 148, 1, 1);
                SP_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
                if (n < 1) return fail(SP_ERR_DEVICE, "no cluster of %d CTAs fits (variant %d)", csize, V);
                nc = (uint64_t)n + 1;
                occ[dev & 63].store(nc);
                if (getenv("SP_DEBUG_CLUSTER"))
                    fprintf(stderr, "[sp] variant %d T=%d: %d active clusters of %d CTAs (smem %zu)\n", V, T, n,
                            csize, smem);
            }
            const int clusters = (int)std::min<int64_t>(a.units, (int64_t)(nc - 1));
            cfg.gridDim = dim3(clusters * csize, 1, 1);
            if constexpr (two_arg) SP_CUDA(cudaLaunchKernelEx(&cfg, kern, map, a));
            else SP_CUDA(cudaLaunchKernelEx(&cfg, kern, map, map_sv, a));
        } else {
            if constexpr (two_arg) kern<<<grid, Pl::NT, smem, stream>>>(map, a);
            else kern<<<grid, Pl::NT, smem, stream>>>(map, map_sv, a);
        }
        g_launches.fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "tb_kernel launch");
        return SP_OK;
    }
}

template <typename R, int T>
int launch_variant(int v, const void* src, const sp_layout* L, const sp::TBArgs& a, int grid,
                   cudaStream_t s) {
    switch (v) {
        case 0: return launch_tb_t<R, T, 0>(src, L, a, grid, s);
        case 1: return launch_tb_t<R, T, 1>(src, L, a, grid, s);
        case 2: return launch_tb_t<R, T, 2>(src, L, a, grid, s);
        case 3: return launch_tb_t<R, T, 3>(src, L, a, grid, s);
        case 4: return launch_tb_t<R, T, 4>(src, L, a, grid, s);
        case 5: return launch_tb_t<R, T, 5>(src, L, a, grid, s);
        case 6: return launch_tb_t<R, T, 6>(src, L, a, grid, s);
        case 7: return launch_tb_t<R, T, 7>(src, L, a, grid, s);
        case 8: return launch_tb_t<R, T, 8>(src, L, a, grid, s);
        case 9: return launch_tb_t<R, T, 9>(src, L, a, grid, s);
        case 10: return launch_tb_t<R, T, 10>(src, L, a, grid, s);
        case 11: return launch_tb_t<R, T, 11>(src, L, a, grid, s);
        case 12: return launch_tb_t<R, T, 12>(src, L, a, grid, s);
        case 13: return launch_tb_t<R, T, 13>(src, L, a, grid, s);
        case 14: return launch_tb_t<R, T, 14>(src, L, a, grid, s);
        case 15: return launch_tb_t<R, T, 15>(src, L, a, grid, s);
        case 16: return launch_tb_t<R, T, 16>(src, L, a, grid, s);
        case 17: return launch_tb_t<R, T, 17>(src, L, a, grid, s);
        case 18: return launch_tb_t<R, T, 18>(src, L, a, grid, s);
        case 19: return launch_tb_t<R, T, 19>(src, L, a, grid, s);
        case 20: return launch_tb_t<R, T, 20>(src, L, a, grid, s);
        case 21: return launch_tb_t<R, T, 21>(src, L, a, grid, s);
        case 22: return launch_tb_t<R, T, 22>(src, L, a, grid, s);
        case 23: return launch_tb_t<R, T, 23>(src, L, a, grid, s);
        case 24: return launch_tb_t<R, T, 24>(src, L, a, grid, s);
        case 25: return launch_tb_t<R, T, 25>(src, L, a, grid, s);
        case 26: return launch_tb_t<R, T, 26>(src, L, a, grid, s);
        case 27: return launch_tb_t<R, T, 27>(src, L, a, grid, s);
        case 28: return launch_tb_t<R, T, 28>(src, L, a, grid, s);
        case 29: return launch_tb_t<R, T, 29>(src, L, a, grid, s);
        case 30: return launch_tb_t<R, T, 30>(src, L, a, grid, s);
        case 31: return launch_tb_t<R, T, 31>(src, L, a, grid, s);
        case 32: return launch_tb_t<R, T, 32>(src, L, a, grid, s);
        case 33: return launch_tb_t<R, T, 33>(src, L, a, grid, s);
        case 34: return launch_tb_t<R, T, 34>(src, L, a, grid, s);
        case 35: return launch_tb_t<R, T, 35>(src, L, a, grid, s);
        case 36: return launch_tb_t<R, T, 36>(src, L, a, grid, s);
        case 37: return launch_tb_t<R, T, 37>(src, L, a, grid, s);
        case 38: return launch_tb_t<R, T, 38>(src, L, a, grid, s);
        case 39: return launch_tb_t<R, T, 39>(src, L, a, grid, s);
        case 40: return launch_tb_t<R, T, 40>(src, L, a, grid, s);
        case 41: return launch_tb_t<R, T, 41>(src, L, a, grid, s);
        case 42: return launch_tb_t<R, T, 42>(src, L, a, grid, s);
        case 43: return launch_tb_t<R, T, 43>(src, L, a, grid, s);
        case 44: return launch_tb_t<R, T, 44>(src, L, a, grid, s);
        case 45: return launch_tb_t<R, T, 45>(src, L, a, grid, s);
        case 46: return launch_tb_t<R, T, 46>(src, L, a, grid, s);
        case 47: return launch_tb_t<R, T, 47>(src, L, a, grid, s);
        case 48: return launch_tb_t<R, T, 48>(src, L, a, grid, s);
        case 49: return launch_tb_t<R, T, 49>(src, L, a, grid, s);
        case 50: return launch_tb_t<R, T, 50>(src, L, a, grid, s);
        case 51: return launch_tb_t<R, T, 51>(src, L, a, grid, s);
        case 52: return launch_tb_t<R, T, 52>(src, L, a, grid, s);
        case 53: return launch_tb_t<R, T, 53>(src, L, a, grid, s);
        case 54: return launch_tb_t<R, T, 54>(src, L, a, grid, s);
        case 55: return launch_tb_t<R, T, 55>(src, L, a, grid, s);
        case 56: return launch_tb_t<R, T, 56>(src, L, a, grid, s);
        case 57: return launch_tb_t<R, T, 57>(src, L, a, grid, s);
        case 58: return launch_tb_t<R, T, 58>(src, L, a, grid, s);
        case 59: return launch_tb_t<R, T, 59>(src, L, a, grid, s);
        case 60: return launch_tb_t<R, T, 60>(src, L, a, grid, s);
        case 61: return launch_tb_t<R, T, 61>(src, L, a, grid, s);
        case 62: return launch_tb_t<R, T, 62>(src, L, a, grid, s);
        case 63: return launch_tb_t<R, T, 63>(src, L, a, grid, s);
        case 64: return launch_tb_t<R, T, 64>(src, L, a, grid, s);
        case 65: return launch_tb_t<R, T, 65>(src, L, a, grid, s);
        case 66: return launch_tb_t<R, T, 66>(src, L, a, grid, s);
        case 67: return launch_tb_t<R, T, 67>(src, L, a, grid, s);
        case 68: return launch_tb_t<R, T, 68>(src, L, a, grid, s);
        case 69: return launch_tb_t<R, T, 69>(src, L, a, grid, s);
        case 70: return launch_tb_t<R, T, 70>(src, L, a, grid, s);
        case 71: return launch_tb_t<R, T, 71>(src, L, a, grid, s);
        case 72: return launch_tb_t<R, T, 72>(src, L, a, grid, s);
        case 73: return launch_tb_t<R, T, 73>(src, L, a, grid, s);
        case 74: return launch_tb_t<R, T, 74>(src, L, a, grid, s);
        case 75: return launch_tb_t<R, T, 75>(src, L, a, grid, s);
        case 76: return launch_tb_t<R, T, 76>(src, L, a, grid, s);
        case 77: return launch_tb_t<R, T, 77>(src, L, a, grid, s);
        case 78: return launch_tb_t<R, T, 78>(src, L, a, grid, s);
        case 79: return launch_tb_t<R, T, 79>(src, L, a, grid, s);
        case 80: return launch_tb_t<R, T, 80>(src, L, a, grid, s);
        case 81: return launch_tb_t<R, T, 81>(src, L, a, grid, s);
        case 82: return launch_tb_t<R, T, 82>(src, L, a, grid, s);
        case 83: return launch_tb_t<R, T, 83>(src, L, a, grid, s);
        case 84: return launch_tb_t<R, T, 84>(src, L, a, grid, s);
        case 85: return launch_tb_t<R, T, 85>(src, L, a, grid, s);
        case 86: return launch_tb_t<R, T, 86>(src, L, a, grid, s);
        case 87: return launch_tb_t<R, T, 87>(src, L, a, grid, s);
        case 88: return launch_tb_t<R, T, 88>(src, L, a, grid, s);
        case 89: return launch_tb_t<R, T, 89>(src, L, a, grid, s);
        case 90: return launch_tb_t<R, T, 90>(src, L, a, grid, s);
        case 91: return launch_tb_t<R, T, 91>(src, L, a, grid, s);
        case 92: return launch_tb_t<R, T, 92>(src, L, a, grid, s);
        case 93: return launch_tb_t<R, T, 93>(src, L, a, grid, s);
        case 94: return launch_tb_t<R, T, 94>(src, L, a, grid, s);
        case 95: return launch_tb_t<R, T, 95>(src, L, a, grid, s);
        case 96: return launch_tb_t<R, T, 96>(src, L, a, grid, s);
        case 97: return launch_tb_t<R, T, 97>(src, L, a, grid, s);
        case 98: return launch_tb_t<R, T, 98>(src, L, a, grid, s);
        case 99: return launch_tb_t<R, T, 99>(src, L, a, grid, s);
        case 100: return launch_tb_t<R, T, 100>(src, L, a, grid, s);
        case 101: return launch_tb_t<R, T, 101>(src, L, a, grid, s);
        case 102: return launch_tb_t<R, T, 102>(src, L, a, grid, s);
        case 103: return launch_tb_t<R, T, 103>(src, L, a, grid, s);
        case 104: return launch_tb_t<R, T, 104>(src, L, a, grid, s);
        case 105: return launch_tb_t<R, T, 105>(src, L, a, grid, s);
        case 106: return launch_tb_t<R, T, 106>(src, L, a, grid, s);
        case 107: return launch_tb_t<R, T, 107>(src, L, a, grid, s);
        case 108: return launch_tb_t<R, T, 108>(src, L, a, grid, s);
        case 109: return launch_tb_t<R, T, 109>(src, L, a, grid, s);
        case 110: return launch_tb_t<R, T, 110>(src, L, a, grid, s);
        case 111: return launch_tb_t<R, T, 111>(src, L, a, grid, s);
        case 112: return launch_tb_t<R, T, 112>(src, L, a, grid, s);
        case 113: return launch_tb_t<R, T, 113>(src, L, a, grid, s);
        case 114: return launch_tb_t<R, T, 114>(src, L, a, grid, s);
        case 115: return launch_tb_t<R, T, 115>(src, L, a, grid, s);
        case 116: return launch_tb_t<R, T, 116>(src, L, a, grid, s);
        case 117: return launch_tb_t<R, T, 117>(src, L, a, grid, s);
        case 118: return launch_tb_t<R, T, 118>(src, L, a, grid, s);
        case 119: return launch_tb_t<R, T, 119>(src, L, a, grid, s);
        case 120: return launch_tb_t<R, T, 120>(src, L, a, grid, s);
        case 121: return launch_tb_t<R, T, 121>(src, L, a, grid, s);
        case 122: return launch_tb_t<R, T, 122>(src, L, a, grid, s);
        case 123: return launch_tb_t<R, T, 123>(src, L, a, grid, s);
        case 124: return launch_tb_t<R, T, 124>(src, L, a, grid, s);
        case 125: return launch_tb_t<R, T, 125>(src, L, a, grid, s);
        case 126: return launch_tb_t<R, T, 126>(src, L, a, grid, s);
        case 127: return launch_tb_t<R, T, 127>(src, L, a, grid, s);
        case 128: return launch_tb_t<R, T, 128>(src, L, a, grid, s);
        case 129: return launch_tb_t<R, T, 129>(src, L, a, grid, s);
        case 130: return launch_tb_t<R, T, 130>(src, L, a, grid, s);
        default: return launch_tb_t<R, T, 131>(src, L, a, grid, s);
    }
}

// Peer-store launches (boundary slabs of a z-slab rank: h planes each, stored a second time
// into the z neighbours' ghost planes) run the depth's default kernel where that is a
// tensor-memory kernel, the fallback tb_kernel variant 0 otherwise.
constexpr int kPeerF64[9] = {0, 0, 0, 89, 130, 110, 112, 112, 112};
constexpr int kPeerF32[9] = {0, 0, 0, 0, 92, 92, 121, 121, 111};
template <typename R, int T>
constexpr int peer_variant() {
    if constexpr (sizeof(R) == 8) return kPeerF64[T];
    else return kPeerF32[T];
}

// In-place passes (compressed storage) are separate instantiations with the
// in-place hooks (keeping their registers out of the two-grid kernels).  The
// per-unit chunk wait costs registers, so they use shapes with headroom: the
// two-grid defaults that sit at the register cap (fp64 T=2 at two CTAs/SM,
// T=3 12x3, T=4 8x4/3, fp32 T=2) would spill.  fp64 T=2,3: 8x4/3 with one
// __syncthreads per step (measured: 562 / 524-538 GLUP/s against 457 / 512
// for 16x2/3 and 8x4/2 with the split barrier; at T=4 it spills: 355 vs 507).
// Since the tensor-memory kernels (tq_kernel) the deeper in-place passes run on their FQ
// forms, whose step body is not register-critical (the hooks cost nothing there).
#ifndef SP_INPL64_T2
#define SP_INPL64_T2 13
#endif
#ifndef SP_INPL64_T3
#define SP_INPL64_T3 111  // FQ 8x8 (round 2, 12x3/2 hoisted: 603 / 620 GLUP/s at chunk 64 / 128)
#endif
#ifndef SP_INPL64_T4
#define SP_INPL64_T4 123  // FQ 12x5 (round 2, 8x4/2: 512)
#endif
constexpr int kInplaceF64[9] = {0, 5, SP_INPL64_T2, SP_INPL64_T3, SP_INPL64_T4, 110, 112, 112, 112};
constexpr int kInplaceF32[9] = {0, 14, 4, 22, 92, 92, 121, 121, 111};

template <typename R, int T>
constexpr int inplace_variant() {
    if constexpr (sizeof(R) == 8) return kInplaceF64[T];
    else return kInplaceF32[T];
}

// One entry per (dtype, T), explicitly instantiated in its own unit:
// kind 0 = the variant table (v), 1 = peer-store boundary pass, 2 = in place.
template <typename R, int T>
int launch_kind(int kind, int v, const void* src, const sp_layout* L, const sp::TBArgs& a, int grid,
                cudaStream_t s) {
    if (kind == 1) return launch_tb_t<R, T, peer_variant<R, T>(), true>(src, L, a, grid, s);
    if (kind == 2) return launch_tb_t<R, T, inplace_variant<R, T>(), false, true>(src, L, a, grid, s);
    return launch_variant<R, T>(v, src, L, a, grid, s);
}

#define SP_LAUNCH_KIND_SIG(R, T)                                                                    \
    int launch_kind<R, T>(int, int, const void*, const sp_layout*, const sp::TBArgs&, int, cudaStream_t)
#define SP_FOR_EACH_RT(X) \
    X(double, 1) X(double, 2) X(double, 3) X(double, 4) X(double, 5) X(double, 6) X(double, 7) X(double, 8) \
    X(float, 1) X(float, 2) X(float, 3) X(float, 4) X(float, 5) X(float, 6) X(float, 7) X(float, 8)
#ifndef SP_INST_UNIT
#define SP_EXTERN_RT(R, T) extern template SP_LAUNCH_KIND_SIG(R, T);
SP_FOR_EACH_RT(SP_EXTERN_RT)
#undef SP_EXTERN_RT
#endif

}  // namespace spi
