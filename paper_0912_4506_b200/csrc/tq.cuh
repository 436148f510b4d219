// tq.cuh -- K2 with the z-queue's older plane in TENSOR MEMORY (`tq_kernel`),
// included by jacobi_kernels.cuh inside namespace sp.
//
// tb_kernel is bound by two things on B200 (ncu, profiles/r02_tuning.md): the
// register file (two planes x T levels of z-queue per cell cap the footprint
// at 8 fp64 cells per thread) and the LSU data pipe that carries SHFL, LDS and
// STS (60-65 % busy at two warps per scheduler; the y-edge exchange costs as
// many wavefronts per thread whatever the patch height).  Tensor memory is a
// second 256 KB per-SM store that a warp reaches lane-for-lane
// (tcgen05.ld/st .32x32b: thread i <-> TMEM lane i) on its own datapath, not
// the LSU pipe.  This kernel keeps v[p-1] of every level there:
//
//   registers  C[ph][l]   = v[p] of level l (ph = step parity), the plane
//                           computed this step lands in C[ph^1][l]: no moves
//   TMEM       M[l]       = v[p-1] of level l: loaded once per step right
//                           before level l+1's z sum, overwritten with v[p]
//                           right after it
//
// so the register state is (T+1) planes instead of 2T+1 and a thread can own
// a taller patch (fp64 T=4: 12 cells instead of 8 -> 64x48 footprints, 1.37
// instead of 1.52 cell-levels per output, and a third fewer y-edge
// wavefronts per cell-level).  Level planes are kept as edge rows only (two
// per warp and level, double-buffered by step parity).
//
// Wavefront, arithmetic, summation order and the Dirichlet/domain rule are
// tb_kernel's (level t trails level t-1 by one plane; bit-identical results).
// No cluster forms; in-place (INPL) and peer-store (PEER) passes as tb_kernel.
// (R/pipeline.py:395-408 is the reference's per-block level loop.)

#define SP_TM_R4(r, o) "=r"(r[o]), "=r"(r[o + 1]), "=r"(r[o + 2]), "=r"(r[o + 3])
#define SP_TM_W4(r, o) "r"(r[o]), "r"(r[o + 1]), "r"(r[o + 2]), "r"(r[o + 3])
#define SP_TM_P4(r, o) "+r"(r[o]), "+r"(r[o + 1]), "+r"(r[o + 2]), "+r"(r[o + 3])

__device__ __forceinline__ void tm_ld2(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a));
}
__device__ __forceinline__ void tm_st2(uint32_t a, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(a), "r"(r[0]), "r"(r[1]) : "memory");
}
__device__ __forceinline__ void tm_ld4(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : SP_TM_R4(r, 0) : "r"(a));
}
__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : SP_TM_R4(r, 0), SP_TM_R4(r, 4)
                 : "r"(a));
}
__device__ __forceinline__ void tm_ld16(uint32_t a, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : SP_TM_R4(r, 0), SP_TM_R4(r, 4), SP_TM_R4(r, 8), SP_TM_R4(r, 12)
        : "r"(a));
}
__device__ __forceinline__ void tm_st4(uint32_t a, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), SP_TM_W4(r, 0) : "memory");
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
                 SP_TM_W4(r, 0), SP_TM_W4(r, 4)
                 : "memory");
}
__device__ __forceinline__ void tm_st16(uint32_t a, const uint32_t* r) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
        SP_TM_W4(r, 0), SP_TM_W4(r, 4), SP_TM_W4(r, 8), SP_TM_W4(r, 12)
        : "memory");
}
// N 32-bit columns per lane, in pieces of 16 / 8 / 4
template <int N>
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t* r) {
    static_assert(N % 2 == 0, "TMEM pieces of 2 columns");
    if constexpr (N >= 16) { tm_ld16(a, r); tm_ld<N - 16>(a + 16, r + 16); }
    else if constexpr (N >= 8) { tm_ld8(a, r); tm_ld<N - 8>(a + 8, r + 8); }
    else if constexpr (N >= 4) { tm_ld4(a, r); tm_ld<N - 4>(a + 4, r + 4); }
    else if constexpr (N >= 2) { tm_ld2(a, r); }
}
template <int N>
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t* r) {
    if constexpr (N >= 16) { tm_st16(a, r); tm_st<N - 16>(a + 16, r + 16); }
    else if constexpr (N >= 8) { tm_st8(a, r); tm_st<N - 8>(a + 8, r + 8); }
    else if constexpr (N >= 4) { tm_st4(a, r); tm_st<N - 4>(a + 4, r + 4); }
    else if constexpr (N >= 2) { tm_st2(a, r); }
}
// tcgen05.wait::ld with the loaded registers as in/out operands: every use of
// them depends on the wait (the compiler may not hoist a use above it)
template <int N>
__device__ __forceinline__ void tm_dep(uint32_t* r) {
    if constexpr (N >= 16) {
        asm volatile("" : SP_TM_P4(r, 0), SP_TM_P4(r, 4), SP_TM_P4(r, 8), SP_TM_P4(r, 12));
        tm_dep<N - 16>(r + 16);
    } else if constexpr (N >= 8) {
        asm volatile("" : SP_TM_P4(r, 0), SP_TM_P4(r, 4));
        tm_dep<N - 8>(r + 8);
    } else if constexpr (N >= 4) {
        asm volatile("" : SP_TM_P4(r, 0));
        tm_dep<N - 4>(r + 4);
    } else if constexpr (N >= 2) {
        asm volatile("" : "+r"(r[0]), "+r"(r[1]));
    }
}
template <int N>
__device__ __forceinline__ void tm_wait_ld(uint32_t* r) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    tm_dep<N>(r);
}
__device__ __forceinline__ void tm_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

template <typename R> struct TmPack;
template <> struct TmPack<double> {
    static constexpr int W = 2;
    __device__ static __forceinline__ void put(uint32_t* r, double v) {
        r[0] = (uint32_t)__double2loint(v);
        r[1] = (uint32_t)__double2hiint(v);
    }
    __device__ static __forceinline__ double get(const uint32_t* r) { return __hiloint2double((int)r[1], (int)r[0]); }
};
template <> struct TmPack<float> {
    static constexpr int W = 1;
    __device__ static __forceinline__ void put(uint32_t* r, float v) { r[0] = __float_as_uint(v); }
    __device__ static __forceinline__ float get(const uint32_t* r) { return __uint_as_float(r[0]); }
};

// FQ: both older planes of every level in TMEM (no z-queue registers at all)
template <typename R, int T, int BY, int PY, int RCAP, int FQ = 0>
struct PlanQ {
    static_assert(T >= 2 && T * PY <= 64 && T * PX <= 32, "domain bitmasks too narrow");
    static constexpr int WY = BY * PY;
    static constexpr int NT = 32 * BY;
    static constexpr int PLANE = WX * WY;
    static constexpr int PLANE_BYTES = PLANE * (int)sizeof(R);
    static constexpr int RROWS = WY;
    static constexpr int RPLANE_BYTES = PLANE_BYTES;
    static constexpr int EDGE = 2 * BY * WX;              // a level plane's edge rows: 2 per warp
    static constexpr int EDGE_BYTES = EDGE * (int)sizeof(R);
    static constexpr int NL = T - 1;                      // levels with edge buffers (1..T-1)
    static constexpr int NR = PY * PX * (int)sizeof(R) / 4;   // TMEM columns per level and thread
    static constexpr int GROUPS = (BY + 3) / 4;           // warps w, w+4, .. share TMEM lanes
    static constexpr int GCOLS = (FQ ? 2 : 1) * T * NR;   // per warp: M[T][NR] (FQ: [T][2][NR])
    static constexpr int COLS = GROUPS * GCOLS;
    // tcgen05.alloc takes a power of two >= 32 columns
    static constexpr int ALLOC = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
    static constexpr int BUDGET = 232448 - 512;
    static constexpr int RING_FIT = (BUDGET - 2 * NL * EDGE_BYTES) / PLANE_BYTES;
    static constexpr int RING = RING_FIT > RCAP ? RCAP : RING_FIT;
    static constexpr bool FITS = RING >= 3 && WY - 2 * T >= 1 && COLS <= 512 && NR % 2 == 0;
    static constexpr int NUID = 16;
    static constexpr size_t SMEM = (size_t)RING * PLANE_BYTES + (size_t)2 * NL * EDGE_BYTES + (RING + 2) * 8 +
                                   NUID * 4 + 16;
};

// HOIST bit 0: level 1's xy sums before the TMA wait; bit 1 (tq form): the deeper levels'
// right after the step barrier (independent chains ahead of the level loop); bit 2 (FQ form,
// FAST steps): the next level's v[p] load is issued after this level's xy sums.
// SG: columns per tcgen05.st (0 = one wide store per level).  FQ: see PlanQ.
// INPL: in-place pass of compressed storage (tb_kernel's hooks: chunk order, z shift of the
// stores, per-chunk completion counters; TBArgs::cdone).  PEER: boundary-slab pass of a z-slab
// rank that also stores its planes into the neighbours' ghost planes.
template <typename R, int T, int BY, int PY, int RCAP, int HOIST, int SG = 0, int FQ = 0, bool INPL = false,
          bool PEER = false>
__global__ void __launch_bounds__(32 * BY, 1)
    tq_kernel(const __grid_constant__ CUtensorMap tmap, const TBArgs a) {
    using A = Arith<R>;
    using V2 = typename A::V2;
    using P = PlanQ<R, T, BY, PY, RCAP, FQ>;
    using TP = TmPack<R>;
    constexpr int WY = P::WY;
    constexpr int PLANE = P::PLANE;
    constexpr int RING_N = P::RING;
    constexpr int NR = P::NR;
    constexpr bool PACK = sizeof(R) == 4;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    R* ring = reinterpret_cast<R*>(smem_raw);
    R* edge = ring + RING_N * PLANE;                       // [buf 0..1][level 1..T-1][2*BY rows][WX]
    uint64_t* full = reinterpret_cast<uint64_t*>(edge + 2 * P::NL * P::EDGE);
    uint64_t* lbar = full + RING_N;                        // [2]: step k complete in every warp, k mod 2
    volatile int* uid = reinterpret_cast<volatile int*>(lbar + 2);
    uint32_t* tbase = const_cast<uint32_t*>(reinterpret_cast<volatile uint32_t*>(uid + P::NUID));

    const int lane = threadIdx.x & 31;
    const int wy = threadIdx.x >> 5;
    const int cx = lane * PX;
    const int cy = wy * PY;
    const int cym = max(cy - 1, 0);
    const int cyp = min(cy + PY, WY - 1);
    constexpr uint32_t kRingBytes = P::RPLANE_BYTES;

    if (wy == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase)),
                     "n"(P::ALLOC)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < RING_N; ++i) mbar_init(&full[i], 1);
        for (int i = 0; i < 2; ++i) mbar_init(&lbar[i], BY);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this thread's TMEM lane and first column: M[l] at tm + l * NR
    // (read through lane 0: the compiler then knows the address is warp-uniform and keeps it in a
    // uniform register instead of converting it before every tcgen05.ld/st)
#ifndef SP_TM_NOUNIFORM
    const uint32_t tm = __shfl_sync(0xffffffffu,
                                    *tbase + ((uint32_t)(32 * (wy & 3)) << 16) + (uint32_t)((wy >> 2) * P::GCOLS), 0);
#else   // A/B builds
    const uint32_t tm = *tbase + ((uint32_t)(32 * (wy & 3)) << 16) + (uint32_t)((wy >> 2) * P::GCOLS);
#endif

    // producer (thread 0): as in tb_kernel
    int pu = -1, pseq = 0, pc0 = 0, pc1 = 0, pc2 = 0, pc2_end = 0;
    bool pdone = false;
    auto producer_unit = [&]() {
        if (a.sched) {
            pu = (int)atomicAdd(a.sched, 1u);
            if (pu == a.units + (int)gridDim.x - 1) atomicExch(a.sched, 0u);
        } else {
            pu = pseq == 0 ? (int)blockIdx.x : pu + (int)gridDim.x;
        }
        uid[pseq++ & (P::NUID - 1)] = pu < a.units ? pu : -1;
        if (pu >= a.units) return;
        const Unit pw = decode_unit<INPL>(a, pu);
        pc0 = footprint_x<R>(a, pw.x0, T) + a.x_off;
        pc1 = pw.y0 - T + a.gy;
        pc2 = pw.zc0 - T + a.gz;
        pc2_end = pw.zc1 + T + a.gz;
    };
    auto produce = [&](int slot) {
        if (pu >= a.units) {
            if (!pdone) mbar_arrive(&full[slot]);
            pdone = true;
            return;
        }
        mbar_expect_tx(&full[slot], kRingBytes);
        tma_load_3d(ring + slot * PLANE, &tmap, &full[slot], pc0, pc1, pc2);
        if (++pc2 == pc2_end) producer_unit();
    };
    if (threadIdx.x == 0) {
        producer_unit();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (int i = 0; i < RING_N - 1; ++i) produce(i);
    }
    if constexpr (INPL) {   // the first unit's dependencies (see the end of the unit loop)
        if (threadIdx.x == 0 && uid[0] >= 0) wait_chunks_read(a, decode_unit<INPL>(a, uid[0]).c);
    }
    __syncwarp();

    const R sixth = A::sixth();
    uint32_t gstep = 0;

    // v[p] of levels 0..T-1 by step parity (see the header); garbage until a
    // unit's pipeline has filled, like every value derived from it
    R C[FQ ? 1 : 2][FQ ? 1 : T][PY][PX];
#pragma unroll
    for (int f = 0; f < (FQ ? 1 : 2); ++f)
#pragma unroll
        for (int t = 0; t < (FQ ? 1 : T); ++t)
#pragma unroll
            for (int j = 0; j < PY; ++j)
#pragma unroll
                for (int i = 0; i < PX; ++i) C[f][t][j][i] = R(0);
    {
        uint32_t z[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) z[i] = 0u;
#pragma unroll
        for (int t = 0; t < (FQ ? 2 : 1) * T; ++t) tm_st<NR>(tm + t * NR, z);
        tm_wait_st();
    }

    for (int cseq = 0;; ++cseq) {
        mbar_wait(&full[gstep % RING_N], (gstep / RING_N) & 1);
        const int u = uid[cseq & (P::NUID - 1)];
        if (u < 0) break;
        const Unit w = decode_unit<INPL>(a, u);
        const int fx = footprint_x<R>(a, w.x0, T), fy = w.y0 - T;
        const int nsteps = (w.zc1 - w.zc0) + 2 * T;

        uint32_t xin = 0;
        uint64_t yin = 0;
        uint32_t fastm = 0;
#pragma unroll
        for (int t = 1; t <= T; ++t) {
            const int ext = T - t;
            int xl = a.lo[2] - a.elo[2] * ext, xh = a.hi[2] + a.ehi[2] * ext;
            int yl = a.lo[1] - a.elo[1] * ext, yh = a.hi[1] + a.ehi[1] * ext;
            bool all = true;
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                int gx = fx + cx + i;
                bool in = gx >= xl && gx < xh;
                all &= in;
                if (in) xin |= 1u << ((t - 1) * PX + i);
            }
#pragma unroll
            for (int j = 0; j < PY; ++j) {
                int gyy = fy + cy + j;
                bool in = gyy >= yl && gyy < yh;
                all &= in;
                if (in) yin |= 1ull << ((t - 1) * PY + j);
            }
            if (__all_sync(0xffffffffu, all)) fastm |= 1u << (t - 1);
        }
        uint32_t wx = 0, wyb = 0;
#pragma unroll
        for (int i = 0; i < PX; ++i) {
            int gx = fx + cx + i;
            wx |= (gx >= w.x0 && gx < min(w.x0 + a.ox, a.ohi[2]) ? 1u : 0u) << i;
        }
#pragma unroll
        for (int j = 0; j < PY; ++j) {
            int gyy = fy + cy + j;
            wyb |= (gyy >= w.y0 && gyy < min(w.y0 + a.oy, a.ohi[1]) ? 1u : 0u) << j;
        }
        R* dcol = reinterpret_cast<R*>(a.dst) + a.origin + (int64_t)(fy + cy) * a.py + (fx + cx);
        const int64_t pz = a.pz, py = a.py;
        // plane q-T of step 0 (INPL: level-T plane p goes to plane p + zshift)
        R* dnext = dcol + (int64_t)(w.zc0 - 2 * T + (INPL ? a.zshift : 0)) * pz;
        const bool vec_store = wx == 3u && ((reinterpret_cast<uintptr_t>(dcol) & (sizeof(V2) - 1)) == 0);
        const bool full_rows = vec_store && wyb == (1u << PY) - 1u;

        // level T: the finished plane p (16-byte streaming stores; lanes outside the tile's
        // columns skip the block).  PEER: planes of the slab's halo depth also go into the z
        // neighbours' ghost planes (peer memory; TBArgs::rd_lo/rd_hi, as tb_kernel)
        auto store_plane = [&](const R(&out)[PY][PX], int p) __attribute__((always_inline)) {
            auto put = [&](R* b) __attribute__((always_inline)) {
                if (full_rows) {
#pragma unroll
                    for (int j = 0; j < PY; ++j) __stcs(reinterpret_cast<V2*>(b + j * py), V2{out[j][0], out[j][1]});
                } else if (vec_store) {
#pragma unroll
                    for (int j = 0; j < PY; ++j)
                        if ((wyb >> j) & 1u) __stcs(reinterpret_cast<V2*>(b + j * py), V2{out[j][0], out[j][1]});
                } else if (wx != 0u) {
#pragma unroll
                    for (int j = 0; j < PY; ++j) {
                        const bool row = (wyb >> j) & 1u;
                        if (row && (wx & 1u)) __stcs(b + j * py, out[j][0]);
                        if (row && (wx & 2u)) __stcs(b + j * py + 1, out[j][1]);
                    }
                }
            };
            put(dnext);
            if constexpr (PEER) {
                if (p < a.rz_lo) put(dnext + a.rd_lo);
                if (p >= a.rz_hi) put(dnext + a.rd_hi);
            }
        };
        auto step = [&](auto phase, auto fast, int st) __attribute__((always_inline)) {
            constexpr int PH = decltype(phase)::value;
            constexpr bool FAST = decltype(fast)::value;
            const int slot = gstep % RING_N;
            const int pslot = (gstep + RING_N - 1) % RING_N;
            const int pslot2 = (gstep + RING_N - 2) % RING_N;
            const int cur = (int)(gstep & 1u), prv = cur ^ 1;
            const int q = w.zc0 - T + st;

            R s[T][PY][PX];
            // s_t = (x- + x+) + (y- + y+) of level t-1 at plane q-t (C[PH][t-1])
            auto xy_sums = [&](int t) __attribute__((always_inline)) {
                const R(&v)[PY][PX] = C[PH][t - 1];
                V2 up, dn;
                if (t == 1) {
                    const R* Pl = ring + pslot * PLANE;
                    up = *reinterpret_cast<const V2*>(Pl + cym * WX + cx);
                    dn = *reinterpret_cast<const V2*>(Pl + cyp * WX + cx);
                } else {
                    // warp w's first row is edge row 2w, its last row 2w+1 (footprint
                    // edges: any value, those cells are halo)
                    const R* E = edge + (prv * P::NL + (t - 2)) * P::EDGE;
                    const int ru = wy > 0 ? 2 * wy - 1 : 0, rd = wy < BY - 1 ? 2 * wy + 2 : 2 * wy + 1;
                    up = *reinterpret_cast<const V2*>(E + ru * WX + cx);
                    dn = *reinterpret_cast<const V2*>(E + rd * WX + cx);
                }
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    R lft = __shfl_up_sync(0xffffffffu, v[j][1], 1);
                    R rgt = __shfl_down_sync(0xffffffffu, v[j][0], 1);
                    R ym0 = (j == 0) ? up.x : v[j > 0 ? j - 1 : 0][0];
                    R ym1 = (j == 0) ? up.y : v[j > 0 ? j - 1 : 0][1];
                    R yp0 = (j == PY - 1) ? dn.x : v[j + 1 < PY ? j + 1 : j][0];
                    R yp1 = (j == PY - 1) ? dn.y : v[j + 1 < PY ? j + 1 : j][1];
                    if constexpr (!PACK) {
                        s[t - 1][j][0] = A::add(A::add(lft, v[j][1]), A::add(ym0, yp0));
                        s[t - 1][j][1] = A::add(A::add(v[j][0], rgt), A::add(ym1, yp1));
                    } else {
                        R x0 = A::add(lft, v[j][1]), x1 = A::add(v[j][0], rgt), y0, y1;
                        A::add2(y0, y1, ym0, ym1, yp0, yp1);
                        A::add2(s[t - 1][j][0], s[t - 1][j][1], x0, x1, y0, y1);
                    }
                }
            };

            uint32_t raw[NR];
            tm_wait_st();                    // the previous step's M[] stores
            tm_ld<NR>(tm, raw);              // M[0]: level 0 at plane q-2
            if constexpr (HOIST & 1) xy_sums(1);
            mbar_wait(&full[slot], (gstep / RING_N) & 1);
            {
                const R* L0 = ring + slot * PLANE;
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    V2 r = *reinterpret_cast<const V2*>(L0 + (cy + j) * WX + cx);
                    C[PH ^ 1][0][j][0] = r.x;
                    C[PH ^ 1][0][j][1] = r.y;
                }
            }
            R out[PY][PX];
#pragma unroll
            for (int t = 1; t <= T; ++t) {
                const R(&cc)[PY][PX] = C[PH][t - 1];
                const R(&nn)[PY][PX] = C[PH ^ 1][t - 1];
                R(&dst)[PY][PX] = (t < T) ? C[PH ^ 1][t < T ? t : 0] : out;
                // z- + z+ as soon as M[t-1] has landed, then the next level's load
                R zs[PY][PX];
                tm_wait_ld<NR>(raw);
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    if constexpr (!PACK) {
#pragma unroll
                        for (int i = 0; i < PX; ++i)
                            zs[j][i] = A::add(TP::get(raw + (j * PX + i) * TP::W), nn[j][i]);
                    } else {
                        A::add2(zs[j][0], zs[j][1], TP::get(raw + (j * PX) * TP::W),
                                TP::get(raw + (j * PX + 1) * TP::W), nn[j][0], nn[j][1]);
                    }
                }
                if (t < T) tm_ld<NR>(tm + t * NR, raw);
                if (t == 1 ? !(HOIST & 1) : !(HOIST & 2)) xy_sums(t);
                uint32_t inm = 0;
                if constexpr (!FAST) {
                    const int p = q - t;
                    const int ext = T - t;
                    const bool zin = p >= a.lo[0] - a.elo[0] * ext && p < a.hi[0] + a.ehi[0] * ext;
                    const uint32_t xb = (xin >> ((t - 1) * PX)) & ((1u << PX) - 1);
                    const uint32_t yb = (uint32_t)(yin >> ((t - 1) * PY)) & ((1u << PY) - 1);
#pragma unroll
                    for (int j = 0; j < PY; ++j)
                        if (zin && ((yb >> j) & 1u)) inm |= xb << (j * PX);
                }
                // v[p] of level t-1 becomes its v[p-1]
                {
                    uint32_t wr[NR];
#pragma unroll
                    for (int j = 0; j < PY; ++j)
#pragma unroll
                        for (int i = 0; i < PX; ++i) TP::put(wr + (j * PX + i) * TP::W, cc[j][i]);
                    // SG columns per tcgen05.st: a wide store wants its sources in consecutive
                    // registers and ptxas gathers them with one move per register; SG = 2 stores
                    // each fp64 value from its own register pair
                    if constexpr (SG == 0 || NR % (SG ? SG : 1) != 0) {
                        tm_st<NR>(tm + (t - 1) * NR, wr);
                    } else {
#pragma unroll
                        for (int c = 0; c < NR; c += SG) tm_st<SG>(tm + (t - 1) * NR + c, wr + c);
                    }
                }
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    R ups[PX];
                    if constexpr (!PACK) {
#pragma unroll
                        for (int i = 0; i < PX; ++i) ups[i] = A::mul(A::add(s[t - 1][j][i], zs[j][i]), sixth);
                    } else {
                        R us[PX];
                        A::add2(us[0], us[1], s[t - 1][j][0], s[t - 1][j][1], zs[j][0], zs[j][1]);
                        A::mul2(ups[0], ups[1], us[0], us[1], sixth);
                    }
#pragma unroll
                    for (int i = 0; i < PX; ++i) {
                        if constexpr (FAST) dst[j][i] = ups[i];
                        else dst[j][i] = ((inm >> (j * PX + i)) & 1u) ? ups[i] : cc[j][i];
                    }
                }
                if (t == 1 && gstep > 0) {
                    // step k-1 is complete in every warp: its edge rows are visible, its
                    // reads of buffer `cur` and of ring plane q-2 are done
                    const uint32_t k1 = gstep - 1;
                    mbar_wait(&lbar[k1 & 1u], (k1 >> 1) & 1u);
                    if (threadIdx.x == 0) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        produce(pslot2);
                    }
                    __syncwarp();
                }
                if constexpr (HOIST & 2) {
                    if (t == 1) {
#pragma unroll
                        for (int tt = 2; tt <= T; ++tt) xy_sums(tt);
                    }
                }
                if (t < T) {
                    R* E = edge + (cur * P::NL + (t - 1)) * P::EDGE;
                    *reinterpret_cast<V2*>(E + (2 * wy) * WX + cx) = V2{dst[0][0], dst[0][1]};
                    *reinterpret_cast<V2*>(E + (2 * wy + 1) * WX + cx) = V2{dst[PY - 1][0], dst[PY - 1][1]};
                }
            }
            if (st >= 2 * T) store_plane(out, q - T);
            dnext += pz;
            __syncwarp();
            if (lane == 0) mbar_arrive(&lbar[gstep & 1u]);
            __syncwarp();
            ++gstep;
        };
        // FQ: one step with every level's v[p-1] and v[p] in TMEM.  Level l's planes live in
        // two TMEM slots that swap roles with the (unit-local) step parity: `sm` holds plane
        // k-2 and receives the plane computed this step, `sc` holds plane k-1.  No register
        // carries a value from one step to the next.
        auto stepf = [&](auto fast, int st) __attribute__((always_inline)) {
            constexpr bool FAST = decltype(fast)::value;
            constexpr bool LATEC = FAST && (HOIST & 4);   // HOIST bit 2: see the loads below
            const int slot = gstep % RING_N;
            const int pslot = (gstep + RING_N - 1) % RING_N;
            const int pslot2 = (gstep + RING_N - 2) % RING_N;
            const int cur = (int)(gstep & 1u), prv = cur ^ 1;
            const int q = w.zc0 - T + st;
            const uint32_t sm = (uint32_t)(st & 1) * NR, sc = NR - sm;
            uint32_t rm[NR], rc[NR];
            tm_wait_st();                    // the previous step's stores
            tm_ld<NR>(tm + sm, rm);
            tm_ld<NR>(tm + sc, rc);
            R lv[T + 1][PY][PX];             // lv[t]: the plane of level t computed this step
            // this step's level-0 plane: wait for its TMA, load own rows
            auto load_l0 = [&]() __attribute__((always_inline)) {
                mbar_wait(&full[slot], (gstep / RING_N) & 1);
                const R* L0 = ring + slot * PLANE;
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    V2 r = *reinterpret_cast<const V2*>(L0 + (cy + j) * WX + cx);
                    lv[0][j][0] = r.x;
                    lv[0][j][1] = r.y;
                }
            };
            if constexpr (!(HOIST & 1)) load_l0();
#pragma unroll
            for (int t = 1; t <= T; ++t) {
                const R(&nn)[PY][PX] = lv[t - 1];
                R(&dst)[PY][PX] = lv[t];
                R cc[PY][PX], zs[PY][PX], sxy[PY][PX];
                tm_wait_ld<NR>(rm);
                tm_dep<NR>(rc);
                // HOIST bit 0: level 1's xy sums (level 0 at plane q-1: TMEM + the ring) before
                // waiting for this step's TMA plane
                const bool early = (HOIST & 1) && t == 1;
                auto xy = [&]() __attribute__((always_inline)) {
                    V2 up, dn;
                    if (t == 1) {
                        const R* Pl = ring + pslot * PLANE;
                        up = *reinterpret_cast<const V2*>(Pl + cym * WX + cx);
                        dn = *reinterpret_cast<const V2*>(Pl + cyp * WX + cx);
                    } else {
                        const R* E = edge + (prv * P::NL + (t - 2)) * P::EDGE;
                        const int ru = wy > 0 ? 2 * wy - 1 : 0, rd = wy < BY - 1 ? 2 * wy + 2 : 2 * wy + 1;
                        up = *reinterpret_cast<const V2*>(E + ru * WX + cx);
                        dn = *reinterpret_cast<const V2*>(E + rd * WX + cx);
                    }
#pragma unroll
                    for (int j = 0; j < PY; ++j) {
                        R lft = __shfl_up_sync(0xffffffffu, cc[j][1], 1);
                        R rgt = __shfl_down_sync(0xffffffffu, cc[j][0], 1);
                        R ym0 = (j == 0) ? up.x : cc[j > 0 ? j - 1 : 0][0];
                        R ym1 = (j == 0) ? up.y : cc[j > 0 ? j - 1 : 0][1];
                        R yp0 = (j == PY - 1) ? dn.x : cc[j + 1 < PY ? j + 1 : j][0];
                        R yp1 = (j == PY - 1) ? dn.y : cc[j + 1 < PY ? j + 1 : j][1];
                        if constexpr (!PACK) {
                            sxy[j][0] = A::add(A::add(lft, cc[j][1]), A::add(ym0, yp0));
                            sxy[j][1] = A::add(A::add(cc[j][0], rgt), A::add(ym1, yp1));
                        } else {
                            R x0 = A::add(lft, cc[j][1]), x1 = A::add(cc[j][0], rgt), y0, y1;
                            A::add2(y0, y1, ym0, ym1, yp0, yp1);
                            A::add2(sxy[j][0], sxy[j][1], x0, x1, y0, y1);
                        }
                    }
                };
                if (early) {
#pragma unroll
                    for (int j = 0; j < PY; ++j)
#pragma unroll
                        for (int i = 0; i < PX; ++i) cc[j][i] = TP::get(rc + (j * PX + i) * TP::W);
                    xy();
                    load_l0();
                }
                // level t-1's new plane replaces its v[p-1] (just loaded)
                {
                    uint32_t wr[NR];
#pragma unroll
                    for (int j = 0; j < PY; ++j)
#pragma unroll
                        for (int i = 0; i < PX; ++i) TP::put(wr + (j * PX + i) * TP::W, nn[j][i]);
                    if constexpr (SG == 0 || NR % (SG ? SG : 1) != 0) {
                        tm_st<NR>(tm + (t - 1) * 2 * NR + sm, wr);
                    } else {
#pragma unroll
                        for (int c = 0; c < NR; c += SG) tm_st<SG>(tm + (t - 1) * 2 * NR + sm + c, wr + c);
                    }
                }
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    if (!early) {
#pragma unroll
                        for (int i = 0; i < PX; ++i) cc[j][i] = TP::get(rc + (j * PX + i) * TP::W);
                    }
                    if constexpr (!PACK) {
#pragma unroll
                        for (int i = 0; i < PX; ++i)
                            zs[j][i] = A::add(TP::get(rm + (j * PX + i) * TP::W), nn[j][i]);
                    } else {
                        A::add2(zs[j][0], zs[j][1], TP::get(rm + (j * PX) * TP::W),
                                TP::get(rm + (j * PX + 1) * TP::W), nn[j][0], nn[j][1]);
                    }
                }
                // next level's v[p-1] now (rm is consumed); its v[p] once the xy sums have
                // consumed this level's (LDTM wants one block of registers: loading it while
                // cc is live costs a copy per register)
                if (t < T) tm_ld<NR>(tm + t * 2 * NR + sm, rm);
                if constexpr (!LATEC) {
                    if (t < T) tm_ld<NR>(tm + t * 2 * NR + sc, rc);
                }
                if (!early) xy();
                if constexpr (LATEC) {
                    if (t < T) tm_ld<NR>(tm + t * 2 * NR + sc, rc);
                }
                uint32_t inm = 0;
                if constexpr (!FAST) {
                    const int p = q - t;
                    const int ext = T - t;
                    const bool zin = p >= a.lo[0] - a.elo[0] * ext && p < a.hi[0] + a.ehi[0] * ext;
                    const uint32_t xb = (xin >> ((t - 1) * PX)) & ((1u << PX) - 1);
                    const uint32_t yb = (uint32_t)(yin >> ((t - 1) * PY)) & ((1u << PY) - 1);
#pragma unroll
                    for (int j = 0; j < PY; ++j)
                        if (zin && ((yb >> j) & 1u)) inm |= xb << (j * PX);
                }
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    R ups[PX];
                    if constexpr (!PACK) {
                        ups[0] = A::mul(A::add(sxy[j][0], zs[j][0]), sixth);
                        ups[1] = A::mul(A::add(sxy[j][1], zs[j][1]), sixth);
                    } else {
                        R u0, u1;
                        A::add2(u0, u1, sxy[j][0], sxy[j][1], zs[j][0], zs[j][1]);
                        A::mul2(ups[0], ups[1], u0, u1, sixth);
                    }
#pragma unroll
                    for (int i = 0; i < PX; ++i) {
                        if constexpr (FAST) dst[j][i] = ups[i];
                        else dst[j][i] = ((inm >> (j * PX + i)) & 1u) ? ups[i] : cc[j][i];
                    }
                }
                if (t == 1 && gstep > 0) {
                    const uint32_t k1 = gstep - 1;
                    mbar_wait(&lbar[k1 & 1u], (k1 >> 1) & 1u);
                    if (threadIdx.x == 0) {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        produce(pslot2);
                    }
                    __syncwarp();
                }
                if (t < T) {
                    R* E = edge + (cur * P::NL + (t - 1)) * P::EDGE;
                    *reinterpret_cast<V2*>(E + (2 * wy) * WX + cx) = V2{dst[0][0], dst[0][1]};
                    *reinterpret_cast<V2*>(E + (2 * wy + 1) * WX + cx) = V2{dst[PY - 1][0], dst[PY - 1][1]};
                }
            }
            const R(&out)[PY][PX] = lv[T];
            if (st >= 2 * T) store_plane(out, q - T);
            dnext += pz;
            __syncwarp();
            if (lane == 0) mbar_arrive(&lbar[gstep & 1u]);
            __syncwarp();
            ++gstep;
        };
#ifndef SP_TQ_FORCE_SLOW
        const bool fast_xy = fastm == (1u << T) - 1u;
#else   // diagnostic builds: every step takes the SLOW (per-cell select) path
        const bool fast_xy = false;
#endif
        using I0 = std::integral_constant<int, 0>;
        using I1 = std::integral_constant<int, 1>;
        // Steps run in pairs (parities 0, 1), so only C[0] is live between pairs; a
        // pair is FAST when both its steps are (steps [fs, fe) are FAST for the whole
        // warp: every cell inside every level's domain).  An odd last step runs alone
        // and moves its new planes back into C[0].
        int fs = nsteps, fe = nsteps;
        if (fast_xy) {
            const int q0 = w.zc0 - T;
            fs = max(0, a.lo[0] + T - q0);
            fe = min(nsteps, a.hi[0] + a.ehi[0] * (T - 1) + 1 - q0);
            if (fe <= fs) fs = fe = nsteps;
        }
        int st = 0;
        if constexpr (FQ) {
            for (; st < fs; ++st) stepf(std::false_type{}, st);
            for (; st < fe; ++st) stepf(std::true_type{}, st);
            for (; st < nsteps; ++st) stepf(std::false_type{}, st);
        }
        for (; st + 2 <= nsteps; st += 2) {
            if (st >= fs && st + 2 <= fe) {
                step(I0{}, std::true_type{}, st);
                step(I1{}, std::true_type{}, st + 1);
            } else {
                step(I0{}, std::false_type{}, st);
                step(I1{}, std::false_type{}, st + 1);
            }
        }
        if (st < nsteps) {
            step(I0{}, std::false_type{}, st);
#pragma unroll
            for (int t = 0; t < T; ++t)
#pragma unroll
                for (int j = 0; j < PY; ++j)
#pragma unroll
                    for (int i = 0; i < PX; ++i) C[0][t][j][i] = C[1][t][j][i];
        }
        if constexpr (INPL) {
            if (threadIdx.x == 0) {
                // this thread consumed the unit's last plane: all its global reads (TMA) are done.
                // The next unit stores over planes chunks c-2, c-3 read: wait for them here; the
                // other warps store only after a step barrier has seen this thread's next arrival.
                asm volatile("fence.proxy.async.global;" ::: "memory");
                __threadfence();
                atomicAdd(a.cdone + w.c, 1u);
                const int nu = uid[(cseq + 1) & (P::NUID - 1)];
                if (nu >= 0) wait_chunks_read(a, decode_unit<INPL>(a, nu).c);
            }
            __syncwarp();
        }
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (wy == 0) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase), "n"(P::ALLOC) : "memory");
    }
}
