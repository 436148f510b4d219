// wave2.cuh -- K2 with a lag-2 z-wavefront (`tb2_kernel`), included by
// jacobi_kernels.cuh inside namespace sp.
//
// In tb_kernel level t trails level t-1 by ONE plane: at step q level 1
// computes plane q-1, level 2 plane q-2, ...  The z+ neighbour level t needs
// is then the plane level t-1 produced in the SAME step, so the T levels of a
// step form one dependent chain ((z- + z+) -> + s -> * 1/6, three FP64
// latencies per level, 3T per step) that no amount of warps per scheduler
// fully hides at two warps.  Here level t >= 1 trails by TWO planes:
//
//     level 1 computes plane q-1,   level t computes plane q-2t+1,
//
// so every input of every level at step q was produced in an EARLIER step and
// the T level updates of a step are independent (T-fold more ILP for the
// same registers).  Per level t-1 >= 1 the thread keeps three planes in a
// rotating register queue (z-, centre, z+: produced 3, 2 and 1 steps ago);
// the level-0 queue holds planes q-2, q-1 and the new TMA plane q.  Levels
// are processed from T down to 1, so level t-1's new plane overwrites its
// oldest slot after level t consumed it.  The y-neighbour edge rows of a
// level plane are read two steps after they were written, so the edge buffers
// are triple-buffered (step mod 3) and synchronised by three step barriers:
// reads at step k need step k-2 complete, writes need step k-1 complete --
// a warp may run almost two steps ahead of the slowest one.
//
// Arithmetic, summation order and the Dirichlet/domain rule are exactly
// tb_kernel's (bit-identical results); the z cone is unchanged (a unit still
// reads planes [zc0 - T, zc1 + T)), only the schedule differs: T - 1 extra
// drain steps per unit, without TMA planes.
// (R/pipeline.py:395-408 is the reference's per-block level loop.)

template <typename R, int T, int BY, int PY, int MINB, int RCAP>
struct Plan2 {
    static_assert(T >= 2 && T * PY <= 64 && T * PX <= 32, "lag-2 wavefront: depth 2..8");
    static constexpr int WY = BY * PY;
    static constexpr int NT = 32 * BY;
    static constexpr int PLANE = WX * WY;
    static constexpr int PLANE_BYTES = PLANE * (int)sizeof(R);
    static constexpr int RROWS = WY;
    static constexpr int RPLANE_BYTES = PLANE_BYTES;
    static constexpr int EDGE = 2 * BY * WX;              // a level plane's edge rows: 2 per warp
    static constexpr int EDGE_BYTES = EDGE * (int)sizeof(R);
    static constexpr int NL = T - 1;                      // levels with edge buffers (1..T-1)
    static constexpr int BUDGET = (MINB == 1 ? 232448 : 233472 / MINB - 1024) - 512;
    static constexpr int RING_FIT = (BUDGET - 3 * NL * EDGE_BYTES) / PLANE_BYTES;
    static constexpr int RING = RING_FIT > RCAP ? RCAP : RING_FIT;
    static constexpr bool FITS = RING >= 4 && WY - 2 * T >= 1;
    static constexpr int NUID = 16;
    static constexpr size_t SMEM = (size_t)RING * PLANE_BYTES + (size_t)3 * NL * EDGE_BYTES + (RING + 3) * 8 +
                                   NUID * 4;
};

template <typename R, int T, int BY, int PY, int MINB, int RCAP>
__global__ void __launch_bounds__(32 * BY, MINB)
    tb2_kernel(const __grid_constant__ CUtensorMap tmap, const TBArgs a) {
    using A = Arith<R>;
    using V2 = typename A::V2;
    using P = Plan2<R, T, BY, PY, MINB, RCAP>;
    constexpr int WY = P::WY;
    constexpr int PLANE = P::PLANE;
    constexpr int RING_N = P::RING;
    constexpr bool PACK = sizeof(R) == 4 && MINB == 1;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    R* ring = reinterpret_cast<R*>(smem_raw);
    R* edge = ring + RING_N * PLANE;                       // [buf 0..2][level 1..T-1][2*BY rows][WX]
    uint64_t* full = reinterpret_cast<uint64_t*>(edge + 3 * P::NL * P::EDGE);
    uint64_t* lbar = full + RING_N;                        // [3]: step k complete (all warps), k mod 3
    volatile int* uid = reinterpret_cast<volatile int*>(lbar + 3);

    const int lane = threadIdx.x & 31;
    const int wy = threadIdx.x >> 5;
    const int cx = lane * PX;
    const int cy = wy * PY;
    const int cym = max(cy - 1, 0);
    const int cyp = min(cy + PY, WY - 1);
    constexpr uint32_t kRingBytes = P::RPLANE_BYTES;

    if (threadIdx.x == 0) {
        for (int i = 0; i < RING_N; ++i) mbar_init(&full[i], 1);
        for (int i = 0; i < 3; ++i) mbar_init(&lbar[i], BY);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // producer (thread 0): as in tb_kernel -- claim units, publish ids ahead of
    // their first TMA plane, walk each unit's planes [zc0 - T, zc1 + T)
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
        const Unit pw = decode_unit(a, pu);
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
        // the slot of plane q-1 is released after step q: prime all but two
        for (int i = 0; i < RING_N - 2; ++i) produce(i);
    }

    const R sixth = A::sixth();
    uint32_t gstep = 0;    // steps so far (barrier phases)
    uint32_t gplane = 0;   // TMA planes consumed so far (ring slots)

    // register queues: Z0[3] = level 0 planes, Q[3][T-1] = levels 1..T-1
    R Z0[3][PY][PX];
    R Q[3][T - 1][PY][PX];
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int j = 0; j < PY; ++j)
#pragma unroll
            for (int i = 0; i < PX; ++i) {
                Z0[f][j][i] = R(0);
#pragma unroll
                for (int t = 0; t < T - 1; ++t) Q[f][t][j][i] = R(0);
            }

    for (int cseq = 0;; ++cseq) {
        mbar_wait(&full[gplane % RING_N], (gplane / RING_N) & 1);
        const int u = uid[cseq & (P::NUID - 1)];
        if (u < 0) break;
        const Unit w = decode_unit(a, u);
        const int fx = footprint_x<R>(a, w.x0, T), fy = w.y0 - T;
        const int nplanes = (w.zc1 - w.zc0) + 2 * T;         // TMA planes of the unit
        const int nsteps = nplanes + T - 1;                    // + drain of levels 2..T

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
        // level-T plane of step 0: (zc0 - T) - 2T + 1
        R* dnext = dcol + (int64_t)(w.zc0 - 3 * T + 1) * pz;
        const bool vec_store = wx == 3u && ((reinterpret_cast<uintptr_t>(dcol) & (sizeof(V2) - 1)) == 0);
        const bool full_rows = vec_store && wyb == (1u << PY) - 1u;
        const bool fast_xy = fastm == (1u << T) - 1u;

        // One step.  PH = step mod 3 (compile time): level-0 slots Z0[PH] = q-2,
        // Z0[PH+1] = q-1, Z0[PH+2] <- q; level l >= 1 slots Q[PH] = oldest (z- of
        // level l+1), Q[PH+1] = centre, Q[PH+2] = newest; level l's new plane goes
        // to Q[PH] once level l+1 has used it.
        auto step = [&](auto phase, auto fast, int st) {
            constexpr int PH = decltype(phase)::value;
            constexpr int F0 = PH, F1 = (PH + 1) % 3, F2 = (PH + 2) % 3;
            constexpr bool FAST = decltype(fast)::value;
            const int q = w.zc0 - T + st;              // newest level-0 plane
            const bool has_plane = st < nplanes;
            const int slot = gplane % RING_N;
            const int pslot = (gplane + RING_N - 1) % RING_N;   // plane q-1
            const uint32_t ebuf_w = gstep % 3, ebuf_r = (gstep + 1) % 3;   // k, k-2

            // step k-2 complete: its edge rows (read below) are visible
            if (gstep >= 2) {
                const uint32_t k2 = gstep - 2;
                mbar_wait(&lbar[k2 % 3], (k2 / 3) & 1);
            }

            R out[PY][PX];
            // levels T..2: from level t-1's queue (all planes of earlier steps)
#pragma unroll
            for (int t = T; t >= 1; --t) {
                const R(&zm)[PY][PX] = t == 1 ? Z0[F0] : Q[F0][t >= 2 ? t - 2 : 0];
                const R(&cc)[PY][PX] = t == 1 ? Z0[F1] : Q[F1][t >= 2 ? t - 2 : 0];
                const R(&zp)[PY][PX] = t == 1 ? Z0[F2] : Q[F2][t >= 2 ? t - 2 : 0];
                if (t == 1) {
                    if (has_plane) {
                        // the new level-0 plane q: wait for its TMA, load own rows
                        mbar_wait(&full[slot], (gplane / RING_N) & 1);
                        const R* L0 = ring + slot * PLANE;
#pragma unroll
                        for (int j = 0; j < PY; ++j) {
                            V2 r = *reinterpret_cast<const V2*>(L0 + (cy + j) * WX + cx);
                            Z0[F2][j][0] = r.x;
                            Z0[F2][j][1] = r.y;
                        }
                    }
                }
                // y-neighbour rows of the centre plane
                V2 up, dn;
                if (t == 1) {
                    const R* Pl = ring + pslot * PLANE;
                    up = *reinterpret_cast<const V2*>(Pl + cym * WX + cx);
                    dn = *reinterpret_cast<const V2*>(Pl + cyp * WX + cx);
                } else {
                    const R* E = edge + ((int)ebuf_r * P::NL + (t - 2)) * P::EDGE;
                    // warp w's first row is edge row 2w, its last row 2w+1
                    const int ru = wy > 0 ? 2 * wy - 1 : 0, rd = wy < BY - 1 ? 2 * wy + 2 : 2 * wy + 1;
                    up = wy > 0 ? *reinterpret_cast<const V2*>(E + ru * WX + cx) : V2{cc[0][0], cc[0][1]};
                    dn = wy < BY - 1 ? *reinterpret_cast<const V2*>(E + rd * WX + cx)
                                     : V2{cc[PY - 1][0], cc[PY - 1][1]};
                }
                uint32_t inm = 0;
                if constexpr (!FAST) {
                    const int p = q - 2 * t + 1;
                    const int ext = T - t;
                    const bool zin = p >= a.lo[0] - a.elo[0] * ext && p < a.hi[0] + a.ehi[0] * ext;
                    const uint32_t xb = (xin >> ((t - 1) * PX)) & ((1u << PX) - 1);
                    const uint32_t yb = (uint32_t)(yin >> ((t - 1) * PY)) & ((1u << PY) - 1);
#pragma unroll
                    for (int j = 0; j < PY; ++j)
                        if (zin && ((yb >> j) & 1u)) inm |= xb << (j * PX);
                }
                R nv[PY][PX];
#pragma unroll
                for (int j = 0; j < PY; ++j) {
                    R lft = __shfl_up_sync(0xffffffffu, cc[j][1], 1);
                    R rgt = __shfl_down_sync(0xffffffffu, cc[j][0], 1);
                    R ym0 = (j == 0) ? up.x : cc[j > 0 ? j - 1 : 0][0];
                    R ym1 = (j == 0) ? up.y : cc[j > 0 ? j - 1 : 0][1];
                    R yp0 = (j == PY - 1) ? dn.x : cc[j + 1 < PY ? j + 1 : j][0];
                    R yp1 = (j == PY - 1) ? dn.y : cc[j + 1 < PY ? j + 1 : j][1];
                    R s0, s1, ups[PX];
                    if constexpr (!PACK) {
                        s0 = A::add(A::add(lft, cc[j][1]), A::add(ym0, yp0));
                        s1 = A::add(A::add(cc[j][0], rgt), A::add(ym1, yp1));
                        ups[0] = A::mul(A::add(s0, A::add(zm[j][0], zp[j][0])), sixth);
                        ups[1] = A::mul(A::add(s1, A::add(zm[j][1], zp[j][1])), sixth);
                    } else {
                        R x0 = A::add(lft, cc[j][1]), x1 = A::add(cc[j][0], rgt), y0, y1, z0, z1, u0, u1;
                        A::add2(y0, y1, ym0, ym1, yp0, yp1);
                        A::add2(s0, s1, x0, x1, y0, y1);
                        A::add2(z0, z1, zm[j][0], zm[j][1], zp[j][0], zp[j][1]);
                        A::add2(u0, u1, s0, s1, z0, z1);
                        A::mul2(ups[0], ups[1], u0, u1, sixth);
                    }
#pragma unroll
                    for (int i = 0; i < PX; ++i) {
                        if constexpr (FAST) nv[j][i] = ups[i];
                        else nv[j][i] = ((inm >> (j * PX + i)) & 1u) ? ups[i] : cc[j][i];
                    }
                }
                if (t == T) {
#pragma unroll
                    for (int j = 0; j < PY; ++j)
#pragma unroll
                        for (int i = 0; i < PX; ++i) out[j][i] = nv[j][i];
                } else {
                    // level t's new plane replaces its oldest (consumed above by level t+1)
#pragma unroll
                    for (int j = 0; j < PY; ++j)
#pragma unroll
                        for (int i = 0; i < PX; ++i) Q[F0][t - 1][j][i] = nv[j][i];
                }
            }

            // step k-1 complete: nobody still reads the edge buffer k mod 3 (= k-3), and
            // the ring slot of plane g-2 (g = this step's plane; last read by the step
            // of plane g-1, at the latest step k-1) may be refilled with plane g-2+RING
            if (gstep >= 1) {
                const uint32_t k1 = gstep - 1;
                mbar_wait(&lbar[k1 % 3], (k1 / 3) & 1);
            }
            if (threadIdx.x == 0 && has_plane) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                produce((gplane + RING_N - 2) % RING_N);
            }
            // this step's edge rows of levels 1..T-1
#pragma unroll
            for (int t = 1; t < T; ++t) {
                R* E = edge + ((int)ebuf_w * P::NL + (t - 1)) * P::EDGE;
                const R(&nw)[PY][PX] = Q[F0][t - 1];
                *reinterpret_cast<V2*>(E + (2 * wy) * WX + cx) = V2{nw[0][0], nw[0][1]};
                *reinterpret_cast<V2*>(E + (2 * wy + 1) * WX + cx) = V2{nw[PY - 1][0], nw[PY - 1][1]};
            }
            // level T: plane q - 2T + 1 once inside the unit's chunk
            const int pT = q - 2 * T + 1;
            if (pT >= w.zc0 && pT < w.zc1) {
                R* b = dnext;
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
            }
            dnext += pz;
            __syncwarp();
            if (lane == 0) mbar_arrive(&lbar[gstep % 3]);
            ++gstep;
            if (has_plane) ++gplane;
        };
        // every level's plane inside its z domain this step (and the warp in x/y)
        auto zin_all = [&](int st) {
            const int q = w.zc0 - T + st;
            return q - 1 < a.hi[0] + a.ehi[0] * (T - 1) && q - 2 * T + 1 >= a.lo[0] - 0;
        };
        auto run = [&](auto phase, int st) {
            if (fast_xy && zin_all(st)) step(phase, std::true_type{}, st);
            else step(phase, std::false_type{}, st);
        };
        // the phase must follow gstep (queues rotate with the global step count)
        int st = 0;
        while (st < nsteps) {
            const uint32_t ph = gstep % 3;
            if (ph == 0) { run(std::integral_constant<int, 0>{}, st); ++st; if (st >= nsteps) break; }
            if (gstep % 3 == 1) { run(std::integral_constant<int, 1>{}, st); ++st; if (st >= nsteps) break; }
            if (gstep % 3 == 2) { run(std::integral_constant<int, 2>{}, st); ++st; }
        }
    }
}
