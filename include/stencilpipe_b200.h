/*
 * stencilpipe_b200.h -- C ABI of the B200-native Jacobi hot path.
 *
 * The reference (`stencilpipe`, pure Python/numpy) has no FFI; its seam is the
 * Python function layer listed per entry point below.  This library replaces
 * the arithmetic under that seam; the Python package paper_0912_4506_b200
 * binds it with ctypes and keeps the reference's API above it.
 * (R = /root/reference/pkg/src/stencilpipe)
 *
 * Conventions
 *  - Plain C types only.  Device buffers are allocated by the caller (PyTorch)
 *    and passed as raw pointers to the START of the allocation; the library
 *    never allocates or frees grid memory.  Streams are cudaStream_t passed as
 *    void* (0 = legacy default stream).
 *  - Every entry point returns 0 (SP_OK) or an SP_ERR_* code; sp_last_error()
 *    returns a thread-local message for the last failure on that thread.
 *  - Grid layout: C order (z, y, x), x contiguous; ghost depths gx/gy/gz are
 *    present on both sides; interior element (z,y,x) lives at
 *    base[origin + z*pz + y*py + x].  TMA needs py*sizeof(elem) % 16 == 0 and a
 *    16-byte-aligned base; sp_layout_make() returns such a layout (interior row
 *    start 128-byte aligned).
 */
#ifndef STENCILPIPE_B200_H
#define STENCILPIPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_OK 0
#define SP_ERR_GRID 1         /* -> GridError(ValueError)          R/grid.py:25      */
#define SP_ERR_SCHEDULE 2     /* -> ScheduleError(ValueError)      R/pipeline.py:30  */
#define SP_ERR_DECOMP 3       /* -> DecompositionError(ValueError) R/decomp.py:26    */
#define SP_ERR_DEVICE 4       /* -> RuntimeError (CUDA failure)                      */
#define SP_ERR_ARG 5          /* -> ValueError (bad argument)                        */

#define SP_F64 0
#define SP_F32 1

typedef struct sp_layout {
    int64_t nx, ny, nz;       /* interior extents (GridDims, R/grid.py:29-51)    */
    int64_t gx, gy, gz;       /* ghost depth present in memory on each side      */
    int64_t py, pz;           /* row / plane pitch, elements                     */
    int64_t origin;           /* element offset of interior (0,0,0) from base    */
} sp_layout;

/* Initial-value pattern, evaluated over GLOBAL coordinates (FillPattern,
 * R/grid.py:66-118; subdomain shift as _ShiftedPattern, R/decomp.py:107-117).
 * kind: 0 constant, 1 linear, 2 hotplate, 3 random(seed), 4 2*random-1.
 * has_faces: cells outside the global interior [0, gn) take faces[] of the
 * first face beyond which they lie, in the order (z-, z+, y-, y+, x-, x+). */
typedef struct sp_pattern {
    int32_t kind;
    int32_t has_faces;
    double value;
    uint64_t seed;
    int64_t gorigin[3];       /* global (z,y,x) of the local interior origin */
    int64_t gn[3];            /* global interior extents (z,y,x)             */
    double faces[6];
} sp_pattern;

/* Library identity / diagnostics. */
int sp_version(void);
const char* sp_last_error(void);
/* Number of device kernels this library has launched since load. */
uint64_t sp_launch_count(void);

/* Padded device layout for a grid (replaces the dense numpy allocation of
 * TwoGrid, R/grid.py:126-134).  *alloc_elems = elements to allocate. */
int sp_layout_make(int64_t nx, int64_t ny, int64_t nz, int64_t gx, int64_t gy,
                   int64_t gz, int dtype, sp_layout* out, int64_t* alloc_elems);

/* K3: fill every cell of the allocation from the pattern (ghost shell
 * included; row padding set to 0).  Replaces FillPattern.evaluate over the
 * ghosted box in TwoGrid.__init__ (R/grid.py:96-134). */
int sp_fill(void* base, int dtype, const sp_layout* L, const sp_pattern* p,
            void* stream);

/* K1: one Jacobi level over the logical box [lo, hi) (z,y,x), dst = stencil(src)
 * there, every other dst cell untouched.  Replaces update_region
 * (R/kernel.py:37-40) and hence sweep_naive / sweep_spatial_blocked /
 * update_block (R/kernel.py:43-80,124-147).  The box may reach into the ghost
 * shell up to depth-1 (R/kernel.py:138-140). */
int sp_update_region(const void* src, void* dst, int dtype, const sp_layout* L,
                     const int64_t lo[3], const int64_t hi[3], void* stream);

/* K2: T levels in one pass over HBM (temporally blocked wavefront), reading
 * src (level 0) and writing level T into dst over [lo, hi) only.  Level t
 * (1..T) updates the domain [lo - ext_lo*(T-t), hi + ext_hi*(T-t)) per axis
 * and keeps every other cell at its previous-level value, so ext = 0 gives
 * Dirichlet walls and ext = 1 the shrinking extended domains of a rank face
 * with a neighbour (level_domains_for_rank, R/decomp.py:192-205).  Equivalent
 * to T node-sweep levels of run_node_sweeps (R/pipeline.py:395-408,459-462).
 * 1 <= T <= 8. */
int sp_sweep_tb(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                const int32_t ext_hi[3], void* stream);

/* K2 restricted to an output sub-box: identical level domains (lo, hi, ext_*)
 * as sp_sweep_tb, but only cells of [out_lo, out_hi) (a subset of [lo, hi))
 * are computed to level T and written.  Used to run a rank's boundary slabs
 * first and its interior while the halo exchange is in flight
 * (outer_step + exchange_halos, R/decomp.py:149-237, with overlap added). */
int sp_sweep_tb_part(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                     const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                     const int32_t ext_hi[3], const int64_t out_lo[3],
                     const int64_t out_hi[3], void* stream);

/* sp_sweep_tb_part that also delivers its z-boundary planes to the z-slab
 * neighbours (fused halo exchange over peer memory; replaces the send half of
 * exchange_halos, R/decomp.py:149-179, for layouts (1,1,P)): every level-T
 * output plane z < halo is stored a second time into peer_lo -- the
 * allocation base of the z- neighbour's destination grid, which has this
 * grid's layout except nz -- at its plane z + peer_lo_shift (= its nz), and
 * every plane z >= nz - halo into peer_hi at plane z + peer_hi_shift
 * (= -nz).  The pointers must be addressable from this device (CUDA IPC /
 * peer access); a null pointer skips that side.  Ordering against the
 * neighbours' own passes is the caller's (SlabRunner: one token per step). */
int sp_sweep_tb_part_peer(const void* src, void* dst, int dtype, const sp_layout* L, int T,
                          const int64_t lo[3], const int64_t hi[3], const int32_t ext_lo[3],
                          const int32_t ext_hi[3], const int64_t out_lo[3],
                          const int64_t out_hi[3], void* peer_lo, int64_t peer_lo_shift,
                          void* peer_hi, int64_t peer_hi_shift, int64_t halo, void* stream);

/* Grid transfers (stream-ordered; host memory should be pinned for
 * asynchrony).  sp_copy_in: the dense ghosted box (nz+2gz, ny+2gy, nx+2gx)
 * -- the reference TwoGrid's array layout, R/grid.py:126-134 -- into the
 * allocation at base_a and, if base_b is given, also base_b (B = copy of A,
 * R/grid.py:132-133).  sp_copy_out: the interior (nz, ny, nx) of the
 * allocation at base into dense host memory (TwoGrid.interior,
 * R/grid.py:151-153).  With a device staging buffer (>= two planes) the
 * data crosses PCIe as linear copies of whole planes through its two halves,
 * repacked on the device (K6) on a library side stream and joined back to
 * `stream`; without one, as a single pitched 3-D DMA.  A staging buffer must
 * not be shared by transfers in flight at the same time. */
int sp_copy_in(const void* host, int dtype, const sp_layout* L, void* base_a, void* base_b,
               void* staging, int64_t staging_elems, void* stream);
int sp_copy_out(const void* base, int dtype, const sp_layout* L, void* host, void* staging,
                int64_t staging_elems, void* stream);

/* Cross-process grid mapping for sp_sweep_tb_part_peer (CUDA IPC).
 * sp_ipc_export: 64-byte handle of the device allocation holding ptr and
 * ptr's byte offset inside it.  sp_ipc_import (another process): map it into
 * the current device (peer access to the owner's GPU enabled on demand) and
 * return the address of the exported byte.  sp_ipc_close unmaps.  Imports
 * are refcounted per (device, handle): buffers exported from one allocation
 * block share one mapping, closed with the last sp_ipc_close. */
int sp_ipc_export(const void* ptr, unsigned char handle[64], int64_t* offset);
int sp_ipc_import(const unsigned char handle[64], int64_t offset, void** ptr);
int sp_ipc_close(void* ptr, int64_t offset);

/* `levels` full-interior sweeps as passes of depth T (last pass shorter),
 * ping-ponging a/b.  *active: in = which array holds the current level
 * (0 = a), out = which holds the result (TwoGrid.active, R/grid.py:136-149).
 * Replaces `levels` calls of sweep_naive (R/kernel.py:43-47). */
int sp_run_sweeps(void* a, void* b, int dtype, const sp_layout* L, int64_t levels,
                  int T, int* active, void* stream);

/* K5: order-independent 64-bit digest of the interior (definition in
 * oracle/jacobi_oracle.c), cell (z,y,x) hashed with linear index
 * index_base + (z*ny + y)*nx + x -- so the digests of a z-slab decomposition
 * (index_base = z0*ny*nx per slab) sum to the digest of the whole grid.
 * Synchronises the stream. */
int sp_digest(const void* base, int dtype, const sp_layout* L, int64_t index_base,
              uint64_t* out, void* stream);

/* Measured FP64 add throughput of this device (DADD/s over all SMs) -- the
 * compute roof of the stencil, which has no fusable multiply-add. */
int sp_probe_fp64(double* dadd_per_s, double* ms);

/* Tuning hook (benchmarks only): kernel-variant override (0 = automatic per
 * dtype/T; k = variant k-1 of the table in csrc/capi.cu, warps x
 * rows-per-thread / z-queue slots; a variant not built for a depth falls back
 * to variant 0; -1 = single-level sweeps on the K1 kernel) and z-chunk count
 * override (0 = automatic).  Returns the previous values encoded as
 * (variant+1)*1000 + chunks.  The setting is THREAD-LOCAL: it applies to the
 * calling host thread's later launches only. */
int sp_set_tuning(int variant, int chunks);

/* Tuning hook (benchmarks only): work-unit schedule of the temporally blocked
 * kernel.  dynamic = 1: persistent CTAs claim (tile, z-chunk) units in order
 * from a device counter, so units in flight at one time are neighbours and
 * share their halo rows through L2; 0: static round-robin.  strip = width in
 * tiles of the column strips units are ordered by (y-major inside a strip;
 * 0 = plain x-major rows).  Negative arguments keep the current value.
 * Returns the previous values encoded as dynamic*1000 + strip.  Thread-local
 * like sp_set_tuning.  The dynamic schedule's unit counter is one per (device,
 * stream): launches on a stream are serial and each leaves it at zero, and
 * launches on different streams never share one. */
int sp_set_schedule(int dynamic, int strip);

/* Compressed single-array storage (R/grid.py:164-208; R/kernel.py:83-121):
 * one temporally blocked pass of depth T IN PLACE over the box [lo, hi) of the
 * allocation `buf` (layout L, walls on every face of the box).  Level-T plane
 * p is stored at plane p - (2*chunk + T) (direction +1, z-chunks in ascending
 * order) or p + (2*chunk + T) (direction -1, descending): no chunk overwrites
 * a plane a chunk still reading it may need, which per-chunk counters in
 * `counters` (device, >= ceil((hi-lo)/chunk) unsigned) enforce.  chunk >= 2T.
 * The box's ghost shell does not move with it: sp_ghost_shell re-scatters it.
 * Replaces update_region_compressed / _refresh_compressed_ghosts. */
int sp_sweep_tb_inplace(void* buf, int dtype, const sp_layout* L, int T, const int64_t lo[3],
                        const int64_t hi[3], int64_t chunk, int direction, void* counters,
                        int64_t ncounters, void* stream);

/* Ghost shell of a ghost-depth-1 box (layout L at `base`) packed into `shell`
 * (sp_ghost_shell_elems elements): to_grid = 0 gathers, 1 scatters. */
int sp_ghost_shell(void* base, int dtype, const sp_layout* L, void* shell, int to_grid, void* stream);
int64_t sp_ghost_shell_elems(int64_t nx, int64_t ny, int64_t nz);

/* Strided 3-D box copy on the device (K6): nz x ny x nx elements from src
 * (row pitch src_py, plane pitch src_pz, in elements) to dst (dst_py,
 * dst_pz).  Packs and unpacks the halo slabs of multi-axis decompositions
 * (the extended slabs of R/decomp.py:137-179) around NCCL send/recv. */
int sp_copy_box(const void* src, void* dst, int dtype, int64_t nz, int64_t ny, int64_t nx, int64_t src_py,
                int64_t src_pz, int64_t dst_py, int64_t dst_pz, void* stream);

/* Scatter only the ghost face cells adjacent to the interior box [lo, hi)
 * (z, y, x): a face only where the box touches it (lo == 0 / hi == n on that
 * axis), within the box's extent on the other axes, edges and corners never.
 * Replaces _refresh_compressed_ghosts (R/kernel.py:83-102) before a
 * compressed update_block (R/kernel.py:124-147). */
int sp_ghost_shell_region(void* base, int dtype, const sp_layout* L, const void* shell, const int64_t lo[3],
                          const int64_t hi[3], void* stream);

/* Introspection (benchmarks, reports): the kernel variant a temporally blocked
 * pass of depth T in dtype runs (after any sp_set_tuning override and the
 * fallback for variants not built for T), and a one-line description of it
 * (CTA shape, z-queue, CTAs per SM, step barrier, cluster form) in buf.
 * Returns the variant index (>= 0) or a negative error code. */
int sp_describe_variant(int dtype, int T, char* buf, int buflen);

/* ---- z-slab multi-GPU behind the ABI (one process per GPU; NCCL bound at run
 * time with dlopen("libnccl.so.2"), override with the environment variable
 * SP_NCCL_LIB).  The overlapped and peer-store transports are driven by the
 * Python SlabRunner; these entry points are the reference's strict
 * alternation of exchange and compute for hosts without PyTorch. ------------- */
#define SP_DIST_ID_BYTES 128
typedef struct sp_dist sp_dist;

/* Rank 0 creates the communicator id (ncclGetUniqueId); the host ships its
 * SP_DIST_ID_BYTES bytes to every rank (the role of the reference's transport
 * rendezvous, R/decomp.py:240-255). */
int sp_dist_unique_id(void* id_out, int64_t len);

/* Join the communicator as `rank` of `world` z-slab ranks on the current CUDA
 * device (ranks are z-ordered: rank r's z- neighbour is r-1). */
int sp_dist_create(const void* id, int rank, int world, sp_dist** out);
int sp_dist_destroy(sp_dist* d);

/* exchange_halos, z phase (R/decomp.py:149-179): the first / last h interior
 * planes of `grid` go to the z- / z+ neighbour's ghost planes, and theirs come
 * into this grid's ghost planes [-h, 0) and [nz, nz + h); whole padded planes,
 * grouped ncclSend/ncclRecv on `stream`.  1 <= h <= L->gz. */
int sp_dist_exchange_z(sp_dist* d, void* grid, int dtype, const sp_layout* L, int64_t h, void* stream);

/* One outer step (R/decomp.py:208-237 after :149-179): exchange the depth-T
 * halos of src, then T levels src -> dst on the rank's extended level domains
 * (level_domains_for_rank, R/decomp.py:192-205: extended by T-t towards each
 * neighbour, Dirichlet at physical walls) in one K2 pass.  The caller swaps
 * src and dst afterwards (dst's ghosts are refreshed by the next step's
 * exchange).  Requires L->gz >= T. */
int sp_dist_step(sp_dist* d, void* src, void* dst, int dtype, const sp_layout* L, int T, void* stream);

#ifdef __cplusplus
}
#endif
#endif
