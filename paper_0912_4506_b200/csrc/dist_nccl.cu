// dist_nccl.cu -- sp_dist_*: the z-slab halo exchange + outer step behind the C ABI
// (SURVEY 8b), so that a host without PyTorch can drive one process per GPU.
//
// sp_dist_step = exchange_halos (z phase, R/decomp.py:149-179) of the current
// grid followed by outer_step (R/decomp.py:208-237): T levels on the rank's
// extended level domains (level_domains_for_rank, R/decomp.py:192-205) in one
// K2 pass.  The exchange is a grouped ncclSend/ncclRecv of h whole padded
// z-planes per neighbour, straight from and into the grid allocations (slab
// ranks' ghost planes are contiguous spans) on the caller's
// stream.  NCCL is bound at run time (dlopen of libnccl.so.2: the copy already
// mapped by the host process, e.g. PyTorch's, or the system library), so the
// library itself has no link-time dependency on it.  The overlapped and
// peer-store transports stay in the Python SlabRunner (dist.py); this is the
// reference's strict alternation of exchange and compute.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/stencilpipe_b200.h"

namespace spi {   // defined in capi.cu (thread-local error string behind the status codes)
int fail(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* where);
}  // namespace spi

namespace {

using spi::fail;

// the slice of nccl.h this file uses (stable since NCCL 2.7)
struct NcclUniqueId { char internal[128]; };
typedef void* NcclComm;
typedef int NcclResult;                       // 0 = ncclSuccess
constexpr int kNcclInt8 = 0;                  // ncclInt8 / ncclChar

struct NcclApi {
    NcclResult (*GetUniqueId)(NcclUniqueId*);
    NcclResult (*CommInitRank)(NcclComm*, int, NcclUniqueId, int);
    NcclResult (*CommDestroy)(NcclComm);
    NcclResult (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t);
    NcclResult (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t);
    NcclResult (*GroupStart)();
    NcclResult (*GroupEnd)();
    const char* (*GetErrorString)(NcclResult);
    bool ok = false;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;
std::string g_nccl_why;

void load_nccl() {
    void* h = nullptr;
    const char* env = getenv("SP_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
        if (!n) continue;
        h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) {
        g_nccl_why = "libnccl.so.2 not found (set SP_NCCL_LIB to its path)";
        return;
    }
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) g_nccl_why = std::string("NCCL symbol missing: ") + name;
        return p;
    };
    g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(sym("ncclGetUniqueId"));
    g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(sym("ncclCommInitRank"));
    g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(sym("ncclCommDestroy"));
    g_nccl.Send = reinterpret_cast<decltype(g_nccl.Send)>(sym("ncclSend"));
    g_nccl.Recv = reinterpret_cast<decltype(g_nccl.Recv)>(sym("ncclRecv"));
    g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(sym("ncclGroupStart"));
    g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(sym("ncclGroupEnd"));
    g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(sym("ncclGetErrorString"));
    g_nccl.ok = g_nccl_why.empty();
}

int need_nccl() {
    std::call_once(g_nccl_once, load_nccl);
    if (!g_nccl.ok) return fail(SP_ERR_DEVICE, "NCCL unavailable: %s", g_nccl_why.c_str());
    return SP_OK;
}

int nccl_fail(NcclResult r, const char* where) {
    return fail(SP_ERR_DEVICE, "%s: %s", where, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "NCCL error");
}

#define SP_NCCL(expr)                                  \
    do {                                               \
        NcclResult _r = (expr);                        \
        if (_r != 0) return nccl_fail(_r, #expr);      \
    } while (0)

}  // namespace

struct sp_dist {
    NcclComm comm;
    int rank, world, device;
};

extern "C" {

int sp_dist_unique_id(void* id_out, int64_t len) {
    if (!id_out || len < SP_DIST_ID_BYTES) return fail(SP_ERR_ARG, "unique id buffer must hold %d bytes", SP_DIST_ID_BYTES);
    if (int rc = need_nccl()) return rc;
    NcclUniqueId id;
    SP_NCCL(g_nccl.GetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return SP_OK;
}

int sp_dist_create(const void* id, int rank, int world, sp_dist** out) {
    if (!id || !out) return fail(SP_ERR_ARG, "null argument");
    if (world < 1 || rank < 0 || rank >= world)
        return fail(SP_ERR_DECOMP, "rank %d outside a world of %d", rank, world);
    if (int rc = need_nccl()) return rc;
    NcclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    sp_dist* d = new sp_dist{nullptr, rank, world, 0};
    cudaError_t e = cudaGetDevice(&d->device);
    if (e != cudaSuccess) { delete d; return spi::cuda_fail(e, "cudaGetDevice"); }
    NcclResult r = g_nccl.CommInitRank(&d->comm, world, uid, rank);
    if (r != 0) { delete d; return nccl_fail(r, "ncclCommInitRank"); }
    *out = d;
    return SP_OK;
}

int sp_dist_destroy(sp_dist* d) {
    if (!d) return SP_OK;
    NcclResult r = d->comm ? g_nccl.CommDestroy(d->comm) : 0;
    delete d;
    return r == 0 ? SP_OK : nccl_fail(r, "ncclCommDestroy");
}

int sp_dist_exchange_z(sp_dist* d, void* grid, int dtype, const sp_layout* L, int64_t h, void* stream) {
    if (!d || !grid || !L) return fail(SP_ERR_ARG, "null argument");
    const int es = dtype == SP_F64 ? 8 : (dtype == SP_F32 ? 4 : 0);
    if (!es) return fail(SP_ERR_ARG, "unknown dtype %d", dtype);
    if (d->world == 1) return SP_OK;   // no neighbour: every face is a physical wall
    if (h < 1 || h > L->gz) return fail(SP_ERR_DECOMP, "halo depth %lld outside 1..gz=%lld", (long long)h, (long long)L->gz);
    if (h > L->nz) return fail(SP_ERR_DECOMP, "slab of %lld planes is thinner than the halo depth %lld", (long long)L->nz, (long long)h);
    cudaStream_t s = (cudaStream_t)stream;
    char* base = static_cast<char*>(grid);
    // whole padded planes [z, z+h) of the allocation: plane z starts at element (z + gz) * pz
    auto planes = [&](int64_t z) { return base + (size_t)(z + L->gz) * (size_t)L->pz * es; };
    const size_t bytes = (size_t)h * (size_t)L->pz * es;
    SP_NCCL(g_nccl.GroupStart());
    if (d->rank > 0) {               // z- neighbour: my first h planes out, its last h planes into my low ghosts
        SP_NCCL(g_nccl.Send(planes(0), bytes, kNcclInt8, d->rank - 1, d->comm, s));
        SP_NCCL(g_nccl.Recv(planes(-h), bytes, kNcclInt8, d->rank - 1, d->comm, s));
    }
    if (d->rank < d->world - 1) {    // z+ neighbour
        SP_NCCL(g_nccl.Send(planes(L->nz - h), bytes, kNcclInt8, d->rank + 1, d->comm, s));
        SP_NCCL(g_nccl.Recv(planes(L->nz), bytes, kNcclInt8, d->rank + 1, d->comm, s));
    }
    SP_NCCL(g_nccl.GroupEnd());
    return SP_OK;
}

int sp_dist_step(sp_dist* d, void* src, void* dst, int dtype, const sp_layout* L, int T, void* stream) {
    if (!d) return fail(SP_ERR_ARG, "null argument");
    if (int rc = sp_dist_exchange_z(d, src, dtype, L, T, stream)) return rc;
    const int64_t lo[3] = {0, 0, 0}, hi[3] = {L->nz, L->ny, L->nx};
    const int32_t elo[3] = {d->rank > 0 ? 1 : 0, 0, 0}, ehi[3] = {d->rank < d->world - 1 ? 1 : 0, 0, 0};
    return sp_sweep_tb(src, dst, dtype, L, T, lo, hi, elo, ehi, stream);
}

}  // extern "C"
