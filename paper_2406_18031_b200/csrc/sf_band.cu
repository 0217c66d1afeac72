// sf_band.cu -- banded mode: row-band decomposition of a tall grid over several contexts
// (config 5).  Each band context holds its owned rows plus `halo` rows on
// each side; one halo exchange per frame (the rows are exact copies of the neighbours' owned
// rows), then an ordinary sf_step on the extended band.  Garbage produced at the band's cut
// edges travels at most halo rows per frame and never reaches the owned rows, so the owned
// rows are bitwise those of a single context over the whole grid.
#include <dlfcn.h>
#include <string.h>

#include "sf_internal.cuh"

extern "C" int32_t sf_band_halo(const sf_config* cfg) {
    const int N = (int)ceilf(cfg->max_flow_px) < 1 ? 1 : (int)ceilf(cfg->max_flow_px);
    return (N > 2 ? N : 2) + 2 * cfg->smooth_iters;
}

extern "C" sf_status sf_band_partition(int32_t gh, int32_t nbands, int32_t band, int32_t halo, int32_t* ext_begin,
                                       int32_t* own_begin, int32_t* own_end, int32_t* ext_end) {
    if (gh < 2 || nbands < 1 || band < 0 || band >= nbands || halo < 0) return SF_E_CONFIG;
    const int base = gh / nbands, rem = gh % nbands;
    const int ob = band * base + (band < rem ? band : rem);
    const int oe = ob + base + (band < rem ? 1 : 0);
    if (nbands > 1 && (oe - ob) < halo) return SF_E_CONFIG;  // a neighbour's halo must lie in one band
    if (own_begin) *own_begin = ob;
    if (own_end) *own_end = oe;
    if (ext_begin) *ext_begin = ob - halo < 0 ? 0 : ob - halo;
    if (ext_end) *ext_end = oe + halo > gh ? gh : oe + halo;
    return SF_OK;
}

// rows [gr0, gr1) (global) of src's current state and Yhat^k into dst's current buffers
static cudaError_t copy_rows(sf_ctx* dst, const sf_ctx* src, int gr0, int gr1) {
    if (gr1 <= gr0) return cudaSuccess;
    const FrameParams& f = dst->fp;
    const int dl = gr0 - dst->ext_begin, sl = gr0 - src->ext_begin, n = gr1 - gr0;
    const size_t W = (size_t)f.W;
    for (int b = 0; b < f.B; ++b) {
        const size_t dpl = (size_t)b * f.H * W, spl = (size_t)b * src->fp.H * W;
        cudaError_t e = cudaMemcpyAsync(dst->state[dst->cur] + dpl + dl * W, src->state[src->cur] + spl + sl * W,
                                        n * W * sizeof(float4), cudaMemcpyDeviceToDevice, dst->stream);
        if (e != cudaSuccess) return e;
        e = cudaMemcpyAsync(dst->yhat[dst->cur] + dpl + dl * W, src->yhat[src->cur] + spl + sl * W,
                            n * W * sizeof(float), cudaMemcpyDeviceToDevice, dst->stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

static bool compatible(const sf_ctx* a, const sf_ctx* b) {
    return a->fp.W == b->fp.W && a->fp.B == b->fp.B && a->global_h == b->global_h;
}

extern "C" sf_status sf_halo_exchange_peer(sf_ctx* c, const sf_ctx* up, const sf_ctx* down) {
    SF_NVTX("sf_halo_exchange_peer");
    if (!c) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->initialized) return SF_E_STATE;
    if (c->pending) return SF_E_STATE;
    if (c->ext_begin < c->own_begin) {  // top halo rows [ext_begin, own_begin) live in `up`
        if (!up || !compatible(c, up) || !up->initialized || up->own_begin > c->ext_begin ||
            up->own_end < c->own_begin)
            return SF_E_DATA;
        if (copy_rows(c, up, c->ext_begin, c->own_begin) != cudaSuccess) return SF_E_CUDA;
    }
    const int ext_end = c->ext_begin + c->fp.H;
    if (ext_end > c->own_end) {  // bottom halo rows [own_end, ext_end) live in `down`
        if (!down || !compatible(c, down) || !down->initialized || down->own_begin > c->own_end ||
            down->own_end < ext_end)
            return SF_E_DATA;
        if (copy_rows(c, down, c->own_end, ext_end) != cudaSuccess) return SF_E_CUDA;
    }
    return SF_OK;
}

// ------------------------------------------------------------------ NCCL (loaded at first use)
namespace {
typedef int nres_t;  // ncclResult_t
struct NcclApi {
    bool ok = false;
    nres_t (*GetUniqueId)(void* id) = nullptr;
    nres_t (*CommInitRank)(void** comm, int n, char id[128], int rank) = nullptr;
    nres_t (*CommDestroy)(void* comm) = nullptr;
    nres_t (*GroupStart)() = nullptr;
    nres_t (*GroupEnd)() = nullptr;
    nres_t (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nres_t (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32 (nccl.h)

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);  // torch's copy if already loaded
        if (!h) return api;
        api.GetUniqueId = (nres_t(*)(void*))dlsym(h, "ncclGetUniqueId");
        api.CommInitRank = (nres_t(*)(void**, int, char*, int))dlsym(h, "ncclCommInitRank");
        api.CommDestroy = (nres_t(*)(void*))dlsym(h, "ncclCommDestroy");
        api.GroupStart = (nres_t(*)())dlsym(h, "ncclGroupStart");
        api.GroupEnd = (nres_t(*)())dlsym(h, "ncclGroupEnd");
        api.Send = (nres_t(*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclSend");
        api.Recv = (nres_t(*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclRecv");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
                 api.Recv;
    }
    return api;
}
}  // namespace

extern "C" sf_status sf_nccl_unique_id(char id[128]) {
    NcclApi& n = nccl();
    if (!n.ok || !id) return SF_E_NCCL;
    return n.GetUniqueId(id) == 0 ? SF_OK : SF_E_NCCL;
}

extern "C" sf_status sf_nccl_comm_init(int32_t nranks, const char id[128], int32_t rank, void** comm) {
    NcclApi& n = nccl();
    if (!n.ok || !id || !comm) return SF_E_NCCL;
    char buf[128];
    memcpy(buf, id, 128);
    return n.CommInitRank(comm, nranks, buf, rank) == 0 ? SF_OK : SF_E_NCCL;
}

extern "C" void sf_nccl_comm_destroy(void* comm) {
    NcclApi& n = nccl();
    if (n.ok && comm) n.CommDestroy(comm);
}

// Band `rank` sends its first `halo_up` owned rows to rank-1 and its last `halo_dn` owned rows to
// rank+1, and receives its own halo rows from them.  Band heights >= halo (sf_band_partition), so
// the rows a neighbour needs are always inside one band; both sides use the same halo size.
extern "C" sf_status sf_halo_exchange_nccl(sf_ctx* c, void* comm, int32_t rank, int32_t nranks) {
    SF_NVTX("sf_halo_exchange_nccl");
    if (!c || !comm) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (!c->initialized || c->pending) return SF_E_STATE;
    NcclApi& n = nccl();
    if (!n.ok) return SF_E_NCCL;
    const FrameParams& f = c->fp;
    const size_t W = (size_t)f.W;
    const int top = c->own_begin - c->ext_begin;                 // halo rows above
    const int bot = (c->ext_begin + f.H) - c->own_end;           // halo rows below
    const int lo = top, hi = c->own_end - c->ext_begin;          // owned rows, local
    if (n.GroupStart() != 0) return SF_E_NCCL;
    for (int b = 0; b < f.B; ++b) {
        float4* st = c->state[c->cur] + (size_t)b * f.H * W;
        float* yh = c->yhat[c->cur] + (size_t)b * f.H * W;
        if (rank > 0 && top > 0) {
            n.Send(st + lo * W, (size_t)top * W * 4, kNcclFloat32, rank - 1, comm, c->stream);
            n.Send(yh + lo * W, (size_t)top * W, kNcclFloat32, rank - 1, comm, c->stream);
            n.Recv(st, (size_t)top * W * 4, kNcclFloat32, rank - 1, comm, c->stream);
            n.Recv(yh, (size_t)top * W, kNcclFloat32, rank - 1, comm, c->stream);
        }
        if (rank < nranks - 1 && bot > 0) {
            n.Send(st + (hi - bot) * W, (size_t)bot * W * 4, kNcclFloat32, rank + 1, comm, c->stream);
            n.Send(yh + (hi - bot) * W, (size_t)bot * W, kNcclFloat32, rank + 1, comm, c->stream);
            n.Recv(st + hi * W, (size_t)bot * W * 4, kNcclFloat32, rank + 1, comm, c->stream);
            n.Recv(yh + hi * W, (size_t)bot * W, kNcclFloat32, rank + 1, comm, c->stream);
        }
    }
    return n.GroupEnd() == 0 ? SF_OK : SF_E_NCCL;
}
