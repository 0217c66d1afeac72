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

// ------------------------------------------------------------------ per-substep exchange
// The north star's banded split: a band context holds its owned rows plus 2 halo rows on each
// cut side, and the halo rows are refreshed at every point of the frame that reads across a row
// boundary -- after each column pass (1 row of (w*, rho*): the row pass reads i +- 1)
// and before each box pass (2 rows of w: the 5x5 box reads i +- 2).  The transport and
// the box run on the per-pass kernels over the owned rows (transport) / the band (box); the
// update's models read the band's own inputs (Y, depth cover the band and its halo rows).
extern "C" int32_t sf_band_halo_substep(const sf_config* cfg) {
    (void)cfg;
    return 2;
}

namespace {
// One exchange point: rows of the float4 plane `buf` ([B][H][W], local rows) -- send own rows
// [lo, lo + r) up and [hi - r, hi) down, receive [lo - r, lo) from up and [hi, hi + r) from down.
sf_status exchange_rows(sf_ctx* c, float4* buf, int r, sf_halo_xfer_fn xfer, void* user, int host_staged,
                        cudaStream_t s) {
    const FrameParams& f = c->fp;
    const size_t W = (size_t)f.W;
    const int lo = c->own_begin - c->ext_begin, hi = c->own_end - c->ext_begin;
    const bool up = lo > 0, dn = hi < f.H;
    const size_t n = (size_t)r * W * 4;  // floats per segment
    for (int b = 0; b < f.B; ++b) {
        float4* base = buf + (size_t)b * f.H * W;
        float* su = up ? reinterpret_cast<float*>(base + lo * W) : nullptr;
        float* ru = up ? reinterpret_cast<float*>(base + (lo - r) * W) : nullptr;
        float* sd = dn ? reinterpret_cast<float*>(base + (hi - r) * W) : nullptr;
        float* rd = dn ? reinterpret_cast<float*>(base + hi * W) : nullptr;
        if (!host_staged) {
            if (xfer(user, su, ru, sd, rd, up ? n : 0, dn ? n : 0) != 0) return SF_E_NCCL;
            continue;
        }
        float* h = c->xhost;  // [send_up | recv_up | send_dn | recv_dn], n floats each
        if (up && cudaMemcpyAsync(h, su, n * sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess) return SF_E_CUDA;
        if (dn && cudaMemcpyAsync(h + 2 * n, sd, n * sizeof(float), cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return SF_E_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return SF_E_CUDA;
        if (xfer(user, up ? h : nullptr, up ? h + n : nullptr, dn ? h + 2 * n : nullptr, dn ? h + 3 * n : nullptr,
                 up ? n : 0, dn ? n : 0) != 0)
            return SF_E_NCCL;
        if (up && cudaMemcpyAsync(ru, h + n, n * sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess) return SF_E_CUDA;
        if (dn && cudaMemcpyAsync(rd, h + 3 * n, n * sizeof(float), cudaMemcpyHostToDevice, s) != cudaSuccess)
            return SF_E_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return SF_E_CUDA;  // the staging is reused next call
    }
    return SF_OK;
}

struct NcclXfer {
    void* comm;
    int rank;
    cudaStream_t stream;
};
int32_t nccl_xfer(void* u, const float* su, float* ru, const float* sd, float* rd, size_t nu, size_t nd) {
    NcclXfer* x = static_cast<NcclXfer*>(u);
    NcclApi& n = nccl();
    if (n.GroupStart() != 0) return 1;
    if (su) {
        n.Send(su, nu, kNcclFloat32, x->rank - 1, x->comm, x->stream);
        n.Recv(ru, nu, kNcclFloat32, x->rank - 1, x->comm, x->stream);
    }
    if (sd) {
        n.Send(sd, nd, kNcclFloat32, x->rank + 1, x->comm, x->stream);
        n.Recv(rd, nd, kNcclFloat32, x->rank + 1, x->comm, x->stream);
    }
    return n.GroupEnd() == 0 ? 0 : 1;
}

sf_status banded_step(sf_ctx* c, const float* Y, const float* D, sf_halo_xfer_fn xfer, void* user, int host_staged,
                      NcclXfer* nx) {
    const FrameParams& f = c->fp;
    const int lo = c->own_begin - c->ext_begin, hi = c->own_end - c->ext_begin;
    if ((lo > 0 && lo < 2) || (hi < f.H && f.H - hi < 2) || hi - lo < 4) return SF_E_CONFIG;
    if (host_staged && !c->xhost) {
        if (cudaMallocHost(&c->xhost, 4 * 2 * (size_t)f.W * 4 * sizeof(float)) != cudaSuccess) {
            c->xhost = nullptr;
            return SF_E_CUDA;
        }
    }
    const bool overlap = nx != nullptr;  // device transport: the row pass's inner rows overlap the exchange
    if (overlap && !c->xstream) {
        cudaStream_t s = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&e0, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) != cudaSuccess) {
            if (s) cudaStreamDestroy(s);
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
            return SF_E_CUDA;
        }
        c->xstream = s;
        c->xev[0] = e0;
        c->xev[1] = e1;
    }
    if (nx) nx->stream = c->xstream;
    // ---- prediction: N x (column pass, exchange 1 row, row pass), owned rows only
    const float4* src = c->state[c->cur];
    for (int n = 0; n < f.N; ++n) {
        SF_TRY(sf_launch_pass(c, 0, src, c->tmp, lo, hi, c->stream));
        if (overlap) {
            SF_TRY(cudaEventRecord(c->xev[0], c->stream));
            SF_TRY(cudaStreamWaitEvent(c->xstream, c->xev[0], 0));
            const sf_status st = exchange_rows(c, c->tmp, 1, xfer, user, 0, c->xstream);
            if (st != SF_OK) return st;
            SF_TRY(cudaEventRecord(c->xev[1], c->xstream));
            SF_TRY(sf_launch_pass(c, 1, c->tmp, c->pred, lo + 1, hi - 1, c->stream));  // rows with no halo read
            SF_TRY(cudaStreamWaitEvent(c->stream, c->xev[1], 0));
            SF_TRY(sf_launch_pass(c, 1, c->tmp, c->pred, lo, lo + 1, c->stream));
            SF_TRY(sf_launch_pass(c, 1, c->tmp, c->pred, hi - 1, hi, c->stream));
        } else {
            const sf_status st = exchange_rows(c, c->tmp, 1, xfer, user, host_staged, c->stream);
            if (st != SF_OK) return st;
            SF_TRY(sf_launch_pass(c, 1, c->tmp, c->pred, lo, hi, c->stream));
        }
        src = c->pred;
    }
    // ---- update: models + LS + fusion over the band, then S x (exchange 2 rows, box pass)
    float4* nxt = c->state[1 - c->cur];
    float4* solved = f.S > 0 ? c->tmp : nxt;
    SF_TRY(sf_launch_update_solve(c, Y, D, solved));
    for (int s = 0; s < f.S; ++s) {
        float4* in = (s & 1) ? c->tmp2 : c->tmp;
        float4* out = s == f.S - 1 ? nxt : ((s & 1) ? c->tmp : c->tmp2);
        if (nx) nx->stream = c->stream;
        const sf_status st = exchange_rows(c, in, 2, xfer, user, host_staged, c->stream);
        if (st != SF_OK) return st;
        SF_TRY(sf_launch_box(c, in, out));
    }
    c->cur = 1 - c->cur;
    return SF_OK;
}
}  // namespace

extern "C" sf_status sf_step_banded(sf_ctx* c, const float* Y, const float* D, sf_halo_xfer_fn xfer, void* user,
                                    int32_t host_staged) {
    SF_NVTX("sf_step_banded");
    if (!c || !Y || !D || !xfer) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels != 1) return SF_E_UNSUPPORTED;
    if (!c->initialized) return sf_update(c, Y, D);  // frame 0: pointwise init of the band (exact on owned rows)
    if (c->pending) return SF_E_STATE;
    return banded_step(c, Y, D, xfer, user, host_staged ? 1 : 0, nullptr);
}

extern "C" sf_status sf_step_banded_nccl(sf_ctx* c, const float* Y, const float* D, void* comm, int32_t rank,
                                         int32_t nranks) {
    SF_NVTX("sf_step_banded_nccl");
    if (!c || !Y || !D || !comm || rank < 0 || rank >= nranks) return SF_E_DATA;
    SF_DEVICE_GUARD(c);
    if (c->levels != 1) return SF_E_UNSUPPORTED;
    if (!nccl().ok) return SF_E_NCCL;
    if (!c->initialized) return sf_update(c, Y, D);
    if (c->pending) return SF_E_STATE;
    NcclXfer x{comm, rank, c->stream};
    return banded_step(c, Y, D, nccl_xfer, &x, 0, &x);
}
