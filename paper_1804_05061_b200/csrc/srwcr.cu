// srwcr.cu -- host runtime and C ABI of the SRWCR hot path (see include/srwcr.h).
//
// Owns device memory, the per-axis B-spline tables (built in fp64 on the host from
// Eq 8 P:99 / Eq 17), the work-item list of the CTA decomposition, the static
// fixed-image counts, the NCCL communicator of the z-slab decomposition, and the
// launch sequence of one evaluation.  No compute of the method happens on the host
// (apart from building the tables and summing the static total mass Z).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/srwcr.h"
#include "srwcr_kernels.cuh"
#include "srwcr_fast.cuh"

using namespace srwcr;

// Host -> device copy of create-time (and other host-built) tables: a pageable cudaMemcpy may
// return before its DMA has landed, and the kernels that read these tables run on the
// context's non-blocking stream, which does not wait for the legacy stream -- so wait for the
// device (under contention from another process the race was real: wrong line lists)
static cudaError_t h2d_sync(void *dst, const void *src, size_t bytes) {
    const cudaError_t e = cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
    return e != cudaSuccess ? e : cudaDeviceSynchronize();
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
    bool ok = false;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    // point-to-point (the halo gradient exchange)
    bool p2p = false;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};
NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.Broadcast = (decltype(api.Broadcast))dlsym(h, "ncclBroadcast");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            api.ok = api.CommInitRank && api.AllReduce && api.CommDestroy && api.GetErrorString && api.Broadcast;
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
            api.p2p = api.ok && api.GroupStart && api.GroupEnd && api.Send && api.Recv;
        }
    }
    return api;
}
}  // namespace

constexpr int NPART = 8;   // pipelined host evaluation: at most this many concurrent parts per pass

struct srwcr_ctx {
    std::string err;
    bool poisoned = false;
    srwcr_options opt{};
    int dev = 0;
    cudaStream_t stream = nullptr;
    Geo g{};
    int nranks = 1, rank = 0;
    int64_t z0 = 0, z1 = 0;
    double delta[3]{}, Delta[3]{};
    int32_t kcells[3]{};
    int64_t R = 0, nparams = 0, nint = 0;
    // host tables (kept for dumps)
    std::vector<int> h_cb[3], h_sb[3];
    std::vector<float4> h_sw[3];
    // device
    float *F = nullptr, *M = nullptr, *phi = nullptr, *phimax = nullptr;
    float4 *MG = nullptr;  // pass 1 -> pass 2: (m, dM/dy) per slab voxel
    int *xlist = nullptr, *xcount = nullptr;  // voxels deferred to k_exact_fix
    int xcap = 0;
    double *params64 = nullptr, *grad64 = nullptr;
    const double *cur_params = nullptr;  // device fp64 params of the current evaluation
    int *cb[3]{}, *sb[3]{};
    float4 *cw[3]{}, *sw[3]{};
    double4 *cw64[3]{};
    Item *items = nullptr, *items_full = nullptr;  // this rank's slab / whole volume
    Item *items2 = nullptr;                          // pass 2 (its own x-chunking)
    int nitems2 = 0, XV2 = 1;
    bool MC = false;   // multi-cell items (fine spatial lattices): several x-cells per item
    int zrn = 4;       //   and their z-regions (z-cells per item + 3)
    ItemW *itemw = nullptr, *itemw_full = nullptr;
    int *slotbins = nullptr;                         // slot lists of both item lists
    int nitems = 0, nitems_full = 0;
    int W = 16, W2 = 16, XV = 1, S = 1, S2 = 2;       // warps per CTA (pass 1, 2), voxels per lane, slots, bin list
    double *SQ = nullptr, *Qt = nullptr;             // stats: [R][B][2] binned, then [R] binless
    double *NQ = nullptr;                            // orientation 1: dynamic counts [R][B][2]
    int gstride = 0;                                 // row stride of the gamma table
    int pz0 = 0, pzb1 = 0, pz1 = 0;                  // node layers the slab reads: [pz0, pz1), bases < pzb1
    int64_t lay[5] = {0, 0, 0, 0, 0};                // srwcr_plan_layers of this rank (3-D)
    bool halo = false;                               // grad_exchange = 1: halo sum instead of the all-reduce
    long long *halo_recv = nullptr;                  //   rank - 1's partial on layers [lay[2], lay[4])
    double *Nlo = nullptr, *Nup = nullptr, *dterm = nullptr, *reg = nullptr, *Dout = nullptr;
    unsigned *ticket = nullptr;   // k_combine's last-CTA ticket
    double *dpart = nullptr;      // k_combine's per-CTA partial sums
    double *S_out = nullptr;   // unshifted S[r][a], written by the combine only for a debug dump
    bool dump_S = false;
    float *shiftc = nullptr, *alpha = nullptr, *beta = nullptr, *gamma = nullptr;
    double Z = 0;
    size_t smem1 = 0, smem2 = 0;
    ncclComm_t comm = nullptr;
    bool external_exchange = false;
    bool begun = false;
    // stats
    int64_t launches = 0;
    cudaGraphExec_t gexec = nullptr;            // captured evaluation (options.use_graph)
    cudaGraphExec_t hexec = nullptr;            // captured pipelined host-buffer evaluation (pinned buffers)
    const void *h_params = nullptr, *h_grad = nullptr;
    int64_t h_kernels = 0;
    const double *g_params = nullptr;           //   for these params / grad pointers
    const double *g_grad = nullptr;
    int64_t g_kernels = 0;                      //   kernels per replay
    bool g_timing = false;                      //   with the per-pass event records
    int launches_per_eval = 0;
    bool timing = false;
    cudaEvent_t ev[5]{};  // pass1 start, pass1 end, combine end, pass2 end, prep start
    // pipelined host-buffer evaluation (one rank): params H2D overlapped with pass 1, the
    // gradient D2H with pass 2, on a second stream
    cudaStream_t cstream = nullptr;
    cudaEvent_t pev[4]{};
    cudaStream_t kst[NPART]{};             // pipelined host evaluation: part j of a pass runs on kst[j],
    cudaEvent_t pex[12]{};                 //   priority decreasing with j (upload / prep / part-done events)
    bool fconc = false;                    //   (concurrent parts, no drain at the boundaries)
    bool fconc2 = false;                   //   (pass 2 too)
    int xparts = 1;                        // exact-path lists of the last evaluation (pinned + 4)
    int *xbeg = nullptr;
    // pass 1 in parts: items [p1_b[j], p1_b[j+1]) need params layers [0, p1_l[j]); pass 2 in
    // parts: after items [0, p2_b[j+1]) the gradient layers [0, p2_l[j]) are final
    std::vector<int> p1_b, p1_l, p2_b, p2_l;
    int p1_split = 0, p2_split = 0;    // first part boundaries (stats; 0: not pipelined)
    float ms[5]{};
    double *pinned = nullptr;  // 2 doubles
    // bending energy / L-BFGS (srwcr_register.inc)
    double *bend_gram = nullptr;  // [3 axes][3 orders][Gmax][7] banded 1-D Gram matrices
    double *bend_ws = nullptr;    // 8 vectors of nparams: Hphi, Z0..Z2, A0..A2, staging
    double *dot_part = nullptr;   // deterministic dot-product partials
    double *dot_host = nullptr;   // pinned, 16 doubles
    int64_t gram_G = 0;
    // round-2 fast passes (coarse spatial lattice, orientation 0; srwcr_fast.cuh)
    bool fast = false;
    int fXV = 1, fW = 16, fS = 0, nfitems = 0;
    size_t fsmem1 = 0;
    FItem *fitems = nullptr;
    ItemW *fitemw = nullptr;
    int *fslotbins = nullptr, *fiflag = nullptr;
    unsigned *frec = nullptr, *floff = nullptr, *flent = nullptr;
    uint4 *frmask = nullptr;
    unsigned long long *SQi = nullptr;   // int64 statistics (units 2^-16), same layout as SQ
    unsigned long long *gradi = nullptr; // int64 gradient (units 2^-k of Z dD/dphi)
    int fW2 = 16, fnpmax = 0;
    size_t fsmem2 = 0;
    float fdxz = 1.f;
    std::vector<FItem> h_fitems;
    // split pass 1: sample half (k_p1w) -> plain m (fMv) -> moment half (k_p1f MODE 2)
    bool fsplit = false;
    float *fMv = nullptr;
    cudaArray_t fMarr = nullptr;            // M as a 2-D layered array (pass 1 textureGather)
    // pipelined host-buffer evaluation of the fast passes: pass 1 parts [fp1_b[j], fp1_b[j+1])
    // need params layers [0, fp1_l[j]); after pass-2 part j the gradient layers [0, fp2_l[j])
    // are final
    std::vector<int> fp1_b, fp1_l, fp2_b, fp2_l;
    float4 *fphi4 = nullptr;                // fp32 phi, one float4 (x, y, z, 0) per node
    std::vector<NBox> h_nboxes;             // whole-volume boxes of the deterministic static counts
    int fzmax = FZMAX;                      // the fast items' longest z-range (sizes the per-slice tables)
    cudaTextureObject_t ftexM = 0;
    int fWw = 8, fMinbW = 3;
    size_t fsmemw = 0;
};

static srwcr_status fail(srwcr_ctx *c, srwcr_status s, const char *fmt, ...) {
    if (c) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        c->err = buf;
        if (s == SRWCR_ECUDA) c->poisoned = true;
    }
    return s;
}

#define CK(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fail(c, SRWCR_ECUDA, "%s failed: %s (%s:%d)", #call,              \
                                           cudaGetErrorString(e_), __FILE__, __LINE__);                 \
    } while (0)
#define CKL()                                                                                           \
    do {                                                                                                \
        c->launches++;                                                                                  \
        cudaError_t e_ = cudaGetLastError();                                                            \
        if (e_ != cudaSuccess) return fail(c, SRWCR_ECUDA, "kernel launch failed: %s (%s:%d)",          \
                                           cudaGetErrorString(e_), __FILE__, __LINE__);                 \
    } while (0)
#define NCK(call)                                                                                       \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess) return fail(c, SRWCR_ENCCL, "%s failed: %s", #call,                      \
                                           nccl().GetErrorString(r_));                                  \
    } while (0)

#define CK0(call)                                   \
    do {                                            \
        if ((call) != cudaSuccess) return SRWCR_ECUDA; \
    } while (0)

#define TRY(x)                                \
    do {                                      \
        srwcr_status s_ = (x);                \
        if (s_ != SRWCR_OK) return s_;        \
    } while (0)

// ------------------------------------------------------------------ host tables
// Eq 8 pieces at t in [0,1), fp64
static void beta4(double t, double w[4]) {
    w[0] = (1.0 - t) * (1.0 - t) * (1.0 - t) / 6.0;
    w[1] = (3.0 * t * t * t - 6.0 * t * t + 4.0) / 6.0;
    w[2] = (-3.0 * t * t * t + 3.0 * t * t + 3.0 * t + 1.0) / 6.0;
    w[3] = t * t * t / 6.0;
}
// voxel index i on a lattice of spacing sp: base floor(i/sp), weights beta(i/sp - base)  (Eq 17)
static void build_axis(int64_t N, double sp, bool degenerate, std::vector<int> &base, std::vector<float4> &w,
                       std::vector<double4> *w64 = nullptr) {
    base.resize(N);
    w.resize(N);
    if (w64) w64->resize(N);
    for (int64_t i = 0; i < N; ++i) {
        double ww[4] = {1.0, 0.0, 0.0, 0.0};
        base[i] = 0;
        if (!degenerate) {
            double s = (double)i / sp, fl = std::floor(s);
            base[i] = (int)fl;
            beta4(s - fl, ww);
        }
        w[i] = make_float4((float)ww[0], (float)ww[1], (float)ww[2], (float)ww[3]);
        if (w64) (*w64)[i] = make_double4(ww[0], ww[1], ww[2], ww[3]);
    }
}

// runs of constant spatial base within [lo, hi), chunked to <= maxlen
static std::vector<std::pair<int, int>> runs(const std::vector<int> &sb, int lo, int hi, int maxlen) {
    std::vector<std::pair<int, int>> out;
    int s = lo;
    while (s < hi) {
        int e = s + 1;
        while (e < hi && sb[e] == sb[s]) ++e;
        int len = e - s, nch = (len + maxlen - 1) / maxlen;
        for (int k = 0; k < nch; ++k) {
            int a = s + (int)((long long)len * k / nch), b = s + (int)((long long)len * (k + 1) / nch);
            if (b > a) out.push_back({a, b - a});
        }
        s = e;
    }
    return out;
}

extern "C" srwcr_status srwcr_plan_slab(int64_t nz, int32_t nranks, int32_t rank, int64_t *z0, int64_t *z1) {
    if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z0 || !z1) return SRWCR_EINVAL;
    *z0 = nz * rank / nranks;
    *z1 = nz * (rank + 1) / nranks;
    return SRWCR_OK;
}

// touched node layers [t0, t1) of the slab [z0, z1): the bases of its first and last slice
// and the 3 further taps (Eq 17), clipped to the lattice
static void slab_layers(const int32_t *cbz, int64_t z0, int64_t z1, int64_t gz, int64_t &t0, int64_t &t1) {
    t0 = cbz[z0];
    t1 = std::min<int64_t>((int64_t)cbz[z1 - 1] + 4, gz);
}

extern "C" srwcr_status srwcr_plan_layers(int64_t nz, int32_t nranks, int32_t rank, const int32_t *cbz, int64_t gz,
                                          int64_t out[5]) {
    if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !cbz || gz < 1 || !out || nz < nranks)
        return SRWCR_EINVAL;
    for (int64_t z = 0; z < nz; ++z)
        if (cbz[z] < 0 || cbz[z] >= gz || (z > 0 && cbz[z] < cbz[z - 1])) return SRWCR_EINVAL;
    // owned layers of rank k: [t0_k, t0_{k+1}) (rank 0 from 0, the last rank to gz); valid
    // iff no rank's touched layers reach past its upper neighbour's owned range, so the only
    // exchange is rank k -> k + 1 (checked for every k: every rank reaches the same verdict)
    std::vector<int64_t> t0(nranks), t1(nranks);
    for (int k = 0; k < nranks; ++k) {
        int64_t z0, z1;
        srwcr_plan_slab(nz, nranks, k, &z0, &z1);
        slab_layers(cbz, z0, z1, gz, t0[k], t1[k]);
    }
    auto own0 = [&](int k) { return k == 0 ? (int64_t)0 : t0[k]; };
    auto own1 = [&](int k) { return k + 1 == nranks ? gz : t0[k + 1]; };
    for (int k = 0; k + 1 < nranks; ++k)
        if (t1[k] > own1(k + 1)) return SRWCR_EINVAL;
    out[0] = t0[rank];
    out[1] = t1[rank];
    out[2] = own0(rank);
    out[3] = own1(rank);
    out[4] = rank == 0 ? out[2] : std::max(out[2], t1[rank - 1]);
    return SRWCR_OK;
}

extern "C" srwcr_status srwcr_grad_layers(const srwcr_ctx *c, int64_t out[5]) {
    if (!c || !out) return SRWCR_EINVAL;
    if (c->g.ndim != 3 || c->lay[1] <= c->lay[0]) return SRWCR_ENOTSUP;
    for (int i = 0; i < 5; ++i) out[i] = c->lay[i];
    return SRWCR_OK;
}

extern "C" srwcr_status srwcr_default_options(srwcr_options *o) {
    if (!o) return SRWCR_EINVAL;
    memset(o, 0, sizeof *o);
    o->struct_size = (int32_t)sizeof *o;
    o->nranks = 1;
    o->eps_mass = 1e-12;
    o->eps_sigma = 1e-6;
    o->moment_shift = 1;
    o->use_graph = 1;
    return SRWCR_OK;
}

static bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static PassArgs pass_args(srwcr_ctx *c) {
    PassArgs a{};
    a.g = c->g;
    for (int i = 0; i < 3; ++i) {
        a.t.cb[i] = c->cb[i]; a.t.cw[i] = c->cw[i]; a.t.cw64[i] = c->cw64[i]; a.t.sb[i] = c->sb[i]; a.t.sw[i] = c->sw[i];
    }
    a.p64 = c->cur_params;
    a.F = c->F; a.M = c->M; a.phi = c->phi; a.shiftc = c->shiftc; a.items = c->items; a.itemw = c->itemw;
    a.tolw = reinterpret_cast<const float4 *>(c->phimax);
    a.MG = c->MG; a.mgz0 = (int)c->z0; a.mgz1 = (int)(c->z1 - c->z0);
    a.zrn = c->zrn;
    a.xlist = c->xlist; a.xcount = c->xcount; a.xcap = c->xcap;
    a.slotbins = c->slotbins; a.SQ = c->SQ; a.Qt = c->Qt; a.W = c->W; a.S = c->S; a.S2 = c->S2;
    a.NQ = c->NQ; a.gstride = c->gstride;
    a.alpha = c->alpha; a.beta = c->beta; a.gamma = c->gamma;
    a.invZ = (float)(1.0 / c->Z);
    a.grad = c->grad64;
    return a;
}

template <int XV>
static srwcr_status launch_pass1_t(srwcr_ctx *c, bool stat, bool full, int i0, int cnt) {
    PassArgs a = pass_args(c);
    int n = full ? c->nitems_full : c->nitems;
    a.items = (full ? c->items_full : c->items) + i0;
    a.itemw = (full ? c->itemw_full : c->itemw) + i0;
    n = cnt >= 0 ? cnt : n - i0;
    if (full) a.MG = nullptr;   // whole-volume create-time passes: no (m, dM/dy) output
    if (n == 0) return SRWCR_OK;
    if (XV == 1 && c->MC) {   // fine lattices: multi-cell items
        const bool small = c->W <= 6;
        if (stat && small) k_pass1<1, true, 192, 0, true><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
        else if (stat) k_pass1<1, true, 512, 0, true><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
        else if (small) k_pass1<1, false, 192, 0, true><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
        else k_pass1<1, false, 512, 0, true><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
    }
    else if (stat) k_pass1<XV, true><<<n, 32 * c->W, c->smem1, c->stream>>>(a);   // fixed-image bins (both orientations)
    else if (c->opt.orientation) k_pass1<XV, false, 512, 1><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
    else if (XV == 1 && c->W <= 6 && !getenv("SRWCR_NOSMALL")) k_pass1<1, false, 192><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
    else k_pass1<XV, false><<<n, 32 * c->W, c->smem1, c->stream>>>(a);
    CKL();
    return SRWCR_OK;
}
// full = true: whole volume (create-time static passes, identical on every rank)
static srwcr_status launch_pass1(srwcr_ctx *c, bool stat, bool full = false, int i0 = 0, int cnt = -1) {
    return c->XV == 2 ? launch_pass1_t<2>(c, stat, full, i0, cnt) : launch_pass1_t<1>(c, stat, full, i0, cnt);
}
// pass 2 over items2 [i0, i0 + cnt) (cnt < 0: to the end), then k_exact_fix over the list
// entries from *xbeg (xmode as in PassArgs); reset = zero the deferred-voxel count first
template <int XV>
static srwcr_status launch_pass2_t(srwcr_ctx *c, double *grad, int i0, int cnt, bool reset, const int *xbeg,
                                   int xmode) {
    PassArgs a = pass_args(c);
    a.grad = grad;
    a.items = c->items2 + i0;
    a.xbeg = xbeg;
    a.xmode = xmode;
    const int n = cnt >= 0 ? cnt : c->nitems2 - i0;
    if (n <= 0) return SRWCR_OK;
    a.W = c->W2;
    if (reset) CK(cudaMemsetAsync(c->xcount, 0, sizeof(int), c->stream));
    const int nitems2 = n;
    if (c->opt.orientation) {
        k_pass2<XV, 512, 1><<<nitems2, 32 * c->W2, c->smem2, c->stream>>>(a);
        CKL();
        k_exact_fix<1><<<1184, 128, 0, c->stream>>>(a);
    } else {
        if (XV == 1 && c->MC && c->W2 <= 6) k_pass2<1, 192, 0, true><<<nitems2, 32 * c->W2, c->smem2, c->stream>>>(a);
        else if (XV == 1 && c->MC) k_pass2<1, 512, 0, true><<<nitems2, 32 * c->W2, c->smem2, c->stream>>>(a);
        else if (XV == 1 && c->W2 <= 6 && !getenv("SRWCR_NOSMALL")) k_pass2<1, 192><<<nitems2, 32 * c->W2, c->smem2, c->stream>>>(a);
        else k_pass2<XV><<<nitems2, 32 * c->W2, c->smem2, c->stream>>>(a);
        CKL();
        k_exact_fix<0><<<1184, 128, 0, c->stream>>>(a);
    }
    CKL();
    return SRWCR_OK;
}
static srwcr_status launch_pass2(srwcr_ctx *c, double *grad, int i0 = 0, int cnt = -1, bool reset = true,
                                 const int *xbeg = nullptr, int xmode = 0) {
    return c->XV2 == 2 ? launch_pass2_t<2>(c, grad, i0, cnt, reset, xbeg, xmode)
                       : launch_pass2_t<1>(c, grad, i0, cnt, reset, xbeg, xmode);
}
// The dynamic-shared-memory ceiling is a per-kernel (process-wide) attribute: set it to the
// device's opt-in maximum so that contexts with different table sizes never race on it
// (each launch still requests exactly its own smem1 / smem2).
template <int XV>
static srwcr_status set_smem_t(int maxsm) {
    CK0(cudaFuncSetAttribute(k_pass1<XV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<XV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<XV, false, 512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass2<XV>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<1, false, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass2<1, 192>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<1, true, 192, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<1, true, 512, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<1, false, 192, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass1<1, false, 512, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass2<1, 192, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass2<1, 512, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    CK0(cudaFuncSetAttribute(k_pass2<XV, 512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    return SRWCR_OK;
}
static srwcr_status set_smem(srwcr_ctx *c) {
    int maxsm = 0;
    CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev));
    if (set_smem_t<1>(maxsm) != SRWCR_OK || set_smem_t<2>(maxsm) != SRWCR_OK)
        return fail(c, SRWCR_ECUDA, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize) failed");
    return SRWCR_OK;
}

// [SQ R][B][2] (ORI 1: then the dynamic counts NQ [R][B][2]) then the binless Q [R]
static size_t stats_count(const srwcr_ctx *c) {
    return (size_t)c->R * c->g.B * (c->opt.orientation ? 4 : 2) + (size_t)c->R;
}

static srwcr_status allreduce(srwcr_ctx *c, double *buf, size_t count) {
    if (c->comm) NCK(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream));
    return SRWCR_OK;
}

static srwcr_status run_combine(srwcr_ctx *c) {
    CombineArgs ca{};
    ca.SQ = c->SQ; ca.Qt = c->Qt; ca.Nlo = c->Nlo; ca.Nup = c->Nup; ca.shiftc = c->shiftc;
    ca.R = (int)c->R; ca.B = c->g.B; ca.Z = c->Z;
    ca.eps_mass = c->opt.eps_mass; ca.eps_sigma = c->opt.eps_sigma;
    ca.dterm = c->dterm; ca.reg = c->reg; ca.S_out = c->dump_S ? c->S_out : nullptr;
    ca.alpha = c->alpha; ca.beta = c->beta; ca.gamma = c->gamma;
    ca.NQ = c->NQ; ca.gstride = c->gstride;
    ca.ticket = c->ticket; ca.Dout = c->Dout; ca.part = c->dpart;   // D reduced by the launch's last CTA
    ca.gbound = c->Dout + 2;
    const unsigned nb = (unsigned)std::min<int64_t>((c->R + 7) / 8, 148 * 8);   // fixed grid (deterministic D)
    if (c->opt.orientation) k_combineA<<<nb, 256, 0, c->stream>>>(ca);
    else k_combine<<<nb, 256, 0, c->stream>>>(ca);
    CKL();
    return SRWCR_OK;
}


// ------------------------------------------------------------------ round-2 fast passes
// Items, static fixed-image records and per-line touched-slot lists of srwcr_fast.cuh.
// Eligible: 3-D, orientation 0, coarse spatial lattice (no multi-cell items), every
// x-chunk reading at most 32 control x-nodes.  SRWCR_NOFAST=1 keeps the round-1 passes.
// pass 1 keeps its per-slice tables at FZMAX (its row-offset stride is a compile-time
// constant: a runtime stride cost ~1 %); pass 2 sizes them by the items' z-range (room for its
// row-buffer copies)
static inline int P1ZM(int zm) { return LTC == 4 ? zm : FZMAX; }   // (4 line-table copies: room from the z-range)
static srwcr_status build_fast(srwcr_ctx *c, int nsm) {
    const Geo &g = c->g;
    if (getenv("SRWCR_NOFAST")) return SRWCR_OK;
    if (g.nz == 1 || c->opt.orientation != 0 || c->MC || c->z1 <= c->z0) return SRWCR_OK;
    int XV = c->XV;
    if (const char *e = getenv("SRWCR_FXV")) XV = std::min(XV, std::max(1, atoi(e)));
    // the split (rows and slices per item) is chosen on the WHOLE volume so that every rank of a
    // z-slab decomposition whose slab boundaries fall on spatial z-cells runs exactly the items
    // of the single-GPU decomposition that lie in its slab (bitwise-equal statistics sums)
    int ymax = 32, zmax = FZMAX;
    // at least 1.5 items per SM over the whole volume (times imul: SRWCR_FITEMS_MUL, experiments
    // with the z-slab decomposition, where each rank gets 1/P of them)
    int imul = 1;
    if (const char *e = getenv("SRWCR_FITEMS_MUL")) imul = std::max(1, atoi(e));
    auto make_items = [&](int zlo, int zhi) {
        std::vector<Item> out;
        auto xr = runs(c->h_sb[0], 0, g.nx, 32 * XV);
        auto yr = runs(c->h_sb[1], 0, g.ny, ymax);
        auto zr = runs(c->h_sb[2], zlo, zhi, zmax);
        for (auto &zz : zr)
            for (auto &yy : yr)
                for (auto &xx : xr) out.push_back(Item{xx.first, xx.second, yy.first, yy.second, zz.first, zz.second, 0, 0, 0.f, 0});
        return out;
    };
    for (;;) {
        const size_t nall = make_items(0, g.nz).size();
        if ((long long)nall * 2 < 3LL * nsm * imul && (ymax > 16 || zmax > 16)) {
            if (ymax > 16) ymax = 16;
            else zmax /= 2;
            continue;
        }
        break;
    }
    std::vector<Item> its = make_items((int)c->z0, (int)c->z1);
    if (its.empty()) return SRWCR_OK;
    for (const Item &it : make_items(0, g.nz)) c->h_nboxes.push_back(NBox{it.x0, it.xlen, it.y0, it.ylen, it.z0, it.zlen});
    int zm = 1;
    for (const Item &it : its) {
        const int nxn = c->h_cb[0][it.x0 + it.xlen - 1] + 4 - c->h_cb[0][it.x0];
        if (nxn > 32 || it.zlen > FZMAX) return SRWCR_OK;   // not eligible: round-1 passes
        zm = std::max(zm, it.zlen);
    }
    if (P1_TEX) {   // the layered copy of M (2-D layered limits: 32768 x 32768 x 2048)
        if (g.nx > 32768 || g.ny > 32768 || g.nz > 2048) return SRWCR_OK;
        cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
        CK(cudaMalloc3DArray(&c->fMarr, &cd, make_cudaExtent(g.nx, g.ny, g.nz), cudaArrayLayered));
        cudaMemcpy3DParms cp{};
        cp.srcPtr = make_cudaPitchedPtr(c->M, sizeof(float) * g.nx, g.nx, g.ny);
        cp.dstArray = c->fMarr;
        cp.extent = make_cudaExtent(g.nx, g.ny, g.nz);
        cp.kind = cudaMemcpyDeviceToDevice;
        CK(cudaMemcpy3DAsync(&cp, c->stream));
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeArray;
        rd.res.array.array = c->fMarr;
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeClamp;
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CK(cudaCreateTextureObject(&c->ftexM, &rd, &td, nullptr));
    }
    const size_t n = its.size();
    // per item: fixed bins present, binless shift, spatial weight sums
    Item *d_it = nullptr;
    unsigned *d_mask = nullptr;
    double *d_sum = nullptr;
    CK(cudaMalloc(&d_it, sizeof(Item) * n));
    CK(cudaMalloc(&d_mask, sizeof(unsigned) * 4 * n));
    CK(cudaMalloc(&d_sum, sizeof(double) * n));
    CK(h2d_sync(d_it, its.data(), sizeof(Item) * n));
    k_item_scan<<<(unsigned)n, 256, 0, c->stream>>>(c->F, c->M, d_it, g, d_mask, d_sum);
    CKL();
    std::vector<unsigned> mask(4 * n);
    std::vector<double> sum(n);
    CK(cudaMemcpyAsync(mask.data(), d_mask, sizeof(unsigned) * 4 * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(sum.data(), d_sum, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_it);
    cudaFree(d_mask);
    cudaFree(d_sum);
    std::vector<FItem> fi(n);
    std::vector<ItemW> w(n);
    std::vector<int> slotbins;
    long long lines = 0, rows = 0;
    int smax = 1;
    for (size_t i = 0; i < n; ++i) {
        const Item &it = its[i];
        FItem &f = fi[i];
        f.x0 = it.x0; f.xlen = it.xlen; f.y0 = it.y0; f.ylen = it.ylen; f.z0 = it.z0; f.zlen = it.zlen;
        f.slot_off = (int)slotbins.size();
        int ns = 0;
        for (int b = 0; b < g.B; ++b)
            if ((mask[4 * i + (b >> 5)] >> (b & 31)) & 1u) { slotbins.push_back(b); ++ns; }
        f.nslots = ns;
        smax = std::max(smax, ns);
        f.line_off = (int)lines;
        f.row_off = (int)rows;
        lines += (long long)it.ylen * it.zlen;
        rows += it.ylen;
        f.cI = (float)(sum[i] / ((double)it.xlen * it.ylen * it.zlen));
        f.pad = 0;
        ItemW &iw = w[i];
        for (int l = 0; l < 8; ++l) iw.sx[l] = iw.sz[l] = 0.0;
        for (int l = 0; l < 4; ++l) iw.sy[l] = 0.0;
        const int lo[3] = {it.x0, it.y0, it.z0}, len[3] = {it.xlen, it.ylen, it.zlen};
        double *dst[3] = {iw.sx, iw.sy, iw.sz};
        for (int ax = 0; ax < 3; ++ax)
            for (int k = lo[ax]; k < lo[ax] + len[ax]; ++k) {
                const float4 q = c->h_sw[ax][k];
                dst[ax][0] += q.x; dst[ax][1] += q.y; dst[ax][2] += q.z; dst[ax][3] += q.w;
            }
    }
    if (lines >= (1LL << 31) || smax + 2 > 255) return SRWCR_OK;
    const int S = smax + 2;   // + binless pseudo-slot + dummy slot of padding lanes
    int maxsm = 0;
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
    int W = 0;
    for (int Wc : {16, 12, 8, 4})
        if (!W && p1_smem(Wc, S, P1ZM(zm)).total <= maxsm) W = Wc;
    if (const char *e = getenv("SRWCR_FW")) {   // experiments: up to 24 warps (XV 1: <= 85 registers)
        const int w = std::max(1, atoi(e));
        if (w <= 16 || (XV == 1 && w <= 24 && p1_smem(w, S, P1ZM(zm)).total <= maxsm)) W = w;
    }
    if (W == 0) return SRWCR_OK;
    // device copies
    CK(cudaMalloc(&c->fitems, sizeof(FItem) * n));
    CK(h2d_sync(c->fitems, fi.data(), sizeof(FItem) * n));
    CK(cudaMalloc(&c->fitemw, sizeof(ItemW) * n));
    CK(h2d_sync(c->fitemw, w.data(), sizeof(ItemW) * n));
    CK(cudaMalloc(&c->fslotbins, sizeof(int) * std::max<size_t>(1, slotbins.size())));
    CK(h2d_sync(c->fslotbins, slotbins.data(), sizeof(int) * slotbins.size()));
    CK(cudaMalloc(&c->fiflag, sizeof(int) * n));
    CK(cudaMemset(c->fiflag, 0, sizeof(int) * n));
    const long long slab = (c->z1 - c->z0) * (long long)g.nxy;
    CK(cudaMalloc(&c->frec, sizeof(unsigned) * slab));
    k_frec<<<(unsigned)n, 256, 0, c->stream>>>(c->F, c->fitems, c->fslotbins, g, (int)c->z0, c->frec);
    CKL();
    // per-line lists: count, prefix sum on the host, write
    std::vector<int> iol(lines);
    for (size_t i = 0; i < n; ++i)
        for (long long k = 0; k < (long long)fi[i].ylen * fi[i].zlen; ++k) iol[fi[i].line_off + k] = (int)i;
    int *d_iol = nullptr;
    unsigned *d_cnt = nullptr;
    CK(cudaMalloc(&d_iol, sizeof(int) * lines));
    CK(cudaMalloc(&d_cnt, sizeof(unsigned) * lines));
    CK(h2d_sync(d_iol, iol.data(), sizeof(int) * lines));
    CK(cudaMalloc(&c->frmask, sizeof(uint4) * rows));
    CK(cudaMemset(c->frmask, 0, sizeof(uint4) * rows));
    const unsigned lb = (unsigned)((lines * 32 + 255) / 256);
    if (XV == 2) k_lists<2><<<lb, 256, 0, c->stream>>>(c->frec, c->fitems, (int)n, g, (int)c->z0, d_iol, d_cnt, nullptr, nullptr, nullptr, lines, 0);
    else k_lists<1><<<lb, 256, 0, c->stream>>>(c->frec, c->fitems, (int)n, g, (int)c->z0, d_iol, d_cnt, nullptr, nullptr, nullptr, lines, 0);
    CKL();
    std::vector<unsigned> cnt(lines), off(lines + 1);
    CK(cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(unsigned) * lines, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    off[0] = 0;
    for (long long i = 0; i < lines; ++i) off[i + 1] = off[i] + cnt[i];
    CK(cudaMalloc(&c->floff, sizeof(unsigned) * (lines + 1)));
    CK(h2d_sync(c->floff, off.data(), sizeof(unsigned) * (lines + 1)));
    CK(cudaMalloc(&c->flent, sizeof(unsigned) * std::max<unsigned>(1, off[lines])));
    if (XV == 2) k_lists<2><<<lb, 256, 0, c->stream>>>(c->frec, c->fitems, (int)n, g, (int)c->z0, d_iol, nullptr, c->floff, c->flent, reinterpret_cast<unsigned *>(c->frmask), lines, 1);
    else k_lists<1><<<lb, 256, 0, c->stream>>>(c->frec, c->fitems, (int)n, g, (int)c->z0, d_iol, nullptr, c->floff, c->flent, reinterpret_cast<unsigned *>(c->frmask), lines, 1);
    CKL();
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_iol);
    cudaFree(d_cnt);
    CK(cudaMalloc(&c->SQi, sizeof(unsigned long long) * stats_count(c)));
    CK(cudaMemset(c->SQi, 0, sizeof(unsigned long long) * stats_count(c)));
    c->fXV = XV;
    c->fW = W;
    c->fS = S;
    c->nfitems = (int)n;
    c->fsmem1 = p1_smem(W, S, P1ZM(zm)).total;
    c->fzmax = zm;
    c->h_fitems = fi;
    // pipelined host-buffer evaluation (one rank).  Items are ordered by z, so every part
    // boundary is a layer prefix.  Concurrent parts (default): see below.  Serial parts
    // (SRWCR_PIPE_CONC=0): pass 1 in parts of one wave, one wave, the rest; pass 2 as all but
    // two waves, then one wave at a time (each boundary drains a wave, so only for >= 6 waves).
    if (c->nranks == 1 && !getenv("SRWCR_NOPIPE")) {
        int wave = nsm;
        if (const char *e = getenv("SRWCR_PIPE_WAVE")) wave = std::max(1, atoi(e));   // tests: small volumes
        const int nn = (int)n;
        c->fconc = !getenv("SRWCR_PIPE_CONC") || atoi(getenv("SRWCR_PIPE_CONC")) != 0;
        c->fconc2 = c->fconc && (!getenv("SRWCR_PIPE_CONC2") || atoi(getenv("SRWCR_PIPE_CONC2")) != 0);
        int q0 = 0;   // items of the first z-run
        while (q0 < nn && fi[q0].z0 == fi[0].z0) ++q0;
        if (c->fconc ? (nn >= wave && nn >= 3 * q0) : nn >= 6 * wave) {
            const int np = std::min(4, std::max(2, atoi(getenv("SRWCR_PIPE_P1") ? getenv("SRWCR_PIPE_P1") : "2")));
            std::vector<int> b = {0}, l;
            if (c->fconc) {
                // concurrent parts (each on its own stream: a part's items fill the SMs the
                // previous part's last wave leaves, so a boundary costs no drain): q, q, 2q items
                // and the rest, q = the items of the first z-run (its layers go up first)
                int q = 0;
                while (q < nn && fi[q].z0 == fi[0].z0) ++q;
                if (const char *e = getenv("SRWCR_PIPE_Q")) q = std::max(1, atoi(e));
                for (int k : {q, 2 * q, 4 * q})
                    if (k < nn) b.push_back(k);
            } else {
                for (int k = 1; k < np; ++k) b.push_back(k * wave);
            }
            b.push_back(nn);
            for (size_t j = 0; j + 1 < b.size(); ++j) {
                int hi = 0;
                for (int i = 0; i < b[j + 1]; ++i) hi = std::max(hi, c->h_cb[2][fi[i].z0 + fi[i].zlen - 1] + 4);
                l.push_back(std::min(hi, g.GzExt));
            }
            l.back() = g.GzExt;
            c->fp1_b = b;
            c->fp1_l = l;
            const int np2 = std::min(5, std::max(2, atoi(getenv("SRWCR_PIPE_P2") ? getenv("SRWCR_PIPE_P2") : "3")));
            // (C5 e2e, pass-1 / pass-2 parts: 3/4 372.6, 2/4 375.0, 3/3 375.6, 3/2 377.6, 2/2
            // 380.1 evals/s; 351.5 without the parts: each part boundary drains a wave; with 2
            // pass-1 parts, pass-2 parts / first boundary in waves from the end: 2/1 378.9,
            // 2/2 381.6, 3/2 383.9, 3/3 381.3)
            // the first pass-2 boundary sits k2 waves before the end (its final layers go back while
            // the last k2 waves run), later ones one wave apart
            const int k2 = std::max(np2 - 1, atoi(getenv("SRWCR_PIPE_P2K") ? getenv("SRWCR_PIPE_P2K") : "2"));
            std::vector<int> b2 = {0}, l2;
            if (c->fconc2) {
                // concurrent parts: the last five z-runs of items one by one (the fewest
                // layers go back after the last kernel, the first ones early), the rest.
                // (C5 e2e, evals/s: serial parts 397; concurrent pass-1 parts 410; + concurrent
                // pass-2 parts, trailing z-runs 1 / 2 / 3 / 5 / 7: 398 / 409 / 421 / 437 / 421 --
                // 7 exceeds the device's 6 stream priorities; without
                // cudaGraphInstantiateFlagUseNodePriority the graph ignores them: 402)
                int q = 0;
                while (q < nn && fi[nn - 1 - q].z0 == fi[nn - 1].z0) ++q;
                if (const char *e = getenv("SRWCR_PIPE_Q2")) q = std::max(1, atoi(e));
                const int nt = std::min(NPART - 1, std::max(1, atoi(getenv("SRWCR_PIPE_P2N") ? getenv("SRWCR_PIPE_P2N") : "5")));
                for (int k = nt; k >= 1; --k)
                    if (nn - k * q > b2.back()) b2.push_back(nn - k * q);
            } else {
                b2.push_back(nn - k2 * wave);
                for (int k = np2 - 2; k >= 1; --k) b2.push_back(nn - k * wave);
            }
            b2.push_back(nn);
            for (size_t j = 0; j + 1 < b2.size(); ++j) {
                int lo = g.GzExt;
                for (int i = b2[j + 1]; i < nn; ++i) lo = std::min(lo, c->h_cb[2][fi[i].z0]);
                l2.push_back(lo);
            }
            l2.back() = g.GzExt;
            for (size_t j = 1; j < l2.size(); ++j) l2[j] = std::max(l2[j], l2[j - 1]);
            c->fp2_b = b2;
            c->fp2_l = l2;
        }
    }
    // split pass 1 (SRWCR_SPLIT=0/1 overrides the default).  Measured on C5 (c18/c19): the
    // halves take 0.82 ms (k_p1w) + 0.87 ms (k_p1f MODE 2) against 1.60 ms fused: off
    c->fsplit = false;
    if (const char *e = getenv("SRWCR_SPLIT")) c->fsplit = atoi(e) != 0;
    if (const char *e = getenv("SRWCR_P1W_MINB")) c->fMinbW = atoi(e) == 2 ? 2 : 3;
    if (const char *e = getenv("SRWCR_P1W_W")) c->fWw = std::min(16, std::max(1, atoi(e)));
    // the split variant's m array (4 B/voxel) only when SRWCR_SPLIT is set at create (then it
    // is re-read per launch: the fused-vs-split test toggles it on one context)
    if (c->fsplit || getenv("SRWCR_SPLIT")) CK(cudaMalloc(&c->fMv, sizeof(float) * slab));
    CK(cudaMalloc(&c->fphi4, sizeof(float4) * (size_t)g.Gx * g.Gy * g.Gz));
    CK(cudaMemset(c->fphi4, 0, sizeof(float4) * (size_t)g.Gx * g.Gy * g.Gz));
    c->fsmemw = p1w_smem(c->fWw, zm).total;
    // pass 2: node window and warps per CTA
    int npmax = 0;
    for (const FItem &f : fi) {
        const int nxn = c->h_cb[0][f.x0 + f.xlen - 1] + 4 - c->h_cb[0][f.x0];
        const int nyn = c->h_cb[1][f.y0 + f.ylen - 1] + 4 - c->h_cb[1][f.y0];
        const int nzn = c->h_cb[2][f.z0 + f.zlen - 1] + 4 - c->h_cb[2][f.z0];
        npmax = std::max(npmax, nzn * 3 * nyn * nxn);
    }
    int W2 = 0;
    for (int Wc : {16, 12, 8, 4})
        if (!W2 && p2_smem(Wc, S, npmax, zm).total <= maxsm) W2 = Wc;
    if (const char *e = getenv("SRWCR_FW2")) W2 = std::min(W2, std::max(1, atoi(e)));
    if (W2 == 0) return SRWCR_OK;
    c->fW2 = W2;
    c->fnpmax = npmax;
    c->fsmem2 = p2_smem(W2, S, npmax, zm).total;
    c->fdxz = (float)((std::ceil(c->delta[0]) + 1.0) * (std::ceil(c->delta[2]) + 1.0));
    CK(cudaMalloc(&c->gradi, sizeof(unsigned long long) * c->nparams));
    CK(cudaMemset(c->gradi, 0, sizeof(unsigned long long) * c->nparams));
    {
        // the attribute is per function and process-wide: every context sets the device maximum
        // (a context-sized value would break the launches of an earlier context with larger
        // tables, e.g. several z-slab ranks in one process)
        const int sm = maxsm;
        const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
        if (XV == 2) {
            CK(cudaFuncSetAttribute(k_p2f<2, 512>, attr, sm));
            CK(cudaFuncSetAttribute(k_p2f<2, 384>, attr, sm));
            CK(cudaFuncSetAttribute(k_p2f<2, 256>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 512>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 384>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 256>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 512, 2>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 384, 2>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<2, 256, 2>, attr, sm));
        } else {
            CK(cudaFuncSetAttribute(k_p2f<1, 512>, attr, sm));
            CK(cudaFuncSetAttribute(k_p2f<1, 384>, attr, sm));
            CK(cudaFuncSetAttribute(k_p2f<1, 256>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 512, 2>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 384, 2>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 256, 2>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 768>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 512>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 384>, attr, sm));
            CK(cudaFuncSetAttribute(k_p1f<1, 256>, attr, sm));
        }
    }
    c->fast = true;
    return SRWCR_OK;
}

static FArgs fast_args(srwcr_ctx *c) {
    FArgs a{};
    a.g = c->g;
    for (int i = 0; i < 3; ++i) {
        a.t.cb[i] = c->cb[i]; a.t.cw[i] = c->cw[i]; a.t.cw64[i] = c->cw64[i]; a.t.sb[i] = c->sb[i]; a.t.sw[i] = c->sw[i];
    }
    a.M = c->M; a.phi = c->phi; a.phi4 = c->fphi4; a.rec = c->frec; a.loff = c->floff; a.lent = c->flent; a.rmask = c->frmask;
    a.items = c->fitems; a.itemw = c->fitemw; a.slotbins = c->fslotbins; a.iflag = c->fiflag; a.shiftc = c->shiftc;
    a.SQi = c->SQi; a.Qi = c->SQi + (size_t)c->R * c->g.B * 2;
    a.MG = c->MG; a.Mv = c->fMv; a.mgz0 = (int)c->z0;
    a.texM = (unsigned long long)c->ftexM;
    a.S = c->fS; a.W = c->fW; a.i0 = 0;
    a.L1 = p1_smem(c->fW, c->fS, P1ZM(c->fzmax));
    a.ablate = 0;
    if (const char *e = getenv("SRWCR_ABLATE")) a.ablate = atoi(e);
    return a;
}

// fast pass 1 over items [i0, i0 + cnt) and the int64 -> fp64 statistics conversion
static srwcr_status launch_fast_pass1(srwcr_ctx *c, int i0 = 0, int cnt = -1, bool convert = true, cudaStream_t st = nullptr) {
    cudaStream_t ks = st ? st : c->stream;
    FArgs a = fast_args(c);
    a.i0 = i0;
    const int n = cnt >= 0 ? cnt : c->nfitems - i0;
    bool split = c->fsplit;
    if (const char *e = getenv("SRWCR_SPLIT")) split = atoi(e) != 0;   // experiments / the fused-vs-split test
    split = split && c->fMv != nullptr;
    if (n > 0 && split) {
        // sample half, then the moment half (same items)
        FArgs aw = a;
        aw.W = c->fWw;
        aw.L1 = p1w_smem(c->fWw, c->fzmax);
        const int Tw = 32 * c->fWw, T = 32 * c->fW;
        const size_t smw = c->fsmemw;
        if (c->fXV == 2) {
            if (Tw <= 256 && c->fMinbW == 3) k_p1w<2, 256, 3><<<n, Tw, smw, ks>>>(aw);
            else if (Tw <= 256) k_p1w<2, 256, 2><<<n, Tw, smw, ks>>>(aw);
            else k_p1w<2, 512, 1><<<n, Tw, smw, ks>>>(aw);
            CKL();
            if (T > 384) k_p1f<2, 512, 2><<<n, T, c->fsmem1, ks>>>(a);
            else if (T > 256) k_p1f<2, 384, 2><<<n, T, c->fsmem1, ks>>>(a);
            else k_p1f<2, 256, 2><<<n, T, c->fsmem1, ks>>>(a);
        } else {
            if (Tw <= 256 && c->fMinbW == 3) k_p1w<1, 256, 3><<<n, Tw, smw, ks>>>(aw);
            else if (Tw <= 256) k_p1w<1, 256, 2><<<n, Tw, smw, ks>>>(aw);
            else k_p1w<1, 512, 1><<<n, Tw, smw, ks>>>(aw);
            CKL();
            if (T > 384) k_p1f<1, 512, 2><<<n, T, c->fsmem1, ks>>>(a);
            else if (T > 256) k_p1f<1, 384, 2><<<n, T, c->fsmem1, ks>>>(a);
            else k_p1f<1, 256, 2><<<n, T, c->fsmem1, ks>>>(a);
        }
        CKL();
    } else if (n > 0) {
        const int T = 32 * c->fW;
        if (c->fXV == 2) {
            if (T > 384) k_p1f<2, 512><<<n, T, c->fsmem1, ks>>>(a);
            else if (T > 256) k_p1f<2, 384><<<n, T, c->fsmem1, ks>>>(a);
            else k_p1f<2, 256><<<n, T, c->fsmem1, ks>>>(a);
        } else {
            if (T > 512) k_p1f<1, 768><<<n, T, c->fsmem1, ks>>>(a);
            else if (T > 384) k_p1f<1, 512><<<n, T, c->fsmem1, ks>>>(a);
            else if (T > 256) k_p1f<1, 384><<<n, T, c->fsmem1, ks>>>(a);
            else k_p1f<1, 256><<<n, T, c->fsmem1, ks>>>(a);
        }
        CKL();
    }
    if (convert) {
        k_stats_convert<<<592, 256, 0, c->stream>>>(c->SQi, c->SQ, (long long)stats_count(c), (long long)c->R * c->g.B * 2);
        CKL();
    }
    return SRWCR_OK;
}

// per-eval flags of the fast items (the fp32 phi itself comes from k_prep_phi_wx)
static srwcr_status launch_fast_prep(srwcr_ctx *c, const double *pd) {
    Tables t{};
    for (int i = 0; i < 3; ++i) { t.cb[i] = c->cb[i]; t.cw[i] = c->cw[i]; t.sb[i] = c->sb[i]; t.sw[i] = c->sw[i]; }
    const int nconv = 296;   // blocks converting the params layers [pz0, pz1) to fp32; then one per item
    k_fprep<<<(unsigned)(nconv + c->nfitems), 256, 0, c->stream>>>(pd, c->fphi4, c->g, c->pz0, c->pz1, nconv, c->fitems,
                                                                    c->nfitems, t, c->fiflag);
    CKL();
    return SRWCR_OK;
}

// fast pass 2 (+ the fp64 exact-path voxels, + the int64 -> fp64 gradient conversion)
static F2Args fast_pass2_args(srwcr_ctx *c) {
    F2Args A{};
    A.f = fast_args(c);
    A.MG = c->MG;
    A.alpha = c->alpha; A.beta = c->beta; A.gamma = c->gamma;
    A.gbound = c->Dout + 2;
    A.dxz = c->fdxz;
    A.gradi = c->gradi;
    A.xlist = c->xlist; A.xcount = c->xcount; A.xcap = c->xcap;
    A.npmax = c->fnpmax;
    A.f.W = c->fW2;
    A.L2 = p2_smem(c->fW2, c->fS, c->fnpmax, c->fzmax);
    return A;
}
static srwcr_status launch_fast_p2f(srwcr_ctx *c, const F2Args &A0, int i0, int n, cudaStream_t st = nullptr) {
    if (n <= 0) return SRWCR_OK;
    F2Args A = A0;
    A.f.i0 = i0;
    const int T = 32 * c->fW2;
    cudaStream_t ks = st ? st : c->stream;
    if (c->fXV == 2) {
        if (T > 384) k_p2f<2, 512><<<n, T, c->fsmem2, ks>>>(A);
        else if (T > 256) k_p2f<2, 384><<<n, T, c->fsmem2, ks>>>(A);
        else k_p2f<2, 256><<<n, T, c->fsmem2, ks>>>(A);
    } else {
        if (T > 384) k_p2f<1, 512><<<n, T, c->fsmem2, ks>>>(A);
        else if (T > 256) k_p2f<1, 384><<<n, T, c->fsmem2, ks>>>(A);
        else k_p2f<1, 256><<<n, T, c->fsmem2, ks>>>(A);
    }
    CKL();
    return SRWCR_OK;
}
// Halo gradient exchange: instead of the all-reduce of the whole int64
// gradient, rank k sends its partial on the layers [o1, t1) that rank k + 1 owns and receives
// rank k - 1's partial on its own layers [o0, r1) (srwcr_plan_layers: no other rank touches
// them), adds it and zeroes every layer it does not own.  Integer adds of the same two
// partials: the owned layers hold the all-reduce's bits; the rank gradients partition the
// full gradient.  One ncclSend / ncclRecv per component (the layers of one component are
// contiguous), grouped; captured in the evaluation graph like the all-reduce.
static srwcr_status halo_exchange(srwcr_ctx *c) {
    const Geo &g = c->g;
    const long long plane = (long long)g.Gx * g.Gy;
    const long long t1 = c->lay[1], o0 = c->lay[2], o1 = c->lay[3], r1 = c->lay[4];
    const long long nsend = std::max(0LL, t1 - o1), nrecv = r1 - o0;
    NCK(nccl().GroupStart());
    for (int d = 0; d < g.ndim; ++d) {
        if (nsend > 0 && c->rank + 1 < c->nranks)
            NCK(nccl().Send(c->gradi + ((long long)d * g.Gz + o1) * plane, (size_t)(nsend * plane), ncclInt64,
                            c->rank + 1, c->comm, c->stream));
        if (nrecv > 0 && c->rank > 0)
            NCK(nccl().Recv(c->halo_recv + (long long)d * nrecv * plane, (size_t)(nrecv * plane), ncclInt64,
                            c->rank - 1, c->comm, c->stream));
    }
    NCK(nccl().GroupEnd());
    const long long t0 = std::min<long long>(c->lay[0], o0), hi = std::max<long long>(t1, o1);
    k_halo_finish<<<592, 256, 0, c->stream>>>(reinterpret_cast<long long *>(c->gradi), c->halo_recv, g.ndim, g.Gz,
                                               plane, t0, hi, o0, o1, c->rank > 0 ? r1 : o0);
    CKL();
    return SRWCR_OK;
}

static srwcr_status launch_fast_pass2(srwcr_ctx *c, double *grad, bool reduce_int64 = false) {
    F2Args A{};
    A.f = fast_args(c);
    A.MG = c->MG;
    A.alpha = c->alpha; A.beta = c->beta; A.gamma = c->gamma;
    A.gbound = c->Dout + 2;
    A.dxz = c->fdxz;
    A.gradi = c->gradi;
    A.xlist = c->xlist; A.xcount = c->xcount; A.xcap = c->xcap;
    A.npmax = c->fnpmax;
    A.f.W = c->fW2;
    A.L2 = p2_smem(c->fW2, c->fS, c->fnpmax, c->fzmax);
    CK(cudaMemsetAsync(c->xcount, 0, sizeof(int), c->stream));
    const int n = c->nfitems, T = 32 * c->fW2;
    if (c->fXV == 2) {
        if (T > 384) k_p2f<2, 512><<<n, T, c->fsmem2, c->stream>>>(A);
        else if (T > 256) k_p2f<2, 384><<<n, T, c->fsmem2, c->stream>>>(A);
        else k_p2f<2, 256><<<n, T, c->fsmem2, c->stream>>>(A);
    } else {
        if (T > 384) k_p2f<1, 512><<<n, T, c->fsmem2, c->stream>>>(A);
        else if (T > 256) k_p2f<1, 384><<<n, T, c->fsmem2, c->stream>>>(A);
        else k_p2f<1, 256><<<n, T, c->fsmem2, c->stream>>>(A);
    }
    CKL();
    PassArgs pa = pass_args(c);
    pa.invZ = 1.f;              // the int64 gradient holds Z dD/dphi
    pa.gradi = c->gradi;
    pa.gbound = c->Dout + 2;
    pa.dxz = c->fdxz;
    k_exact_fix<0><<<1184, 128, 0, c->stream>>>(pa);
    CKL();
    // z-slabs: the int64 gradient partials are summed across ranks before the conversion
    // (exact: the same gradient bits for every rank count)
    if (reduce_int64 && c->halo) TRY(halo_exchange(c));
    else if (reduce_int64) NCK(nccl().AllReduce(c->gradi, c->gradi, (size_t)c->nparams, ncclInt64, ncclSum, c->comm, c->stream));
    k_grad_convert<<<592, 256, 0, c->stream>>>(c->gradi, grad, (long long)c->nparams, c->Dout + 2, c->fdxz, 1.0 / c->Z);
    CKL();
    return SRWCR_OK;
}

static srwcr_status create_impl(srwcr_ctx *c, const float *fixed, const float *moving, const int64_t dims[3],
                                const double sp[3], int32_t bins, const int32_t sbins[3], const double csp[3]) {
    const srwcr_options &o = c->opt;
    if (!fixed) return fail(c, SRWCR_EINVAL, "fixed is NULL");
    if (!moving) return fail(c, SRWCR_EINVAL, "moving is NULL");
    if (!dims || !sp || !sbins || !csp) return fail(c, SRWCR_EINVAL, "dims/spacing_mm/spatial_bins/control_spacing_mm is NULL");
    if (dims[0] < 2 || dims[1] < 2 || dims[2] < 1) return fail(c, SRWCR_EINVAL, "dims: need Nx >= 2, Ny >= 2, Nz >= 1");
    if (dims[0] > (1 << 20) || dims[1] > (1 << 20) || dims[2] > (1 << 20)) return fail(c, SRWCR_EINVAL, "dims too large");
    if (dims[0] * dims[1] * dims[2] > INT32_MAX)   // the passes index voxels with 32-bit offsets
        return fail(c, SRWCR_EINVAL, "volume too large: %lld voxels, at most 2^31 - 1",
                    (long long)(dims[0] * dims[1] * dims[2]));
    if (bins < 2 || bins > 128) return fail(c, SRWCR_EINVAL, "intensity_bins must be in [2, 128], got %d", bins);
    if (o.orientation != 0 && o.orientation != 1) return fail(c, SRWCR_EINVAL, "orientation must be 0 or 1");
    if (o.nranks < 1 || o.rank < 0 || o.rank >= o.nranks) return fail(c, SRWCR_EINVAL, "rank/nranks out of range");
    for (int i = 0; i < 3; ++i) {
        if (!(sp[i] > 0)) return fail(c, SRWCR_EINVAL, "spacing_mm[%d] must be > 0", i);
        if (!(csp[i] > 0)) return fail(c, SRWCR_EINVAL, "control_spacing_mm[%d] must be > 0", i);
        if (sbins[i] < 0 || sbins[i] > dims[i]) return fail(c, SRWCR_EINVAL, "spatial_bins[%d] must be in [0, dims]", i);
    }
    const bool is2d = dims[2] == 1;
    Geo &g = c->g;
    g.nx = (int)dims[0]; g.ny = (int)dims[1]; g.nz = (int)dims[2];
    g.nxy = (long long)g.nx * g.ny;
    g.L = bins - 1; g.B = bins;
    g.ndim = is2d ? 2 : 3;
    int64_t G[3];
    for (int i = 0; i < 3; ++i) {
        c->delta[i] = csp[i] / sp[i];
        G[i] = (is2d && i == 2) ? 1 : (int64_t)std::floor((double)(dims[i] - 1) / c->delta[i]) + 4;
        c->kcells[i] = (is2d && i == 2) ? 0 : sbins[i];
    }
    for (int i = 0; i < 2 + !is2d; ++i)
        if (c->delta[i] < 1.2) return fail(c, SRWCR_EINVAL, "control spacing along axis %d is %.3f voxels; >= 1.2 required", i, c->delta[i]);
    g.Gx = (int)G[0]; g.Gy = (int)G[1]; g.GzExt = (int)G[2];
    g.nxy32 = (int)g.nxy;
    g.nxm2 = std::max(g.nx - 2, 0); g.nym2 = std::max(g.ny - 2, 0); g.nzm2 = std::max(g.nz - 2, 0);
    g.dzo = g.nz > 1 ? g.nxy32 : 0;
    g.Gz = is2d ? 4 : (int)G[2];
    g.Kx = c->kcells[0] > 0 ? c->kcells[0] + 3 : 4;
    g.Ky = c->kcells[1] > 0 ? c->kcells[1] + 3 : 4;
    g.Kz = c->kcells[2] > 0 ? c->kcells[2] + 3 : 4;
    c->R = (int64_t)g.Kx * g.Ky * g.Kz;
    c->nparams = (int64_t)g.ndim * G[0] * G[1] * G[2];
    c->nint = 3LL * g.Gx * g.Gy * g.Gz;
    c->pz0 = 0; c->pzb1 = g.Gz; c->pz1 = g.Gz;   // refined below once the slab and tap tables exist

    c->dev = o.device;
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (int i = 0; i < 5; ++i) CK(cudaEventCreate(&c->ev[i]));
    CK(cudaMallocHost(&c->pinned, (4 + NPART / 2) * sizeof(double)));   // a copy of Dout (D, #retained, ..., counts)
    CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 4; ++i) CK(cudaEventCreateWithFlags(&c->pev[i], cudaEventDisableTiming));
    {   // part streams: the earlier part's CTAs are dispatched first, a later part fills the SMs
        // its last wave leaves
        int least = 0, greatest = 0;
        CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        for (int i = 0; i < NPART; ++i)
            CK(cudaStreamCreateWithPriority(&c->kst[i], cudaStreamNonBlocking, std::min(least, greatest + i)));
    }
    for (int i = 0; i < 12; ++i) CK(cudaEventCreateWithFlags(&c->pex[i], cudaEventDisableTiming));
    CK(cudaMalloc(&c->xbeg, sizeof(int)));
    memset(c->pinned, 0, (4 + NPART / 2) * sizeof(double));

    // per-axis tables (fp64 on host -> device), control and spatial lattices
    for (int ax = 0; ax < 3; ++ax) {
        std::vector<float4> w;
        std::vector<double4> w64;
        build_axis(dims[ax], c->delta[ax], is2d && ax == 2, c->h_cb[ax], w, &w64);
        CK(cudaMalloc(&c->cb[ax], sizeof(int) * dims[ax]));
        CK(cudaMalloc(&c->cw[ax], sizeof(float4) * dims[ax]));
        CK(cudaMalloc(&c->cw64[ax], sizeof(double4) * dims[ax]));
        CK(h2d_sync(c->cw64[ax], w64.data(), sizeof(double4) * dims[ax]));
        CK(h2d_sync(c->cb[ax], c->h_cb[ax].data(), sizeof(int) * dims[ax]));
        CK(h2d_sync(c->cw[ax], w.data(), sizeof(float4) * dims[ax]));
        const bool deg = c->kcells[ax] == 0;
        c->Delta[ax] = deg ? 0.0 : (double)dims[ax] / (double)c->kcells[ax];
        build_axis(dims[ax], c->Delta[ax], deg, c->h_sb[ax], w);
        c->h_sw[ax] = w;
        CK(cudaMalloc(&c->sb[ax], sizeof(int) * dims[ax]));
        CK(cudaMalloc(&c->sw[ax], sizeof(float4) * dims[ax]));
        CK(h2d_sync(c->sb[ax], c->h_sb[ax].data(), sizeof(int) * dims[ax]));
        CK(h2d_sync(c->sw[ax], w.data(), sizeof(float4) * dims[ax]));
    }
    // max lanes sharing a control x-base inside a 32-lane chunk -> segmented-reduction steps
    // volumes: upload (host or device source) and normalise
    const long long nvox = (long long)g.nx * g.ny * g.nz;
    CK(cudaMalloc(&c->F, sizeof(float) * nvox));
    CK(cudaMalloc(&c->M, sizeof(float) * nvox));
    float *raw = nullptr;
    CK(cudaMalloc(&raw, sizeof(float) * nvox));
    int *mm = nullptr;
    CK(cudaMalloc(&mm, 2 * sizeof(int)));
    for (int v = 0; v < 2; ++v) {
        const float *src = v == 0 ? fixed : moving;
        float *dst = v == 0 ? c->F : c->M;
        CK(cudaMemcpy(raw, src, sizeof(float) * nvox, cudaMemcpyDefault));
        int init[2] = {0x7f800000, (int)(0xff800000u ^ 0x7fffffffu)};
        CK(h2d_sync(mm, init, sizeof init));
        k_minmax<<<296, 256>>>(raw, nvox, reinterpret_cast<float *>(mm));
        CKL();
        int key[2];
        CK(cudaMemcpy(key, mm, sizeof key, cudaMemcpyDeviceToHost));
        float lohi[2];
        for (int k = 0; k < 2; ++k) {
            int bits = key[k] >= 0 ? key[k] : key[k] ^ 0x7fffffff;
            memcpy(&lohi[k], &bits, 4);
        }
        if (!std::isfinite(lohi[0]) || !std::isfinite(lohi[1]))
            return fail(c, SRWCR_EINVAL, "%s contains non-finite values", v == 0 ? "fixed" : "moving");
        if (o.inputs_normalized) {
            if (lohi[0] < 0.f || lohi[1] > (float)g.L)
                return fail(c, SRWCR_EINVAL, "%s not in [0, L=%d] although inputs_normalized = 1", v == 0 ? "fixed" : "moving", g.L);
            CK(cudaMemcpy(dst, raw, sizeof(float) * nvox, cudaMemcpyDeviceToDevice));
        } else {
            const double lo = lohi[0], hi = lohi[1];
            const bool constant = !(hi > lo);
            const double scale = constant ? 0.0 : (double)g.L / (hi - lo);
            k_normalize<<<1184, 256>>>(raw, dst, nvox, lo, scale, (float)g.L, constant ? 1 : 0);
            CKL();
        }
    }
    CK(cudaDeviceSynchronize());
    cudaFree(raw);
    cudaFree(mm);

    // z-slab of this rank and the work items (each inside one spatial cell)
    c->nranks = o.nranks;
    c->rank = o.rank;
    srwcr_plan_slab(g.nz, c->nranks, c->rank, &c->z0, &c->z1);
    if (c->z1 > c->z0 && !is2d) {   // node layers read by the slab's taps (3 beyond the last base)
        c->pz0 = c->h_cb[2][c->z0];
        c->pzb1 = c->h_cb[2][c->z1 - 1] + 1;
        c->pz1 = std::min(c->h_cb[2][c->z1 - 1] + 4, g.Gz);
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->dev);
    // voxels per lane: 2 when every spatial x-cell is at least 48 voxels wide
    {
        int minw = g.nx;
        auto xr = runs(c->h_sb[0], 0, g.nx, 1 << 30);
        for (auto &r : xr) minw = std::min(minw, r.second);
        c->XV = minw >= 48 ? 2 : 1;
        // ... and every 64-voxel x-chunk reads at most 32 control x-nodes (the FFD layer
        // loads are one node per lane): otherwise 32-voxel chunks (delta_x <= ~2.25 voxels)
        if (c->XV == 2)
            for (auto &r : runs(c->h_sb[0], 0, g.nx, 64))
                if (c->h_cb[0][r.first + r.second - 1] + 4 - c->h_cb[0][r.first] > 32) c->XV = 1;
        if (const char *e = getenv("SRWCR_XV")) c->XV = std::min(c->XV, std::max(1, atoi(e)));
        c->XV2 = c->XV;  // pass 2 amortises its per-line gamma/alpha/beta contractions over XV2 x 32 voxels
        if (const char *e = getenv("SRWCR_XV2")) c->XV2 = std::min(c->XV, std::max(1, atoi(e)));
        // fine spatial lattices: pack whole x-cells into one 32-voxel item when at least two fit
        int maxw = 0;
        for (auto &r : xr) maxw = std::max(maxw, r.second);
        c->MC = o.orientation == 0 && c->XV == 1 && c->XV2 == 1 && 2 * maxw <= 32 && !getenv("SRWCR_NOMC");
    }
    const int xmax = 32 * c->XV;
    int ymax = 64, zmax = 64;
    const bool yfirst = true;  // pass 1: split rows before z (longer z-marches), measured ~1% on C5
    const bool yfirst2 = true; // pass 2 likewise (C5 pass 2 -7 %)
    long long ips1 = 6, ips2 = 6;   // minimum items per SM (load balance vs per-item overhead)
    if (const char *e = getenv("SRWCR_IPS1")) ips1 = std::max(1, atoi(e));
    if (const char *e = getenv("SRWCR_IPS2")) ips2 = std::max(1, atoi(e));
    int zmin = 20;
    if (const char *e = getenv("SRWCR_ZMIN")) zmin = atoi(e);
    std::vector<Item> items, items_full, items2;
    size_t npmax = 0;
    // MC: consecutive whole cells along an axis, at most XRN - 3 of them and len voxels per item
    auto cruns_mc = [&](const std::vector<int> &sb, int lo, int hi, int len, int maxcells) {
        std::vector<std::pair<int, int>> out;
        auto cells = runs(sb, lo, hi, 1 << 30);
        size_t i = 0;
        while (i < cells.size()) {
            int x0 = cells[i].first, w = cells[i].second, k = 1;
            while (i + k < cells.size() && k < maxcells && w + cells[i + k].second <= len) w += cells[i + k++].second;
            if (w > len) {   // one cell longer than len: split it
                for (auto &r : runs(sb, x0, x0 + w, len)) out.push_back(r);
            } else {
                out.push_back({x0, w});
            }
            i += k;
        }
        return out;
    };
    int mcz = 3;   // MC: z-cells per item (tables grow with it; measured best 3-5)
    if (const char *e = getenv("SRWCR_MCZ")) mcz = std::min(MC_ZRN - 3, std::max(1, atoi(e)));
    c->zrn = mcz + 3;
    auto build_items = [&](int zlo, int zhi, std::vector<Item> &out, int xm) {
        auto xr = c->MC ? cruns_mc(c->h_sb[0], 0, g.nx, xm, MC_XRN - 3) : runs(c->h_sb[0], 0, g.nx, xm);
        auto yr = runs(c->h_sb[1], 0, g.ny, ymax);
        auto zr = c->MC ? cruns_mc(c->h_sb[2], zlo, zhi, std::min(zmax, 64), mcz) : runs(c->h_sb[2], zlo, zhi, zmax);
        for (auto &zz : zr)
            for (auto &yy : yr)
                for (auto &xx : xr) {
                    Item it{xx.first, xx.second, yy.first, yy.second, zz.first, zz.second, 0, 0, 0.f, 0};
                    out.push_back(it);
                    size_t nxn = c->h_cb[0][it.x0 + it.xlen - 1] + 4 - c->h_cb[0][it.x0];
                    size_t nyn = c->h_cb[1][it.y0 + it.ylen - 1] + 4 - c->h_cb[1][it.y0];
                    size_t nzn = c->h_cb[2][it.z0 + it.zlen - 1] + 4 - c->h_cb[2][it.z0];
                    npmax = std::max(npmax, nzn * 3 * nyn * nxn);
                    if (nxn > 32) npmax = SIZE_MAX;   // ffd_layer contracts y for <= 32 x-nodes
                }
    };
    for (;;) {
        items.clear();
        npmax = 0;
        build_items((int)c->z0, (int)c->z1, items, xmax);
        const bool small = (long long)items.size() < ips1 * nsm;
        const bool big_np = npmax > 12288;
        // z-marches shorter than ~20 slices re-load the 4-layer FFD window too often: accept
        // 3 items per SM rather than split z below that (C5 on 8 ranks: -14 % per rank)
        if (!big_np && ymax <= 16 && zmax / 2 < zmin && (long long)items.size() >= 3LL * nsm) break;
        if ((small || big_np) && (ymax > 16 || zmax > 4)) {
            if (yfirst && ymax > 16) ymax /= 2;
            else if (zmax >= ymax / 2 && zmax > 4) zmax /= 2;
            else if (ymax > 16) ymax /= 2;
            else zmax /= 2;
            continue;
        }
        break;
    }
    if (npmax == SIZE_MAX)
        return fail(c, SRWCR_EINVAL, "control lattice too fine along x: a voxel line reads more than 32 control x-nodes");
    build_items(0, g.nz, items_full, xmax);
    // pass 2 has its own (narrower) x-chunks, hence more items: keep its z-marches as
    // long as the load balance allows (fewer FFD-layer loads and retires per voxel)
    ymax = 64;
    zmax = 64;
    for (;;) {
        items2.clear();
        npmax = 0;
        build_items((int)c->z0, (int)c->z1, items2, 32 * c->XV2);
        const bool small = (long long)items2.size() < ips2 * nsm;
        if (npmax <= 16384 && ymax <= 16 && zmax / 2 < zmin && (long long)items2.size() >= 3LL * nsm) break;
        if ((small || npmax > 16384) && (ymax > 16 || zmax > 4)) {
            if (yfirst2 && ymax > 16) ymax /= 2;
            else if (zmax >= ymax / 2 && zmax > 4) zmax /= 2;
            else if (ymax > 16) ymax /= 2;
            else zmax /= 2;
            continue;
        }
        break;
    }
    if (npmax > 16384) return fail(c, SRWCR_EINVAL, "control lattice too fine for the node window (%zu)", npmax);
    c->nitems = (int)items.size();
    c->nitems_full = (int)items_full.size();
    c->nitems2 = (int)items2.size();
    // pipelined host-buffer evaluation (one rank, 3-D): pass 1's first two waves of items
    // start once their params layers have arrived; the gradient layers no item of pass 2's
    // last two waves touches go back to the host while those run
    if (c->nranks == 1 && !is2d && !getenv("SRWCR_NOPIPE")) {
        int wave = nsm;
        if (const char *e = getenv("SRWCR_PIPE_WAVE")) wave = std::max(1, atoi(e));   // tests: small volumes
        // parts are whole waves (a part boundary at a z-run start instead needs fewer layers
        // but adds a partial wave: measured slower on C5)
        // pass 1: one wave, one wave, the rest (the first upload part is as small as one
        // wave's layers; later parts arrive while earlier waves run)
        if (c->nitems >= 4 * wave) {
            std::vector<int> b = {0, wave, 2 * wave, c->nitems}, l;
            for (size_t j = 0; j + 1 < b.size(); ++j) {
                int hi = 0;
                for (int i = 0; i < b[j + 1]; ++i) hi = std::max(hi, c->h_cb[2][items[i].z0 + items[i].zlen - 1] + 4);
                l.push_back(std::min(hi, g.GzExt));
            }
            if (l[0] < g.GzExt) { c->p1_b = b; c->p1_l = l; c->p1_split = b[1]; }
        }
        // pass 2: all but three waves, then one wave at a time (the gradient layers final
        // after each part go back while the next runs)
        if (c->nitems2 >= 5 * wave) {
            const int n = c->nitems2;
            std::vector<int> b = {0, n - 3 * wave, n - 2 * wave, n - wave, n}, l;
            for (size_t j = 0; j + 1 < b.size(); ++j) {
                int lo = g.GzExt;
                for (int i = b[j + 1]; i < n; ++i) lo = std::min(lo, c->h_cb[2][items2[i].z0]);
                l.push_back(lo);
            }
            if (l[0] > 0) { c->p2_b = b; c->p2_l = l; c->p2_split = b[1]; }
        }
    }

    // per item: fixed bins present (slot lists), binless shift cI, spatial weight sums
    std::vector<int> slotbins;
    int smax = 1, s2max = 2;
    auto scan_items = [&](std::vector<Item> &its, ItemW **dw, bool pass2) -> srwcr_status {
        const size_t n = its.size();
        if (n == 0) return SRWCR_OK;
        Item *d_it = nullptr;
        unsigned *d_mask = nullptr;
        double *d_sum = nullptr;
        CK(cudaMalloc(&d_it, sizeof(Item) * n));
        CK(cudaMalloc(&d_mask, sizeof(unsigned) * 4 * n));
        CK(cudaMalloc(&d_sum, sizeof(double) * n));
        CK(h2d_sync(d_it, its.data(), sizeof(Item) * n));
        k_item_scan<<<(unsigned)n, 256>>>(c->F, c->M, d_it, g, d_mask, d_sum);
        CKL();
        std::vector<unsigned> mask(4 * n);
        std::vector<double> sum(n);
        CK(cudaMemcpy(mask.data(), d_mask, sizeof(unsigned) * 4 * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sum.data(), d_sum, sizeof(double) * n, cudaMemcpyDeviceToHost));
        cudaFree(d_it);
        cudaFree(d_mask);
        cudaFree(d_sum);
        std::vector<ItemW> w(n);
        for (size_t i = 0; i < n; ++i) {
            Item &it = its[i];
            it.slot_off = (int)slotbins.size();
            int ns = 0;
            if (o.orientation == 1) {   // model bins come from m: every bin (dense lists)
                const int cnt = pass2 ? 3 * (g.B + 2) : g.L;      // pass 2: 3 table columns per bin -1..L+1
                for (int b = 0; b < cnt; ++b) slotbins.push_back(b);
                ns = cnt;
                if (pass2) s2max = std::max(s2max, ns);
                else smax = std::max(smax, 2 * ns);               // two slot groups per bin
            } else if (!pass2) {   // pass 1: the fixed bins a0 present in the item ("slots")
                for (int b = 0; b < g.B; ++b)
                    if ((mask[4 * i + (b >> 5)] >> (b & 31)) & 1u) { slotbins.push_back(b); ++ns; }
                smax = std::max(smax, ns);
            } else {        // pass 2: every a0 present and a0 + 1, sorted, no duplicates
                int last = -1;
                for (int b = 0; b < g.B; ++b)
                    if ((mask[4 * i + (b >> 5)] >> (b & 31)) & 1u) {
                        if (b != last) { slotbins.push_back(b); ++ns; }
                        slotbins.push_back(b + 1);
                        ++ns;
                        last = b + 1;
                    }
                s2max = std::max(s2max, ns);
            }
            it.nslots = ns;
            it.cI = (float)(sum[i] / ((double)it.xlen * it.ylen * it.zlen));
            ItemW &iw = w[i];
            for (int l = 0; l < 8; ++l) iw.sx[l] = iw.sz[l] = 0.0;
            for (int l = 0; l < 4; ++l) iw.sy[l] = 0.0;
            const int lo[3] = {it.x0, it.y0, it.z0}, len[3] = {it.xlen, it.ylen, it.zlen};
            double *dst[3] = {iw.sx, iw.sy, iw.sz};
            for (int ax = 0; ax < 3; ++ax)
                for (int k = lo[ax]; k < lo[ax] + len[ax]; ++k) {
                    const float4 q = c->h_sw[ax][k];
                    // x, z: per relative region (the voxel's cell offset in a multi-cell item)
                    const int off = ax == 1 ? 0 : c->h_sb[ax][k] - c->h_sb[ax][lo[ax]];
                    dst[ax][off + 0] += q.x; dst[ax][off + 1] += q.y; dst[ax][off + 2] += q.z; dst[ax][off + 3] += q.w;
                }
        }
        CK(cudaMalloc(dw, sizeof(ItemW) * n));
        CK(h2d_sync(*dw, w.data(), sizeof(ItemW) * n));
        return SRWCR_OK;
    };
    TRY(scan_items(items, &c->itemw, false));
    TRY(scan_items(items_full, &c->itemw_full, false));
    {
        ItemW *tmpw = nullptr;
        TRY(scan_items(items2, &tmpw, true));
        if (tmpw) cudaFree(tmpw);
    }
    c->S = smax + (c->MC ? 1 : 0);   // MC: + the binless slot
    c->S2 = s2max;
    CK(cudaMalloc(&c->slotbins, sizeof(int) * std::max<size_t>(1, slotbins.size())));
    CK(h2d_sync(c->slotbins, slotbins.data(), sizeof(int) * slotbins.size()));
    if (c->nitems) {
        CK(cudaMalloc(&c->items, sizeof(Item) * items.size()));
        CK(h2d_sync(c->items, items.data(), sizeof(Item) * items.size()));
    }
    if (c->nitems2) {
        CK(cudaMalloc(&c->items2, sizeof(Item) * items2.size()));
        CK(h2d_sync(c->items2, items2.data(), sizeof(Item) * items2.size()));
    }
    CK(cudaMalloc(&c->items_full, sizeof(Item) * items_full.size()));
    CK(h2d_sync(c->items_full, items_full.data(), sizeof(Item) * items_full.size()));

    // buffers
    const long long RB = c->R * g.B;
    CK(cudaMalloc(&c->phi, sizeof(float) * c->nint));
    // [0, 4G) float4 tolerances, [4G, 7G) and [7G, 10G) scratch of the window-max passes
    CK(cudaMalloc(&c->phimax, sizeof(float) * (size_t)g.Gx * g.Gy * g.Gz * 10));
    CK(cudaMemset(c->phimax, 0, sizeof(float) * (size_t)g.Gx * g.Gy * g.Gz * 10));
    {   // deferred exact-path voxels: 1/16 of the slab (more falls back to an MG scan)
        const int64_t sv = std::max<int64_t>(1, (c->z1 - c->z0) * (int64_t)g.nxy);
        c->xcap = (int)std::min<int64_t>(std::max<int64_t>(4096, sv / 16), 1 << 30);
        if (const char *e = getenv("SRWCR_XCAP")) c->xcap = std::max(1, atoi(e));  // tests: force the scan fallback
        CK(cudaMalloc(&c->xlist, sizeof(int) * (size_t)c->xcap));
    }
    CK(cudaMalloc(&c->MG, sizeof(float4) * (size_t)std::max<int64_t>(1, (c->z1 - c->z0) * (int64_t)g.nxy)));
    CK(cudaMalloc(&c->params64, sizeof(double) * c->nparams));
    CK(cudaMalloc(&c->grad64, sizeof(double) * c->nparams));
    CK(cudaMalloc(&c->SQ, sizeof(double) * stats_count(c)));
    const bool ori1 = o.orientation == 1;
    c->NQ = ori1 ? c->SQ + RB * 2 : nullptr;
    c->Qt = c->SQ + RB * (ori1 ? 4 : 2);
    c->gstride = ori1 ? 3 * (g.B + 2) : g.B;
    CK(cudaMalloc(&c->Nlo, sizeof(double) * RB));
    CK(cudaMalloc(&c->Nup, sizeof(double) * RB));
    CK(cudaMalloc(&c->S_out, sizeof(double) * RB));
    CK(cudaMalloc(&c->dterm, sizeof(double) * c->R));
    CK(cudaMalloc(&c->reg, sizeof(double) * c->R * 6));
    // D, #retained, gradient bound (fast pass 2), spare, then the exact-path list counts
    // (xcount: [0] the list, [1..] the pipelined parts): one 64-byte copy returns them all
    CK(cudaMalloc(&c->Dout, sizeof(double) * (4 + NPART / 2)));
    CK(cudaMemset(c->Dout, 0, sizeof(double) * (4 + NPART / 2)));
    c->xcount = reinterpret_cast<int *>(c->Dout + 4);
    CK(cudaMalloc(&c->ticket, sizeof(unsigned)));
    CK(cudaMalloc(&c->dpart, sizeof(double) * 3 * (size_t)std::min<int64_t>((c->R + 7) / 8, 148 * 8)));
    CK(cudaMemset(c->ticket, 0, sizeof(unsigned)));
    CK(cudaMalloc(&c->shiftc, sizeof(float) * g.B));
    CK(cudaMalloc(&c->alpha, sizeof(float) * c->R));
    CK(cudaMalloc(&c->beta, sizeof(float) * c->R));
    CK(cudaMalloc(&c->gamma, sizeof(float) * (size_t)c->R * c->gstride));
    CK(cudaMemset(c->phi, 0, sizeof(float) * c->nint));
    CK(cudaMemset(c->params64, 0, sizeof(double) * c->nparams));
    c->cur_params = c->params64;

    // shared memory and warps per CTA of each pass: the largest W in {16, 12, 8, 6, 4} that fits
    int maxsm = 0;
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev);
    // (2 and 1: orientation 1 at > 83 bins, whose 2 (L) slots per item fill the tables)
    const int Wc[10] = {32, 24, 20, 16, 12, 8, 6, 4, 2, 1};
    // a CTA's warps own whole rows of its item: no more warps than the tallest item has
    // rows (fine spatial lattices -- small items -- then fit several CTAs per SM)
    auto wcap = [&](const std::vector<Item> &its) {
        int ym = 1;
        for (const Item &it : its) ym = std::max(ym, it.ylen);
        for (int W : {4, 6, 8, 12, 16})
            if (W >= ym) return W;
        return 16;
    };
    int w1max = wcap(items), w2max = wcap(items2);
    if (const char *e = getenv("SRWCR_W1")) w1max = atoi(e);
    if (const char *e = getenv("SRWCR_W2")) w2max = atoi(e);
    c->W = c->W2 = 0;
    for (int W : Wc) {
        const size_t ltsv = c->MC ? 2 * MC_XRN + 1 : LTS, ks = c->MC ? 8 * MC_XRN : 32;
        const size_t cts = c->MC ? 4 * (size_t)c->zrn * 2 * MC_XRN : 4 * ks;
        const size_t s1 = sizeof(int) * (((size_t)W * c->S * ltsv + 3) & ~(size_t)3) + sizeof(float) * (size_t)W * c->S * ks +
                          sizeof(float) * ((size_t)c->S * cts + 128 + g.B) + (size_t)g.B + 16 + 2048 + 256;
        if (!c->W && W <= w1max && W != 32 && W != 20 && (int)s1 <= maxsm) { c->W = W; c->smem1 = s1; }
        const size_t xrn = c->MC ? MC_XRN : 4, zrn = c->MC ? c->zrn : 4, gys = c->MC ? MC_XRN + 1 : GYS;
        const size_t s2 = sizeof(float4) * (size_t)W * c->S2 * (gys + xrn / 4) +
                          sizeof(float) * (4 * zrn * xrn * (size_t)c->S2 + (c->S2 + 1) + 8 * zrn * xrn + W * 192 + (o.orientation ? g.B : 0)) +
                          2 * (((o.orientation ? 3 * (g.B + 2) : g.B) + 7) & ~7) +
                          sizeof(float) * npmax;
        if (!c->W2 && W <= w2max && (int)s2 <= maxsm) { c->W2 = W; c->smem2 = s2; }
    }
    if (c->W == 0 || c->W2 == 0) return fail(c, SRWCR_EINVAL, "shared memory too small for %d bins / %d slots", g.B, c->S);
    // the pipelined parts are whole waves of one resident CTA per SM (16 warps x 128
    // registers fill the register file); with several resident CTAs they would not be
    if (c->W != 16 && !getenv("SRWCR_PIPE_WAVE")) { c->p1_b.clear(); c->p1_l.clear(); c->p1_split = 0; }
    if (c->W2 != 16 && !getenv("SRWCR_PIPE_WAVE")) { c->p2_b.clear(); c->p2_l.clear(); c->p2_split = 0; }
    TRY(set_smem(c));

    // NCCL communicator for the z-slab decomposition (also built for nranks = 1 when an id
    // is given: the same code path, exercised on a single GPU by the tests)
    if (c->nranks > 1 || o.nccl_id) {
        if (o.nccl_id) {
            if (!nccl().ok) return fail(c, SRWCR_ENCCL, "libnccl.so.2 could not be loaded");
            ncclUniqueId id;
            memcpy(&id, o.nccl_id, sizeof id);
            NCK(nccl().CommInitRank(&c->comm, c->nranks, id, c->rank));
        } else {
            c->external_exchange = true;
        }
    }

    // static weighted counts N[r][a] (lower / upper Parzen half) over the whole volume
    // (every rank holds the full F, so no create-time collective is needed).  The work above
    // ran on the legacy stream (uploads, normalisation, scans, memsets): order it before the
    // context stream's first launch.
    CK(cudaDeviceSynchronize());
    CK(cudaMemsetAsync(c->SQ, 0, sizeof(double) * stats_count(c), c->stream));
    TRY(launch_pass1(c, true, true));
    k_split_counts<<<512, 256, 0, c->stream>>>(c->SQ, c->Nlo, c->Nup, RB);
    CKL();
    {
        std::vector<double> nl(RB), nu(RB);
        CK(cudaMemcpyAsync(nl.data(), c->Nlo, sizeof(double) * RB, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(nu.data(), c->Nup, sizeof(double) * RB, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        double Z = 0;
        for (long long i = 0; i < RB; ++i) Z += nl[i] + nu[i];
        c->Z = Z;
    }
    // per-bin moment shift: bin index, then (option) conditional means at Phi = 0
    {
        std::vector<float> sh(g.B);
        for (int b = 0; b < g.B; ++b) sh[b] = (float)b;
        CK(h2d_sync(c->shiftc, sh.data(), sizeof(float) * g.B));
        if (o.moment_shift) {
            CK(cudaMemsetAsync(c->SQ, 0, sizeof(double) * stats_count(c), c->stream));
            TRY(launch_pass1(c, false, true));
            float *tmp = nullptr;
            CK(cudaMalloc(&tmp, sizeof(float) * g.B));
            if (o.orientation)
                k_shift_updateA<<<(g.B + 127) / 128, 128, 0, c->stream>>>(c->SQ, c->NQ, c->shiftc, tmp, (int)c->R, g.B);
            else
                k_shift_update<<<(g.B + 127) / 128, 128, 0, c->stream>>>(c->SQ, c->Nlo, c->Nup, c->shiftc, tmp, (int)c->R, g.B);
            CKL();
            CK(cudaMemcpyAsync(c->shiftc, tmp, sizeof(float) * g.B, cudaMemcpyDeviceToDevice, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            cudaFree(tmp);
        }
    }
    c->launches_per_eval = 6;  // prep (phi + x-max, y/z-max), pass 1, combine (+ D), pass 2, exact fix
    TRY(build_fast(c, nsm));
    if (c->fast && !c->h_nboxes.empty() && !getenv("SRWCR_NONDET_N")) {
        // the fast contexts replace N, Z and the moment shifts by the deterministic whole-volume
        // computation (k_static_N): bitwise the same in every context, rank count and run
        const size_t nb = c->h_nboxes.size();
        NBox *d_nb = nullptr;
        unsigned long long *Ni = nullptr, *Ci = nullptr;
        CK(cudaMalloc(&d_nb, sizeof(NBox) * nb));
        CK(h2d_sync(d_nb, c->h_nboxes.data(), sizeof(NBox) * nb));
        CK(cudaMalloc(&Ni, sizeof(unsigned long long) * 2 * RB));
        CK(cudaMalloc(&Ci, sizeof(unsigned long long) * 4 * g.B));
        CK(cudaMemsetAsync(Ni, 0, sizeof(unsigned long long) * 2 * RB, c->stream));
        CK(cudaMemsetAsync(Ci, 0, sizeof(unsigned long long) * 4 * g.B, c->stream));
        Tables t{};
        for (int i = 0; i < 3; ++i) { t.cb[i] = c->cb[i]; t.cw[i] = c->cw[i]; t.sb[i] = c->sb[i]; t.sw[i] = c->sw[i]; }
        const int sm = (int)(sizeof(double) * 132 * (size_t)g.B);
        int maxsm = 0;
        CK(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->dev));
        CK(cudaFuncSetAttribute(k_static_N, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
        k_static_N<<<(unsigned)nb, 32, sm, c->stream>>>(c->F, c->M, d_nb, t, g, Ni, Ci);
        CKL();
        k_static_N_convert<<<296, 256, 0, c->stream>>>(Ni, Ci, c->Nlo, c->Nup, c->shiftc, RB, g.B);
        CKL();
        std::vector<double> nl(RB), nu(RB);
        CK(cudaMemcpyAsync(nl.data(), c->Nlo, sizeof(double) * RB, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(nu.data(), c->Nup, sizeof(double) * RB, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        double Z = 0;
        for (long long i = 0; i < RB; ++i) Z += nl[i] + nu[i];
        c->Z = Z;
        cudaFree(d_nb);
        cudaFree(Ni);
        cudaFree(Ci);
    }
    if (c->comm && c->nranks > 1) {
        // z-slab ranks: every rank computed the whole-volume static counts and moment shifts
        // (fp32 shared / fp64 global atomics: equal to rounding, not bitwise); rank 0's copy is
        // broadcast so that the replicated combine -- and so D, the coefficient tables and the
        // gradient -- are bitwise identical on every rank
        const long long RBn = c->R * g.B;
        NCK(nccl().Broadcast(c->Nlo, c->Nlo, (size_t)RBn, ncclFloat64, 0, c->comm, c->stream));
        NCK(nccl().Broadcast(c->Nup, c->Nup, (size_t)RBn, ncclFloat64, 0, c->comm, c->stream));
        NCK(nccl().Broadcast(c->shiftc, c->shiftc, (size_t)g.B, ncclFloat32, 0, c->comm, c->stream));
        double *zb = nullptr;
        CK(cudaMalloc(&zb, sizeof(double)));
        CK(h2d_sync(zb, &c->Z, sizeof(double)));
        NCK(nccl().Broadcast(zb, zb, 1, ncclFloat64, 0, c->comm, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        CK(cudaMemcpy(&c->Z, zb, sizeof(double), cudaMemcpyDeviceToHost));
        cudaFree(zb);
    }
    if (c->fast) c->launches_per_eval = c->fsplit ? 8 : 7;   // prep, pass 1 (split: 2 kernels), stats conversion, combine, pass 2, exact fix, gradient conversion
    // node-layer plan of the slab (srwcr_grad_layers) and the halo gradient exchange
    if (o.grad_exchange != 0 && o.grad_exchange != 1) return fail(c, SRWCR_EINVAL, "grad_exchange must be 0 or 1");
    bool plan_ok = false;
    if (!is2d) {
        std::vector<int32_t> cbz(c->h_cb[2].begin(), c->h_cb[2].end());
        plan_ok = srwcr_plan_layers(g.nz, c->nranks, c->rank, cbz.data(), g.Gz, c->lay) == SRWCR_OK;
    }
    if (o.grad_exchange == 1) {
        if (!c->comm) return fail(c, SRWCR_EINVAL, "grad_exchange = 1 needs nccl_id (with the caller-driven exchange the caller sums the partials)");
        if (is2d || !c->fast) return fail(c, SRWCR_ENOTSUP, "grad_exchange = 1: 3-D configurations of the fast passes only");
        if (!nccl().p2p) return fail(c, SRWCR_ENCCL, "libnccl has no ncclSend/ncclRecv");
        if (!plan_ok) return fail(c, SRWCR_EINVAL, "grad_exchange = 1: slabs too thin (a rank's node layers reach past its neighbour's)");
        c->halo = true;
        const size_t nrecv = (size_t)g.ndim * (size_t)(c->lay[4] - c->lay[2]) * g.Gx * g.Gy;
        CK(cudaMalloc(&c->halo_recv, sizeof(long long) * std::max<size_t>(nrecv, 1)));
        c->launches_per_eval += 1;   // k_halo_finish
    }
    CK(cudaStreamSynchronize(c->stream));
    return SRWCR_OK;
}

extern "C" srwcr_status srwcr_create(srwcr_ctx **out, const float *fixed, const float *moving, const int64_t dims[3],
                                     const double spacing_mm[3], int32_t intensity_bins, const int32_t spatial_bins[3],
                                     const double control_spacing_mm[3], const srwcr_options *opt) {
    if (!out) return SRWCR_EINVAL;
    *out = nullptr;
    srwcr_ctx *c = new (std::nothrow) srwcr_ctx();
    if (!c) return SRWCR_ENOMEM;
    if (opt) {
        if (opt->struct_size != (int32_t)sizeof(srwcr_options)) {
            *out = c;
            return fail(c, SRWCR_EINVAL, "opt->struct_size mismatch (use srwcr_default_options)");
        }
        c->opt = *opt;
    } else {
        srwcr_default_options(&c->opt);
    }
    srwcr_status s = create_impl(c, fixed, moving, dims, spacing_mm, intensity_bins, spatial_bins, control_spacing_mm);
    *out = c;  // returned even on failure so srwcr_last_error can be read; caller destroys
    return s;
}

extern "C" srwcr_status srwcr_num_params(const srwcr_ctx *c, int64_t *n, int64_t grid_dims[3]) {
    if (!c) return SRWCR_EINVAL;
    if (n) *n = c->nparams;
    if (grid_dims) { grid_dims[0] = c->g.Gx; grid_dims[1] = c->g.Gy; grid_dims[2] = c->g.GzExt; }
    return SRWCR_OK;
}

// per-pass timing event: an external event-record node when the stream is being captured
// into the evaluation graph (the flag is invalid outside a capture)
static cudaError_t record_ev(srwcr_ctx *c, int i) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(c->ev[i], c->stream, cudaEventRecordExternal)
                                               : cudaEventRecord(c->ev[i], c->stream);
}

static srwcr_status eval_begin_impl(srwcr_ctx *c, const double *params, int pdev = -1) {
    if (c->poisoned) return fail(c, SRWCR_ESTATE, "context poisoned by an earlier CUDA error");
    if (!params) return fail(c, SRWCR_EINVAL, "params is NULL");
    CK(cudaSetDevice(c->dev));
    const double *pd = params;
    if (!(pdev < 0 ? is_device_ptr(params) : pdev != 0)) {
        CK(cudaMemcpyAsync(c->params64, params, sizeof(double) * c->nparams, cudaMemcpyHostToDevice, c->stream));
        pd = c->params64;
    }
    c->cur_params = pd;
    if (c->timing) CK(record_ev(c, 4));
    // only the node layers this rank's slab reads: taps of slices [z0, z1) (all of them on
    // one rank), converted to fp32, and their tap-window max |phi_c| (x, y into scratch,
    // z -> float4) for pass 1's rounding bound
    if (!c->fast) {
        const size_t G = (size_t)c->g.Gx * c->g.Gy * c->g.Gz;
        float *s1 = c->phimax + 4 * G;
        k_prep_phi_wx<<<592, 256, 0, c->stream>>>(pd, c->phi, s1, c->g, c->pz0, c->pz1);
        CKL();
        k_prep_tol<<<592, 256, 0, c->stream>>>(s1, reinterpret_cast<float4 *>(c->phimax), c->g, c->pz0, c->pzb1,
                                               c->pz1);
        CKL();
    }
    if (c->fast) {
        TRY(launch_fast_prep(c, pd));
        if (c->timing) CK(record_ev(c, 0));
        // with a communicator the int64 statistics are summed across ranks before the
        // conversion: exact, so every rank count gives bitwise the same statistics
        TRY(launch_fast_pass1(c, 0, -1, c->comm == nullptr));
        if (c->comm) {
            NCK(nccl().AllReduce(c->SQi, c->SQi, stats_count(c), ncclInt64, ncclSum, c->comm, c->stream));
            k_stats_convert<<<592, 256, 0, c->stream>>>(c->SQi, c->SQ, (long long)stats_count(c), (long long)c->R * c->g.B * 2);
            CKL();
        }
    } else {
        CK(cudaMemsetAsync(c->SQ, 0, sizeof(double) * stats_count(c), c->stream));
        if (c->timing) CK(record_ev(c, 0));
        TRY(launch_pass1(c, false));
    }
    if (c->timing) CK(record_ev(c, 1));
    return SRWCR_OK;
}

// combine, pass 2 and the result copies (stream-ordered, no host synchronisation:
// also the body of the captured evaluation graph)
static srwcr_status eval_end_enqueue(srwcr_ctx *c, double *grad, bool reduce_grad, int gdev = -1) {
    TRY(run_combine(c));
    if (c->timing) CK(record_ev(c, 2));
    double *gd = nullptr;
    const bool grad_dev = grad && (gdev < 0 ? is_device_ptr(grad) : gdev != 0);
    if (grad) {
        gd = grad_dev ? grad : c->grad64;
        if (c->fast) {
            TRY(launch_fast_pass2(c, gd, reduce_grad && c->comm));
        } else {
            CK(cudaMemsetAsync(gd, 0, sizeof(double) * c->nparams, c->stream));
            TRY(launch_pass2(c, gd));
            if (reduce_grad) TRY(allreduce(c, gd, (size_t)c->nparams));
        }
    }
    if (c->timing) CK(record_ev(c, 3));
    CK(cudaMemcpyAsync(c->pinned, c->Dout, (grad ? 4 + NPART / 2 : 2) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (grad && !grad_dev) CK(cudaMemcpyAsync(grad, c->grad64, sizeof(double) * c->nparams, cudaMemcpyDeviceToHost, c->stream));
    return SRWCR_OK;
}

static srwcr_status eval_finish(srwcr_ctx *c, double *value) {
    CK(cudaStreamSynchronize(c->stream));
    if (c->timing) {
        cudaEventElapsedTime(&c->ms[0], c->ev[0], c->ev[1]);
        cudaEventElapsedTime(&c->ms[1], c->ev[1], c->ev[2]);
        cudaEventElapsedTime(&c->ms[2], c->ev[2], c->ev[3]);
        cudaEventElapsedTime(&c->ms[4], c->ev[4], c->ev[0]);
        c->ms[3] = c->ms[4] + c->ms[0] + c->ms[1] + c->ms[2];
    }
    if (value) *value = c->pinned[0];
    if (c->pinned[1] < 0.5) {
        if (value) *value = 0.0;
        return fail(c, SRWCR_EDEGENERATE, "no spatial bin passed the retention test (reading c12)");
    }
    return SRWCR_OK;
}

static srwcr_status eval_end_impl(srwcr_ctx *c, double *value, double *grad, bool reduce_grad) {
    TRY(eval_end_enqueue(c, grad, reduce_grad));
    return eval_finish(c, value);
}

// One evaluation as a CUDA graph (options.use_graph, single rank, device params and
// gradient): the 6 kernels, 3 memsets, 2 result copies (and, with timing on, the per-pass
// event records) are captured once per (params, grad, timing) and replayed with one
// cudaGraphLaunch.
static srwcr_status eval_graph(srwcr_ctx *c, const double *params, double *value, double *grad) {
    CK(cudaSetDevice(c->dev));
    if (!c->gexec || c->g_params != params || c->g_grad != grad || c->g_timing != c->timing) {
        if (c->gexec) cudaGraphExecDestroy(c->gexec);
        c->gexec = nullptr;
        const int64_t l0 = c->launches;
        CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        srwcr_status st = eval_begin_impl(c, params, 1);
        // z-slab ranks: the NCCL collectives are captured into the graph with the kernels
        if (st == SRWCR_OK && c->comm && !c->fast) st = allreduce(c, c->SQ, stats_count(c));
        if (st == SRWCR_OK) st = eval_end_enqueue(c, grad, c->comm != nullptr, 1);
        cudaGraph_t gr = nullptr;
        const cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
        c->g_kernels = c->launches - l0;
        c->launches = l0;
        if (st != SRWCR_OK || e != cudaSuccess) {
            if (gr) cudaGraphDestroy(gr);
            return st != SRWCR_OK ? st : fail(c, SRWCR_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
        }
        const cudaError_t e2 = cudaGraphInstantiate(&c->gexec, gr, 0);
        cudaGraphDestroy(gr);
        if (e2 != cudaSuccess) {
            c->gexec = nullptr;
            return fail(c, SRWCR_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e2));
        }
        c->g_params = params;
        c->g_grad = grad;
        c->g_timing = c->timing;
    }
    CK(cudaGraphLaunch(c->gexec, c->stream));
    c->launches += c->g_kernels;
    return eval_finish(c, value);
}

// Host params and host gradient on one rank: the H2D of the params runs on a second
// stream in two parts -- the layers the first two waves of pass-1 items read, then the
// rest -- and the prep + pass 1 of those items start after the first part; pass 2 runs in
// two parts too, and the gradient layers final after the first part (all but the layers
// the last two waves of items touch; their deferred exact voxels fixed first) are copied
// back while the second part runs.  Same kernels, same results as srwcr_eval's plain path.
static srwcr_status eval_host_pipelined(srwcr_ctx *c, const double *params, double *value, double *grad) {
    if (c->poisoned) return fail(c, SRWCR_ESTATE, "context poisoned by an earlier CUDA error");
    CK(cudaSetDevice(c->dev));
    const Geo &g = c->g;
    const size_t plane = (size_t)g.Gx * g.Gy, cs = plane * g.GzExt;
    auto copy_layers = [&](double *dst, const double *src, int l0, int l1, cudaMemcpyKind kind, cudaStream_t st) {
        for (int k = 0; k < g.ndim; ++k)
            if (l1 > l0)
                CK(cudaMemcpyAsync(dst + k * cs + l0 * plane, src + k * cs + l0 * plane, sizeof(double) * plane * (l1 - l0),
                                   kind, st));
        return SRWCR_OK;
    };
    const size_t G = (size_t)g.Gx * g.Gy * g.Gz;
    float *s1 = c->phimax + 4 * G;
    auto prep = [&](int l0, int l1, int b0, int b1) {
        if (l1 > l0) {
            k_prep_phi_wx<<<592, 256, 0, c->stream>>>(c->params64, c->phi, s1, g, l0, l1);
            CKL();
        }
        if (b1 > b0) {
            k_prep_tol<<<592, 256, 0, c->stream>>>(s1, reinterpret_cast<float4 *>(c->phimax), g, b0, b1, c->pz1);
            CKL();
        }
        return SRWCR_OK;
    };
    // ---- params upload in parts (copy stream), each followed by its prep and pass-1 items
    CK(cudaEventRecord(c->pev[3], c->stream));
    CK(cudaStreamWaitEvent(c->cstream, c->pev[3], 0));
    std::vector<int> b1 = c->p1_b, l1 = c->p1_l;
    if (b1.empty()) { b1 = {0, c->nitems}; l1 = {g.GzExt}; }
    l1.back() = g.GzExt;
    const int np1 = (int)l1.size();
    c->cur_params = c->params64;
    CK(cudaMemsetAsync(c->SQ, 0, sizeof(double) * stats_count(c), c->stream));
    int lo_l = 0, lo_b = c->pz0;
    for (int j = 0; j < np1; ++j) {
        TRY(copy_layers(c->params64, params, lo_l, l1[j], cudaMemcpyHostToDevice, c->cstream));
        CK(cudaEventRecord(c->pev[0], c->cstream));
        CK(cudaStreamWaitEvent(c->stream, c->pev[0], 0));
        // fp32 phi of the new layers; tolerance of the base layers whose 4-layer window is here
        const int hi_b = j + 1 == np1 ? c->pzb1 : std::min(c->pzb1, std::max(lo_b, l1[j] - 3));
        TRY(prep(std::max(lo_l, c->pz0), j + 1 == np1 ? c->pz1 : l1[j], lo_b, hi_b));
        TRY(launch_pass1(c, false, false, b1[j], b1[j + 1] - b1[j]));
        lo_l = l1[j];
        lo_b = hi_b;
    }
    TRY(run_combine(c));
    CK(cudaMemcpyAsync(c->pinned, c->Dout, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    bool parts2 = false;
    if (grad) {
        CK(cudaMemsetAsync(c->grad64, 0, sizeof(double) * c->nparams, c->stream));
        if (!c->p2_b.empty()) {
            // ---- pass 2 in parts: the layers final after a part go back during the next
            parts2 = true;
            CK(cudaMemsetAsync(c->xbeg, 0, sizeof(int), c->stream));
            const int np2 = (int)c->p2_l.size();
            int done = 0;
            for (int j = 0; j < np2; ++j) {
                const bool last = j + 1 == np2;
                TRY(launch_pass2(c, c->grad64, c->p2_b[j], c->p2_b[j + 1] - c->p2_b[j], j == 0, c->xbeg, last ? 0 : 1));
                if (last) {
                    TRY(copy_layers(grad, c->grad64, done, g.GzExt, cudaMemcpyDeviceToHost, c->stream));
                } else {
                    CK(cudaMemcpyAsync(c->xbeg, c->xcount, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
                    CK(cudaEventRecord(c->pev[2], c->stream));
                    CK(cudaStreamWaitEvent(c->cstream, c->pev[2], 0));
                    TRY(copy_layers(grad, c->grad64, done, c->p2_l[j], cudaMemcpyDeviceToHost, c->cstream));
                    done = std::max(done, c->p2_l[j]);
                }
            }
        } else {
            TRY(launch_pass2(c, c->grad64));
            TRY(copy_layers(grad, c->grad64, 0, g.GzExt, cudaMemcpyDeviceToHost, c->stream));
        }
        CK(cudaMemcpyAsync(c->pinned + 4, c->xcount, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->cstream));
    CK(cudaStreamSynchronize(c->stream));
    if (parts2) {   // list overflow: the last launch scanned the whole slab, after the early
        int xc = 0;   // gradient layers had gone back -- copy the whole gradient again
        memcpy(&xc, c->pinned + 4, sizeof(int));
        if (xc > c->xcap) CK(cudaMemcpy(grad, c->grad64, sizeof(double) * c->nparams, cudaMemcpyDeviceToHost));
    }
    return eval_finish(c, value);
}

// Host-buffer evaluation of the fast passes on one rank with the copies overlapped: params
// go up in parts, each part's fp32 conversion, interior flags and pass-1 items starting as soon
// as it has arrived; pass 2 runs in parts, and after each part the gradient layers no later
// item touches (their deferred exact-path voxels fixed first) are converted and go back while
// the next part runs.  The same kernels as srwcr_eval on device buffers, on item ranges.
static srwcr_status enqueue_host_pipelined_fast(srwcr_ctx *c, const double *params, double *grad) {
    const Geo &g = c->g;
    const size_t plane = (size_t)g.Gx * g.Gy, cs = plane * g.GzExt;
    auto copy_layers = [&](double *dst, const double *src, int l0, int l1, cudaMemcpyKind kind, cudaStream_t st) {
        for (int k = 0; k < g.ndim; ++k)
            if (l1 > l0)
                CK(cudaMemcpyAsync(dst + k * cs + l0 * plane, src + k * cs + l0 * plane, sizeof(double) * plane * (l1 - l0),
                                   kind, st));
        return SRWCR_OK;
    };
    Tables t{};
    for (int i = 0; i < 3; ++i) { t.cb[i] = c->cb[i]; t.cw[i] = c->cw[i]; t.sb[i] = c->sb[i]; t.sw[i] = c->sw[i]; }
    // ---- params in parts (copy stream), each followed by its prep and pass-1 items
    CK(cudaEventRecord(c->pev[3], c->stream));
    CK(cudaStreamWaitEvent(c->cstream, c->pev[3], 0));
    c->cur_params = c->params64;
    const int np1 = (int)c->fp1_l.size();
    // concurrent parts: part j > 0 on its own stream, after its upload and the previous part's
    // prep (its items read the fp32 layers the earlier preps converted); the int64 statistics
    // adds of the parts commute, so the result is the same bits in any interleaving
    const bool conc = c->fconc && np1 <= 4;   // (pex: 4 uploads, 4 preps, 4 part ends)
    if (conc)
        for (int j = 0; j < np1; ++j) CK(cudaStreamWaitEvent(c->kst[j], c->pev[3], 0));
    int lo = 0;
    for (int j = 0; j < np1; ++j) {
        const int hi = c->fp1_l[j];
        cudaStream_t ks = conc ? c->kst[j] : c->stream;
        TRY(copy_layers(c->params64, params, lo, hi, cudaMemcpyHostToDevice, c->cstream));
        cudaEvent_t up = conc ? c->pex[j] : c->pev[0];
        CK(cudaEventRecord(up, c->cstream));
        CK(cudaStreamWaitEvent(ks, up, 0));
        if (conc && j > 0) CK(cudaStreamWaitEvent(ks, c->pex[4 + j - 1], 0));
        const int b0 = c->fp1_b[j], nb = c->fp1_b[j + 1] - b0;
        const int zl = std::max(lo, c->pz0), zh = j + 1 == np1 ? c->pz1 : std::min(hi, c->pz1);
        const int nconv = zh > zl ? 296 : 0;
        k_fprep<<<(unsigned)(nconv + nb), 256, 0, ks>>>(c->params64, c->fphi4, g, zl, std::max(zl, zh), nconv,
                                                      c->fitems + b0, nb, t, c->fiflag + b0);
        CKL();
        if (conc) CK(cudaEventRecord(c->pex[4 + j], ks));
        TRY(launch_fast_pass1(c, b0, nb, false, ks));
        if (conc) CK(cudaEventRecord(c->pex[8 + j], ks));
        lo = hi;
    }
    if (conc)
        for (int j = 0; j < np1; ++j) CK(cudaStreamWaitEvent(c->stream, c->pex[8 + j], 0));
    k_stats_convert<<<592, 256, 0, c->stream>>>(c->SQi, c->SQ, (long long)stats_count(c), (long long)c->R * c->g.B * 2);
    CKL();
    TRY(run_combine(c));
    CK(cudaMemcpyAsync(c->pinned, c->Dout, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (grad) {
        const F2Args A = fast_pass2_args(c);
        PassArgs pa = pass_args(c);
        pa.invZ = 1.f;
        pa.gradi = c->gradi;
        pa.gbound = c->Dout + 2;
        pa.dxz = c->fdxz;
        pa.xbeg = c->xbeg;
        const int np2 = (int)c->fp2_l.size();
        if (c->fconc2 && np2 <= NPART) {
            // concurrent parts: part j on its own stream with its own exact-path list (a quarter
            // of the capacity: no kernel reads a list another part is still appending to); after
            // part j and the fix / conversion of part j - 1, part j's deferred voxels are fixed,
            // the layers final after part j converted and sent back.  An overflow of any part's
            // list is detected on the host and the evaluation redone without parts.
            const int cap = c->xcap / NPART;
            CK(cudaMemsetAsync(c->xcount, 0, NPART * sizeof(int), c->stream));
            CK(cudaEventRecord(c->pev[2], c->stream));
            int done = 0;
            for (int j = 0; j < np2; ++j) {
                cudaStream_t ks = c->kst[j];
                CK(cudaStreamWaitEvent(ks, c->pev[2], 0));
                F2Args Aj = A;
                Aj.xlist = c->xlist + (size_t)j * cap;
                Aj.xcount = c->xcount + j;
                Aj.xcap = cap;
                TRY(launch_fast_p2f(c, Aj, c->fp2_b[j], c->fp2_b[j + 1] - c->fp2_b[j], ks));
                if (j > 0) CK(cudaStreamWaitEvent(ks, c->pex[j - 1], 0));   // part j - 1 fixed and converted
                PassArgs pj = pa;
                pj.xlist = Aj.xlist;
                pj.xcount = Aj.xcount;
                pj.xcap = cap;
                pj.xbeg = nullptr;
                pj.xmode = 1;
                k_exact_fix<0><<<1184, 128, 0, ks>>>(pj);
                CKL();
                const int hi = c->fp2_l[j];
                if (hi > done) {
                    k_grad_convert_layers<<<592, 256, 0, ks>>>(c->gradi, c->grad64, (long long)plane, (long long)cs, g.ndim,
                                                               done, hi, c->Dout + 2, c->fdxz, 1.0 / c->Z);
                    CKL();
                }
                CK(cudaEventRecord(c->pex[j], ks));
                CK(cudaStreamWaitEvent(c->cstream, c->pex[j], 0));
                TRY(copy_layers(grad, c->grad64, done, hi, cudaMemcpyDeviceToHost, c->cstream));
                done = std::max(done, hi);
            }
            for (int j = 0; j < np2; ++j) CK(cudaStreamWaitEvent(c->stream, c->pex[j], 0));
            CK(cudaMemcpyAsync(c->pinned + 4, c->xcount, NPART * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        } else {
        CK(cudaMemsetAsync(c->xcount, 0, sizeof(int), c->stream));
        CK(cudaMemsetAsync(c->xbeg, 0, sizeof(int), c->stream));
        int done = 0;
        for (int j = 0; j < np2; ++j) {
            const bool last = j + 1 == np2;
            TRY(launch_fast_p2f(c, A, c->fp2_b[j], c->fp2_b[j + 1] - c->fp2_b[j]));
            pa.xmode = last ? 0 : 1;   // a list overflow scans the slab in the last part only
            k_exact_fix<0><<<1184, 128, 0, c->stream>>>(pa);
            CKL();
            const int hi = c->fp2_l[j];
            if (hi > done) {
                k_grad_convert_layers<<<592, 256, 0, c->stream>>>(c->gradi, c->grad64, (long long)plane, (long long)cs, g.ndim,
                                                                  done, hi, c->Dout + 2, c->fdxz, 1.0 / c->Z);
                CKL();
            }
            if (last) {
                TRY(copy_layers(grad, c->grad64, done, hi, cudaMemcpyDeviceToHost, c->stream));
            } else {
                CK(cudaMemcpyAsync(c->xbeg, c->xcount, sizeof(int), cudaMemcpyDeviceToDevice, c->stream));
                CK(cudaEventRecord(c->pev[2], c->stream));
                CK(cudaStreamWaitEvent(c->cstream, c->pev[2], 0));
                TRY(copy_layers(grad, c->grad64, done, hi, cudaMemcpyDeviceToHost, c->cstream));
            }
            done = std::max(done, hi);
        }
        CK(cudaMemcpyAsync(c->pinned + 4, c->xcount, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        }
    }
    // join the copy stream back (a graph capture must end on its origin stream)
    CK(cudaEventRecord(c->pev[1], c->cstream));
    CK(cudaStreamWaitEvent(c->stream, c->pev[1], 0));
    return SRWCR_OK;
}
static bool is_pinned_host(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
static srwcr_status eval_host_pipelined_fast(srwcr_ctx *c, const double *params, double *value, double *grad) {
    if (c->poisoned) return fail(c, SRWCR_ESTATE, "context poisoned by an earlier CUDA error");
    CK(cudaSetDevice(c->dev));
    if (c->opt.use_graph && is_pinned_host(params) && (!grad || is_pinned_host(grad))) {
        // pinned host buffers: the parts' copies, kernels and events as one CUDA graph,
        // captured once per (params, grad) pair (one launch instead of ~30 API calls)
        if (!c->hexec || c->h_params != params || c->h_grad != grad) {
            if (c->hexec) cudaGraphExecDestroy(c->hexec);
            c->hexec = nullptr;
            const int64_t l0 = c->launches;
            CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
            const srwcr_status st = enqueue_host_pipelined_fast(c, params, grad);
            cudaGraph_t gr = nullptr;
            const cudaError_t e = cudaStreamEndCapture(c->stream, &gr);
            c->h_kernels = c->launches - l0;
            c->launches = l0;
            if (st != SRWCR_OK || e != cudaSuccess) {
                if (gr) cudaGraphDestroy(gr);
                return st != SRWCR_OK ? st : fail(c, SRWCR_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
            }
            const cudaError_t e2 = cudaGraphInstantiate(&c->hexec, gr, cudaGraphInstantiateFlagUseNodePriority);
            cudaGraphDestroy(gr);
            if (e2 != cudaSuccess) {
                c->hexec = nullptr;
                return fail(c, SRWCR_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e2));
            }
            c->h_params = params;
            c->h_grad = grad;
        }
        CK(cudaGraphLaunch(c->hexec, c->stream));
        c->launches += c->h_kernels;
    } else {
        TRY(enqueue_host_pipelined_fast(c, params, grad));
    }
    CK(cudaStreamSynchronize(c->cstream));
    CK(cudaStreamSynchronize(c->stream));
    if (grad) {
        int xc[NPART] = {};
        memcpy(xc, c->pinned + 4, sizeof xc);
        const int np2 = (int)c->fp2_l.size();
        bool over = xc[0] > c->xcap;
        if (c->fconc2 && np2 <= NPART) {
            over = false;
            for (int j = 0; j < np2; ++j) over = over || xc[j] > c->xcap / NPART;
        }
        c->xparts = c->fconc2 && np2 <= NPART ? np2 : 1;
        if (over) {
            c->xparts = 1;
            // list overflow: voxels of layers already converted were fixed by the last part's
            // scan after their conversion (their int64 adds are still in gradi) -- rare;
            // clear the int64 gradient and evaluate again without the parts
            CK(cudaMemsetAsync(c->gradi, 0, sizeof(unsigned long long) * c->nparams, c->stream));
            TRY(eval_begin_impl(c, params));
            return eval_end_impl(c, value, grad, true);
        }
    }
    return eval_finish(c, value);
}

extern "C" srwcr_status srwcr_eval(srwcr_ctx *c, const double *params, double *value, double *grad) {
    if (!c) return SRWCR_EINVAL;
    c->xparts = 1;
    if (c->external_exchange) return fail(c, SRWCR_ESTATE, "caller-driven exchange: use srwcr_eval_begin/end");
    if (c->opt.use_graph && !c->poisoned && params && is_device_ptr(params) &&
        (!grad || is_device_ptr(grad)))
        return eval_graph(c, params, value, grad);
    if (!c->comm && !c->timing && !c->poisoned && !c->fast && params && (c->p1_split > 0 || c->p2_split > 0) &&
        !is_device_ptr(params) && (!grad || !is_device_ptr(grad)))
        return eval_host_pipelined(c, params, value, grad);
    if (!c->comm && !c->timing && !c->poisoned && c->fast && params && !c->fp1_b.empty() && !is_device_ptr(params) &&
        (!grad || !is_device_ptr(grad)) && !getenv("SRWCR_NOPIPE"))
        return eval_host_pipelined_fast(c, params, value, grad);
    TRY(eval_begin_impl(c, params));
    if (!c->fast) TRY(allreduce(c, c->SQ, stats_count(c)));   // (fast: int64 sum inside eval_begin)
    return eval_end_impl(c, value, grad, true);
}

extern "C" srwcr_status srwcr_eval_begin(srwcr_ctx *c, const double *params) {
    if (!c) return SRWCR_EINVAL;
    TRY(eval_begin_impl(c, params));
    CK(cudaStreamSynchronize(c->stream));
    c->begun = true;
    return SRWCR_OK;
}
extern "C" srwcr_status srwcr_stats_buffer(srwcr_ctx *c, double **dev_ptr, size_t *count) {
    if (!c || !dev_ptr || !count) return SRWCR_EINVAL;
    *dev_ptr = c->SQ;
    *count = stats_count(c);
    return SRWCR_OK;
}
extern "C" srwcr_status srwcr_eval_end(srwcr_ctx *c, double *value, double *grad) {
    if (!c) return SRWCR_EINVAL;
    if (!c->begun) return fail(c, SRWCR_ESTATE, "srwcr_eval_end without srwcr_eval_begin");
    c->begun = false;
    // the caller summed the statistics in place, possibly with copies on another stream or a
    // pageable cudaMemcpy whose DMA can still be in flight when it returns: wait for all of it
    CK(cudaDeviceSynchronize());
    c->xparts = 1;
    return eval_end_impl(c, value, grad, false);
}

// ------------------------------------------------------------------ debug dumps
extern "C" srwcr_status srwcr_debug_size(const srwcr_ctx *c, int32_t what, size_t *bytes) {
    if (!c || !bytes) return SRWCR_EINVAL;
    const long long nvox = (long long)c->g.nx * c->g.ny * c->g.nz, RB = c->R * c->g.B;
    switch (what) {
        case SRWCR_DUMP_FIXED: case SRWCR_DUMP_MOVING: *bytes = sizeof(float) * nvox; break;
        case SRWCR_DUMP_A0: *bytes = sizeof(short) * nvox; break;
        case SRWCR_DUMP_CTRL_TAPS: case SRWCR_DUMP_SPAT_TAPS: *bytes = sizeof(int) * (c->g.nx + c->g.ny + c->g.nz); break;
        case SRWCR_DUMP_N: *bytes = sizeof(double) * RB; break;
        case SRWCR_DUMP_SQ: *bytes = sizeof(double) * (RB + c->R); break;
        case SRWCR_DUMP_REGIONS: *bytes = sizeof(double) * c->R * 6; break;
        case SRWCR_DUMP_COEFS: *bytes = sizeof(float) * (2 * c->R + RB); break;
        case SRWCR_DUMP_WARPED: *bytes = sizeof(float4) * (size_t)((c->z1 - c->z0) * (long long)c->g.nxy); break;
        default: return SRWCR_EINVAL;
    }
    return SRWCR_OK;
}

extern "C" srwcr_status srwcr_debug_dump(srwcr_ctx *c, int32_t what, void *out, size_t bytes) {
    if (!c || !out) return SRWCR_EINVAL;
    if (c->poisoned) return fail(c, SRWCR_ESTATE, "context poisoned");
    size_t need = 0;
    if (srwcr_debug_size(c, what, &need) != SRWCR_OK) return fail(c, SRWCR_EINVAL, "unknown dump %d", what);
    if (bytes < need) return fail(c, SRWCR_EINVAL, "bytes %zu < %zu", bytes, need);
    CK(cudaSetDevice(c->dev));
    CK(cudaStreamSynchronize(c->stream));
    const long long nvox = (long long)c->g.nx * c->g.ny * c->g.nz, RB = c->R * c->g.B;
    switch (what) {
        case SRWCR_DUMP_FIXED: CK(cudaMemcpy(out, c->F, need, cudaMemcpyDeviceToHost)); break;
        case SRWCR_DUMP_MOVING: CK(cudaMemcpy(out, c->M, need, cudaMemcpyDeviceToHost)); break;
        case SRWCR_DUMP_A0: {
            short *d = nullptr;
            CK(cudaMalloc(&d, need));
            k_a0_map<<<1184, 256>>>(c->F, d, nvox, c->g.L);
            CKL();
            CK(cudaMemcpy(out, d, need, cudaMemcpyDeviceToHost));
            cudaFree(d);
            break;
        }
        case SRWCR_DUMP_CTRL_TAPS: case SRWCR_DUMP_SPAT_TAPS: {
            int *o = (int *)out;
            for (int ax = 0; ax < 3; ++ax) {
                const std::vector<int> &v = what == SRWCR_DUMP_CTRL_TAPS ? c->h_cb[ax] : c->h_sb[ax];
                memcpy(o, v.data(), sizeof(int) * v.size());
                o += v.size();
            }
            break;
        }
        case SRWCR_DUMP_N: {
            std::vector<double> lo(RB), up(RB);
            CK(cudaMemcpy(lo.data(), c->Nlo, sizeof(double) * RB, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(up.data(), c->Nup, sizeof(double) * RB, cudaMemcpyDeviceToHost));
            double *o = (double *)out;
            const int B = c->g.B;
            for (long long r = 0; r < c->R; ++r)
                for (int b = 0; b < B; ++b) o[r * B + b] = lo[r * B + b] + (b > 0 ? up[r * B + b - 1] : 0.0);
            break;
        }
        case SRWCR_DUMP_SQ: {
            // re-run the (deterministic) combine of the last statistics with the S output on
            c->dump_S = true;
            const srwcr_status st = run_combine(c);
            c->dump_S = false;
            if (st != SRWCR_OK) return st;
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaMemcpy(out, c->S_out, sizeof(double) * RB, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy((double *)out + RB, c->Qt, sizeof(double) * c->R, cudaMemcpyDeviceToHost));
            break;
        }
        case SRWCR_DUMP_REGIONS: CK(cudaMemcpy(out, c->reg, need, cudaMemcpyDeviceToHost)); break;
        case SRWCR_DUMP_WARPED: CK(cudaMemcpy(out, c->MG, need, cudaMemcpyDeviceToHost)); break;
        case SRWCR_DUMP_COEFS:
            CK(cudaMemcpy(out, c->alpha, sizeof(float) * c->R, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy((float *)out + c->R, c->beta, sizeof(float) * c->R, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy((float *)out + 2 * c->R, c->gamma, sizeof(float) * RB, cudaMemcpyDeviceToHost));
            break;
    }
    return SRWCR_OK;
}

extern "C" srwcr_status srwcr_set_timing(srwcr_ctx *c, int32_t enable) {
    if (!c) return SRWCR_EINVAL;
    c->timing = enable != 0;
    return SRWCR_OK;
}
extern "C" srwcr_status srwcr_get_stats(const srwcr_ctx *c, srwcr_stats *out) {
    if (!c || !out) return SRWCR_EINVAL;
    out->launches_total = c->launches;
    out->launches_per_eval = c->launches_per_eval;
    out->ms_pass1 = c->ms[0];
    out->ms_combine = c->ms[1];
    out->ms_pass2 = c->ms[2];
    out->ms_total = c->ms[3];
    out->warps_per_cta = c->W;
    out->slot_capacity = c->S;
    out->voxels_per_lane = c->XV;
    out->items = c->nitems;
    out->ms_prep = c->ms[4];
    out->warps_per_cta2 = c->W2;
    out->items2 = c->nitems2;
    out->exact_capacity = c->xcap;
    out->pipe_items1 = c->p1_split;
    out->pipe_items2 = c->p2_split;
    out->exact_voxels = 0;
    for (int j = 0; c->pinned && j < c->xparts; ++j) out->exact_voxels += reinterpret_cast<const int *>(c->pinned + 4)[j];
    out->fast_path = c->fast ? 1 : 0;
    out->fast_items = c->nfitems;
    out->fast_warps = c->fW;
    out->fast_slots = c->fS;
    return SRWCR_OK;
}
extern "C" srwcr_status srwcr_stream(const srwcr_ctx *c, void **stream) {
    if (!c || !stream) return SRWCR_EINVAL;
    *stream = (void *)c->stream;
    return SRWCR_OK;
}
extern "C" const char *srwcr_last_error(const srwcr_ctx *c) { return c ? c->err.c_str() : "null context"; }

extern "C" void srwcr_destroy(srwcr_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->dev);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm && nccl().ok) nccl().CommDestroy(c->comm);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    if (c->hexec) cudaGraphExecDestroy(c->hexec);
    if (c->cstream) cudaStreamSynchronize(c->cstream);
    if (c->ftexM) cudaDestroyTextureObject(c->ftexM);
    if (c->fMarr) cudaFreeArray(c->fMarr);
    for (int i = 0; i < 4; ++i)
        if (c->pev[i]) cudaEventDestroy(c->pev[i]);
    for (int i = 0; i < 12; ++i)
        if (c->pex[i]) cudaEventDestroy(c->pex[i]);
    for (int i = 0; i < NPART; ++i)
        if (c->kst[i]) cudaStreamDestroy(c->kst[i]);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    void *bufs[] = {c->F, c->M, c->phi, c->phimax, c->MG, c->xlist, c->params64, c->grad64, c->items, c->items_full, c->items2, c->itemw, c->itemw_full,
                    c->slotbins, c->SQ, c->Nlo, c->Nup, c->dterm, c->reg, c->Dout, c->S_out, c->shiftc, c->alpha,
                    c->beta, c->gamma, c->ticket, c->dpart, c->xbeg, c->fitems, c->fitemw, c->fslotbins,
                    c->fiflag, c->frec, c->floff, c->flent, c->frmask, c->SQi, c->gradi, c->fMv, c->fphi4, c->halo_recv};
    for (void *p : bufs)
        if (p) cudaFree(p);
    for (int i = 0; i < 3; ++i) {
        if (c->cb[i]) cudaFree(c->cb[i]);
        if (c->cw[i]) cudaFree(c->cw[i]);
        if (c->cw64[i]) cudaFree(c->cw64[i]);
        if (c->sb[i]) cudaFree(c->sb[i]);
        if (c->sw[i]) cudaFree(c->sw[i]);
    }
    for (int i = 0; i < 5; ++i)
        if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->dot_host) cudaFreeHost(c->dot_host);
    for (double *p : {c->bend_gram, c->bend_ws, c->dot_part})
        if (p) cudaFree(p);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// ------------------------------------------------------------------ L-BFGS
#include "srwcr_register.inc"
// ------------------------------------------- fields / pyramid utilities (row F4)
#include "srwcr_fields.inc"
