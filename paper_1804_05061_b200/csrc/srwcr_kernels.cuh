// srwcr_kernels.cuh -- sm_100a kernels of the SRWCR hot path (arXiv 1804.05061).
//
// One SRWCR evaluation = pass 1 (k_pass1: FFD + trilinear warp + Parzen moments +
// privatised histogram), combine (k_combine, D reduced by its last CTA: per-region correlation
// ratios, D and the backward coefficient tables), pass 2 (k_pass2: pass 1's (m, dM/dy)
// per voxel + dD/dm + adjoint B-spline scatter onto the control lattice), k_exact_fix
// (the voxels whose derivative the fp64 definition must decide).
// Per-voxel intermediates stay in registers except one float4 (m, dM/dy) per voxel that
// pass 1 streams to pass 2 (the paper's kernels 1-4 materialise the warped image and the
// derivative volumes).  DESIGN.md s5-s6 describe the data flow,
// the roofline of each kernel and what differs from the paper's GPU design.
//
// Work decomposition: a CTA owns one "item" = a box of voxels inside ONE spatial cell
// (all its voxels share the same 4x4x4 = 64 regions of Eq 7) -- or, on fine spatial
// lattices (MC variants), up to 5 x-cells by 3 z-cells with per-lane region offsets.  Each warp owns
// whole rows of the item: lane = x (XV voxels per lane: x0+lane, x0+lane+32), and the
// warp marches z through the item independently of the other warps (no CTA barrier
// inside the march).  CTA-level tables are touched only at row and item ends.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace srwcr {

constexpr unsigned FULL = 0xffffffffu;
constexpr int LTS = 9;          // line-table slot stride: 8 entries (4 x-taps x {lo, hi}) + 1 pad
constexpr int GYS = 5;          // pass-2 per-warp gamma table: float4 per (bin, x-tap), 4 + 1 pad per bin
constexpr int MAXW = 16;        // max warps per CTA
constexpr int MC_XRN = 8;       // multi-cell items: x-regions per item (<= 5 spatial x-cells)
constexpr int MC_ZRN = 8;       //                   z-regions per item (<= 5 spatial z-cells)

struct Tables {                 // per-axis B-spline taps, index = voxel coordinate on that axis
    const int *cb[3];           // control lattice: tap base floor(i/delta)          (Eq 17)
    const float4 *cw[3];        //                  beta_0..3(i/delta - base)         (Eq 8)
    const double4 *cw64[3];     //                  same weights in fp64 (exact-sample path)
    const int *sb[3];           // spatial lattice: tap base floor(i/Delta)          (Eq 7)
    const float4 *sw[3];
};

struct Geo {
    int nx, ny, nz;
    long long nxy;
    int L, B;                   // maximal bin L_eps and bin count L+1
    int Gx, Gy, Gz;             // internal control grid (Gz padded to 4 in 2-D)
    int Kx, Ky, Kz;             // regions per axis
    int ndim, GzExt;            // external components (2 or 3) and external Gz
    int nxy32, nxm2, nym2, nzm2, dzo;  // host-precomputed: nx*ny, max(N-2, 0) per axis, z stride (0 in 2-D)
};

struct Item {
    int x0, xlen, y0, ylen, z0, zlen;
    int slot_off, nslots;       // the item's fixed bins a0 (static slot list in slotbins)
    float cI;                   // binless moment shift of the item (mean of M over the box)
    int pad;
};
// per-item sums of the fp32 spatial weights: sx per relative x-region (MC items span cells)
struct ItemW { double sx[8], sy[4], sz[8]; };

struct PassArgs {
    Geo g;
    Tables t;
    const float *F;             // normalised fixed image  (model image A)
    const float *M;             // normalised moving image (estimated image B after warping)
    const float *phi;           // fp32 displacements [3][Gz][Gy][Gx]
    const float *shiftc;        // per-fixed-bin shift c_a of the binned first moment
    const Item *items;
    const ItemW *itemw;
    const int *slotbins;        // concatenated per-item slot -> bin lists
    double *SQ;                 // pass 1 out: [R][B][2] shifted binned first moments (lo, hi)
    double *Qt;                 // pass 1 out: [R] binless second moments sum_x w_r g2(m)
    double *NQ;                 // pass 1 out (ORI 1): [R][B][2] dynamic counts N' (lo, hi halves)
    int gstride;                // pass 2: row stride of the gamma table (B; ORI 1: 3 (B + 2))
    int W, S, S2;               // warps per CTA, slot capacity, pass-2 bin-list capacity
    const double *p64;          // pass 2: fp64 params, external layout (exact-sample path)
    const float4 *tolw;         // pass 1: [Gz][Gy][Gx] 2e-6 max |phi_c| over the tap window (c = x,y,z)
    int *xlist, *xcount;        // pass 2: slab-linear indices of the voxels deferred to k_exact_fix
    const int *xbeg;            // k_exact_fix: first list entry to process (null: 0)
    int xmode;                  // k_exact_fix on overflow: 0 scan the slab, 1 nothing (a later launch scans)
    int xcap;                   //         capacity of xlist
    int mgz1;                   //         slab slices (k_exact_fix scan fallback)
    int zrn;                    // multi-cell items: z-regions per item (z-cells + 3, <= MC_ZRN)
    float4 *MG;                 // pass 1 out / pass 2 in: per slab voxel (m, dM/dy) -- m < 0
    int mgz0;                   //   encodes -1 - m for voxels that need the fp64 exact path
    const float *alpha, *beta, *gamma;  // pass 2 in: [R], [R], [R][B]
    float invZ;
    double *grad;               // pass 2 out: [ndim][GzExt][Gy][Gx] (fp64)
    unsigned long long *gradi;  // fast pass 2: int64 gradient (units 2^-k, without 1/Z), or null
    const double *gbound;       //   the combine's per-voxel bound (k = grad_shift(*gbound, dxz))
    float dxz;                  //   delta_x * delta_z (+1 each): per-add bound factor
};

// Fixed-point shift k of fast pass 2's gradient accumulation: one node-window add is at most
// (delta_x + 1)(delta_z + 1) gbound in magnitude (the B-spline weights of a node sum to about
// delta per axis); k keeps it below 2^40 so that the int32 (hi, lo) pair of the node window and
// the int64 global sums are exact.
__device__ __forceinline__ int grad_shift(double b1, float dxz) {
    const double bnd = b1 * (double)dxz * 1.1;
    if (!(bnd > 0.0) || !(bnd < 1e300)) return 40;
    int e;
    frexp(bnd, &e);   // bnd < 2^e
    return max(-200, min(60, 40 - e));
}

__device__ __forceinline__ float f4(const float4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ float dot4(const float4 &a, const float4 &b) {
    return fmaf(a.w, b.w, fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x)));
}
// streaming load (read once: do not allocate in L1, keep L1 for the gathers of M)
__device__ __forceinline__ float ld_stream(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_stream4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
// streaming store (written once, read once by the next pass)
__device__ __forceinline__ void st_stream4(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

// 2^k as a float, k in [-126, 127]
__device__ __forceinline__ float exp2i(int k) { return __int_as_float((k + 127) << 23); }

// ---------------------------------------------------------------- FFD
// Contribution of control layer gz to the displacements of this lane's XV voxels,
// contracted over the 4x4 (x, y) taps: U[v][c] = sum_{l,m} cwx_l cwy_m phi[c][gz][cby+m][cbx_v+l].
// The warp shares one row y, so lanes j < nxn first contract y for x-node xn0+j
// (coalesced loads), then every lane gathers its 4 x-taps per voxel by shuffle.
template <int XV, int NC = 3>
__device__ __forceinline__ void ffd_layer(const float *__restrict__ phi, const Geo &g, int gz, int cby, float4 cwy,
                                          int xn0, int nxn, const int (&relx)[XV], const float4 (&cwx)[XV],
                                          int lane, float (&U)[XV][NC]) {
    float p[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) p[c] = 0.f;
    if (lane < nxn) {
        const long long plane = (long long)g.Gx * g.Gy;
        const long long cs = plane * g.Gz;
        const float *q = phi + (long long)gz * plane + (long long)cby * g.Gx + xn0 + lane;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float w = f4(cwy, m);
#pragma unroll
            for (int c = 0; c < NC; ++c) p[c] = fmaf(w, __ldg(q + c * cs + m * g.Gx), p[c]);
        }
    }
#pragma unroll
    for (int v = 0; v < XV; ++v) {
#pragma unroll
        for (int c = 0; c < NC; ++c) U[v][c] = 0.f;
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int src = relx[v] + l;
            const float w = f4(cwx[v], l);
#pragma unroll
            for (int c = 0; c < NC; ++c) U[v][c] = fmaf(w, __shfl_sync(FULL, p[c], src), U[v][c]);
        }
    }
}

// ------------------------------------------------ backward warping (c1-c3)
// Split sample coordinate along one axis: position i + u with i integer.  The cell is
// formed as the integer i + floor(u) and t = u - floor(u) stays a small fp32 fraction
// (never i + u in fp32: SURVEY H11).  Out-of-domain positions clamp to [0, N-1] and
// report `clamped` (their derivative is 0, reading c2); cell = min(floor y, N-2).
__device__ __forceinline__ void axis_cell(int i, float u, int N, int &c0, float &t, bool &cl) {
    if (N == 1) { c0 = 0; t = 0.f; cl = true; return; }
    const float fu = floorf(u);
    const int c = i + (int)fu;
    const float tt = u - fu;
    if (c < 0) { c0 = 0; t = 0.f; cl = true; }
    else if (c >= N - 1) { c0 = N - 2; t = 1.f; cl = !(c == N - 1 && tt == 0.f); }
    else { c0 = c; t = tt; cl = false; }
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

// trilinear value (nested lerps) and, if GRAD, the analytic gradient of the interpolant
template <bool GRAD>
__device__ __forceinline__ float sample_m(const float *__restrict__ M, const Geo &g, int x, int y, int z,
                                          float ux, float uy, float uz, float &gx, float &gy, float &gz) {
    int cx, cy, cz;
    float tx, ty, tz;
    bool clx, cly, clz;
    axis_cell(x, ux, g.nx, cx, tx, clx);
    axis_cell(y, uy, g.ny, cy, ty, cly);
    axis_cell(z, uz, g.nz, cz, tz, clz);
    const long long dyo = g.nx, dzo = g.nz > 1 ? g.nxy : 0;
    const float *b = M + (long long)cz * g.nxy + (long long)cy * g.nx + cx;
    const float c000 = __ldg(b), c100 = __ldg(b + 1), c010 = __ldg(b + dyo), c110 = __ldg(b + dyo + 1);
    const float c001 = __ldg(b + dzo), c101 = __ldg(b + dzo + 1), c011 = __ldg(b + dzo + dyo),
                c111 = __ldg(b + dzo + dyo + 1);
    const float e00 = lerpf(c000, c100, tx), e10 = lerpf(c010, c110, tx);
    const float e01 = lerpf(c001, c101, tx), e11 = lerpf(c011, c111, tx);
    const float f0 = lerpf(e00, e10, ty), f1 = lerpf(e01, e11, ty);
    if (GRAD) {
        const float dx0 = lerpf(c100 - c000, c110 - c010, ty), dx1 = lerpf(c101 - c001, c111 - c011, ty);
        const float dy0 = lerpf(c010 - c000, c110 - c100, tx), dy1 = lerpf(c011 - c001, c111 - c101, tx);
        gx = clx ? 0.f : lerpf(dx0, dx1, tz);
        gy = cly ? 0.f : lerpf(dy0, dy1, tz);
        gz = clz ? 0.f : (f1 - f0);
    }
    return lerpf(f0, f1, tz);
}

// ------------------------------------------------------------ Parzen (Eq 5)
// weights of the two active bins a0 = min(floor v, L-1) and a0+1 at fraction f:
// h(f) and h(1-f), written so that f = 0 and f = 1 give exact zeros (reading c5).
__device__ __forceinline__ void parzen_pair(float f, float &hlo, float &hhi) {
    if (f < 0.5f) {
        const float w = f * fmaf(1.8f, f, 0.1f);
        hhi = w;
        hlo = 1.0f - w;
    } else {
        const float s = 1.0f - f;
        const float w = s * fmaf(1.8f, s, 0.1f);
        hlo = w;
        hhi = 1.0f - w;
    }
}

// Parzen pair of the FIXED image with h_hi rounded to a multiple of 2^-23 (|error| <= 2^-24,
// fp32-rounding size): the static record of the fast passes stores h_hi in 24 bits, and every
// pass, the static counts N and the exact path use the same weights, so that S and N (whose
// ratio is the conditional mean of Eq 10) are accumulated with identical h.
__device__ __forceinline__ void parzen_pair_F(float f, float &hlo, float &hhi) {
    float lo, hi;
    parzen_pair(f, lo, hi);
    // the zero pattern is kept: a nonzero weight never rounds to 0 (nor its complement)
    float k = rintf(hi * 8388608.f);
    k = hi > 0.f ? fmaxf(k, 1.f) : k;
    k = lo > 0.f ? fminf(k, 8388607.f) : k;
    hhi = k * (1.f / 8388608.f);
    hlo = 1.0f - hhi;
}

// recursive-halving warp reduction of 8 per-lane values: afterwards every lane holds
// the warp total of value (lane >> 2)   (9 shuffles)
__device__ __forceinline__ float halving8(const float (&v)[8], int lane) {
    float r4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = (lane & 16) ? v[i] : v[i + 4], keep = (lane & 16) ? v[i + 4] : v[i];
        r4[i] = keep + __shfl_xor_sync(FULL, send, 16);
    }
    float r2[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = (lane & 8) ? r4[i] : r4[i + 2], keep = (lane & 8) ? r4[i + 2] : r4[i];
        r2[i] = keep + __shfl_xor_sync(FULL, send, 8);
    }
    const float send = (lane & 4) ? r2[0] : r2[1], keep = (lane & 4) ? r2[1] : r2[0];
    float r = keep + __shfl_xor_sync(FULL, send, 4);
    r += __shfl_xor_sync(FULL, r, 2);
    r += __shfl_xor_sync(FULL, r, 1);
    return r;
}

// position of the r-th (0-based) set bit of w (branch-free 5-step select)
__device__ __forceinline__ int select_bit(unsigned w, int r) {
    int pos = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const unsigned lo = w & ((1u << s) - 1u);
        const int c = __popc(lo);
        const bool up = r >= c;
        r = up ? r - c : r;
        w = up ? (w >> s) : lo;
        pos += up ? s : 0;
    }
    return pos;
}
// the j-th set bit of a (<= 32 NWD-bit) mask, or -1
template <int NWD>
__device__ __forceinline__ int mask_select(const unsigned (&bits)[NWD], int nw, int j) {
    int pos = -1, base = 0;
#pragma unroll
    for (int k = 0; k < NWD; ++k) {
        if (k < nw) {
            const int c = __popc(bits[k]);
            if (pos < 0 && j >= base && j < base + c) pos = 32 * k + select_bit(bits[k], j - base);
            base += c;
        }
    }
    return pos;
}

// sample cell along one axis (pass 1: no clamp flag), branch free; nm2 = max(N-2, 0)
__device__ __forceinline__ int axis_fast(int i, float u, int nm2, float &t) {
    const float fu = floorf(u);
    const int c = i + (int)fu;
    const float tt = u - fu;
    t = c < 0 ? 0.f : (c > nm2 ? 1.f : tt);
    return min(max(c, 0), nm2);
}
// branch-free, with the clamp flag of reading c2 and the near-integer flag (below)
__device__ __forceinline__ int axis_fast_fl(int i, float u, int nm2, float tol, float &t, bool &cl, bool &near) {
    const float fu = floorf(u);
    const int c = i + (int)fu;
    const float tt = u - fu;
    const bool lo = c < 0, hi = c > nm2;
    t = lo ? 0.f : (hi ? 1.f : tt);
    // clamped iff the position c + tt lies outside [0, N-1]: 2c + (tt > 0) outside [0, 2(N-1)]
    cl = (unsigned)(2 * c + (tt > 0.f ? 1 : 0)) > (unsigned)(2 * nm2 + 2);
    // (far outside the volume the flag may be raised needlessly: harmless, the fp64 path
    // then confirms the clamp)
    near = fabsf(u - rintf(u)) < tol;
    return min(max(c, 0), nm2);
}
// same (branchy) with the clamp flag of reading c2 (derivative 0 along a clamped axis) and a
// flag telling that the fp32 position lies within tol of an integer, i.e. of a cell or
// clamp boundary where the derivative of the interpolant jumps.  tol bounds |u32 - u64|
// (see k_pass2); tol = 0 (all tap nodes of the component at rest) never flags.
__device__ __forceinline__ int axis_fast_cl(int i, float u, int nm2, float tol, float &t, bool &cl, bool &near) {
    const float fu = floorf(u);
    int c = i + (int)fu;
    t = u - fu;
    cl = false;
    // cell and clamp boundaries sit at integer u; u - rint(u) is exact in fp32
    near = fabsf(u - rintf(u)) < tol;
    if ((unsigned)c > (unsigned)nm2) {       // rare: outside [0, N-2]
        if (c < 0) { near = near && c == -1; c = 0; t = 0.f; cl = true; }
        else { near = near && c == nm2 + 1; cl = !(c == nm2 + 1 && t == 0.f); c = nm2; t = 1.f; }
    }
    return c;
}

// ---------------------------------------------------------------- pass 1
// Moving-as-B orientation: the fixed-image bins and the spatial weights are static, so
// the combine needs, per region r,
//   binned (per fixed bin a):  S_ra = sum_x w_r h_a(F) g1(m),  g1 = sum_b b h(b - m)
//   binless:                   Q_r  = sum_x w_r g2(m),          g2 = sum_b b^2 h(b - m)
// (Eq 3 P:73 rewritten as moments; V_r = Q_r - sum_a S_ra^2/N_ra needs
// Q only per region).  Per voxel the binned part is keyed by a0 (the lower Parzen bin of
// F) with two channels  lo = h_lo (g1 - c_a0),  hi = h_hi (g1 - c_a0)  (c_a: per-bin
// shift), times the 4 spatial x-taps -> 8 values.  The binless part is q' = (g1 - cI)^2
// + w1 (1 - w1) and g1 - cI (cI: per-item shift), times the 4 x-taps.
//
// Privatisation, all per warp, no CTA barrier inside the march:
//   line  : LT[warp][slot][8]  int32 fixed point (native ATOMS; warp-uniform bins reduce
//           in registers), one 32/64-voxel line = one (row, z)
//   column: K[warp][slot][8][4 z-taps]  fp32, after every line; 4 slots per instruction
//   cell  : CT[slot][4 y-taps][32]  fp32 (CTA), after every row: K x wy, float atomics
//   global: SQ[r][bin][2] fp64 atomics, once per item
// STATIC mode accumulates the weighted counts (lo = h_lo, hi = h_hi) in fp32 (float
// line tables) so that the zero pattern of N is exact.
// Lanes past the item's x-extent sample the item's last column with zero weights, so
// the voxel loop has no divergent branches.
// ORI = 1 (moving image as the model image A, Eq 20-21): the bins come from
// m (dynamic, n = min(floor m, L-1)), the item's slot list is every bin, and each voxel
// feeds two slot groups: 2*slot(n) the counts N'_{r,n|n+1} = sum w h_{n|n+1}(m) and
// 2*slot(n)+1 the first moments S'_{r,n|n+1} = sum w h_{n|n+1}(m) (g1(F) - c_n); the
// second moments of F are static (no binless channel).
// MAXT <= 256 (small items of fine spatial lattices, few warps per CTA): register budget for
// 4 resident CTAs per SM -- their latency is otherwise exposed at 2 CTAs (Table VIII
// 256x256x99: 4.1 -> 2.9 ms per evaluation with pass 2 at 5 CTAs)
// MC (multi-cell items, fine spatial lattices, ORI 0): an item spans up to MC_CELLS
// spatial x-cells; every lane keeps its own cell offset lcx, the tables are indexed by the
// relative x-region xr = lcx + l (XRN = 8 of them: 16 entries per slot), the warp-uniform
// halving path is off, and the binless channels (q', g1 - cI) are one more slot of the
// line tables (index ns) with their own fixed-point exponents.
template <int XV, bool STATIC, int MAXT = 512, int ORI = 0, bool MC = false>
__global__ void __launch_bounds__(MAXT, MAXT <= 256 ? (MC ? 3 : 4) : 1) k_pass1(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int XRN = MC ? MC_XRN : 4;      // x-regions per item
    constexpr int E = 2 * XRN;                // line-table entries per slot
    constexpr int LTSV = MC ? 2 * MC_XRN + 1 : LTS;
    constexpr int KS = 4 * E;                 // column-table floats per slot (entry*4 + n)
    const int ZR = MC ? a.zrn : 4;            // z-regions of the item's cell table
    const int CTS = MC ? 4 * ZR * E : 4 * KS; // cell-table floats per slot
    const Geo &g = a.g;
    const int B = g.B, W = a.W, S = a.S;
    const int ltsz = (W * S * LTSV + 3) & ~3;                     // keep K 16-byte aligned
    int *LT = reinterpret_cast<int *>(smem);                      // [W][S][LTSV]
    float *K = reinterpret_cast<float *>(LT + ltsz);              // [W][S][KS]
    float *CT = K + W * S * KS;                                   // [S][4][KS]  (MC: [S][4 m][ZRN zr][E])
    float *CB = CT + S * CTS;                                     // [4][32] binless cell table (!MC)
    float4 *ZT = reinterpret_cast<float4 *>(CB + 128);            // [2][64] the item's z-tap tables
    int *ZB = reinterpret_cast<int *>(ZT + 128);                  // [64] control-tap bases, MC: | z-cell offset << 20
    float *shc = reinterpret_cast<float *>(ZB + 64);              // [B]
    unsigned char *smap = reinterpret_cast<unsigned char *>(shc + B);  // [B] bin -> slot

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Item it = a.items[blockIdx.x];
    const int ns = it.nslots;                       // list entries (ORI 1: every bin)
    const int nsl = ORI ? 2 * ns : ns + (MC ? 1 : 0); // slots (ORI 1: two groups per bin; MC: + binless)
    const int nwords = (nsl + 31) >> 5;
    constexpr int NW = ORI ? 8 : 4;                 // slot-mask words (ORI 1: 2 slots per bin, B <= 128)

    for (int i = threadIdx.x; i < ltsz; i += blockDim.x) LT[i] = 0;
    for (int i = threadIdx.x; i < W * S * KS; i += blockDim.x) K[i] = 0.f;
    for (int i = threadIdx.x; i < nsl * CTS + 128; i += blockDim.x) (i < nsl * CTS ? CT[i] : CB[i - nsl * CTS]) = 0.f;
    for (int i = threadIdx.x; i < B; i += blockDim.x) {
        shc[i] = STATIC ? 0.f : a.shiftc[i];
        smap[i] = 0xFF;
    }
    for (int i = threadIdx.x; i < it.zlen; i += blockDim.x) {   // z-tap tables in shared memory
        ZT[i] = a.t.cw[2][it.z0 + i];
        ZT[64 + i] = a.t.sw[2][it.z0 + i];
        ZB[i] = a.t.cb[2][it.z0 + i] | (MC ? (a.t.sb[2][it.z0 + i] - a.t.sb[2][it.z0]) << 20 : 0);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) smap[a.slotbins[it.slot_off + s]] = (unsigned char)s;

    const int cx = a.t.sb[0][it.x0], cy = a.t.sb[1][it.y0], cz = a.t.sb[2][it.z0];
    const int xn0 = a.t.cb[0][it.x0];
    const int nxn = a.t.cb[0][it.x0 + it.xlen - 1] + 4 - xn0;
    int xv[XV], relx[XV], lcx[XV];
    float4 cwx[XV], swx[XV];
#pragma unroll
    for (int v = 0; v < XV; ++v) {
        const bool ok = lane + 32 * v < it.xlen;
        xv[v] = ok ? it.x0 + lane + 32 * v : it.x0 + it.xlen - 1;
        lcx[v] = MC ? a.t.sb[0][xv[v]] - cx : 0;
        relx[v] = a.t.cb[0][xv[v]] - xn0;
        cwx[v] = a.t.cw[0][xv[v]];
        swx[v] = ok ? a.t.sw[0][xv[v]] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // fixed-point exponents (dynamic mode): value v_c * wx_l is scaled by 2^(274 - El - EA)
    // where 2^(El-126) bounds max_lanes wx_l (static per item) and 2^(EA-126) bounds
    // max_lanes |g1 - c| (per line): |scaled| < 2^22 (exact magic-number conversion) and a
    // 64-value lane sum stays < 2^28.
    int El[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        float mx = 0.f;
#pragma unroll
        for (int v = 0; v < XV; ++v) mx = fmaxf(mx, f4(swx[v], l));
        El[l] = (int)(__reduce_max_sync(FULL, __float_as_uint(mx)) >> 23);
    }
    if (MC) {   // one exponent for all x-taps: an entry mixes lanes of different cells (taps)
        const int em = max(max(El[0], El[1]), max(El[2], El[3]));
#pragma unroll
        for (int l = 0; l < 4; ++l) El[l] = em;
    }
    const int le = (lane & 7) >> 1;                               // fold lane's x-tap
    const int El_e = le == 0 ? El[0] : le == 1 ? El[1] : le == 2 ? El[2] : El[3];
    // mixed-bin path: lane q = lane & 3 visits the x-taps in the rotated order (k + q) & 3,
    // so runs of up to 4 neighbouring lanes with the same bin hit distinct line-table
    // entries in each atomic instruction (same-address lanes serialise)
    const int q4 = lane & 3;
    float4 swr[XV];
    int Elr[4];
#pragma unroll
    for (int v = 0; v < XV; ++v) {
        const float4 w = swx[v];
        swr[v] = q4 == 0 ? w : q4 == 1 ? make_float4(w.y, w.z, w.w, w.x)
                             : q4 == 2 ? make_float4(w.z, w.w, w.x, w.y) : make_float4(w.w, w.x, w.y, w.z);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int src = (k + q4) & 3;
        Elr[k] = src == 0 ? El[0] : src == 1 ? El[1] : src == 2 ? El[2] : El[3];
    }
    const float cI = it.cI;
    const int nx = g.nx, nxy = g.nxy32, nxm2 = g.nxm2, nym2 = g.nym2, nzm2 = g.nzm2;
    const int dzo = g.dzo;
    const float *__restrict__ Mv = a.M;
    __syncthreads();

    int *LTw = LT + warp * S * LTSV;
    float *Kw = K + warp * S * KS;

    for (int y = it.y0 + warp; y < it.y0 + it.ylen; y += W) {
        const int cby = a.t.cb[1][y];
        const float4 cwy = a.t.cw[1][y];
        const float4 swy = a.t.sw[1][y];
        const float *__restrict__ Frow = a.F + y * nx;
        int gzl = a.t.cb[2][it.z0];
        float U[4][XV][3];
        if (!STATIC) {
#pragma unroll
            for (int n = 0; n < 4; ++n) ffd_layer<XV>(a.phi, g, gzl + n, cby, cwy, xn0, nxn, relx, cwx, lane, U[n]);
        }
        float bacc = 0.f;
        unsigned wmask[NW];
#pragma unroll
        for (int k = 0; k < NW; ++k) wmask[k] = 0u;
        // fold the column table with the row's y-weights into the cell table (MC: at z-region
        // offset lcz -- called at every crossed z-cell of a multi-cell item and at row end)
        // (MC only: a by-reference lambda in the coarse kernel costs it registers)
        auto foldK = [&](int lcz) {
          if constexpr (MC) {
#pragma unroll
            for (int k = 0; k < NW; ++k) {
                unsigned bw = k < nwords ? wmask[k] : 0u;
                wmask[k] = 0u;
                while (bw) {
                    const int s = 32 * k + __ffs(bw) - 1;
                    bw &= bw - 1;
#pragma unroll
                    for (int jj = lane; jj < KS; jj += 32) {
                        // lane -> (z-tap n, entry) with the 16 entries of one z-tap on
                        // consecutive lanes: the cell-table atomics hit 32 distinct banks
                        const int j = (jj & 15) * 4 + (jj >> 4);
                        const float val = Kw[s * KS + j];
                        Kw[s * KS + j] = 0.f;
                        if (val != 0.f) {
                            float *ct = CT + s * CTS + (lcz + (j & 3)) * E + (j >> 2);
#pragma unroll
                            for (int mm = 0; mm < 4; ++mm) atomicAdd(ct + mm * ZR * E, f4(swy, mm) * val);
                        }
                    }
                }
            }
          }
        };
        int lczr = 0;   // MC: z-cell offset of the column table's contents
        // F is software-pipelined one slice ahead (its DRAM latency is otherwise exposed:
        // the bin a0 it decides gates the whole line's accumulation)
        float Fnext[XV];
#pragma unroll
        for (int v = 0; v < XV; ++v) Fnext[v] = ld_stream(Frow + it.z0 * nxy + xv[v]);
        // The 8 M gathers of every voxel are software-pipelined one slice ahead too: issued
        // for slice z+1 right after slice z's sample arithmetic, so their latency overlaps
        // the line-table, fold and binless work of slice z.
        float C[XV][8], T[XV][3];
        int fl[XV];   // bits: clamp x,y,z (0-2), near-integer coordinate x,y,z (3-5)
        auto gather = [&](int zz) {
            const float4 cw = ZT[zz - it.z0];
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                const float ux = fmaf(cw.w, U[3][v][0], fmaf(cw.z, U[2][v][0], fmaf(cw.y, U[1][v][0], cw.x * U[0][v][0])));
                const float uy = fmaf(cw.w, U[3][v][1], fmaf(cw.z, U[2][v][1], fmaf(cw.y, U[1][v][1], cw.x * U[0][v][1])));
                const float uz = fmaf(cw.w, U[3][v][2], fmaf(cw.z, U[2][v][2], fmaf(cw.y, U[1][v][2], cw.x * U[0][v][2])));
                // rounding bound of u_c: |u32 - u64| <= gamma_16 max_taps |phi_c| ~ 9.5e-7
                // max |phi_c| (16 roundings on any path: fp32 phi and the 3 weights, 3 x 4
                // fma levels; weights >= 0 sum to 1); tolerance 2e-6, 2.1x that.  The max is
                // over this voxel's own 4x4x4 tap window (k_prep_tol).
                const float4 tl = __ldg(a.tolw + (gzl * g.Gy + cby) * g.Gx + relx[v] + xn0);
                bool clx, cly, clz, nrx, nry, nrz;
                const int ccx = axis_fast_fl(xv[v], ux, nxm2, tl.x, T[v][0], clx, nrx);
                const int ccy = axis_fast_fl(y, uy, nym2, tl.y, T[v][1], cly, nry);
                const int ccz = axis_fast_fl(zz, uz, nzm2, tl.z, T[v][2], clz, nrz);
                fl[v] = (int)clx | (int)cly << 1 | (int)clz << 2 | (int)nrx << 3 | (int)nry << 4 | (int)nrz << 5;
                const int o0 = ccz * nxy + ccy * nx + ccx, o1 = o0 + nx, o2 = o0 + dzo, o3 = o2 + nx;
                C[v][0] = __ldg(Mv + o0); C[v][1] = __ldg(Mv + o0 + 1);
                C[v][2] = __ldg(Mv + o1); C[v][3] = __ldg(Mv + o1 + 1);
                C[v][4] = __ldg(Mv + o2); C[v][5] = __ldg(Mv + o2 + 1);
                C[v][6] = __ldg(Mv + o3); C[v][7] = __ldg(Mv + o3 + 1);
            }
        };
        if (!STATIC) gather(it.z0);

        for (int z = it.z0; z < it.z0 + it.zlen; ++z) {
            if (MC) {   // crossed into the next z-cell: its z-taps are other regions
                const int lz = ZB[z - it.z0] >> 20;
                if (lz != lczr) {
                    __syncwarp();
                    foldK(lczr);
                    __syncwarp();
                    lczr = lz;
                }
            }
            float Fcur[XV];
            {
                const int nz1 = z + 1 < it.z0 + it.zlen ? nxy : 0;
#pragma unroll
                for (int v = 0; v < XV; ++v) {
                    Fcur[v] = Fnext[v];
                    Fnext[v] = ld_stream(Frow + z * nxy + nz1 + xv[v]);
                }
            }
            const float4 wz = ZT[64 + z - it.z0];
            float4 *MGrow = a.MG + ((long long)(z - a.mgz0) * g.ny + y) * nx;
            int a0[XV], slot[XV];
            float lo[XV], hi[XV], lo2[XV], hi2[XV];
            float qv[XV], abv[XV];   // MC: binless channels per voxel
            float bq[4] = {0.f, 0.f, 0.f, 0.f}, ba[4] = {0.f, 0.f, 0.f, 0.f};
            float amax = 0.f, amax2 = 0.f;
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                const float Fv = Fcur[v];
                a0[v] = min((int)Fv, g.L - 1);
                slot[v] = smap[a0[v]];
                float hlo, hhi;
                parzen_pair_F(Fv - (float)a0[v], hlo, hhi);
                if (STATIC) {
                    lo[v] = hlo;
                    hi[v] = hhi;
                } else {
                    const float tx = T[v][0], ty = T[v][1], tz = T[v][2];
                    const float c000 = C[v][0], c100 = C[v][1], c010 = C[v][2], c110 = C[v][3];
                    const float c001 = C[v][4], c101 = C[v][5], c011 = C[v][6], c111 = C[v][7];
                    const float e00 = lerpf(c000, c100, tx), e10 = lerpf(c010, c110, tx);
                    const float e01 = lerpf(c001, c101, tx), e11 = lerpf(c011, c111, tx);
                    const float f0 = lerpf(e00, e10, ty);
                    const float f1 = lerpf(e01, e11, ty);
                    const float m = lerpf(f0, f1, tz);
                    const int n = min(max((int)floorf(m), 0), g.L - 1);
                    float w1l, w1;
                    parzen_pair(m - (float)n, w1l, w1);
                    {   // (m, dM/dy) for pass 2 (Eq 16-17 chain); the fp64 path is needed where
                        // the per-voxel derivative jumps: a sample coordinate within rounding of
                        // an integer (cell / clamp boundary) or m within 5e-5 of an integer (the
                        // Parzen kink, reading c4) unless the cell is flat (m exact in fp32)
                        float dgx = lerpf(lerpf(c100 - c000, c110 - c010, ty), lerpf(c101 - c001, c111 - c011, ty), tz);
                        float dgy = lerpf(e10 - e00, e11 - e01, tz);
                        float dgz = f1 - f0;
                        dgx = (fl[v] & 1) ? 0.f : dgx;
                        dgy = (fl[v] & 2) ? 0.f : dgy;
                        dgz = ((fl[v] & 4) || dzo == 0) ? 0.f : dgz;
                        const float fm = m - (float)n;
                        bool ex = (fl[v] & 0x18) || ((fl[v] & 0x20) && dzo != 0);
                        if (!ex && (fm < 5e-5f || fm > 1.0f - 5e-5f))   // rare: the flatness test
                            ex = !(c100 == c000 && c010 == c000 && c110 == c000 && c001 == c000 &&
                                   c101 == c000 && c011 == c000 && c111 == c000);
                        if (a.MG && lane + 32 * v < it.xlen)
                            st_stream4(MGrow + xv[v], make_float4(ex ? -1.0f - m : m, dgx, dgy, dgz));
                    }
                    if (ORI == 0) {
                        const float A = ((float)n - shc[a0[v]]) + w1;      // g1 - c_a0
                        const float Ab = ((float)n - cI) + w1;            // g1 - cI
                        const float q = fmaf(Ab, Ab, w1 * w1l);           // sum_b (b - cI)^2 h(b - m)
                        lo[v] = hlo * A;
                        hi[v] = hhi * A;
                        amax = fmaxf(amax, fabsf(A));
                        if (MC) {
                            qv[v] = q;
                            abv[v] = Ab;
                        } else {
#pragma unroll
                            for (int l = 0; l < 4; ++l) {
                                bq[l] = fmaf(f4(swx[v], l), q, bq[l]);
                                ba[l] = fmaf(f4(swx[v], l), Ab, ba[l]);
                            }
                        }
                    } else {   // model bins from m; F gives the moment g1(F) = a0 + w1(F - a0)
                        slot[v] = 2 * smap[n];
                        lo[v] = w1l;                                      // N' halves
                        hi[v] = w1;
                        const float A = ((float)a0[v] + hhi) - shc[n];   // g1(F) - c_n
                        lo2[v] = w1l * A;                                 // S' halves
                        hi2[v] = w1 * A;
                        amax = fmaxf(amax, fmaxf(w1l, w1));
                        amax2 = fmaxf(amax2, fabsf(A));
                    }
                }
            }
            if (!STATIC && z + 1 < it.z0 + it.zlen) {   // next slice: slide the layer window, issue its gathers
                const int bz1 = MC ? ZB[z + 1 - it.z0] & 0xFFFFF : ZB[z + 1 - it.z0];
                while (gzl < bz1) {
#pragma unroll
                    for (int n = 0; n < 3; ++n)
#pragma unroll
                        for (int v = 0; v < XV; ++v) { U[n][v][0] = U[n + 1][v][0]; U[n][v][1] = U[n + 1][v][1]; U[n][v][2] = U[n + 1][v][2]; }
                    ++gzl;
                    ffd_layer<XV>(a.phi, g, gzl + 3, cby, cwy, xn0, nxn, relx, cwx, lane, U[3]);
                }
                gather(z + 1);
            }
            // ---- binless: warp-reduce (x-tap, channel) and fold the z-taps into bacc
            float iscQ = 1.f, iscB = 1.f;
            if (!STATIC && ORI == 0 && MC) {   // binless slot ns: entry 2 xr + {0: q', 1: g1 - cI}
                float mq = 0.f, mb = 0.f;
#pragma unroll
                for (int v = 0; v < XV; ++v) { mq = fmaxf(mq, qv[v]); mb = fmaxf(mb, fabsf(abv[v])); }
                const int EQ = (int)(__reduce_max_sync(FULL, __float_as_uint(mq)) >> 23);
                const int EB = (int)(__reduce_max_sync(FULL, __float_as_uint(mb)) >> 23);
                const float scQ = exp2i(min(274 - El[0] - EQ, 120)), scB = exp2i(min(274 - El[0] - EB, 120));
                iscQ = exp2i(-min(274 - El[0] - EQ, 120));
                iscB = exp2i(-min(274 - El[0] - EB, 120));
                const int chA = (lane >> 2) & 1;
#pragma unroll
                for (int v = 0; v < XV; ++v) {
                    int *row = LTw + ns * LTSV + 2 * lcx[v] + chA;
                    const float va = chA ? abv[v] * scB : qv[v] * scQ, vb = chA ? qv[v] * scQ : abv[v] * scB;
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const int lr = (l + q4) & 3;
                        const float w = f4(swr[v], l);
                        atomicAdd(row + 2 * lr, __float_as_int(fmaf(va, w, 12582912.f)) - 0x4B400000);
                        atomicAdd(row + 2 * lr + 1 - 2 * chA, __float_as_int(fmaf(vb, w, 12582912.f)) - 0x4B400000);
                    }
                }
            }
            if (!STATIC && ORI == 0 && !MC) {
                const float bv[8] = {bq[0], ba[0], bq[1], ba[1], bq[2], ba[2], bq[3], ba[3]};
                const float tot = halving8(bv, lane);          // value (lane>>2) = 2*l + ch
                bacc = fmaf(f4(wz, lane & 3), tot, bacc);
            }
            // ---- binned: line table (ORI 1: two slot groups per voxel, each with its own scale)
            float isc_g[2] = {1.f, 1.f};
            bool uniform = true;
#pragma unroll
            for (int gi = 0; gi < (ORI ? 2 : 1); ++gi) {
            if (gi == 1) {
#pragma unroll
                for (int v = 0; v < XV; ++v) { slot[v] += 1; lo[v] = lo2[v]; hi[v] = hi2[v]; }
                amax = amax2;
            }
            float sc[4] = {1.f, 1.f, 1.f, 1.f}, isc_e = 1.f;
            int EA = 0;
            if (!STATIC) {
                EA = (int)(__reduce_max_sync(FULL, __float_as_uint(amax)) >> 23);
#pragma unroll
                for (int l = 0; l < 4; ++l) sc[l] = exp2i(min(274 - El[l] - EA, 120));
                isc_e = exp2i(-min(274 - El_e - EA, 120));
            }
            isc_g[gi] = isc_e;
            int amx = ORI ? slot[0] : a0[0];
#pragma unroll
            for (int v = 1; v < XV; ++v) amx = max(amx, ORI ? slot[v] : a0[v]);
            const int af = (int)__reduce_max_sync(FULL, (unsigned)amx);
            bool same = true;
#pragma unroll
            for (int v = 0; v < XV; ++v) same = same && (ORI ? slot[v] : a0[v]) == af;
            uniform = !MC && __all_sync(FULL, same);
            if (uniform) {
                float vv[8];
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    float sl = 0.f, sh = 0.f;
#pragma unroll
                    for (int v = 0; v < XV; ++v) {
                        sl = fmaf(f4(swx[v], l), lo[v], sl);
                        sh = fmaf(f4(swx[v], l), hi[v], sh);
                    }
                    vv[2 * l] = sl;
                    vv[2 * l + 1] = sh;
                }
                const float tot = halving8(vv, lane);
                if ((lane & 3) == 0) {   // one bin: straight into the column table (no line table, no fold)
                    const int ent = lane >> 2;
                    float4 *kp = reinterpret_cast<float4 *>(Kw + slot[0] * KS + ent * 4);
                    float4 k4 = *kp;
                    k4.x = fmaf(wz.x, tot, k4.x);
                    k4.y = fmaf(wz.y, tot, k4.y);
                    k4.z = fmaf(wz.z, tot, k4.z);
                    k4.w = fmaf(wz.w, tot, k4.w);
                    *kp = k4;
                }
            } else if (STATIC) {
#pragma unroll
                for (int v = 0; v < XV; ++v) {
                    float *row = reinterpret_cast<float *>(LTw + slot[v] * LTSV + 2 * lcx[v]);
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const int lr = (l + q4) & 3;
                        atomicAdd(row + 2 * lr, f4(swr[v], l) * lo[v]);
                        atomicAdd(row + 2 * lr + 1, f4(swr[v], l) * hi[v]);
                    }
                }
            } else {
                float scr[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) scr[k] = exp2i(min(274 - Elr[k] - EA, 120));
                // lanes 4-7 (mod 8) also swap the channel order: 8 neighbouring lanes of one
                // bin touch 8 distinct entries per instruction
                const int chA = (lane >> 2) & 1;
#pragma unroll
                for (int v = 0; v < XV; ++v) {
                    int *row = LTw + slot[v] * LTSV + 2 * lcx[v] + chA;
                    const float va = chA ? hi[v] : lo[v], vb = chA ? lo[v] : hi[v];
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const int lr = (l + q4) & 3;
                        const float ws = f4(swr[v], l) * scr[l];
                        atomicAdd(row + 2 * lr, __float_as_int(fmaf(va, ws, 12582912.f)) - 0x4B400000);
                        atomicAdd(row + 2 * lr + 1 - 2 * chA, __float_as_int(fmaf(vb, ws, 12582912.f)) - 0x4B400000);
                    }
                }
            }
            if (ORI && gi == 1) {   // both groups' slots are marked (uniform lines) / folded below
#pragma unroll
                for (int v = 0; v < XV; ++v) slot[v] -= 1;
            }
            if (uniform && ORI) {
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    if (((slot[0] + gi) >> 5) == k) wmask[k] |= 1u << ((slot[0] + gi) & 31);
            }
            }
            // ---- fold the line into the warp's column table, 4 slots per instruction:
            //      K[slot][ent][n] += wz_n * LT[slot][ent]
            unsigned bits[NW];
#pragma unroll
            for (int k = 0; k < NW; ++k) bits[k] = 0u;
            int cnt = 0;
            if (MC && !STATIC) {   // the binless slot is touched by every line
                bits[ns >> 5] |= 1u << (ns & 31);
                wmask[ns >> 5] |= 1u << (ns & 31);
                cnt = 1;
            }
            if (uniform && !ORI) {
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    if ((slot[0] >> 5) == k) wmask[k] |= 1u << (slot[0] & 31);
            }
#pragma unroll
            for (int k = 0; k < NW; ++k) {
                if (k < nwords && !uniform) {
                    unsigned mine = 0u;
#pragma unroll
                    for (int v = 0; v < XV; ++v) {
                        mine |= ((slot[v] >> 5) == k) ? 1u << (slot[v] & 31) : 0u;
                        if (ORI) mine |= (((slot[v] + 1) >> 5) == k) ? 1u << ((slot[v] + 1) & 31) : 0u;
                    }
                    bits[k] |= __reduce_or_sync(FULL, mine);
                    wmask[k] |= bits[k];
                }
            }
            if (!uniform) {
                cnt = 0;
#pragma unroll
                for (int k = 0; k < NW; ++k) cnt += __popc(bits[k]);
            }
            const int nwf = MC ? max(nwords, (ns >> 5) + 1) : nwords;
            __syncwarp();
            const int ent = lane & (E - 1);
            for (int c0 = 0; c0 < cnt; c0 += 32) {
                const int myslot = mask_select(bits, nwf, c0 + lane);
                const int rmax = min(cnt - c0, 32);
                for (int r = 0; r < rmax; r += 32 / E) {
                    const int idx = r + lane / E;
                    const int s = __shfl_sync(FULL, myslot, idx & 31);
                    if (idx < rmax) {
                        int *lp = LTw + s * LTSV + ent;
                        const int iv = *lp;
                        *lp = 0;
                        float isc = isc_g[ORI ? (s & 1) : 0];
                        if (MC && s == ns) isc = (ent & 1) ? iscB : iscQ;
                        const float val = STATIC ? __int_as_float(iv) : (float)iv * isc;
                        float4 *kp = reinterpret_cast<float4 *>(Kw + s * KS + ent * 4);
                        float4 k4 = *kp;
                        k4.x = fmaf(wz.x, val, k4.x);
                        k4.y = fmaf(wz.y, val, k4.y);
                        k4.z = fmaf(wz.z, val, k4.z);
                        k4.w = fmaf(wz.w, val, k4.w);
                        *kp = k4;
                    }
                }
            }
            __syncwarp();
        }
        // ---- row done: fold the column table with the row's y-weights into the cell table
        if constexpr (MC) {
            __syncwarp();
            foldK(lczr);
        } else {
#pragma unroll
            for (int k = 0; k < NW; ++k) {
                unsigned bw = k < nwords ? wmask[k] : 0u;
                while (bw) {
                    const int s = 32 * k + __ffs(bw) - 1;
                    bw &= bw - 1;
#pragma unroll
                    for (int j = lane; j < KS; j += 32) {
                        const float val = Kw[s * KS + j];
                        Kw[s * KS + j] = 0.f;
                        if (val != 0.f) {
#pragma unroll
                            for (int mm = 0; mm < 4; ++mm) atomicAdd(CT + (s * 4 + mm) * KS + j, f4(swy, mm) * val);
                        }
                    }
                }
            }
        }
        if (!STATIC && !MC && bacc != 0.f) {
#pragma unroll
            for (int mm = 0; mm < 4; ++mm) atomicAdd(CB + mm * 32 + lane, f4(swy, mm) * bacc);
        }
        __syncwarp();
    }
    __syncthreads();
    // ---- item done: flush to global.  CT entry (s, m, e): e = 8*l + 4*ch + n
    for (int t = threadIdx.x; t < nsl * CTS; t += blockDim.x) {
        const float val = CT[t];
        const int s = t / CTS;
        int mm, l, ch, n;
        if (MC) {   // [s][m][zr][E], entry = 2 xr + ch
            const int rem = t - s * CTS;
            mm = rem / (ZR * E);
            n = (rem / E) % ZR;
            l = (rem % E) >> 1;
            ch = rem & 1;
        } else {    // [s][m][8 l + 4 ch + n]
            const int e = t % KS;
            mm = (t / KS) & 3;
            l = e >> 3;
            ch = (e >> 2) & 1;
            n = e & 3;
        }
        const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        if (MC && !STATIC && s == ns) {   // binless: Q_r += Q' + 2 cI S' + cI^2 N
            if (ch == 0) {
                const ItemW &iw = a.itemw[blockIdx.x];
                const double N = iw.sx[l] * iw.sy[mm] * iw.sz[n];
                if (N > 0.0) {
                    const double c = cI;
                    atomicAdd(a.Qt + r, (double)val + 2.0 * c * (double)CT[t + 1] + c * c * N);
                }
            }
            continue;
        }
        if (val == 0.f) continue;
        if (ORI)   // slot 2k: counts N' -> NQ, slot 2k+1: first moments S' -> SQ
            atomicAdd(((s & 1) ? a.SQ : a.NQ) + (r * B + a.slotbins[it.slot_off + (s >> 1)]) * 2 + ch, (double)val);
        else
            atomicAdd(a.SQ + (r * B + a.slotbins[it.slot_off + s]) * 2 + ch, (double)val);
    }
    if (!STATIC && ORI == 0 && !MC && threadIdx.x < 64) {
        // binless: Q_r += Q' + 2 cI S' + cI^2 N  with N = sum of the item's spatial weights
        const int l = threadIdx.x >> 4, mm = (threadIdx.x >> 2) & 3, n = threadIdx.x & 3;
        const double Qp = CB[mm * 32 + (2 * l) * 4 + n], Sp = CB[mm * 32 + (2 * l + 1) * 4 + n];
        const ItemW &iw = a.itemw[blockIdx.x];
        const double N = iw.sx[l] * iw.sy[mm] * iw.sz[n];
        if (N > 0.0) {
            const double c = cI;
            const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
            atomicAdd(a.Qt + r, Qp + 2.0 * c * Sp + c * c * N);
        }
    }
}

// ---------------------------------------------------------------- combine
// One warp per region r (Eq 9-12 P:111-127 in moment form):
//   N_ra = Nlo[r][a] + Nup[r][a-1];  S_ra unshifted from the binned pass-1 moments;
//   mu_ra = S_ra/N_ra, mu_r = S_r/N_r;  T_r = Q_r - S_r^2/N_r (binless Q_r);
//   V_r = T_r - sum_{a:N_ra>0} N_ra (mu_ra - mu_r)^2  (= Q_r - sum_a S_ra^2/N_ra);
//   retained iff N_r/Z > eps_mass and sigma_r^2 = T_r/N_r > eps_sigma (reading c12);
//   dterm[r] = N_r V_r / T_r (so D = sum dterm / Z), and the coefficients
//   alpha_r = CR_r/sigma_r^2, beta_r = (1-CR_r) mu_r/sigma_r^2, gamma_ra = mu_r(a)/sigma_r^2.
struct CombineArgs {
    const double *SQ;           // [R][B][2]
    const double *Qt;           // [R]
    const double *Nlo, *Nup;    // [R][B]
    const float *shiftc;        // [B]
    int R, B;
    double Z, eps_mass, eps_sigma;
    double *dterm;              // [R]
    double *reg;                // [R][6] {p(r), sigma2, mu, 1-CR, retained, Z}
    double *S_out;              // [R][B] unshifted (debug / parity), may be null
    float *alpha, *beta, *gamma;
    const double *NQ;           // ORI 1: [R][B][2] dynamic counts N' (lo, hi halves)
    int gstride;                // ORI 1: row stride of gamma = 3 (B + 2)
    unsigned *ticket;           // last-CTA ticket (0 between launches)
    double *part;               // [3 * gridDim] per-CTA partial sums of dterm, retained; max q_r
    double *Dout;               // [2] D, #retained regions
    double *gbound;             // [1] bound on |dD/dm * dM/dy_c| * Z per voxel (fast pass 2's fixed point)
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// D = (1/Z) sum_r dterm[r], deterministic: each CTA sums its regions' dterm and retained
// flags in warp order into part[2*blockIdx]; the last CTA (atomic ticket) sums the
// partials in block order into Dout = {D, #retained} and re-arms the ticket.
// The third value is a max: q_r = (2L+1)|alpha_r| + 2|beta_r| + 2 max_a |gamma_ra| over the
// regions, giving gbound = 1.9 L max_r q_r >= |Z dD/dm dM/dy_c| per voxel (|g1'| <= 1.9, the
// spatial weights sum to 1, |dM/dy_c| <= L): the scale of fast pass 2's fixed point.
__device__ __forceinline__ void combine_tail(const CombineArgs &a, double dt, double rt, double mq = 0.0) {
    __shared__ bool last;
    __shared__ double sd[256], sc[256], sq[256];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) { sd[warp] = dt; sc[warp] = rt; sq[warp] = mq; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0, c = 0, q = 0;
        for (int w = 0; w < nw; ++w) { s += sd[w]; c += sc[w]; q = fmax(q, sq[w]); }
        a.part[3 * blockIdx.x] = s;
        a.part[3 * blockIdx.x + 1] = c;
        a.part[3 * blockIdx.x + 2] = q;
        __threadfence();
        last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0, c = 0, q = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        s += __ldcg(a.part + 3 * i);
        c += __ldcg(a.part + 3 * i + 1);
        q = fmax(q, __ldcg(a.part + 3 * i + 2));
    }
    sd[threadIdx.x] = s;
    sc[threadIdx.x] = c;
    sq[threadIdx.x] = q;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sd[threadIdx.x] += sd[threadIdx.x + o];
            sc[threadIdx.x] += sc[threadIdx.x + o];
            sq[threadIdx.x] = fmax(sq[threadIdx.x], sq[threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.Dout[0] = sd[0] / a.Z;
        a.Dout[1] = sc[0];
        if (a.gbound) a.gbound[0] = 1.9 * (double)(a.B - 1) * sq[0];
        *a.ticket = 0u;
    }
}

__device__ __forceinline__ void bin_NS(const CombineArgs &a, int r, int b, double &N, double &S) {
    const int B = a.B;
    const double *q = a.SQ + ((long long)r * B + b) * 2;
    const double nlo = a.Nlo[(long long)r * B + b];
    N = nlo;
    S = q[0] + (double)a.shiftc[b] * nlo;
    if (b > 0) {
        const double nup = a.Nup[(long long)r * B + b - 1];
        N += nup;
        S += (q - 2)[1] + (double)a.shiftc[b - 1] * nup;
    }
}

// returns (in dt, rt; lane 0 of the region's warp) the region's dterm and retained flag, and
// (every lane) the region's q_r of combine_tail
__device__ __forceinline__ void combine_region(const CombineArgs &a, int r, double &dt, double &rt, double &mq) {
    const int lane = threadIdx.x & 31;
    dt = rt = 0.0;
    mq = 0.0;
    if (r >= a.R) return;
    const int B = a.B;
    double Nv[4], Sv[4];    // this lane's bins b = lane + 32 k (B <= 128)
    double Nr = 0, Sr = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int b = lane + 32 * k;
        Nv[k] = Sv[k] = 0.0;
        if (b < B) {
            bin_NS(a, r, b, Nv[k], Sv[k]);
            if (a.S_out) a.S_out[(long long)r * B + b] = Sv[k];
        }
        Nr += Nv[k];
        Sr += Sv[k];
    }
    Nr = warp_sum_d(Nr);
    Sr = warp_sum_d(Sr);
    const double mu = Nr > 0 ? Sr / Nr : 0.0;
    double btw = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (Nv[k] > 0.0) {
            const double d = Sv[k] / Nv[k] - mu;
            btw += Nv[k] * d * d;
        }
    btw = warp_sum_d(btw);
    const double pr = Nr / a.Z;
    double sig2 = 0, omcr = 0;
    bool ret = false;
    if (pr > a.eps_mass) {
        const double Tr = a.Qt[r] - Sr * Sr / Nr, Vr = Tr - btw;
        sig2 = Tr / Nr;
        if (sig2 > a.eps_sigma) { ret = true; omcr = Vr / Tr; }
    }
    if (lane == 0) {
        dt = ret ? Nr * omcr : 0.0;
        rt = ret ? 1.0 : 0.0;
        a.dterm[r] = dt;
        a.alpha[r] = ret ? (float)((1.0 - omcr) / sig2) : 0.f;
        a.beta[r] = ret ? (float)(omcr * mu / sig2) : 0.f;
        double *rg = a.reg + (long long)r * 6;
        rg[0] = pr; rg[1] = sig2; rg[2] = mu; rg[3] = omcr; rg[4] = rt; rg[5] = a.Z;
    }
    const double is2 = ret ? 1.0 / sig2 : 0.0;
    float gmax = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int b = lane + 32 * k;
        const float gv = (ret && Nv[k] > 0.0) ? (float)((Sv[k] / Nv[k]) * is2) : 0.f;
        if (b < B) a.gamma[(long long)r * B + b] = gv;
        gmax = fmaxf(gmax, b < B ? fabsf(gv) : 0.f);
    }
    gmax = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(gmax)));
    if (ret) mq = (2.0 * (B - 1) + 1.0) * fabs((1.0 - omcr) / sig2) + 2.0 * fabs(omcr * mu / sig2) + 2.0 * (double)gmax;
}


// ORI 1 (moving image as the model image A; Eq 20-21, App. II in moment form, reading
// c23), one warp per region: the estimated image is F, so N_r, S_r = sum_a a N^F_ra and
// Q_r = sum_a a^2 N^F_ra are static (from the fixed-bin counts, exact: g1(F), g2(F) are
// the Parzen moments); the model bins are m's:
//   N'_ra = NQ[r][a][0] + NQ[r][a-1][1],  S'_ra unshifted likewise (shift c_a, c_{a-1});
//   V_r = Q_r - sum_{a: N'_ra > 0} S'_ra^2 / N'_ra,  T_r = Q_r - S_r^2/N_r.
// Pass 2's table, per region and bin a = -1..L+1 (column 3(a+1) + {0,1,2}), written so
// that the fp32 derivative has no cancellation: psi_ra(g) = (mu_ra - g)^2/sigma_r^2 - g^2/
// sigma_r^2 for a populated bin and -g^2/sigma_r^2 for an empty or virtual one (c23); the
// -g^2 terms cancel exactly in dD/dm (the two bins' dh/dm are opposite), so only
//   psi'_ra(g) = [populated] (delta^2 + 2 delta (c_a - g) + (c_a - g)^2) / sigma_r^2,
//   delta = mu_ra - c_a (c_a: the bin's moment shift, near the conditional mean)
// is needed: columns {1/sigma^2, delta/sigma^2, delta^2/sigma^2} for a populated bin of a
// retained region, zeros otherwise.
__device__ __forceinline__ void bin_NS_A(const CombineArgs &a, int r, int b, double &N, double &S) {
    const int B = a.B;
    const double *n = a.NQ + ((long long)r * B + b) * 2;
    const double *q = a.SQ + ((long long)r * B + b) * 2;
    N = n[0];
    S = q[0] + (double)a.shiftc[b] * n[0];
    if (b > 0) {
        N += (n - 2)[1];
        S += (q - 2)[1] + (double)a.shiftc[b - 1] * (n - 2)[1];
    }
}

__device__ __forceinline__ void combineA_region(const CombineArgs &a, int r, double &dt, double &rt) {
    const int lane = threadIdx.x & 31;
    dt = rt = 0.0;
    if (r >= a.R) return;
    const int B = a.B;
    double Nr = 0, Sr = 0, Qr = 0, s2n = 0;
    for (int b = lane; b < B; b += 32) {
        const double nf = a.Nlo[(long long)r * B + b] + (b > 0 ? a.Nup[(long long)r * B + b - 1] : 0.0);
        Nr += nf;
        Sr += (double)b * nf;
        Qr += (double)b * (double)b * nf;
        double N, S;
        bin_NS_A(a, r, b, N, S);
        if (a.S_out) a.S_out[(long long)r * B + b] = S;
        if (N > 0.0) s2n += S * S / N;
    }
    Nr = warp_sum_d(Nr);
    Sr = warp_sum_d(Sr);
    Qr = warp_sum_d(Qr);
    s2n = warp_sum_d(s2n);
    const double pr = Nr / a.Z;
    double sig2 = 0, omcr = 0;
    bool ret = false;
    if (pr > a.eps_mass) {
        const double Tr = Qr - Sr * Sr / Nr, Vr = Qr - s2n;
        sig2 = Tr / Nr;
        if (sig2 > a.eps_sigma) { ret = true; omcr = Vr / Tr; }
    }
    if (lane == 0) {
        dt = ret ? Nr * omcr : 0.0;
        rt = ret ? 1.0 : 0.0;
        a.dterm[r] = dt;
        a.alpha[r] = 0.f;
        a.beta[r] = 0.f;
        double *rg = a.reg + (long long)r * 6;
        rg[0] = pr; rg[1] = sig2; rg[2] = Nr > 0 ? Sr / Nr : 0.0; rg[3] = omcr; rg[4] = ret ? 1.0 : 0.0; rg[5] = a.Z;
    }
    float *row = a.gamma + (long long)r * a.gstride;
    for (int j = lane; j < B + 2; j += 32) {   // bin a = j - 1
        const int b = j - 1;
        float T0 = 0.f, T1 = 0.f, T2 = 0.f;
        if (ret && b >= 0 && b < B) {
            double N = 0.0, S = 0.0;
            bin_NS_A(a, r, b, N, S);
            if (N > 0.0) {
                const double dl = S / N - (double)a.shiftc[b];
                T0 = (float)(1.0 / sig2);
                T1 = (float)(dl / sig2);
                T2 = (float)(dl * dl / sig2);
            }
        }
        row[3 * j] = T0;
        row[3 * j + 1] = T1;
        row[3 * j + 2] = T2;
    }
}

// a fixed grid: warp w of CTA b takes regions b*8 + w, then + 8*gridDim (fine lattices have
// 10^5-10^6 regions; one CTA per 8 regions made the last-CTA ticket a serial hot spot)
__global__ void __launch_bounds__(256) k_combine(CombineArgs a) {
    double dt = 0, rt = 0, mq = 0;
    for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < a.R; r += gridDim.x * 8) {
        double d1, r1, q1;
        combine_region(a, r, d1, r1, q1);
        dt += d1;
        rt += r1;
        mq = fmax(mq, q1);
    }
    combine_tail(a, dt, rt, mq);
}
__global__ void __launch_bounds__(256) k_combineA(CombineArgs a) {
    double dt = 0, rt = 0;
    for (int r = blockIdx.x * 8 + (threadIdx.x >> 5); r < a.R; r += gridDim.x * 8) {
        double d1, r1;
        combineA_region(a, r, d1, r1);
        dt += d1;
        rt += r1;
    }
    combine_tail(a, dt, rt);
}


// ----------------------------------------------- pass 2: exact-sample path (fp64)
__device__ __forceinline__ double d4(const double4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// fp64 sample coordinate along one axis, exactly as the definition (c2, c3)
__device__ __forceinline__ void axis64(int i, double u, int N, long long &c0, double &t, bool &cl) {
    double yv = (double)i + u;
    const double N1 = (double)(N - 1);
    cl = (yv < 0.0 || yv > N1);
    yv = yv < 0.0 ? 0.0 : (yv > N1 ? N1 : yv);
    if (N == 1) { c0 = 0; t = 0.0; return; }
    long long fl = (long long)floor(yv);
    if (fl > N - 2) fl = N - 2;
    c0 = fl;
    t = yv - (double)fl;
}

struct ExactGeo { int nx, ny, nz, L, Gx, Gy, GzExt, ndim; };

// Taken by the rare lanes whose fp32 sample position lies within 1e-4 voxel of an
// integer (a trilinear cell or clamp boundary) or whose warped intensity lies within
// 1e-4 of an integer (the Parzen kink of c4): there the per-voxel derivative is
// discontinuous and the side must be decided as the fp64 definition decides it.
// (returned by value: reference outputs would force the caller's locals into local memory)
// Called by a group of 16 lanes (half a warp, mask gm) for one voxel: the lanes stage the
// 64 x ndim control values in the group's shared buffer sp[3][64] (independent loads in
// flight together), then every lane sums them in the definition's order (identical result
// in every lane).
struct ExactOut { float gx, gy, gz, g1p, c2; };
__device__ __forceinline__ ExactOut exact_sample(ExactGeo g, const double *__restrict__ p64, const float *__restrict__ M,
                                                 const double4 *__restrict__ cwx64, const double4 *__restrict__ cwy64,
                                                 const double4 *__restrict__ cwz64, int bx, int by, int bz, int x,
                                                 int y, int z, double *sp, int gl, unsigned gm) {
    const double4 wx = cwx64[x], wy = cwy64[y], wz = cwz64[z];
    ExactOut o;
    const long long plane = (long long)g.Gx * g.Gy, cs = plane * g.GzExt;
    const long long nxy = (long long)g.nx * g.ny;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int tp = gl + 16 * h, n = tp >> 4, mm = (tp >> 2) & 3, l = tp & 3;
        const long long s = (long long)(bz + n) * plane + (long long)(by + mm) * g.Gx + bx + l;
        const bool in = bz + n < g.GzExt;
#pragma unroll
        for (int c = 0; c < 3; ++c) sp[c * 64 + tp] = (in && c < g.ndim) ? p64[c * cs + s] : 0.0;
    }
    __syncwarp(gm);
    double u[3] = {0.0, 0.0, 0.0};
    for (int n = 0; n < 4; ++n) {
        const double wn = d4(wz, n);
        if (wn == 0.0 || bz + n >= g.GzExt) continue;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm) {
            const double wm = d4(wy, mm);
            if (wm == 0.0) continue;
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const double wl = d4(wx, l);
                if (wl == 0.0) continue;
                const double w = wl * wm * wn;
                const int tp = n * 16 + mm * 4 + l;
                u[0] += w * sp[tp];
                u[1] += w * sp[64 + tp];
                if (g.ndim == 3) u[2] += w * sp[128 + tp];
            }
        }
    }
    long long cx, cy, cz;
    double tx, ty, tz;
    bool clx, cly, clz;
    axis64(x, u[0], g.nx, cx, tx, clx);
    axis64(y, u[1], g.ny, cy, ty, cly);
    axis64(z, u[2], g.nz, cz, tz, clz);
    const long long dzo = g.nz > 1 ? nxy : 0;
    const float *b = M + cz * nxy + cy * g.nx + cx;
    const double c000 = b[0], c100 = b[1], c010 = b[g.nx], c110 = b[g.nx + 1];
    const double c001 = b[dzo], c101 = b[dzo + 1], c011 = b[dzo + g.nx], c111 = b[dzo + g.nx + 1];
    const double e00 = c000 + tx * (c100 - c000), e10 = c010 + tx * (c110 - c010);
    const double e01 = c001 + tx * (c101 - c001), e11 = c011 + tx * (c111 - c011);
    const double f0 = e00 + ty * (e10 - e00), f1 = e01 + ty * (e11 - e01);
    const double m = f0 + tz * (f1 - f0);
    const double gx = (1 - ty) * (1 - tz) * (c100 - c000) + ty * (1 - tz) * (c110 - c010) +
                      (1 - ty) * tz * (c101 - c001) + ty * tz * (c111 - c011);
    const double gy = (1 - tx) * (1 - tz) * (c010 - c000) + tx * (1 - tz) * (c110 - c100) +
                      (1 - tx) * tz * (c011 - c001) + tx * tz * (c111 - c101);
    const double gz = (1 - tx) * (1 - ty) * (c001 - c000) + tx * (1 - ty) * (c101 - c100) +
                      (1 - tx) * ty * (c011 - c010) + tx * ty * (c111 - c110);
    o.gx = clx ? 0.f : (float)gx;
    o.gy = cly ? 0.f : (float)gy;
    o.gz = (clz || g.nz == 1) ? 0.f : (float)gz;
    int n = (int)floor(m);
    n = n > g.L - 1 ? g.L - 1 : (n < 0 ? 0 : n);
    const double f = m - (double)n;
    if (m == floor(m)) { o.g1p = 0.1f; o.c2 = (float)(2.0 * m); }
    else { o.g1p = (float)(f < 0.5 ? 0.1 + 3.6 * f : 3.7 - 3.6 * f); o.c2 = (float)(2.0 * n + 1.0); }
    return o;
}

__device__ __forceinline__ bool near_integer(float v, float tol) { return fabsf(v - rintf(v)) < tol; }

// ---------------------------------------------------------------- pass 2
// Per voxel (equal to Eq 27 P:475 after the b-sum):
//   dD/dm = (g1'/Z) [c2 A~ - 2 G~ + 2 B~],  A~ = sum_r w_r alpha_r,  B~ = sum_r w_r beta_r,
//   G~ = sum_r w_r (h_lo gamma_{r,a0} + h_hi gamma_{r,a0+1});  g1' = w1'(f), c2 = 2n+1,
//   and at integer m: g1' = 0.1, c2 = 2m (reading c4).
// Then d_c = dD/dm * dM/dy_c and the adjoint of the FFD (Eq 16-17):
//   dD/dphi_{s,c} += d_c * cwx_l cwy_m cwz_n, accumulated along the z-march in registers
//   (4 active control layers), x-contracted across lanes when a layer retires (segmented
//   shuffle), y-contracted into a CTA node window in shared memory, flushed with fp64
//   atomics at the end of the item.
// The warp's row is fixed during its z-march: gamma, alpha, beta are contracted over the
// y-taps once per row (GY[bin][xtap] = float4 over the z-taps); per line the bins the
// line touches are contracted over z cooperatively (GZ[bin] = float4 over the x-taps),
// so a voxel reads two float4.
// ORI = 1 (moving image as the model image A): dD/dm = (1/Z) sum_r w_r sum_a (dh_a/dm)
// psi'_ra(g1(F)) (k_combineA's table, 3 columns per bin, bins -1..L+1): bins n, n+1 with
// -/+ w1'(f), or at integer m = k bins k-1, k+1 with -/+ 0.05 (reading c4); no alpha /
// beta terms.
// MC (multi-cell items, ORI 0): the region tables are indexed (n, m, xr) with XRN
// relative x-regions; per line the item's bins are contracted over z per x-region
// (GZs[bin][xr]) and each voxel sums its own 4 x-regions lcx..lcx+3.
template <int XV, int MAXT = 512, int ORI = 0, bool MC = false>
__global__ void __launch_bounds__(MAXT, MAXT <= 256 ? (MC ? 3 : 5) : 1) k_pass2(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int XRN = MC ? MC_XRN : 4;
    const int ZRN = MC ? a.zrn : 4;           // z-regions per item
    constexpr int GYSV = MC ? MC_XRN + 1 : GYS;
    const Geo &g = a.g;
    const int B = g.B, W = a.W;
    const Item it = a.items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const int xn0 = a.t.cb[0][it.x0];
    const int nxn = a.t.cb[0][it.x0 + it.xlen - 1] + 4 - xn0;
    const int yn0 = a.t.cb[1][it.y0];
    const int nyn = a.t.cb[1][it.y0 + it.ylen - 1] + 4 - yn0;
    const int zn0 = a.t.cb[2][it.z0];
    const int nzn = a.t.cb[2][it.z0 + it.zlen - 1] + 4 - zn0;

    // gamma tables are indexed by the item's bin list (a0 and a0+1 of every slot,
    // sorted, so bin a0+1 always sits right after a0): capacity GB = a.S2
    const int GB = a.S2;
    float4 *GY = reinterpret_cast<float4 *>(smem);                // [W][GB][GYSV]
    float4 *GZ = GY + W * GB * GYSV;                              // [W][GB] (MC: [W][GB][XRN] floats)
    float *gl = reinterpret_cast<float *>(GZ + W * GB * (XRN / 4)); // [4 ZRN XRN][GB] gamma of the regions
    int *gbins = reinterpret_cast<int *>(gl + 4 * ZRN * XRN * GB); // [GB+1] the bin list, count
    unsigned short *gmap = reinterpret_cast<unsigned short *>(gbins + GB + 1);  // [B] bin -> list index
    float *al = reinterpret_cast<float *>(gmap + (((ORI ? 3 * (B + 2) : B) + 7) & ~7)); // [4 ZRN XRN]
    float *bl = al + 4 * ZRN * XRN;                               // [4 ZRN XRN]
    float *shc2 = bl + 4 * ZRN * XRN;                             // [B] (ORI 1) the bins' moment shifts
    float *RB = shc2 + (ORI ? B : 0);                             // [W][3][64] retiring-layer row buffer
    float *NP = RB + W * 192;                                     // [nzn][3][nyn][nxn] node window

    const int cx = a.t.sb[0][it.x0], cy = a.t.sb[1][it.y0], cz = a.t.sb[2][it.z0];
    // bin list of the item (host-built): every a0 present and a0+1, sorted, no duplicates
    const int nb2 = it.nslots;
    for (int i = threadIdx.x; i < nb2; i += blockDim.x) {
        const int b = a.slotbins[it.slot_off + i];
        gbins[i] = b;
        gmap[b] = (unsigned short)i;
    }
    __syncthreads();
    // region (n, m, l) of the item (l, n: relative x-, z-regions) at index (n * 4 + m) * XRN + l
    for (int i = threadIdx.x; i < 4 * ZRN * XRN * nb2; i += blockDim.x) {
        const int reg = i / nb2, k = i - reg * nb2;
        const int l = reg % XRN, mm = (reg / XRN) & 3, n = reg / (4 * XRN);
        const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        gl[reg * GB + k] = cx + l < g.Kx && cz + n < g.Kz ? __ldg(a.gamma + r * a.gstride + gbins[k]) : 0.f;
    }
    for (int i = threadIdx.x; i < 4 * ZRN * XRN; i += blockDim.x) {
        const int l = i % XRN, mm = (i / XRN) & 3, n = i / (4 * XRN);
        const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        const bool in = cx + l < g.Kx && cz + n < g.Kz;
        al[i] = in ? __ldg(a.alpha + r) : 0.f;
        bl[i] = in ? __ldg(a.beta + r) : 0.f;
    }
    if (ORI)
        for (int i = threadIdx.x; i < B; i += blockDim.x) shc2[i] = a.shiftc[i];
    const int npsz = nzn * 3 * nyn * nxn;
    for (int i = threadIdx.x; i < npsz; i += blockDim.x) NP[i] = 0.f;
    for (int i = threadIdx.x; i < W * 192; i += blockDim.x) RB[i] = 0.f;

    bool lok[XV];
    int xv[XV], relx[XV], cbx[XV], lcx[XV];
    float4 swx[XV], cwr[XV];
    const int q4 = lane & 3;
#pragma unroll
    for (int v = 0; v < XV; ++v) {
        lok[v] = lane + 32 * v < it.xlen;
        xv[v] = lok[v] ? it.x0 + lane + 32 * v : it.x0 + it.xlen - 1;
        cbx[v] = a.t.cb[0][xv[v]];
        relx[v] = cbx[v] - xn0;
        lcx[v] = MC ? a.t.sb[0][xv[v]] - cx : 0;
        swx[v] = a.t.sw[0][xv[v]];
        const float4 w = a.t.cw[0][xv[v]];
        cwr[v] = q4 == 0 ? w : q4 == 1 ? make_float4(w.y, w.z, w.w, w.x)
                             : q4 == 2 ? make_float4(w.z, w.w, w.x, w.y) : make_float4(w.w, w.x, w.y, w.z);
    }
    const int nx = g.nx, nxy = (int)g.nxy;
    float *rbw = RB + warp * 192;
    float4 *GYw = GY + warp * GB * GYSV;
    float4 *GZw = GZ + warp * GB * (XRN / 4);
    float *GZs = reinterpret_cast<float *>(GZw);   // MC: [GB][XRN]
    __syncthreads();

    for (int y = it.y0 + warp; y < it.y0 + it.ylen; y += W) {
        const int cby = a.t.cb[1][y];
        const float4 cwy = a.t.cw[1][y];
        const float4 swy = a.t.sw[1][y];
        const float *__restrict__ Frow = a.F + y * nx;

        // gamma of the item's bins contracted over the y-taps, for the z-cell at offset lcz:
        // GYw[k][l] = float4_n( sum_m wy_m gamma[(lcz + n, m, l)][bin k] )
        // alpha (lanes 0-15) / beta (lanes 16-31) contracted over y: lane = 16*ab + 4*l + n
        // (MC: alpha in abY, beta in abY2, lane = 4*xr + n)
        float abY = 0.f, abY2 = 0.f;
        auto rowTables = [&](int lcz) {
            for (int i = lane; i < nb2 * 4 * XRN; i += 32) {
                const int k = i / (4 * XRN), l = (i >> 2) % XRN, n = i & 3;
                const float *src = gl + ((lcz + n) * 4 * XRN + l) * GB + k;   // region (n, m, l): (n*4 + m)*XRN + l
                const float val = swy.x * src[0] + swy.y * src[XRN * GB] + swy.z * src[2 * XRN * GB] + swy.w * src[3 * XRN * GB];
                reinterpret_cast<float *>(GYw + k * GYSV + l)[n] = val;
            }
            if (ORI == 0 && !MC) {
                const int l = (lane >> 2) & 3, n = lane & 3;
                const float *src = (lane < 16 ? al : bl) + n * 16 + l;
                abY = swy.x * src[0] + swy.y * src[4] + swy.z * src[8] + swy.w * src[12];
            } else if (ORI == 0) {
                const int l = lane >> 2, n = lane & 3;
                const float *sa = al + (lcz + n) * 4 * XRN + l, *sb2 = bl + (lcz + n) * 4 * XRN + l;
                abY = swy.x * sa[0] + swy.y * sa[XRN] + swy.z * sa[2 * XRN] + swy.w * sa[3 * XRN];
                abY2 = swy.x * sb2[0] + swy.y * sb2[XRN] + swy.z * sb2[2 * XRN] + swy.w * sb2[3 * XRN];
            }
        };
        rowTables(0);
        int lczr = 0;   // MC: z-cell offset the row tables are built for
        __syncwarp();

        int gzl = zn0;
        float Ad[4][XV][3];
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int v = 0; v < XV; ++v) Ad[n][v][0] = Ad[n][v][1] = Ad[n][v][2] = 0.f;

        // retire control layer gzr with this lane's accumulated adjoints R[v][3]
        auto retire = [&](int gzr, const float (&R)[XV][3]) {
            // x-contraction across lanes into the row buffer as int32 fixed point (native
            // ATOMS.ADD): 2^(EA-126) bounds max |R| over the warp, so |w R 2^ks| < 2^22
            // (exact magic-number conversion) and a node's <= 32 contributions stay < 2^27.
            // Lane q = lane & 3 visits the x-taps in rotated order so neighbouring lanes of
            // one control cell hit distinct nodes in each atomic instruction.
            float mx = 0.f;
#pragma unroll
            for (int v = 0; v < XV; ++v)
#pragma unroll
                for (int c = 0; c < 3; ++c) mx = fmaxf(mx, fabsf(R[v][c]));
            const int EA = (int)(__reduce_max_sync(FULL, __float_as_uint(mx)) >> 23);
            if (EA == 0) return;   // all adjoints zero (or denormal): nothing to retire
            const int ks = min(148 - EA, 120);
            const float sc = exp2i(ks);
            int *rbi = reinterpret_cast<int *>(rbw);
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                const float R0 = R[v][0] * sc, R1 = R[v][1] * sc, R2 = R[v][2] * sc;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const int nd = relx[v] + ((l + q4) & 3);
                    const float w = f4(cwr[v], l);
                    atomicAdd(rbi + nd, __float_as_int(fmaf(w, R0, 12582912.f)) - 0x4B400000);
                    atomicAdd(rbi + 64 + nd, __float_as_int(fmaf(w, R1, 12582912.f)) - 0x4B400000);
                    atomicAdd(rbi + 128 + nd, __float_as_int(fmaf(w, R2, 12582912.f)) - 0x4B400000);
                }
            }
            __syncwarp();
            const float isc = exp2i(-ks);
            // y-contraction of the row buffer into the CTA node window
            const int lz = gzr - zn0;
            for (int i = lane; i < 3 * nxn; i += 32) {
                const int c = i / nxn, gxl = i - c * nxn;
                const float rv = (float)rbi[c * 64 + gxl] * isc;
                rbi[c * 64 + gxl] = 0;
                if (rv != 0.f) {
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float w = f4(cwy, mm);
                        if (w != 0.f) atomicAdd(NP + ((lz * 3 + c) * nyn + (cby + mm - yn0)) * nxn + gxl, w * rv);
                    }
                }
            }
            __syncwarp();
        };

        float4 cwzn = a.t.cw[2][it.z0], wzn = a.t.sw[2][it.z0];
        int bzn = a.t.cb[2][it.z0];
        float Fn[XV];   // F one slice ahead
#pragma unroll
        for (int v = 0; v < XV; ++v) Fn[v] = ld_stream(Frow + (long long)it.z0 * nxy + xv[v]);
        for (int z = it.z0; z < it.z0 + it.zlen; ++z) {
            const int bz = bzn;
            bzn = a.t.cb[2][min(z + 1, it.z0 + it.zlen - 1)];
            while (gzl < bz) {
                retire(gzl, Ad[0]);
#pragma unroll
                for (int n = 0; n < 3; ++n)
#pragma unroll
                    for (int v = 0; v < XV; ++v)
#pragma unroll
                        for (int c = 0; c < 3; ++c) Ad[n][v][c] = Ad[n + 1][v][c];
#pragma unroll
                for (int v = 0; v < XV; ++v) Ad[3][v][0] = Ad[3][v][1] = Ad[3][v][2] = 0.f;
                ++gzl;
            }
            if (MC) {   // crossed into the next z-cell: rebuild the row tables for its z-regions
                const int lz = a.t.sb[2][z] - cz;
                if (lz != lczr) {
                    __syncwarp();
                    rowTables(lz);
                    __syncwarp();
                    lczr = lz;
                }
            }
            const float4 cwz = cwzn, wz = wzn;     // this slice's z taps (loaded one slice ahead)
            {
                const int z1 = min(z + 1, it.z0 + it.zlen - 1);
                cwzn = a.t.cw[2][z1];
                wzn = a.t.sw[2][z1];
            }
            const float *__restrict__ Fz = Frow + z * nxy;
            const float4 *__restrict__ MGz = a.MG + ((long long)(z - a.mgz0) * g.ny + y) * nx;
            // issue this line's streaming loads first: their latency overlaps the per-line
            // alpha/beta/gamma contractions below
            float Fl[XV];
            float4 mgl[XV];
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                Fl[v] = Fn[v];
                Fn[v] = ld_stream(Fz + (z + 1 < it.z0 + it.zlen ? nxy : 0) + xv[v]);
                mgl[v] = ld_stream4(MGz + xv[v]);
            }
            // alpha~/beta~ of this line: reduce lane values over the z-taps, then broadcast
            float ay[4], by4[4];
            float tA = 0.f, tB = 0.f;   // MC: lane 4 xr holds alpha~ / beta~ of x-region xr
            if (ORI == 0 && !MC) {
                float t = f4(wz, lane & 3) * abY;
                t += __shfl_xor_sync(FULL, t, 1);
                t += __shfl_xor_sync(FULL, t, 2);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    ay[l] = __shfl_sync(FULL, t, 4 * l);
                    by4[l] = __shfl_sync(FULL, t, 16 + 4 * l);
                }
            } else if (ORI == 0) {
                tA = f4(wz, lane & 3) * abY;
                tB = f4(wz, lane & 3) * abY2;
                tA += __shfl_xor_sync(FULL, tA, 1);
                tB += __shfl_xor_sync(FULL, tB, 1);
                tA += __shfl_xor_sync(FULL, tA, 2);
                tB += __shfl_xor_sync(FULL, tB, 2);
            }
            // gamma of the item's bins contracted over z for this line: GZw[bin] = float4_l
            // (MC: GZs[bin][xr])
            for (int i = lane; i < XRN * nb2; i += 32) {
                const int k = i / XRN, l = i % XRN;
                if (MC) GZs[i] = dot4(wz, GYw[k * GYSV + l]);
                else reinterpret_cast<float *>(GZw + k)[l] = dot4(wz, GYw[k * GYSV + l]);
            }
            int a0[XV];
            float hlo[XV], hhi[XV];
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                const float Fv = Fl[v];
                a0[v] = min((int)Fv, g.L - 1);
                parzen_pair_F(Fv - (float)a0[v], hlo[v], hhi[v]);
            }
            __syncwarp();
#pragma unroll
            for (int v = 0; v < XV; ++v) {
                // (m, dM/dy) of this voxel from pass 1 (same fp32 arithmetic); m < 0 flags the
                // voxels whose per-voxel derivative is decided by the fp64 definition
                const float4 mg = mgl[v];
                float m = mg.x, dgx = mg.y, dgy = mg.z, dgz = mg.w;
                bool ex = m < 0.f;
                m = ex ? -1.0f - m : m;
                if (ex) {   // rare: a tap window at rest (u = 0 exactly in fp32 and fp64: t = 0, m = the
                            // voxel's own value on both sides) cannot have flagged a coordinate, and
                            // its Parzen-kink side is decided identically -- no fp64 recompute needed
                    const float4 tl = __ldg(a.tolw + ((long long)bz * g.Gy + cby) * g.Gx + cbx[v]);
                    ex = !(tl.x == 0.f && tl.y == 0.f && tl.z == 0.f);
                }
                const float4 sw = swx[v];
                const int n = min(max((int)floorf(m), 0), g.L - 1);
                const float fm = m - (float)n;
                float dval;   // dD/dm * Z
                if (ORI == 0) {
                    const int gk = gmap[a0[v]];
                    float4 G0, G1;
                    if (MC) {
                        const float *g0 = GZs + gk * XRN + lcx[v];
                        G0 = make_float4(g0[0], g0[1], g0[2], g0[3]);
                        G1 = make_float4(g0[XRN], g0[XRN + 1], g0[XRN + 2], g0[XRN + 3]);
#pragma unroll
                        for (int l = 0; l < 4; ++l) {
                            ay[l] = __shfl_sync(FULL, tA, 4 * (lcx[v] + l));
                            by4[l] = __shfl_sync(FULL, tB, 4 * (lcx[v] + l));
                        }
                    } else {
                        G0 = GZw[gk];
                        G1 = GZw[gk + 1];
                    }
                    const float At = fmaf(sw.w, ay[3], fmaf(sw.z, ay[2], fmaf(sw.y, ay[1], sw.x * ay[0])));
                    const float Bt = fmaf(sw.w, by4[3], fmaf(sw.z, by4[2], fmaf(sw.y, by4[1], sw.x * by4[0])));
                    const float Gt = fmaf(hlo[v], dot4(sw, G0), hhi[v] * dot4(sw, G1));
                    float g1p, c2;
                    if (m == floorf(m)) { g1p = 0.1f; c2 = 2.0f * m; }
                    else { g1p = fm < 0.5f ? fmaf(3.6f, fm, 0.1f) : fmaf(-3.6f, fm, 3.7f); c2 = 2.0f * (float)n + 1.0f; }
                    dval = g1p * fmaf(c2, At, 2.0f * (Bt - Gt));
                } else {
                    const float gF = (float)a0[v] + hhi[v];       // g1(F)
                    int jm, jp;                                     // table columns 3 (bin + 1)
                    float dm, dp;
                    if (m == floorf(m)) { const int k = (int)m; jm = 3 * k; jp = 3 * (k + 2); dm = -0.05f; dp = 0.05f; }
                    else {
                        jm = 3 * (n + 1); jp = 3 * (n + 2);
                        dp = fm < 0.5f ? fmaf(3.6f, fm, 0.1f) : fmaf(-3.6f, fm, 3.7f);
                        dm = -dp;
                    }
                    const int km = gmap[jm], kp = gmap[jp];
                    // psi' = T2~ + 2 (c_a - g) T1~ + (c_a - g)^2 T0~ (see k_combineA)
                    const int am = jm / 3 - 1, ap = jp / 3 - 1;
                    const float em = (am >= 0 && am < B ? shc2[am] : 0.f) - gF, ep = (ap < B ? shc2[ap] : 0.f) - gF;
                    const float psm = fmaf(em * em, dot4(sw, GZw[km]), fmaf(2.0f * em, dot4(sw, GZw[km + 1]), dot4(sw, GZw[km + 2])));
                    const float psp = fmaf(ep * ep, dot4(sw, GZw[kp]), fmaf(2.0f * ep, dot4(sw, GZw[kp + 1]), dot4(sw, GZw[kp + 2])));
                    dval = fmaf(dm, psm, dp * psp);
                }
                if (ex) {   // deferred to k_exact_fix (fp64); contributes nothing here
                    if (lok[v]) {
                        const int pos = atomicAdd(a.xcount, 1);
                        if (pos < a.xcap) a.xlist[pos] = ((z - a.mgz0) * g.ny + y) * nx + xv[v];
                    }
                    dgx = dgy = dgz = 0.f;
                }
                const float d = lok[v] ? a.invZ * dval : 0.f;
                const float d0 = d * dgx, d1 = d * dgy, d2 = d * dgz;
#pragma unroll
                for (int n2 = 0; n2 < 4; ++n2) {
                    const float w = f4(cwz, n2);
                    Ad[n2][v][0] = fmaf(w, d0, Ad[n2][v][0]);
                    Ad[n2][v][1] = fmaf(w, d1, Ad[n2][v][1]);
                    Ad[n2][v][2] = fmaf(w, d2, Ad[n2][v][2]);
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int n = 0; n < 4; ++n) retire(gzl + n, Ad[n]);
        __syncwarp();
    }
    __syncthreads();
    // ---- flush the node window: grad[c][gz][gy][gx] (external layout)
    for (int i = threadIdx.x; i < npsz; i += blockDim.x) {
        const float v = NP[i];
        if (v == 0.f) continue;
        const int gxl = i % nxn;
        int t = i / nxn;
        const int gyl = t % nyn;
        t /= nyn;
        const int c = t % 3, lz = t / 3;
        const int gzn = zn0 + lz;
        if (c >= g.ndim || gzn >= g.GzExt) continue;
        atomicAdd(a.grad + (((long long)c * g.GzExt + gzn) * g.Gy + (yn0 + gyl)) * g.Gx + (xn0 + gxl), (double)v);
    }
}

// The voxels pass 2 deferred (fp32 sample coordinate within rounding of a cell/clamp
// boundary, or m at the Parzen kink of a non-flat cell): the whole per-voxel derivative
// in the fp64 definition (exact_sample), its a8 weight dD/dm from the same fp32 alpha,
// beta, gamma tables and spatial weights (contracted directly over the 64 regions), and
// its adjoint scattered onto the 64 control nodes with fp64 atomics.  When more voxels
// were flagged than the list holds, the kernel scans the slab's MG flags instead.
// One warp per deferred voxel: the 64 tap loads of each stage are spread over the lanes
// (a thread-per-voxel version was a serial chain of ~250 dependent-latency loads, ~120 us).
template <int ORI>
__device__ __forceinline__ void exact_fix_voxel(const PassArgs &a, long long idx, double *sp, int gl, unsigned gm) {
    const Geo &g = a.g;
    const int x = (int)(idx % g.nx);
    const long long t = idx / g.nx;
    const int y = (int)(t % g.ny), z = (int)(t / g.ny) + a.mgz0;
    const int bx = a.t.cb[0][x], by = a.t.cb[1][y], bz = a.t.cb[2][z];
    // everything that does not depend on the fp64 sample is read before it (fewer serial
    // round trips per voxel): F and its bins, the spatial taps, and (ORI 0) this lane's
    // 4 region coefficients
    const float Fv = a.F[(long long)z * g.nxy + (long long)y * g.nx + x];
    const int a0 = min((int)Fv, g.L - 1);
    float hlo, hhi;
    parzen_pair_F(Fv - (float)a0, hlo, hhi);
    const int cx = a.t.sb[0][x], cy = a.t.sb[1][y], cz = a.t.sb[2][z];
    const float4 sx = a.t.sw[0][x], sy = a.t.sw[1][y], sz = a.t.sw[2][z];
    float al[4], be[4], ga[4];
    long long rr[4];
    float ww[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int tp = gl + 16 * h, nn = tp >> 4, mm = (tp >> 2) & 3, l = tp & 3;
        ww[h] = f4(sz, nn) * f4(sy, mm) * f4(sx, l);
        rr[h] = ((long long)(cz + nn) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        al[h] = be[h] = ga[h] = 0.f;
        if (ORI == 0 && ww[h] != 0.f) {
            al[h] = a.alpha[rr[h]];
            be[h] = a.beta[rr[h]];
            ga[h] = fmaf(hlo, a.gamma[rr[h] * a.gstride + a0], hhi * a.gamma[rr[h] * a.gstride + a0 + 1]);
        }
    }
    const ExactOut e = exact_sample(ExactGeo{g.nx, g.ny, g.nz, g.L, g.Gx, g.Gy, g.GzExt, g.ndim}, a.p64, a.M,
                                    a.t.cw64[0], a.t.cw64[1], a.t.cw64[2], bx, by, bz, x, y, z, sp, gl, gm);
    // ORI 1: exact_sample's c2 is 2m at integer m (even) and 2n + 1 otherwise (odd)
    int jm = 0, jp = 0;
    float dm = 0.f, dp = 0.f, em = 0.f, ep = 0.f;
    if (ORI == 1) {
        const int c2i = (int)e.c2;
        if ((c2i & 1) == 0) { const int k = c2i / 2; jm = 3 * k; jp = 3 * (k + 2); dm = -0.05f; dp = 0.05f; }
        else { const int nb = (c2i - 1) / 2; jm = 3 * (nb + 1); jp = 3 * (nb + 2); dm = -e.g1p; dp = e.g1p; }
        const float gF = (float)a0 + hhi;
        const int am = jm / 3 - 1, ap = jp / 3 - 1;
        em = (am >= 0 && am < g.B ? a.shiftc[am] : 0.f) - gF;
        ep = (ap < g.B ? a.shiftc[ap] : 0.f) - gF;
    }
    float At = 0.f, Bt = 0.f, Gt = 0.f;   // ORI 1 accumulates into At only
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const float w = ww[h];
        if (w == 0.f) continue;
        if (ORI == 0) {
            At = fmaf(w, al[h], At);
            Bt = fmaf(w, be[h], Bt);
            Gt = fmaf(w, ga[h], Gt);
        } else {
            const float *row = a.gamma + rr[h] * a.gstride;
            const float pm = fmaf(em * em, row[jm], fmaf(2.0f * em, row[jm + 1], row[jm + 2]));
            const float pp = fmaf(ep * ep, row[jp], fmaf(2.0f * ep, row[jp + 1], row[jp + 2]));
            At = fmaf(w, fmaf(dm, pm, dp * pp), At);
        }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
        At += __shfl_xor_sync(gm, At, o);
        if (ORI == 0) {
            Bt += __shfl_xor_sync(gm, Bt, o);
            Gt += __shfl_xor_sync(gm, Gt, o);
        }
    }
    const float d = ORI == 0 ? e.g1p * a.invZ * fmaf(e.c2, At, 2.0f * (Bt - Gt)) : a.invZ * At;
    const float dc[3] = {d * e.gx, d * e.gy, d * e.gz};
    const float4 wx = a.t.cw[0][x], wy = a.t.cw[1][y], wz = a.t.cw[2][z];
    const double unit = a.gradi ? ldexp(1.0, grad_shift(*a.gbound, a.dxz)) : 1.0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int tp = gl + 16 * h, nn = tp >> 4, mm = (tp >> 2) & 3, l = tp & 3;
        if (bz + nn >= g.GzExt || f4(wz, nn) == 0.f) continue;
        const float w = f4(wz, nn) * f4(wy, mm) * f4(wx, l);
        for (int c = 0; c < g.ndim; ++c) {
            const long long gi = (((long long)c * g.GzExt + bz + nn) * g.Gy + by + mm) * g.Gx + bx + l;
            if (a.gradi) atomicAdd(a.gradi + gi, (unsigned long long)__double2ll_rn((double)(w * dc[c]) * unit));
            else atomicAdd(a.grad + gi, (double)(w * dc[c]));
        }
    }
    __syncwarp(gm);   // sp is reused by the group's next voxel
}

// Two voxels per warp (one per half-warp group of 16 lanes).
template <int ORI = 0>
__global__ void __launch_bounds__(128) k_exact_fix(PassArgs a) {
    __shared__ double spb[8][3 * 64];
    const Geo &g = a.g;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, half = lane >> 4, gl = lane & 15;
    const unsigned gm = half ? 0xffff0000u : 0x0000ffffu;
    double *sp = spb[2 * wib + half];
    const int cnt = *a.xcount;
    const long long gid = (blockIdx.x * 4LL + wib) * 2 + half, ng = gridDim.x * 8LL;
    if (cnt <= a.xcap) {
        const int beg = a.xbeg ? *a.xbeg : 0;
        for (long long i = beg + gid; i < cnt; i += ng) {
            const int idx = a.xlist[i];
            exact_fix_voxel<ORI>(a, idx, sp, gl, gm);
            // clear the flag: a later overflow scan (pass 2 run in parts) must not fix it again
            if (gl == 0) a.MG[idx].x = -1.0f - a.MG[idx].x;
        }
        return;
    }
    if (a.xmode == 1) return;
    // list overflowed: scan the slab's MG flags, 32 voxels per warp step, the flagged ones
    // two at a time (one per half-warp)
    const long long slab = (long long)g.nxy * a.mgz1;
    const long long wid = blockIdx.x * 4LL + wib, nw = gridDim.x * 4LL;
    for (long long b = wid * 32; b < slab; b += nw * 32) {
        const long long i = b + lane;
        unsigned fl = __ballot_sync(0xffffffffu, i < slab && a.MG[i].x < 0.f);
        while (fl) {
            const int k0 = __ffs(fl) - 1;
            fl &= fl - 1;
            const int k1 = fl ? __ffs(fl) - 1 : -1;
            if (k1 >= 0) fl &= fl - 1;
            const int k = half ? k1 : k0;
            if (k >= 0) exact_fix_voxel<ORI>(a, b + k, sp, gl, gm);
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------- small kernels

// fp64 external params [ndim][GzExt][Gy][Gx] -> fp32 internal [3][Gz][Gy][Gx] (zeros padded)
// phi[c][Gz][Gy][Gx] fp32 (internal layout, Gz padded to 4 in 2-D with zeros)
__global__ void k_params_to_f32(const double *__restrict__ p, float *__restrict__ phi, Geo g, int zlo, int zhi) {
    // node layers [zlo, zhi) only: a rank converts the layers its slab's taps read
    const long long plane = (long long)g.Gx * g.Gy;
    const long long cs = (long long)g.Gz * plane, span = (long long)(zhi - zlo) * plane;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < span; j += (long long)gridDim.x * blockDim.x) {
        const long long i = (long long)zlo * plane + j;
        const long long gz = i / plane, xy = i - gz * plane;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double v = 0.0;
            if (c < g.ndim && gz < g.GzExt) v = p[(c * g.GzExt + gz) * plane + xy];
            phi[c * cs + i] = (float)v;
        }
    }
}


// Prep, step 1: fp64 params -> fp32 phi (as k_params_to_f32) and, per node, the max
// |phi_c| over the 4 nodes [k, k+3] along x, node layers [zlo, zhi)
__global__ void k_prep_phi_wx(const double *__restrict__ p, float *__restrict__ phi, float *__restrict__ wx, Geo g,
                              int zlo, int zhi) {
    const long long plane = (long long)g.Gx * g.Gy;
    const long long cs = (long long)g.Gz * plane, span = (long long)(zhi - zlo) * plane;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < span; j += (long long)gridDim.x * blockDim.x) {
        const long long i = (long long)zlo * plane + j;
        const long long gz = i / plane, xy = i - gz * plane;
        const int gx = (int)(xy % g.Gx);
        const bool live = gz < g.GzExt;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double *q = p + (c * g.GzExt + gz) * plane + xy;
            float v = 0.f, m = 0.f;
            if (c < g.ndim && live) {
                v = (float)q[0];
                m = fabsf(v);
#pragma unroll
                for (int d = 1; d < 4; ++d)
                    if (gx + d < g.Gx) m = fmaxf(m, fabsf((float)q[d]));
            }
            phi[c * cs + i] = v;
            wx[c * cs + i] = m;
        }
    }
}

// Prep, step 2: the y and z window max of step 1's x-max in one pass (-> the 4x4x4 tap
// window max keyed by the base node), base layers [zlo, zb) reading node layers up to zhi
__global__ void k_prep_tol(const float *__restrict__ wx, float4 *__restrict__ out, Geo g, int zlo, int zb, int zhi) {
    const long long plane = (long long)g.Gx * g.Gy, cs = (long long)g.Gz * plane, span = (long long)(zb - zlo) * plane;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < span; j += (long long)gridDim.x * blockDim.x) {
        const long long i = (long long)zlo * plane + j;
        const int k = (int)(i / plane), gy = (int)((i - (long long)k * plane) / g.Gx);
        float m[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int dz = 0; dz < 4; ++dz)
#pragma unroll
                for (int dy = 0; dy < 4; ++dy)
                    if (k + dz < zhi && gy + dy < g.Gy)
                        m[c] = fmaxf(m[c], __ldg(wx + c * cs + i + dz * plane + dy * g.Gx));
        out[i] = make_float4(2e-6f * m[0], 2e-6f * m[1], 2e-6f * m[2], 0.f);
    }
}


// min / max of a volume (exact; order independent)
__global__ void k_minmax(const float *__restrict__ v, long long n, float *out /*[2] encoded keys*/) {
    float lo = INFINITY, hi = -INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float x = v[i];
        lo = fminf(lo, x);
        hi = fmaxf(hi, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        // monotone int keys of the floats, so integer atomics order them correctly
        const int ilo = __float_as_int(lo), ihi = __float_as_int(hi);
        const int klo = ilo >= 0 ? ilo : ilo ^ 0x7fffffff, khi = ihi >= 0 ? ihi : ihi ^ 0x7fffffff;
        atomicMin(reinterpret_cast<int *>(out), klo);
        atomicMax(reinterpret_cast<int *>(out) + 1, khi);
    }
}

// v' = (float)(((double)v - lo) * ((double)L / (hi - lo))), clamped to [0, L]  (reading c1)
// computed with explicit round-to-nearest fp64 ops (no contraction) so it matches the oracle bit for bit.
__global__ void k_normalize(const float *__restrict__ in, float *__restrict__ out, long long n, double lo, double scale,
                            float Lf, int constant) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (constant) { out[i] = 0.f; continue; }
        float f = __double2float_rn(__dmul_rn(__dsub_rn((double)in[i], lo), scale));
        f = f < 0.f ? 0.f : (f > Lf ? Lf : f);
        out[i] = f;
    }
}

// fixed-image bin map a0 (debug / parity dump)
__global__ void k_a0_map(const float *__restrict__ F, short *__restrict__ out, long long n, int L) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (short)min((int)F[i], L - 1);
}

// per item: the set of fixed bins a0 present (bitmask, B <= 128) and the sum of the
// normalised moving image over the box (for the item's binless shift)
__global__ void k_item_scan(const float *__restrict__ F, const float *__restrict__ M, const Item *items, Geo g,
                            unsigned *masks /*[items][4]*/, double *msum /*[items]*/) {
    __shared__ unsigned sm[4];
    __shared__ double ss[32];
    const Item it = items[blockIdx.x];
    if (threadIdx.x < 4) sm[threadIdx.x] = 0u;
    __syncthreads();
    double s = 0;
    const long long n = (long long)it.xlen * it.ylen * it.zlen;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const int x = it.x0 + (int)(i % it.xlen);
        const long long t = i / it.xlen;
        const int y = it.y0 + (int)(t % it.ylen), z = it.z0 + (int)(t / it.ylen);
        const long long idx = (long long)z * g.nxy + (long long)y * g.nx + x;
        const int a0 = min((int)F[idx], g.L - 1);
        atomicOr(&sm[a0 >> 5], 1u << (a0 & 31));
        s += M[idx];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if ((threadIdx.x & 31) == 0) ss[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 4) masks[blockIdx.x * 4 + threadIdx.x] = sm[threadIdx.x];
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ss[w];
        msum[blockIdx.x] = t;
    }
}

// per-bin moment shift c_a = global conditional mean of the moving image given fixed bin a
// (from an identity-transform pass 1 with shift = bin index); bins without mass keep c_a = a
__global__ void k_shift_update(const double *SQ, const double *Nlo, const double *Nup, const float *shift_in,
                               float *shift_out, int R, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double N = 0, S = 0;
    const double c = shift_in[b], cp = b > 0 ? shift_in[b - 1] : 0.0;
    for (int r = 0; r < R; ++r) {
        const double nlo = Nlo[(long long)r * B + b];
        N += nlo;
        S += SQ[((long long)r * B + b) * 2 + 0] + c * nlo;
        if (b > 0) {
            const double nup = Nup[(long long)r * B + b - 1];
            N += nup;
            S += SQ[((long long)r * B + b - 1) * 2 + 1] + cp * nup;
        }
    }
    shift_out[b] = N > 0.0 ? (float)(S / N) : (float)b;
}


// ORI 1: the per-bin shift c_b = conditional mean of g1(F) over the voxels whose m falls in
// bin b (all regions), from an identity pass with shifts shift_in
__global__ void k_shift_updateA(const double *SQ, const double *NQ, const float *shift_in, float *shift_out,
                                int R, int B) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double N = 0, S = 0;
    const double c = shift_in[b], cp = b > 0 ? shift_in[b - 1] : 0.0;
    for (int r = 0; r < R; ++r) {
        const long long i = ((long long)r * B + b) * 2;
        N += NQ[i];
        S += SQ[i] + c * NQ[i];
        if (b > 0) {
            N += NQ[i - 1];
            S += SQ[i - 1] + cp * NQ[i - 1];
        }
    }
    shift_out[b] = N > 0.0 ? (float)(S / N) : (float)b;
}

// split the static-pass table into Nlo / Nup
__global__ void k_split_counts(const double *SQ, double *Nlo, double *Nup, long long RB) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < RB; i += (long long)gridDim.x * blockDim.x) {
        Nlo[i] = SQ[i * 2 + 0];
        Nup[i] = SQ[i * 2 + 1];
    }
}

}  // namespace srwcr
