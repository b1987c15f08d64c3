// srwcr_kernels.cuh -- sm_100a kernels of the SRWCR hot path (arXiv 1804.05061).
//
// One SRWCR evaluation = pass 1 (k_pass1: FFD + trilinear warp + Parzen moments +
// privatised histogram), combine (k_combine + k_reduce_D: per-region correlation
// ratios, D and the backward coefficient tables), pass 2 (k_pass2: FFD + trilinear
// value and gradient + dD/dm + adjoint B-spline scatter onto the control lattice).
// The warped image and every per-voxel intermediate stay in registers (the paper's
// kernels 1-4 materialise them).  DESIGN.md s5-s6 describe the data flow,
// the roofline of each kernel and what differs from the paper's GPU design.
//
// Work decomposition: a CTA of 16 warps owns one "item" = a box of voxels inside
// ONE spatial cell (so all its voxels share the same 4x4x4 = 64 regions of Eq 7).
// Lane = x (<= 32 voxels), warp = one row y of a 16-row chunk, and the CTA marches
// z through the item one slice at a time.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace srwcr {

constexpr int NW = 16;          // warps per CTA
constexpr int NT = NW * 32;     // threads per CTA
constexpr unsigned FULL = 0xffffffffu;
constexpr int LT_STRIDE = 17;   // line-table row stride (16 entries + 1 pad: conflict-free rows)

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
};

struct Item { int x0, xlen, y0, ylen, z0, zlen; };

struct PassArgs {
    Geo g;
    Tables t;
    const float *F;             // normalised fixed image  (model image A)
    const float *M;             // normalised moving image (estimated image B after warping)
    const float *phi;           // fp32 displacements [3][Gz][Gy][Gx]
    const float *shiftc;        // per-fixed-bin moment shift c_a (pass 1)
    const Item *items;
    double *SQ;                 // pass 1 out: [R][B][4] shifted partial moments (fp64)
    float scaleA, scaleB;       // pass 1 fixed-point scales of the line tables
    const double *p64;          // pass 2: fp64 params, external layout (exact-sample path)
    const float *alpha, *beta, *gamma;  // pass 2 in: [R], [R], [R][B]
    float invZ;
    double *grad;               // pass 2 out: [ndim][GzExt][Gy][Gx] (fp64)
    int segsteps;               // pass 2: shuffle steps of the segmented x-reduction
};

__device__ __forceinline__ float f4(const float4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// ---------------------------------------------------------------- FFD
// Contribution of control layer gz to this lane's displacement, contracted over the
// 4x4 (x, y) taps: U[c] = sum_{l,m} cwx_l cwy_m phi[c][gz][cby+m][cbx+l].  The warp
// shares one row y, so lanes j < nxn first contract y for x-node xn0+j (coalesced
// loads), then every lane gathers its 4 x-taps by shuffle.
__device__ __forceinline__ void ffd_layer(const float *__restrict__ phi, const Geo &g, int gz, int cby,
                                          float4 cwy, int xn0, int nxn, int relx, float4 cwx, int lane,
                                          float U[3]) {
    float p0 = 0.f, p1 = 0.f, p2 = 0.f;
    if (lane < nxn) {
        const long long plane = (long long)g.Gx * g.Gy;
        const long long cs = plane * g.Gz;
        const float *p = phi + (long long)gz * plane + (long long)cby * g.Gx + xn0 + lane;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            float w = f4(cwy, m);
            p0 = fmaf(w, __ldg(p + m * g.Gx), p0);
            p1 = fmaf(w, __ldg(p + cs + m * g.Gx), p1);
            p2 = fmaf(w, __ldg(p + 2 * cs + m * g.Gx), p2);
        }
    }
    U[0] = U[1] = U[2] = 0.f;
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        int src = relx + l;
        float w = f4(cwx, l);
        U[0] = fmaf(w, __shfl_sync(FULL, p0, src), U[0]);
        U[1] = fmaf(w, __shfl_sync(FULL, p1, src), U[1]);
        U[2] = fmaf(w, __shfl_sync(FULL, p2, src), U[2]);
    }
}

// ------------------------------------------------ backward warping (c1-c3)
// Split sample coordinate along one axis: position i + u with i integer.  The cell is
// formed as the integer i + floor(u) and t = u - floor(u) stays a small fp32 fraction
// (never i + u in fp32: SURVEY H11).  Out-of-domain positions clamp to [0, N-1] and
// report `clamped` (their derivative is 0, reading c2); cell = min(floor y, N-2).
__device__ __forceinline__ void axis_cell(int i, float u, int N, int &c0, float &t, bool &cl) {
    if (N == 1) { c0 = 0; t = 0.f; cl = true; return; }
    float fu = floorf(u);
    int c = i + (int)fu;
    float tt = u - fu;
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
    float c000 = __ldg(b), c100 = __ldg(b + 1), c010 = __ldg(b + dyo), c110 = __ldg(b + dyo + 1);
    float c001 = __ldg(b + dzo), c101 = __ldg(b + dzo + 1), c011 = __ldg(b + dzo + dyo),
          c111 = __ldg(b + dzo + dyo + 1);
    float e00 = lerpf(c000, c100, tx), e10 = lerpf(c010, c110, tx);
    float e01 = lerpf(c001, c101, tx), e11 = lerpf(c011, c111, tx);
    float f0 = lerpf(e00, e10, ty), f1 = lerpf(e01, e11, ty);
    if (GRAD) {
        float dx0 = lerpf(c100 - c000, c110 - c010, ty), dx1 = lerpf(c101 - c001, c111 - c011, ty);
        float dy0 = lerpf(c010 - c000, c110 - c100, tx), dy1 = lerpf(c011 - c001, c111 - c101, tx);
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
        float w = f * fmaf(1.8f, f, 0.1f);
        hhi = w;
        hlo = 1.0f - w;
    } else {
        float s = 1.0f - f;
        float w = s * fmaf(1.8f, s, 0.1f);
        hlo = w;
        hhi = 1.0f - w;
    }
}

// ---------------------------------------------------------------- pass 1
// Accumulates, per region r and fixed bin a0 (the lower of the two Parzen bins of F),
// the four shifted moments  T0 = sum w_r h_lo (g1 - c), T1 = sum w_r h_hi (g1 - c),
// T2 = sum w_r h_lo q', T3 = sum w_r h_hi q'  with g1 = sum_b b h(b - m) and
// q' = sum_b (b - c)^2 h(b - m) = (g1 - c)^2 + w1 (1 - w1)  (Eq 3 P:73 rewritten as
// moments; c = c_{a0}).  STATIC mode accumulates the weighted counts
// (T0 = sum w_r h_lo, T1 = sum w_r h_hi) instead, in fp32 so that the zero pattern of
// N is exact.
//
// Privatisation: per voxel, 16 values (4 spatial x-taps x 4 channels)
// go into the warp's line table LT[warp][a0][16] (int32 fixed point, native ATOMS;
// a warp whose 32 lanes share a0 reduces in registers first).  After each slice the
// CTA folds the 16 line tables into register accumulators owned by half-warps (half-
// warp h owns bins h, h+32, ...; lane e owns entry e = 4*xtap + channel), applying
// the row's y-weights; at the end of the slice the z-weights; at the end of the item
// the owners flush 64 regions x owned bins x 16 entries to SQ with fp64 atomics.
template <int KB, bool STATIC>
__global__ void __launch_bounds__(NT, 1) k_pass1(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo &g = a.g;
    const int B = g.B;
    int *LT = reinterpret_cast<int *>(smem);                       // [NW][B][LT_STRIDE]
    unsigned *mask = reinterpret_cast<unsigned *>(LT + NW * B * LT_STRIDE);  // [NW][4]
    int *lexp = reinterpret_cast<int *>(mask + NW * 4);            // [NW][2] line exponents (A, q')
    float4 *wyrow = reinterpret_cast<float4 *>(lexp + NW * 2);     // [NW]
    float *shc = reinterpret_cast<float *>(wyrow + NW);            // [B]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const Item it = a.items[blockIdx.x];
    const int hw = warp * 2 + (lane >> 4), e = lane & 15;

    for (int i = threadIdx.x; i < NW * B * LT_STRIDE; i += NT) LT[i] = 0;
    for (int i = threadIdx.x; i < B; i += NT) shc[i] = STATIC ? 0.f : a.shiftc[i];

    const int cx = a.t.sb[0][it.x0], cy = a.t.sb[1][it.y0], cz = a.t.sb[2][it.z0];
    const int x = it.x0 + lane;
    const bool lane_ok = lane < it.xlen;
    const int xc = min(x, g.nx - 1);
    const int cbx = a.t.cb[0][xc];
    const float4 cwx = a.t.cw[0][xc];
    const float4 swx = a.t.sw[0][xc];
    const int xn0 = a.t.cb[0][it.x0];
    const int nxn = a.t.cb[0][it.x0 + it.xlen - 1] + 4 - xn0;
    const int relx = cbx - xn0;
    // fixed-point exponents of the line tables (dynamic mode): a value v_c * wx_l is
    // scaled by 2^(274 - El - Ec) where 2^(El-126) bounds max_lanes wx_l (static per
    // item) and 2^(Ec-126) bounds max_lanes |v_c| (per line), so |scaled| < 2^22
    // (exact magic-number conversion) and a 32-lane sum stays < 2^27.
    int El[4];
#pragma unroll
    for (int l = 0; l < 4; ++l)
        El[l] = (int)(__reduce_max_sync(FULL, lane_ok ? __float_as_uint(f4(swx, l)) : 0u) >> 23);
    const int El_e = El[0] * ((e >> 2) == 0) + El[1] * ((e >> 2) == 1) + El[2] * ((e >> 2) == 2) + El[3] * ((e >> 2) == 3);

    float C[KB][16];
    float acc[KB][4];
#pragma unroll
    for (int k = 0; k < KB; ++k) {
#pragma unroll
        for (int i = 0; i < 16; ++i) C[k][i] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[k][i] = 0.f;
    }
    __syncthreads();

    for (int ys = it.y0; ys < it.y0 + it.ylen; ys += NW) {
        const int y = ys + warp;
        const bool row_ok = y < it.y0 + it.ylen;
        const int yc = min(y, g.ny - 1);
        const int cby = a.t.cb[1][yc];
        const float4 cwy = a.t.cw[1][yc];
        if (lane == 0) wyrow[warp] = row_ok ? a.t.sw[1][yc] : make_float4(0.f, 0.f, 0.f, 0.f);
        const bool ok = lane_ok && row_ok;

        int gzl = a.t.cb[2][it.z0];
        float U[4][3];
#pragma unroll
        for (int n = 0; n < 4; ++n) ffd_layer(a.phi, g, gzl + n, cby, cwy, xn0, nxn, relx, cwx, lane, U[n]);

        for (int z = it.z0; z < it.z0 + it.zlen; ++z) {
            const int bz = a.t.cb[2][z];
            while (gzl < bz) {                           // slide the 4-layer window
#pragma unroll
                for (int n = 0; n < 3; ++n) { U[n][0] = U[n + 1][0]; U[n][1] = U[n + 1][1]; U[n][2] = U[n + 1][2]; }
                ++gzl;
                ffd_layer(a.phi, g, gzl + 3, cby, cwy, xn0, nxn, relx, cwx, lane, U[3]);
            }
            const float4 cwz = a.t.cw[2][z];
            float ux = 0.f, uy = 0.f, uz = 0.f;
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                float w = f4(cwz, n);
                ux = fmaf(w, U[n][0], ux);
                uy = fmaf(w, U[n][1], uy);
                uz = fmaf(w, U[n][2], uz);
            }
            int a0 = 0;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (ok) {
                const long long idx = (long long)z * g.nxy + (long long)y * g.nx + x;
                const float Fv = __ldg(a.F + idx);
                a0 = min((int)Fv, g.L - 1);
                float hlo, hhi;
                parzen_pair(Fv - (float)a0, hlo, hhi);
                if (STATIC) {
                    v[0] = hlo;
                    v[1] = hhi;
                } else {
                    float dgx, dgy, dgz;
                    const float m = sample_m<false>(a.M, g, x, y, z, ux, uy, uz, dgx, dgy, dgz);
                    const int n = min(max((int)floorf(m), 0), g.L - 1);
                    const float fm = m - (float)n;
                    float w1l, w1;
                    parzen_pair(fm, w1l, w1);
                    const float A = ((float)n - shc[a0]) + w1;       // g1 - c
                    const float Bq = fmaf(A, A, w1 * w1l);           // (g1-c)^2 + w1(1-w1)
                    v[0] = hlo * A;
                    v[1] = hhi * A;
                    v[2] = hlo * Bq;
                    v[3] = hhi * Bq;
                }
            }
            // ---- line table update
            const unsigned okm = __ballot_sync(FULL, ok);
            float sc[4][2];                                    // scale per (x-tap, channel group)
            if (!STATIC) {
                const int EA = (int)(__reduce_max_sync(FULL, __float_as_uint(fabsf(v[0]) + fabsf(v[1]))) >> 23);
                const int EB = (int)(__reduce_max_sync(FULL, __float_as_uint(fabsf(v[2]) + fabsf(v[3]))) >> 23);
                if (lane == 0) { lexp[warp * 2] = EA; lexp[warp * 2 + 1] = EB; }
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    sc[l][0] = __int_as_float((min(274 - El[l] - EA, 120) + 127) << 23);
                    sc[l][1] = __int_as_float((min(274 - El[l] - EB, 120) + 127) << 23);
                }
            }
            if (okm) {
                const int a0f = __shfl_sync(FULL, a0, __ffs(okm) - 1);
                const bool uni = __all_sync(FULL, !ok || a0 == a0f);
                int *row = LT + (warp * B + (uni ? a0f : a0)) * LT_STRIDE;
                if (uni) {
                    // recursive-halving warp reduction of the 16 values (x-tap l, channel c)
                    float r8[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        int li = i >> 2, ci = i & 3;           // value i and i+8 (x-tap li+2)
                        float lo = f4(swx, li) * v[ci], hi = f4(swx, li + 2) * v[ci];
                        float send = (lane & 16) ? lo : hi, keep = (lane & 16) ? hi : lo;
                        r8[i] = keep + __shfl_xor_sync(FULL, send, 16);
                    }
                    float r4[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float send = (lane & 8) ? r8[i] : r8[i + 4], keep = (lane & 8) ? r8[i + 4] : r8[i];
                        r4[i] = keep + __shfl_xor_sync(FULL, send, 8);
                    }
                    float r2[2];
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        float send = (lane & 4) ? r4[i] : r4[i + 2], keep = (lane & 4) ? r4[i + 2] : r4[i];
                        r2[i] = keep + __shfl_xor_sync(FULL, send, 4);
                    }
                    float send = (lane & 2) ? r2[0] : r2[1], keep = (lane & 2) ? r2[1] : r2[0];
                    float r1 = keep + __shfl_xor_sync(FULL, send, 2);
                    r1 += __shfl_xor_sync(FULL, r1, 1);
                    // after the 5 halvings lane holds value index 8*b4 + 4*b3 + 2*b2 + b1 = lane>>1,
                    // i.e. entry 4*xtap + channel (step 1 split the x-taps {0,1} | {2,3})
                    const int ent = lane >> 1;
                    if ((lane & 1) == 0) {
                        if (STATIC) reinterpret_cast<float *>(row)[ent] += r1;
                        // a 32-voxel sum can exceed the 2^22 range of the magic-number conversion
                        else row[ent] += __float2int_rn(r1 * sc[ent >> 2][(ent & 3) >> 1]);
                    }
                } else if (ok) {
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const float wl = f4(swx, l);
#pragma unroll
                        for (int c = 0; c < (STATIC ? 2 : 4); ++c) {
                            const float val = wl * v[c];
                            if (STATIC) atomicAdd(reinterpret_cast<float *>(row) + l * 4 + c, val);
                            else atomicAdd(row + l * 4 + c, __float_as_int(fmaf(val, sc[l][c >> 1], 12582912.f)) - 0x4B400000);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                unsigned bits = __reduce_or_sync(FULL, (ok && (a0 >> 5) == k) ? (1u << (a0 & 31)) : 0u);
                if (lane == 0) mask[warp * 4 + k] = bits;
            }
            __syncthreads();
            // ---- fold the 16 line tables into the owners' registers
            const float4 wz = a.t.sw[2][z];
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                const int bin = hw + 32 * k;
                const unsigned mw = mask[(lane & 15) * 4 + k];
                const unsigned bal = __ballot_sync(FULL, bin < B && ((mw >> hw) & 1u));
                const unsigned mine = (lane < 16) ? (bal & 0xFFFFu) : (bal >> 16);
                unsigned uni = (bal & 0xFFFFu) | (bal >> 16);
                while (uni) {
                    const int j = __ffs(uni) - 1;
                    uni &= uni - 1;
                    if ((mine >> j) & 1u) {
                        int *p = LT + (j * B + bin) * LT_STRIDE + e;
                        float val;
                        if (STATIC) val = __int_as_float(*p);
                        else val = (float)(*p) * __int_as_float((127 - min(274 - El_e - lexp[j * 2 + ((e & 3) >> 1)], 120)) << 23);
                        *p = 0;
                        const float4 wy = wyrow[j];
                        acc[k][0] = fmaf(wy.x, val, acc[k][0]);
                        acc[k][1] = fmaf(wy.y, val, acc[k][1]);
                        acc[k][2] = fmaf(wy.z, val, acc[k][2]);
                        acc[k][3] = fmaf(wy.w, val, acc[k][3]);
                    }
                }
                if (mine) {
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        C[k][mm * 4 + 0] = fmaf(wz.x, acc[k][mm], C[k][mm * 4 + 0]);
                        C[k][mm * 4 + 1] = fmaf(wz.y, acc[k][mm], C[k][mm * 4 + 1]);
                        C[k][mm * 4 + 2] = fmaf(wz.z, acc[k][mm], C[k][mm * 4 + 2]);
                        C[k][mm * 4 + 3] = fmaf(wz.w, acc[k][mm], C[k][mm * 4 + 3]);
                        acc[k][mm] = 0.f;
                    }
                }
            }
            __syncthreads();
        }
        __syncthreads();
    }
    // ---- flush: region (cz+n, cy+m, cx+l), bin, channel
    const int l_e = e >> 2, ch = e & 3;
#pragma unroll
    for (int k = 0; k < KB; ++k) {
        const int bin = hw + 32 * k;
        if (bin >= B) continue;
#pragma unroll
        for (int mm = 0; mm < 4; ++mm)
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const float val = C[k][mm * 4 + n];
                if (val != 0.f) {
                    const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l_e);
                    atomicAdd(a.SQ + (r * B + bin) * 4 + ch, (double)val);
                }
            }
    }
}

// ---------------------------------------------------------------- combine
// One warp per region r (Eq 9-12 P:111-127 in moment form):
//   N_ra = Nlo[r][a] + Nup[r][a-1];  S_ra, Q_ra unshifted from the pass-1 moments;
//   T_r = Q_r - S_r^2/N_r;  V_r = Q_r - sum_{a:N_ra>0} S_ra^2/N_ra;
//   retained iff N_r/Z > eps_mass and sigma_r^2 = T_r/N_r > eps_sigma (reading c12);
//   dterm[r] = N_r V_r / T_r (so D = sum dterm / Z), and the coefficients
//   alpha_r = CR_r/sigma_r^2, beta_r = (1-CR_r) mu_r/sigma_r^2, gamma_ra = mu_r(a)/sigma_r^2.
struct CombineArgs {
    const double *SQ;           // [R][B][4]
    const double *Nlo, *Nup;    // [R][B]
    const float *shiftc;        // [B]
    int R, B;
    double Z, eps_mass, eps_sigma;
    double *dterm;              // [R]
    double *reg;                // [R][6] {p(r), sigma2, mu, 1-CR, retained, Z}
    double *S_out, *Q_out;      // [R][B] unshifted (debug / parity), may be null
    float *alpha, *beta, *gamma;
};

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

__global__ void __launch_bounds__(256) k_combine(CombineArgs a) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= a.R) return;
    const int B = a.B;
    double Nr = 0, Sr = 0, Qr = 0, s2n = 0;
    for (int b = lane; b < B; b += 32) {
        const double *q = a.SQ + ((long long)r * B + b) * 4;
        const double c = a.shiftc[b];
        const double nlo = a.Nlo[(long long)r * B + b];
        double N = nlo, S = q[0] + c * nlo, Q = q[2] + 2.0 * c * q[0] + c * c * nlo;
        if (b > 0) {
            const double *qp = q - 4;
            const double cp = a.shiftc[b - 1];
            const double nup = a.Nup[(long long)r * B + b - 1];
            N += nup;
            S += qp[1] + cp * nup;
            Q += qp[3] + 2.0 * cp * qp[1] + cp * cp * nup;
        }
        if (a.S_out) { a.S_out[(long long)r * B + b] = S; a.Q_out[(long long)r * B + b] = Q; }
        Nr += N; Sr += S; Qr += Q;
        if (N > 0.0) s2n += S * S / N;
    }
    Nr = warp_sum_d(Nr); Sr = warp_sum_d(Sr); Qr = warp_sum_d(Qr); s2n = warp_sum_d(s2n);
    const double pr = Nr / a.Z;
    double sig2 = 0, mu = 0, omcr = 0;
    bool ret = false;
    if (pr > a.eps_mass) {
        const double Tr = Qr - Sr * Sr / Nr, Vr = Qr - s2n;
        sig2 = Tr / Nr;
        mu = Sr / Nr;
        if (sig2 > a.eps_sigma) { ret = true; omcr = Vr / Tr; }
    }
    if (lane == 0) {
        a.dterm[r] = ret ? Nr * omcr : 0.0;
        a.alpha[r] = ret ? (float)((1.0 - omcr) / sig2) : 0.f;
        a.beta[r] = ret ? (float)(omcr * mu / sig2) : 0.f;
        double *rg = a.reg + (long long)r * 6;
        rg[0] = pr; rg[1] = sig2; rg[2] = mu; rg[3] = omcr; rg[4] = ret ? 1.0 : 0.0; rg[5] = a.Z;
    }
    for (int b = lane; b < B; b += 32) {
        const double *q = a.SQ + ((long long)r * B + b) * 4;
        const double c = a.shiftc[b];
        const double nlo = a.Nlo[(long long)r * B + b];
        double N = nlo, S = q[0] + c * nlo;
        if (b > 0) {
            const double cp = a.shiftc[b - 1];
            const double nup = a.Nup[(long long)r * B + b - 1];
            N += nup;
            S += (q - 4)[1] + cp * nup;
        }
        a.gamma[(long long)r * B + b] = (ret && N > 0.0) ? (float)((S / N) / sig2) : 0.f;
    }
}

// D = (1/Z) sum_r dterm[r] in a fixed order (deterministic); out[0] = D, out[1] = #retained
__global__ void __launch_bounds__(1024) k_reduce_D(const double *dterm, const double *reg, int R, double Z,
                                                    double *out) {
    __shared__ double sd[1024];
    __shared__ double sc[1024];
    double s = 0, c = 0;
    for (int r = threadIdx.x; r < R; r += blockDim.x) { s += dterm[r]; c += reg[(long long)r * 6 + 4]; }
    sd[threadIdx.x] = s;
    sc[threadIdx.x] = c;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) { sd[threadIdx.x] += sd[threadIdx.x + o]; sc[threadIdx.x] += sc[threadIdx.x + o]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { out[0] = sd[0] / Z; out[1] = sc[0]; }
}


__device__ __forceinline__ double d4(const double4 &v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}

// Exact-sample path of pass 2 (fp64), taken by the rare lanes whose fp32 sample
// position lies within 1e-4 voxel of an integer (a trilinear cell or clamp boundary)
// or whose warped intensity lies within 1e-4 of an integer (the Parzen kink of c4):
// there the per-voxel derivative is discontinuous and the side must be decided as
// the fp64 definition decides it.  Outputs m's gradient, g1' and c2.
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

__device__ __noinline__ void exact_sample(ExactGeo g, const double *__restrict__ p64, const float *__restrict__ M,
                                          int bx, int by, int bz, double4 wx, double4 wy, double4 wz, int x,
                                          int y, int z, float &gxo, float &gyo, float &gzo, float &g1po,
                                          float &c2o) {
    const long long plane = (long long)g.Gx * g.Gy, cs = plane * g.GzExt;
    const long long nxy = (long long)g.nx * g.ny;
    double u[3] = {0.0, 0.0, 0.0};
#pragma unroll
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
                const long long s = (long long)(bz + n) * plane + (long long)(by + mm) * g.Gx + bx + l;
                u[0] += w * p64[s];
                u[1] += w * p64[cs + s];
                if (g.ndim == 3) u[2] += w * p64[2 * cs + s];
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
    gxo = clx ? 0.f : (float)gx;
    gyo = cly ? 0.f : (float)gy;
    gzo = (clz || g.nz == 1) ? 0.f : (float)gz;
    int n = (int)floor(m);
    n = n > g.L - 1 ? g.L - 1 : (n < 0 ? 0 : n);
    const double f = m - (double)n;
    if (m == floor(m)) { g1po = 0.1f; c2o = (float)(2.0 * m); }
    else { g1po = (float)(f < 0.5 ? 0.1 + 3.6 * f : 3.7 - 3.6 * f); c2o = (float)(2.0 * n + 1.0); }
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
template <int KB>
__global__ void __launch_bounds__(NT, 1) k_pass2(PassArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Geo &g = a.g;
    const int B = g.B;
    const Item it = a.items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const int xn0 = a.t.cb[0][it.x0];
    const int nxn = a.t.cb[0][it.x0 + it.xlen - 1] + 4 - xn0;
    const int yn0 = a.t.cb[1][it.y0];
    const int nyn = a.t.cb[1][it.y0 + it.ylen - 1] + 4 - yn0;
    const int zn0 = a.t.cb[2][it.z0];
    const int nzn = a.t.cb[2][it.z0 + it.zlen - 1] + 4 - zn0;

    float *gl = reinterpret_cast<float *>(smem);          // [64][B] gamma of the 64 regions
    float *gz_t = gl + 64 * B;                            // [16][B] z-contracted gamma (m,l) x bin
    float4 *GY = reinterpret_cast<float4 *>(gz_t + 16 * B);  // [NW][B] per-line y,z-contracted gamma
    float *al = reinterpret_cast<float *>(GY + NW * B);   // [64]
    float *bl = al + 64;                                  // [64]
    float *abz = bl + 64;                                 // [32]: alpha_z[m][l], beta_z[m][l]
    float *RB = abz + 32;                                 // [NW][3][32] retiring-layer row buffer
    float *NP = RB + NW * 96;                             // [nzn][3][nyn][nxn] node window

    const int cx = a.t.sb[0][it.x0], cy = a.t.sb[1][it.y0], cz = a.t.sb[2][it.z0];
    for (int i = threadIdx.x; i < 64 * B; i += NT) {
        const int reg = i / B, bin = i - reg * B;
        const int l = reg & 3, mm = (reg >> 2) & 3, n = reg >> 4;
        const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        gl[i] = __ldg(a.gamma + r * B + bin);
    }
    for (int i = threadIdx.x; i < 64; i += NT) {
        const int l = i & 3, mm = (i >> 2) & 3, n = i >> 4;
        const long long r = ((long long)(cz + n) * g.Ky + (cy + mm)) * g.Kx + (cx + l);
        al[i] = __ldg(a.alpha + r);
        bl[i] = __ldg(a.beta + r);
    }
    const int npsz = nzn * 3 * nyn * nxn;
    for (int i = threadIdx.x; i < npsz; i += NT) NP[i] = 0.f;
    for (int i = threadIdx.x; i < NW * 96; i += NT) RB[i] = 0.f;

    const int x = it.x0 + lane;
    const bool lane_ok = lane < it.xlen;
    const int xc = min(x, g.nx - 1);
    const int cbx = a.t.cb[0][xc];
    const float4 cwx = a.t.cw[0][xc];
    const float4 swx = a.t.sw[0][xc];
    const int relx = cbx - xn0;
    // segment heads of equal control x-base (for the adjoint x-contraction)
    const int cbx_prev = __shfl_up_sync(FULL, cbx, 1);
    const bool head = lane == 0 || cbx_prev != cbx;
    float *rbw = RB + warp * 96;
    __syncthreads();

    for (int ys = it.y0; ys < it.y0 + it.ylen; ys += NW) {
        const int y = ys + warp;
        const bool row_ok = y < it.y0 + it.ylen;
        const int yc = min(y, g.ny - 1);
        const int cby = a.t.cb[1][yc];
        const float4 cwy = a.t.cw[1][yc];
        const float4 swy = a.t.sw[1][yc];
        const bool ok = lane_ok && row_ok;

        int gzl = zn0;
        float U[4][3], Ad[4][3];
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            ffd_layer(a.phi, g, gzl + n, cby, cwy, xn0, nxn, relx, cwx, lane, U[n]);
            Ad[n][0] = Ad[n][1] = Ad[n][2] = 0.f;
        }

        // retire control layer gzr with this lane's accumulated adjoint R[3]
        auto retire = [&](int gzr, const float R[3]) {
            float val[4][3];
#pragma unroll
            for (int l = 0; l < 4; ++l)
#pragma unroll
                for (int c = 0; c < 3; ++c) val[l][c] = f4(cwx, l) * R[c];
            for (int s = 0, off = 1; s < a.segsteps; ++s, off <<= 1) {
                const int nb = __shfl_down_sync(FULL, cbx, off);
                const bool same = (lane + off < 32) && nb == cbx;
#pragma unroll
                for (int l = 0; l < 4; ++l)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const float t = __shfl_down_sync(FULL, val[l][c], off);
                        if (same) val[l][c] += t;
                    }
            }
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                if (head)
#pragma unroll
                    for (int c = 0; c < 3; ++c) rbw[c * 32 + relx + l] += val[l][c];
                __syncwarp();
            }
            // y-contraction of the row buffer into the CTA node window
            const int lz = gzr - zn0;
            for (int i = lane; i < 3 * nxn; i += 32) {
                const int c = i / nxn, gxl = i - c * nxn;
                const float rv = rbw[c * 32 + gxl];
                rbw[c * 32 + gxl] = 0.f;
                if (rv != 0.f && row_ok) {
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float w = f4(cwy, mm);
                        if (w != 0.f) atomicAdd(NP + ((lz * 3 + c) * nyn + (cby + mm - yn0)) * nxn + gxl, w * rv);
                    }
                }
            }
            __syncwarp();
        };

        for (int z = it.z0; z < it.z0 + it.zlen; ++z) {
            const int bz = a.t.cb[2][z];
            while (gzl < bz) {
                retire(gzl, Ad[0]);
#pragma unroll
                for (int n = 0; n < 3; ++n)
#pragma unroll
                    for (int c = 0; c < 3; ++c) { U[n][c] = U[n + 1][c]; Ad[n][c] = Ad[n + 1][c]; }
                Ad[3][0] = Ad[3][1] = Ad[3][2] = 0.f;
                ++gzl;
                ffd_layer(a.phi, g, gzl + 3, cby, cwy, xn0, nxn, relx, cwx, lane, U[3]);
            }
            // ---- per-slice region tables: gamma_z[(m,l)][bin], alpha_z, beta_z
            const float4 swz = a.t.sw[2][z];
            __syncthreads();
            for (int i = threadIdx.x; i < 16 * B; i += NT) {
                const int ml = i / B, bin = i - ml * B;
                float s = swz.x * gl[ml * B + bin];
                s = fmaf(swz.y, gl[(16 + ml) * B + bin], s);
                s = fmaf(swz.z, gl[(32 + ml) * B + bin], s);
                s = fmaf(swz.w, gl[(48 + ml) * B + bin], s);
                gz_t[i] = s;
            }
            if (threadIdx.x < 32) {
                const float *src = threadIdx.x < 16 ? al : bl;
                const int ml = threadIdx.x & 15;
                abz[threadIdx.x] = swz.x * src[ml] + swz.y * src[16 + ml] + swz.z * src[32 + ml] + swz.w * src[48 + ml];
            }
            __syncthreads();

            const float4 cwz = a.t.cw[2][z];
            float ux = 0.f, uy = 0.f, uz = 0.f;
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const float w = f4(cwz, n);
                ux = fmaf(w, U[n][0], ux);
                uy = fmaf(w, U[n][1], uy);
                uz = fmaf(w, U[n][2], uz);
            }
            int a0 = 0;
            float hlo = 0.f, hhi = 0.f, m = 0.f, dgx = 0.f, dgy = 0.f, dgz = 0.f;
            if (ok) {
                const long long idx = (long long)z * g.nxy + (long long)y * g.nx + x;
                const float Fv = __ldg(a.F + idx);
                a0 = min((int)Fv, g.L - 1);
                parzen_pair(Fv - (float)a0, hlo, hhi);
                m = sample_m<true>(a.M, g, x, y, z, ux, uy, uz, dgx, dgy, dgz);
            }
            // ---- the line's gamma, contracted over (m, n) for the bins it touches
            unsigned bits[KB];
            int tot = 0;
#pragma unroll
            for (int k = 0; k < KB; ++k) {
                unsigned mine = 0u;
                if (ok) {
                    if ((a0 >> 5) == k) mine |= 1u << (a0 & 31);
                    if (((a0 + 1) >> 5) == k) mine |= 1u << ((a0 + 1) & 31);
                }
                bits[k] = __reduce_or_sync(FULL, mine);
                tot += __popc(bits[k]);
            }
            for (int o = lane; o < 4 * tot; o += 32) {
                int bi = o >> 2;
                const int l = o & 3;
                int bin = 0;
#pragma unroll
                for (int k = 0; k < KB; ++k) {
                    const int c = __popc(bits[k]);
                    if (bi >= 0 && bi < c) {
                        unsigned w = bits[k];
                        int pos = 0, r = bi;
#pragma unroll
                        for (int s = 16; s > 0; s >>= 1) {
                            const unsigned lo = w & ((1u << s) - 1u);
                            const int cnt = __popc(lo);
                            if (r >= cnt) { r -= cnt; w >>= s; pos += s; } else { w = lo; }
                        }
                        bin = 32 * k + pos;
                    }
                    bi -= c;
                }
                float s = swy.x * gz_t[(0 + l) * B + bin];
                s = fmaf(swy.y, gz_t[(4 + l) * B + bin], s);
                s = fmaf(swy.z, gz_t[(8 + l) * B + bin], s);
                s = fmaf(swy.w, gz_t[(12 + l) * B + bin], s);
                reinterpret_cast<float *>(GY + warp * B + bin)[l] = s;
            }
            // alpha/beta contracted over (m, n) for this line, x-taps 0..3
            float abv = 0.f;
            if (lane < 8) {
                const int l = lane & 3, off = (lane >> 2) * 16;
                abv = swy.x * abz[off + l] + swy.y * abz[off + 4 + l] + swy.z * abz[off + 8 + l] + swy.w * abz[off + 12 + l];
            }
            __syncwarp();
            float At = 0.f, Bt = 0.f;
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                At = fmaf(f4(swx, l), __shfl_sync(FULL, abv, l), At);
                Bt = fmaf(f4(swx, l), __shfl_sync(FULL, abv, 4 + l), Bt);
            }
            if (ok) {
                const float4 G0 = GY[warp * B + a0], G1 = GY[warp * B + a0 + 1];
                float Gt = 0.f;
#pragma unroll
                for (int l = 0; l < 4; ++l) Gt = fmaf(f4(swx, l), fmaf(hlo, f4(G0, l), hhi * f4(G1, l)), Gt);
                const int n = min(max((int)floorf(m), 0), g.L - 1);
                const float fm = m - (float)n;
                float g1p, c2;
                if (m == floorf(m)) { g1p = 0.1f; c2 = 2.0f * m; }
                else { g1p = fm < 0.5f ? fmaf(3.6f, fm, 0.1f) : fmaf(-3.6f, fm, 3.7f); c2 = 2.0f * (float)n + 1.0f; }
                // discontinuities of the per-voxel derivative: decide them in fp64
                const float tolu = 1e-4f;
                if (near_integer(ux, tolu + 1e-6f * fabsf(ux)) || near_integer(uy, tolu + 1e-6f * fabsf(uy)) ||
                    near_integer(uz, tolu + 1e-6f * fabsf(uz)) || near_integer(m, 1e-4f))
                    exact_sample(ExactGeo{g.nx, g.ny, g.nz, g.L, g.Gx, g.Gy, g.GzExt, g.ndim}, a.p64, a.M, cbx,
                                 cby, a.t.cb[2][z], a.t.cw64[0][x], a.t.cw64[1][y], a.t.cw64[2][z], x, y, z, dgx,
                                 dgy, dgz, g1p, c2);
                const float d = g1p * a.invZ * (fmaf(c2, At, 2.0f * (Bt - Gt)));
                const float d0 = d * dgx, d1 = d * dgy, d2 = d * dgz;
#pragma unroll
                for (int n2 = 0; n2 < 4; ++n2) {
                    const float w = f4(cwz, n2);
                    Ad[n2][0] = fmaf(w, d0, Ad[n2][0]);
                    Ad[n2][1] = fmaf(w, d1, Ad[n2][1]);
                    Ad[n2][2] = fmaf(w, d2, Ad[n2][2]);
                }
            }
            __syncwarp();
        }
#pragma unroll
        for (int n = 0; n < 4; ++n) retire(gzl + n, Ad[n]);
    }
    __syncthreads();
    // ---- flush the node window: grad[c][gz][gy][gx] (external layout)
    for (int i = threadIdx.x; i < npsz; i += NT) {
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

// ---------------------------------------------------------------- small kernels

// fp64 external params [ndim][GzExt][Gy][Gx] -> fp32 internal [3][Gz][Gy][Gx] (zeros padded)
__global__ void k_params_to_f32(const double *__restrict__ p, float *__restrict__ phi, Geo g) {
    const long long plane = (long long)g.Gx * g.Gy;
    const long long total = 3LL * g.Gz * plane;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / (g.Gz * plane);
        const long long rem = i - c * g.Gz * plane;
        const long long gz = rem / plane, xy = rem - gz * plane;
        float v = 0.f;
        if (c < g.ndim && gz < g.GzExt) v = (float)p[(c * g.GzExt + gz) * plane + xy];
        phi[i] = v;
    }
}

// min / max of a volume (exact; order independent)
__global__ void k_minmax(const float *__restrict__ v, long long n, float *out /*[2], init +inf,-inf*/) {
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
        // float ordering == int ordering for non-negative; use CAS-free atomics on encoded keys
        int ilo = __float_as_int(lo), ihi = __float_as_int(hi);
        int klo = ilo >= 0 ? ilo : ilo ^ 0x7fffffff, khi = ihi >= 0 ? ihi : ihi ^ 0x7fffffff;
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
        S += SQ[((long long)r * B + b) * 4 + 0] + c * nlo;
        if (b > 0) {
            const double nup = Nup[(long long)r * B + b - 1];
            N += nup;
            S += SQ[((long long)r * B + b - 1) * 4 + 1] + cp * nup;
        }
    }
    shift_out[b] = N > 0.0 ? (float)(S / N) : (float)b;
}

// split the static-pass table into Nlo / Nup
__global__ void k_split_counts(const double *SQ, double *Nlo, double *Nup, long long RB) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < RB; i += (long long)gridDim.x * blockDim.x) {
        Nlo[i] = SQ[i * 4 + 0];
        Nup[i] = SQ[i * 4 + 1];
    }
}

}  // namespace srwcr
