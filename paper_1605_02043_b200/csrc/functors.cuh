// functors.cuh -- per-edge "interaction between two adjacent particles" and the
// per-vertex update, as device code shared by the staged (EP) kernel and the naive
// (default-schedule) comparator so both evaluate the same fp32 expression per edge.
//
// Reading Z9: Rodinia Euler3D-style face flux, gamma = 1.4, sigma = 0.2,
// forward Euler U' = U + dt F. Per vertex: u = m/rho, p = (gamma-1)(E - rho|u|^2/2),
// c = sqrt(gamma p / rho); per edge (a, b) with area-normal n out of a:
//   f   = -|n| sigma (|u_a| + |u_b| + c_a + c_b) / 2
//   Phi = f (U_a - U_b) - n.(G(U_a) + G(U_b)) / 2,   F_a += Phi, F_b -= Phi,
// G_rho = m, G_m = m u^T + p I, G_E = (E + p) u.
#pragma once

#include <stdint.h>

namespace epg {

constexpr float kGamma = 1.4f;
constexpr float kSigma = 0.2f;

// float4 slot of half h (0/1) of 32-byte record r in shared memory. XOR-ing h with bit 2
// of r spreads 8 consecutive records over all 8 16-byte bank groups, so the 128-bit
// loads of a quarter-warp do not collide two-way on the even groups (measured: removing
// it costs ~0.6 us per partition on C2).
__device__ __forceinline__ int rec4(int r, int h) { return 2 * r + (h ^ ((r >> 2) & 1)); }

// Staged per-vertex quantities of the cfd functor (8 floats; SoA in shared memory).
struct CfdVertex {
    float rho, mx, my, mz, E, p, speed, rinv;  // speed = |u| + c, rinv = 1 / rho
};

// MUFU reciprocal square root / reciprocal, flush-to-zero forms: rsqrtf / __fdividef add a
// denormal range check and rescale around the MUFU op (an FSETP and a predicated FMUL each);
// the staged values are never denormal (densities, energies, squared speeds and face areas)
__device__ __forceinline__ float rsqrt_ftz(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// sqrt(x) for x >= 0 through the MUFU reciprocal square root (no IEEE fix-up branch);
// relative error ~1e-7, far inside the 1e-5 parity tolerance
__device__ __forceinline__ float sqrt_nb(float x) { return x > 0.0f ? x * rsqrt_ftz(x) : 0.0f; }

__device__ __forceinline__ CfdVertex cfd_derive(float rho, float mx, float my, float mz, float E) {
    CfdVertex d;
    d.rho = rho; d.mx = mx; d.my = my; d.mz = mz; d.E = E;
    d.rinv = __fdividef(1.0f, rho);
    const float ux = mx * d.rinv, uy = my * d.rinv, uz = mz * d.rinv;
    const float uu = ux * ux + uy * uy + uz * uz;
    d.p = (kGamma - 1.0f) * (E - 0.5f * rho * uu);
    d.speed = sqrt_nb(uu) + sqrt_nb(kGamma * d.p * d.rinv);
    return d;
}

// Phi[0..4] for edge (a, b) with normal n out of a.
__device__ __forceinline__ void cfd_phi(const CfdVertex &a, const CfdVertex &b, float nx, float ny, float nz,
                                        float phi[5]) {
    const float nlen = sqrt_nb(nx * nx + ny * ny + nz * nz);
    const float f = -nlen * kSigma * 0.5f * (a.speed + b.speed);
    const float mna = a.mx * nx + a.my * ny + a.mz * nz;
    const float mnb = b.mx * nx + b.my * ny + b.mz * nz;
    const float una = mna * a.rinv, unb = mnb * b.rinv;  // u . n
    phi[0] = f * (a.rho - b.rho) - 0.5f * (mna + mnb);
    phi[1] = f * (a.mx - b.mx) - 0.5f * (a.mx * una + b.mx * unb + (a.p + b.p) * nx);
    phi[2] = f * (a.my - b.my) - 0.5f * (a.my * una + b.my * unb + (a.p + b.p) * ny);
    phi[3] = f * (a.mz - b.mz) - 0.5f * (a.mz * una + b.mz * unb + (a.p + b.p) * nz);
    phi[4] = f * (a.E - b.E) - 0.5f * ((a.E + a.p) * una + (b.E + b.p) * unb);
}

// ---------------------------------------------------------------------------------
// Functor policy classes used by the kernels.
//   ROW   floats per state row (input and output)
//   NV    staged floats per local vertex (SoA in shared memory, stride Lcap)
//   NPHI  floats stored per edge (SoA in shared memory, stride Scap)
//   stage(row, V, j, Lcap)            derive and store vertex j
//   edge(V, Lcap, a, b, payload, e, Phi, Scap, i)
//   gather(Phi, Scap, i, side, acc)   add edge i's contribution to its endpoint `side`
//   finish_smem(V, Lcap, j, acc, c, out_row)  result of a staged vertex (c = vertex const)
//   finish_row(in_row, acc, c, out_row)       result of a vertex from global memory
//   untouched(in_row, out_row)
// ---------------------------------------------------------------------------------
struct CfdFlux {
    static constexpr int ROW = 5, NV = 8, NPHI = 5;
    __device__ __forceinline__ static void stage(const float *__restrict__ row, float *V, int j, int Lcap) {
        CfdVertex d = cfd_derive(row[0], row[1], row[2], row[3], row[4]);
        V[0 * Lcap + j] = d.rho; V[1 * Lcap + j] = d.mx; V[2 * Lcap + j] = d.my; V[3 * Lcap + j] = d.mz;
        V[4 * Lcap + j] = d.E; V[5 * Lcap + j] = d.p; V[6 * Lcap + j] = d.speed; V[7 * Lcap + j] = d.rinv;
    }
    __device__ __forceinline__ static CfdVertex load(const float *V, int j, int Lcap) {
        CfdVertex d;
        d.rho = V[0 * Lcap + j]; d.mx = V[1 * Lcap + j]; d.my = V[2 * Lcap + j]; d.mz = V[3 * Lcap + j];
        d.E = V[4 * Lcap + j]; d.p = V[5 * Lcap + j]; d.speed = V[6 * Lcap + j]; d.rinv = V[7 * Lcap + j];
        return d;
    }
    __device__ __forceinline__ static void edge(const float *V, int Lcap, int a, int b,
                                                const float *__restrict__ payload, int64_t e, float *Phi, int Scap,
                                                int i) {
        const float nx = __ldg(payload + 3 * e), ny = __ldg(payload + 3 * e + 1), nz = __ldg(payload + 3 * e + 2);
        float phi[5];
        cfd_phi(load(V, a, Lcap), load(V, b, Lcap), nx, ny, nz, phi);
#pragma unroll
        for (int c = 0; c < 5; c++) Phi[c * Scap + i] = phi[c];
    }
    __device__ __forceinline__ static void gather(const float *Phi, int Scap, int i, int side, float acc[5]) {
        const float sgn = side ? -1.0f : 1.0f;
#pragma unroll
        for (int c = 0; c < 5; c++) acc[c] = fmaf(sgn, Phi[c * Scap + i], acc[c]);
    }
    __device__ __forceinline__ static void finish_smem(const float *V, int Lcap, int j, const float acc[5], float dt,
                                                       float *__restrict__ out) {
#pragma unroll
        for (int c = 0; c < 5; c++) out[c] = fmaf(dt, acc[c], V[c * Lcap + j]);
    }
    __device__ __forceinline__ static void finish_row(const float *__restrict__ in, const float acc[5], float dt,
                                                      float *__restrict__ out) {
#pragma unroll
        for (int c = 0; c < 5; c++) out[c] = fmaf(dt, acc[c], in[c]);
    }
    __device__ __forceinline__ static void untouched(const float *__restrict__ in, float *__restrict__ out) {
#pragma unroll
        for (int c = 0; c < 5; c++) out[c] = in[c];
    }
    // naive comparator: one edge straight from global memory, global atomics
    __device__ __forceinline__ static void naive_edge(const float *__restrict__ state, int32_t a, int32_t b,
                                                      const float *__restrict__ payload, int64_t e,
                                                      float *__restrict__ F) {
        const float *ra = state + 5 * (int64_t)a, *rb = state + 5 * (int64_t)b;
        CfdVertex da = cfd_derive(__ldg(ra), __ldg(ra + 1), __ldg(ra + 2), __ldg(ra + 3), __ldg(ra + 4));
        CfdVertex db = cfd_derive(__ldg(rb), __ldg(rb + 1), __ldg(rb + 2), __ldg(rb + 3), __ldg(rb + 4));
        float phi[5];
        cfd_phi(da, db, __ldg(payload + 3 * e), __ldg(payload + 3 * e + 1), __ldg(payload + 3 * e + 2), phi);
#pragma unroll
        for (int c = 0; c < 5; c++) {
            atomicAdd(F + 5 * (int64_t)a + c, phi[c]);
            atomicAdd(F + 5 * (int64_t)b + c, -phi[c]);
        }
    }
    // ---- staged kernels. Per local vertex a 32-byte derived record
    // {rho, m_x, m_y, m_z | E, p, |u|+c, 1/rho} read with two 128-bit shared loads at
    // swizzled float4 slots (rec4()); per edge a 24-byte Phi record of three float2.
    static constexpr int PAYW = 3;
    static constexpr int REC = 8;      // floats per derived record
    static constexpr int PHIREC = 6;   // floats per Phi record (5 used)
    __device__ __forceinline__ static void derive_rec(const float *row, float *recs, int j) {
        const CfdVertex d = cfd_derive(row[0], row[1], row[2], row[3], row[4]);
        float4 *r = reinterpret_cast<float4 *>(recs);
        r[rec4(j, 0)] = make_float4(d.rho, d.mx, d.my, d.mz);
        r[rec4(j, 1)] = make_float4(d.E, d.p, d.speed, d.rinv);
    }
    __device__ __forceinline__ static CfdVertex load_rec(const float *recs, int j) {
        const float4 *r = reinterpret_cast<const float4 *>(recs);
        const float4 x = r[rec4(j, 0)], y = r[rec4(j, 1)];
        CfdVertex d;
        d.rho = x.x; d.mx = x.y; d.my = x.z; d.mz = x.w;
        d.E = y.x; d.p = y.y; d.speed = y.z; d.rinv = y.w;
        return d;
    }
    // the conserved state U of record j
    __device__ __forceinline__ static void rec_state(const float *recs, int j, float U[5]) {
        const float4 *r = reinterpret_cast<const float4 *>(recs);
        const float4 x = r[rec4(j, 0)];
        U[0] = x.x; U[1] = x.y; U[2] = x.z; U[3] = x.w;
        U[4] = r[rec4(j, 1)].x;
    }
    // payload of the edge already in registers
    __device__ __forceinline__ static void edge_rec_pw(const float *recs, int a, int b, const float pw[3], int i,
                                                       float *phis) {
        float phi[5];
        cfd_phi(load_rec(recs, a), load_rec(recs, b), pw[0], pw[1], pw[2], phi);
        float2 *r = reinterpret_cast<float2 *>(phis) + 3 * i;
        r[0] = make_float2(phi[0], phi[1]);
        r[1] = make_float2(phi[2], phi[3]);
        r[2] = make_float2(phi[4], 0.0f);
    }
    __device__ __forceinline__ static void edge_rec(const float *recs, int a, int b, const float *pay, int i,
                                                    float *phis) {
        const float pw[3] = {pay[3 * i], pay[3 * i + 1], pay[3 * i + 2]};
        edge_rec_pw(recs, a, b, pw, i, phis);
    }
    __device__ __forceinline__ static void zero_phi(float *phis, int i) {
        float2 *r = reinterpret_cast<float2 *>(phis) + 3 * i;
        r[0] = r[1] = r[2] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ static void gather_rec(const float *phis, int i, int side, float acc[5]) {
        const float2 *r = reinterpret_cast<const float2 *>(phis) + 3 * i;
        const float2 x = r[0], y = r[1], z = r[2];
        const float sgn = side ? -1.0f : 1.0f;
        acc[0] = fmaf(sgn, x.x, acc[0]); acc[1] = fmaf(sgn, x.y, acc[1]); acc[2] = fmaf(sgn, y.x, acc[2]);
        acc[3] = fmaf(sgn, y.y, acc[3]); acc[4] = fmaf(sgn, z.x, acc[4]);
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[5], float dt) {
#pragma unroll
        for (int c = 0; c < 5; c++) out[c] = fmaf(dt, acc[c], out[c]);
    }
    // ---- occupancy kernel (k_edge_occ). Its derived record folds the flux's constant factors
    // into the per-vertex values, {rho, m_x, m_y, m_z | E, -p/2, -(sigma/2)(|u| + c), -1/(2 rho)},
    // so that with u' = (m.n)(-1/(2 rho)) = -(u.n)/2 and P' = -(p_a + p_b)/2 the face flux is
    //   Phi = f (U_a - U_b) + U_a u'_a + U_b u'_b + (0, P' n, -2 (p'_a u'_a + p'_b u'_b)),
    // f = |n| (s'_a + s'_b) -- the same expression as cfd_phi (the factors -1/2 are exact),
    // evaluated with sm_100's packed fp32x2 FMA/ADD (FFMA2 / FADD2) on component pairs
    // (rho, m_x), (m_y, m_z), (E, p'): ~32 FP instructions per edge instead of ~47.
    // The occupancy kernel stores the record as two halves in separate float4 arrays, A = recs
    // and B = recsB (both indexed by j): half h of record j lands in bank group (j mod 8) of its
    // array, so the placement's in-group positions still decide the bank groups (the rec4
    // swizzle is not needed) and both loads of an endpoint share one offset register.
    __device__ __forceinline__ static void derive_occ(const float *row, float *recs, int j, float *recsB) {
        const float rho = row[0], mx = row[1], my = row[2], mz = row[3], E = row[4];
        const float rinv = rcp_ftz(rho);
        const float ux = mx * rinv, uy = my * rinv, uz = mz * rinv;
        const float uu = ux * ux + uy * uy + uz * uz;
        const float p = (kGamma - 1.0f) * (E - 0.5f * rho * uu);
        const float speed = sqrt_nb(uu) + sqrt_nb(kGamma * p * rinv);
        float4 *r = reinterpret_cast<float4 *>(recs);
        r[j] = make_float4(rho, mx, my, mz);
        reinterpret_cast<float4 *>(recsB)[j] = make_float4(E, -0.5f * p, -(kSigma * 0.5f) * speed, -0.5f * rinv);
    }
    // the conserved state of record j; its last component (E) is the caller's register copy of
    // the staged row (a 32-bit load from the 16-byte-strided B array would conflict 4-way)
    __device__ __forceinline__ static void rec_state_occ(const float *recs, int j, float U[5], float last) {
        const float4 x = reinterpret_cast<const float4 *>(recs)[j];
        U[0] = x.x; U[1] = x.y; U[2] = x.z; U[3] = x.w;
        U[4] = last;
    }
    // split Phi layout of the occupancy kernel: a float4 array (Phi_0..3) and a float array
    // (Phi_4) at phisB -- 20 B per edge, conflict-free stores and
    // one 128-bit + one 32-bit shared load per incidence entry instead of three 64-bit
    static constexpr int PHIBYTES = 20;
    __device__ __forceinline__ static void edge_split(const float *recs, int a, int b, const float pw[3], int i,
                                                      float *phis, float *phisB, const float *recsB) {
        const float4 *r = reinterpret_cast<const float4 *>(recs), *rb = reinterpret_cast<const float4 *>(recsB);
        const float4 xa = r[a], ya = rb[a], xb = r[b], yb = rb[b];
        const float nx = pw[0], ny = pw[1], nz = pw[2];
        const float nlen = sqrt_nb(nx * nx + ny * ny + nz * nz);
        const float f = nlen * (ya.z + yb.z);
        const float ua = (xa.y * nx + xa.z * ny + xa.w * nz) * ya.w;    // -(u_a . n) / 2
        const float ub = (xb.y * nx + xb.z * ny + xb.w * nz) * yb.w;
        const float P = ya.y + yb.y;                                    // -(p_a + p_b) / 2
        const float2 A01 = make_float2(xa.x, xa.y), A23 = make_float2(xa.z, xa.w);
        const float2 B01 = make_float2(xb.x, xb.y), B23 = make_float2(xb.z, xb.w);
        const float2 A4 = make_float2(ya.x, ya.y), B4 = make_float2(yb.x, yb.y);
        const float2 U2a = make_float2(ua, ua), U2b = make_float2(ub, ub), F2 = make_float2(f, f);
        float2 c01 = __ffma2_rn(B01, U2b, __ffma2_rn(A01, U2a, make_float2(0.0f, P * nx)));
        float2 c23 = __ffma2_rn(B23, U2b, __ffma2_rn(A23, U2a, __fmul2_rn(make_float2(ny, nz), make_float2(P, P))));
        const float2 e = __ffma2_rn(A4, U2a, __fmul2_rn(B4, U2b));     // (E_a u'_a + E_b u'_b, p'_a u'_a + p'_b u'_b)
        const float2 p01 = __ffma2_rn(F2, __fadd2_rn(A01, make_float2(-B01.x, -B01.y)), c01);
        const float2 p23 = __ffma2_rn(F2, __fadd2_rn(A23, make_float2(-B23.x, -B23.y)), c23);
        const float p4 = fmaf(f, ya.x - yb.x, fmaf(-2.0f, e.y, e.x));
        reinterpret_cast<float4 *>(phis)[i] = make_float4(p01.x, p01.y, p23.x, p23.y);
        phisB[i] = p4;
    }
    __device__ __forceinline__ static void zero_split(float *phis, int i, float *phisB) {
        reinterpret_cast<float4 *>(phis)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        phisB[i] = 0.f;
    }
    __device__ __forceinline__ static void gather_split(const float *phis, int i, int side, float acc[5],
                                                        const float *phisB) {
        const float4 x = reinterpret_cast<const float4 *>(phis)[i];
        const float y = phisB[i];
        const float sgn = side ? -1.0f : 1.0f;
        const float2 S2 = make_float2(sgn, sgn);
        const float2 a01 = __ffma2_rn(S2, make_float2(x.x, x.y), make_float2(acc[0], acc[1]));
        const float2 a23 = __ffma2_rn(S2, make_float2(x.z, x.w), make_float2(acc[2], acc[3]));
        acc[0] = a01.x; acc[1] = a01.y; acc[2] = a23.x; acc[3] = a23.y;
        acc[4] = fmaf(sgn, y, acc[4]);
    }
    // U + dt F for a staged (owned) vertex
    __device__ __forceinline__ static void finish_occ(const float U[5], const float acc[5], float dt, float out[5]) {
        const float2 D2 = make_float2(dt, dt);
        const float2 o01 = __ffma2_rn(D2, make_float2(acc[0], acc[1]), make_float2(U[0], U[1]));
        const float2 o23 = __ffma2_rn(D2, make_float2(acc[2], acc[3]), make_float2(U[2], U[3]));
        out[0] = o01.x; out[1] = o01.y; out[2] = o23.x; out[3] = o23.y;
        out[4] = fmaf(dt, acc[4], U[4]);
    }
    static constexpr bool kUsesConst = true;
};

// y_a += w x_b, y_b += w x_a  (config C4, gather-scatter over an undirected graph)
struct GatherScatter {
    static constexpr int ROW = 1, NV = 1, NPHI = 2;
    __device__ __forceinline__ static void stage(const float *__restrict__ row, float *V, int j, int) { V[j] = row[0]; }
    __device__ __forceinline__ static void edge(const float *V, int, int a, int b, const float *__restrict__ payload,
                                                int64_t e, float *Phi, int Scap, int i) {
        const float w = payload ? __ldg(payload + e) : 1.0f;
        Phi[i] = w * V[b];
        Phi[Scap + i] = w * V[a];
    }
    __device__ __forceinline__ static void gather(const float *Phi, int Scap, int i, int side, float acc[1]) {
        acc[0] += Phi[side * Scap + i];
    }
    __device__ __forceinline__ static void finish_smem(const float *, int, int, const float acc[1], float,
                                                       float *__restrict__ out) { out[0] = acc[0]; }
    __device__ __forceinline__ static void finish_row(const float *__restrict__, const float acc[1], float,
                                                      float *__restrict__ out) { out[0] = acc[0]; }
    __device__ __forceinline__ static void untouched(const float *__restrict__, float *__restrict__ out) { out[0] = 0.0f; }
    __device__ __forceinline__ static void naive_edge(const float *__restrict__ x, int32_t a, int32_t b,
                                                      const float *__restrict__ payload, int64_t e,
                                                      float *__restrict__ F) {
        const float w = payload ? __ldg(payload + e) : 1.0f;
        atomicAdd(F + a, w * __ldg(x + b));
        atomicAdd(F + b, w * __ldg(x + a));
    }
    static constexpr int PAYW = 1;
    static constexpr int REC = 1, PHIREC = 2;
    __device__ __forceinline__ static void derive_rec(const float *row, float *recs, int j) { recs[j] = row[0]; }
    __device__ __forceinline__ static void rec_state(const float *recs, int j, float U[1]) { U[0] = recs[j]; }
    // pw[0] is the weight (1 when the run has no payload)
    __device__ __forceinline__ static void edge_rec_pw(const float *recs, int a, int b, const float pw[1], int i,
                                                       float *phis) {
        reinterpret_cast<float2 *>(phis)[i] = make_float2(pw[0] * recs[b], pw[0] * recs[a]);
    }
    __device__ __forceinline__ static void edge_rec(const float *recs, int a, int b, const float *pay, int i,
                                                    float *phis) {
        const float pw[1] = {pay ? pay[i] : 1.0f};
        edge_rec_pw(recs, a, b, pw, i, phis);
    }
    __device__ __forceinline__ static void zero_phi(float *phis, int i) {
        reinterpret_cast<float2 *>(phis)[i] = make_float2(0.f, 0.f);
    }
    __device__ __forceinline__ static void gather_rec(const float *phis, int i, int side, float acc[1]) {
        acc[0] += phis[2 * i + side];
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[1], float) {
        out[0] += acc[0];
    }
    static constexpr int PHIBYTES = 8;   // same layout as the records above (stride unused)
    __device__ __forceinline__ static void edge_split(const float *recs, int a, int b, const float pw[1], int i,
                                                      float *phis, float *, const float *) { edge_rec_pw(recs, a, b, pw, i, phis); }
    __device__ __forceinline__ static void zero_split(float *phis, int i, float *) { zero_phi(phis, i); }
    __device__ __forceinline__ static void gather_split(const float *phis, int i, int side, float acc[1], const float *) {
        gather_rec(phis, i, side, acc);
    }
    // occupancy-kernel hooks (same record as derive_rec)
    __device__ __forceinline__ static void derive_occ(const float *row, float *recs, int j, float *) { derive_rec(row, recs, j); }
    __device__ __forceinline__ static void rec_state_occ(const float *, int, float U[1], float last) { U[0] = last; }
    __device__ __forceinline__ static void finish_occ(const float U[1], const float acc[1], float dt, float out[1]) {
        finish_row(U, acc, dt, out);
    }
    static constexpr bool kUsesConst = false;
};

// y_i += A[i,j] x_j on the bipartite graph, edge = (column vertex j, row vertex i)  (C5)
struct Spmv {
    static constexpr int ROW = 1, NV = 1, NPHI = 1;
    __device__ __forceinline__ static void stage(const float *__restrict__ row, float *V, int j, int) { V[j] = row[0]; }
    __device__ __forceinline__ static void edge(const float *V, int, int a, int, const float *__restrict__ payload,
                                                int64_t e, float *Phi, int, int i) {
        Phi[i] = __ldg(payload + e) * V[a];
    }
    __device__ __forceinline__ static void gather(const float *Phi, int, int i, int side, float acc[1]) {
        if (side) acc[0] += Phi[i];
    }
    __device__ __forceinline__ static void finish_smem(const float *, int, int, const float acc[1], float,
                                                       float *__restrict__ out) { out[0] = acc[0]; }
    __device__ __forceinline__ static void finish_row(const float *__restrict__, const float acc[1], float,
                                                      float *__restrict__ out) { out[0] = acc[0]; }
    __device__ __forceinline__ static void untouched(const float *__restrict__, float *__restrict__ out) { out[0] = 0.0f; }
    __device__ __forceinline__ static void naive_edge(const float *__restrict__ x, int32_t a, int32_t b,
                                                      const float *__restrict__ payload, int64_t e,
                                                      float *__restrict__ F) {
        atomicAdd(F + b, __ldg(payload + e) * __ldg(x + a));
    }
    static constexpr int PAYW = 1;
    static constexpr int REC = 1, PHIREC = 1;
    __device__ __forceinline__ static void derive_rec(const float *row, float *recs, int j) { recs[j] = row[0]; }
    __device__ __forceinline__ static void rec_state(const float *recs, int j, float U[1]) { U[0] = recs[j]; }
    __device__ __forceinline__ static void edge_rec_pw(const float *recs, int a, int, const float pw[1], int i,
                                                       float *phis) {
        phis[i] = pw[0] * recs[a];
    }
    __device__ __forceinline__ static void edge_rec(const float *recs, int a, int b, const float *pay, int i,
                                                    float *phis) {
        const float pw[1] = {pay[i]};
        edge_rec_pw(recs, a, b, pw, i, phis);
    }
    __device__ __forceinline__ static void zero_phi(float *phis, int i) { phis[i] = 0.0f; }
    __device__ __forceinline__ static void gather_rec(const float *phis, int i, int side, float acc[1]) {
        if (side) acc[0] += phis[i];
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[1], float) {
        out[0] += acc[0];
    }
    static constexpr int PHIBYTES = 4;
    __device__ __forceinline__ static void edge_split(const float *recs, int a, int b, const float pw[1], int i,
                                                      float *phis, float *, const float *) { edge_rec_pw(recs, a, b, pw, i, phis); }
    __device__ __forceinline__ static void zero_split(float *phis, int i, float *) { zero_phi(phis, i); }
    __device__ __forceinline__ static void gather_split(const float *phis, int i, int side, float acc[1], const float *) {
        gather_rec(phis, i, side, acc);
    }
    // occupancy-kernel hooks (same record as derive_rec)
    __device__ __forceinline__ static void derive_occ(const float *row, float *recs, int j, float *) { derive_rec(row, recs, j); }
    __device__ __forceinline__ static void rec_state_occ(const float *, int, float U[1], float last) { U[0] = last; }
    __device__ __forceinline__ static void finish_occ(const float U[1], const float acc[1], float dt, float out[1]) {
        finish_row(U, acc, dt, out);
    }
    static constexpr bool kUsesConst = false;
};

}  // namespace epg
