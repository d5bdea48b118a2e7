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

// Staged per-vertex quantities of the cfd functor (8 floats; SoA in shared memory).
struct CfdVertex {
    float rho, mx, my, mz, E, p, speed, rinv;  // speed = |u| + c, rinv = 1 / rho
};

__device__ __forceinline__ CfdVertex cfd_derive(float rho, float mx, float my, float mz, float E) {
    CfdVertex d;
    d.rho = rho; d.mx = mx; d.my = my; d.mz = mz; d.E = E;
    d.rinv = 1.0f / rho;
    const float ux = mx * d.rinv, uy = my * d.rinv, uz = mz * d.rinv;
    const float uu = ux * ux + uy * uy + uz * uz;
    d.p = (kGamma - 1.0f) * (E - 0.5f * rho * uu);
    d.speed = sqrtf(uu) + sqrtf(kGamma * d.p * d.rinv);
    return d;
}

// Phi[0..4] for edge (a, b) with normal n out of a.
__device__ __forceinline__ void cfd_phi(const CfdVertex &a, const CfdVertex &b, float nx, float ny, float nz,
                                        float phi[5]) {
    const float nlen = sqrtf(nx * nx + ny * ny + nz * nz);
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
    // ---- pipelined (TMA-staged) kernel: rows are the staged AoS state rows, one derived
    // float per local vertex (|u| + c); rinv and p are recomputed per endpoint.
    static constexpr int PAYW = 3;
    static constexpr bool kDerived = true;
    __device__ __forceinline__ static float derive(const float *row) {
        return cfd_derive(row[0], row[1], row[2], row[3], row[4]).speed;
    }
    __device__ __forceinline__ static CfdVertex load_row(const float *rows, int j, float speed) {
        const float *r = rows + 5 * j;
        CfdVertex d;
        d.rho = r[0]; d.mx = r[1]; d.my = r[2]; d.mz = r[3]; d.E = r[4];
        d.rinv = 1.0f / d.rho;
        const float ux = d.mx * d.rinv, uy = d.my * d.rinv, uz = d.mz * d.rinv;
        d.p = (kGamma - 1.0f) * (d.E - 0.5f * d.rho * (ux * ux + uy * uy + uz * uz));
        d.speed = speed;
        return d;
    }
    __device__ __forceinline__ static void edge2(const float *rows, const float *spd, int a, int b,
                                                 const float *pay, int i, float *Phi, int Scap) {
        float phi[5];
        cfd_phi(load_row(rows, a, spd[a]), load_row(rows, b, spd[b]), pay[3 * i], pay[3 * i + 1], pay[3 * i + 2],
                phi);
#pragma unroll
        for (int c = 0; c < 5; c++) Phi[c * Scap + i] = phi[c];
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[5], float dt) {
#pragma unroll
        for (int c = 0; c < 5; c++) out[c] = fmaf(dt, acc[c], out[c]);
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
    static constexpr bool kDerived = false;
    __device__ __forceinline__ static float derive(const float *) { return 0.0f; }
    __device__ __forceinline__ static void edge2(const float *rows, const float *, int a, int b, const float *pay,
                                                 int i, float *Phi, int Scap) {
        const float w = pay ? pay[i] : 1.0f;
        Phi[i] = w * rows[b];
        Phi[Scap + i] = w * rows[a];
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[1], float) {
        out[0] += acc[0];
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
    static constexpr bool kDerived = false;
    __device__ __forceinline__ static float derive(const float *) { return 0.0f; }
    __device__ __forceinline__ static void edge2(const float *rows, const float *, int a, int, const float *pay,
                                                 int i, float *Phi, int) {
        Phi[i] = pay[i] * rows[a];
    }
    __device__ __forceinline__ static void finalise_add(float *__restrict__ out, const float acc[1], float) {
        out[0] += acc[0];
    }
    static constexpr bool kUsesConst = false;
};

}  // namespace epg
