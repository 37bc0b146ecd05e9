// fused2d.cuh -- the nested-parallel ("patch-wise") flavour for 2D patches:
// one warp owns G = 32*C/p patches at a time, each lane owns C adjacent
// interior columns of one patch.  The default launch (pencil.cu) is C = 1,
// one warp per CTA, 12 CTAs per SM; C = 2 is a measured-slower variant.
//
// Reference realisation: run_patchwise (pkg/src/patchbench/executors.py:390-445)
// runs every step of a patch inside one parallel region over the union range
// [-1,p]^d with masks.  Here the whole step chain of a patch (copy, flux_x,
// flux_y, lambda_x, lambda_y, acc_x, acc_y, reduce) is fused into one pass of
// a column "pencil" walk along y; no scratch ever touches HBM:
//
//   * memory: each warp streams its patch rows (and, one group ahead, the
//     halo columns of its next patch group) through a RING-slot shared-memory
//     ring with cp.async, RING-1 rows ahead of the compute, across group
//     boundaries -- loads never stall the FP64 work and cost no registers;
//   * y-direction: lane j walks rows Y = -1..P, keeping, per column, the
//     previous row's state, y-flux, y-wave-speed, x-updated value and lower
//     y-face in registers (two alternating Row sets), so every y-face is
//     computed exactly once;
//   * x-direction: faces between a lane's own columns are computed in
//     registers; the face right of its last column uses the next lane's
//     state (ring) and x-flux / wave speed (shuffles) and is handed to that
//     lane through a per-warp shared-memory exchange row, so every interior
//     x-face is computed once;
//     the two x-boundary faces of each row (halo column -1 | 0 and
//     P-1 | halo P) are computed up front in "phase H" (lane j takes rows
//     C*j..C*j+C-1) and parked in shared memory;
//   * update order is the reference's: Q + s*dX first (axis 0), then + s*dY;
//   * reduce: max_n lambda_n(Q_new) of every finished cell, shuffle max,
//     one 64-bit atomicMax per warp per launch.  Without per-patch maxima
//     the reduction is filtered (common.cuh LamFilter, Euler::lambda_below):
//     a warp evaluates the eigenvalues of a finished row only if some lane's
//     cell may exceed the warp's running maximum -- a few rows per warp.
//   Lanes of a partly filled warp (32 % (p/C) != 0, or the batch's last
//   group) run on a stand-in patch and never store, vote for a redo or feed
//   the reduction.
//
// Arithmetic: the group is first computed with R = XReal (CUDA's fp64
// division / sqrt fast paths written out, reciprocal of rho shared) on
// states the domain policy certifies with fast_path_safe(); if any lane of
// the warp met an uncertified state, the whole group is recomputed with
// R = double (plain IEEE, direct loads) and the stores are overwritten.
// Either way every value is the reference's expression on the reference's
// operands, so output and eigenvalue are bit-identical to run_sequential
// (tests/test_gpu_parity.py).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "physics.cuh"

namespace fvb {

namespace pencil {

template <int N>
struct Cell {
    double q[N];    // state
    double fy[N];   // y-flux
    double ly;      // y-wave speed
    double acc[N];  // Q + s*dX (x-updated value)
    double gy[N];   // lower y-face G_{Y-1/2}
};

template <int C, int N>
struct Row {
    Cell<N> c[C];
};

// With R = XReal the state must satisfy the domain's fast-path precondition;
// a violation marks the warp's group for the IEEE redo.
template <class R, class Eq, int N>
__device__ __forceinline__ void certify(const Eq& eq, const R (&s)[N], bool& bad) {
    if constexpr (std::is_same<R, XReal>::value) bad |= !eq.fast_path_safe(s);
}

// Evaluate the microkernels of one state with scalar type R.
template <class R, bool X, bool Y, class Eq, int N>
__device__ __forceinline__ void eval(const Eq& eq, const double (&q)[N], double (&fx)[N],
                                     double& lx, double (&fy)[N], double& ly, bool& bad) {
    R s[N];
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
    certify(eq, s, bad);
    if (X) {
        R f[N];
        eq.flux(s, 0, f);
        const R l = eq.max_eigenvalue(s, 0);
#pragma unroll
        for (int k = 0; k < N; ++k) fx[k] = val(f[k]);
        lx = val(l);
    }
    if (Y) {
        R f[N];
        eq.flux(s, 1, f);
        const R l = eq.max_eigenvalue(s, 1);
#pragma unroll
        for (int k = 0; k < N; ++k) fy[k] = val(f[k]);
        ly = val(l);
    }
}

template <class R, class Eq, int N>
__device__ __forceinline__ double cell_lambda(const Eq& eq, const double (&q)[N], bool& bad) {
    R s[N];
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
    certify(eq, s, bad);
    const R a = eq.max_eigenvalue(s, 0);
    const R b = eq.max_eigenvalue(s, 1);
    return py_max(val(a), val(b));
}

// ---- cp.async (LDGSTS) helpers ---------------------------------------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const double* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// ---- geometry and per-warp shared memory ------------------------------------
template <int P, int C>
struct Geo {
    static_assert(P % C == 0, "columns per lane must divide p");
    static constexpr int L = P / C;                // lanes per patch
    static constexpr int G = 32 / L;               // patches per warp
    static constexpr bool FULL = (G * L == 32);    // every lane used
    // boundary-face row: patch s uses [s*(P+1), s*(P+1)+P); unused lanes get slot G
    static constexpr int BND = (FULL ? G : G + 1) * (P + 1);
    // face exchange row: [0,32) the right face of each lane's last column,
    // [32, 32+BND) left boundary faces, [32+BND, 32+2*BND) right boundary faces
    static constexpr int XL = 32, XR = 32 + BND, XS = 32 + 2 * BND;
    // shared-memory rows padded to 128 B so a warp's 256 B row access is two wavefronts
    static constexpr int XSP = (XS + 15) / 16 * 16;
    static constexpr int RW = 48;  // ring row: 32 lanes + the right neighbour of lane 31, padded
};

template <int P, int C, int RING, int N>
struct alignas(128) WarpSmem {
    using Gm = Geo<P, C>;
    double ring[RING][N][C][Gm::RW];  // streamed rows, [k][column c of the lane][lane (+ pad)]
    double hq[4 * N * C][32];         // halo-column states of the group: C rows x N x 4 cells
    double xf[N][Gm::XSP];            // x-face exchange + boundary faces (see Geo)
};

// Per-warp context of one patch group.  LS: distance between the cells of
// a row in the batch arrays (1: SoA / AoSoA, N: AoS).
template <int P, int C, int RING, int LS, int N>
struct Ctx {
    const double* __restrict__ qi;  // this lane's patch, haloed input
    double* __restrict__ qo;        // this lane's patch, output
    mutable double* orow;           // this lane's first output cell of the next row to finish
    long long sIn, sOut;            // unknown strides of the batch arrays
    double scale, hscale;           // dt/h and 0.5*dt/h (folded faces)
    int j, lane, hbase;             // lane within patch, lane, smem index of the patch's row 0
    bool valid;
    bool out16;                     // AoS output cells by 16-byte unknown pairs (aligned batch)
    WarpSmem<P, C, RING, N>* sm;       // ring / halo columns (cp.async source)
    double (*xf)[Geo<P, C>::XSP];      // x-face exchange row + boundary faces
};

// ---- row sources -------------------------------------------------------------
// RingSrc: rows of the current group come from the smem ring; begin(r) keeps
// the prefetch RING-1 rows ahead (continuing into the next group, whose halo
// columns ride along with its first row).  DirectSrc: plain loads (the IEEE
// redo path, which must not disturb the ring).
// Per-warp prefetch state that persists across patch groups.
struct Stream {
    int cur;             // ring slot of the current row
    const double* pf;    // this lane's first column of the next row to prefetch (unknown 0)
    int pf_left;         // rows of the current group still to prefetch
};

// V16 (AoS batches, even N, 16-byte aligned): a cell's unknowns are
// contiguous, so each lane moves them in 16-byte pairs (cp.async 16, half the
// copies) and the ring / halo slots hold [unknown pair][column][lane] of
// double2 (128-bit shared loads, conflict-free across a quarter-warp).
template <int P, int C, int RING, int LS, int N, bool V16 = false>
struct RingSrc {
    static constexpr int D = RING - 1;  // prefetch distance in rows
    static constexpr int ROWS = P + 2;  // rows per group: Y = -1..P
    static constexpr int RW = Geo<P, C>::RW;
    static_assert(!V16 || (LS == N && N % 2 == 0), "16-byte copies need AoS cells of an even unknown count");
    using Cx = Ctx<P, C, RING, LS, N>;
    const Cx& c;
    const double* next_qi;  // next group's patch (this lane), or null
    Stream& st;

    __device__ __forceinline__ static double2 (*ring2(const Cx& c, int slot))[C][RW] {
        return reinterpret_cast<double2(*)[C][RW]>(&c.sm->ring[slot][0][0][0]);
    }
    __device__ __forceinline__ static double2 (*hq2(const Cx& c))[32] {
        return reinterpret_cast<double2(*)[32]>(&c.sm->hq[0][0]);
    }
    __device__ __forceinline__ static void issue_row(const Cx& c, const double* p, int slot) {
        if constexpr (V16) {
#pragma unroll
            for (int kp = 0; kp < N / 2; ++kp)
#pragma unroll
                for (int cc = 0; cc < C; ++cc) cp_async16(&ring2(c, slot)[kp][cc][c.lane], p + 2 * kp + cc * LS);
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k, p += c.sIn)
#pragma unroll
                for (int cc = 0; cc < C; ++cc) cp_async8(&c.sm->ring[slot][k][cc][c.lane], p + cc * LS);
        }
    }
    __device__ __forceinline__ static void issue_halo(const Cx& c, const double* qi) {
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            const double* row = qi + (C * c.j + cc + 1) * (P + 2) * LS;
            if constexpr (V16) {
#pragma unroll
                for (int kp = 0; kp < N / 2; ++kp) {
                    double2(*h)[32] = &hq2(c)[4 * (N / 2) * cc + 4 * kp];
                    cp_async16(&h[0][c.lane], row + 2 * kp);
                    cp_async16(&h[1][c.lane], row + LS + 2 * kp);
                    cp_async16(&h[2][c.lane], row + P * LS + 2 * kp);
                    cp_async16(&h[3][c.lane], row + (P + 1) * LS + 2 * kp);
                }
            } else {
#pragma unroll
                for (int k = 0; k < N; ++k, row += c.sIn) {
                    double* h = &c.sm->hq[4 * N * cc + 4 * k][c.lane];
                    cp_async8(h, row);
                    cp_async8(h + 32, row + LS);
                    cp_async8(h + 64, row + P * LS);
                    cp_async8(h + 96, row + (P + 1) * LS);
                }
            }
        }
    }
    // Prologue for the first group of a warp: halo + rows 0..D-1 into slots
    // 0..D-1, one commit group each.
    __device__ __forceinline__ static Stream prologue(const Cx& c) {
        Stream s;
        issue_halo(c, c.qi);
        s.pf = c.qi + (C * c.j + 1) * LS;
#pragma unroll
        for (int r = 0; r < D; ++r, s.pf += (P + 2) * LS) {
            issue_row(c, s.pf, r);
            cp_commit();
        }
        s.pf_left = ROWS - D;
        s.cur = RING - 1;
        return s;
    }
    __device__ __forceinline__ void halo(int cc, double (&q0)[N], double (&q1)[N], double (&q2)[N],
                                         double (&q3)[N]) const {
        if (cc == 0) {
            cp_wait<D - 1>();  // the oldest pending group holds the halo + row 0
            __syncwarp();
        }
        if constexpr (V16) {
#pragma unroll
            for (int kp = 0; kp < N / 2; ++kp) {
                const double2(*h)[32] = &hq2(c)[4 * (N / 2) * cc + 4 * kp];
                const double2 a = h[0][c.lane], b = h[1][c.lane], d = h[2][c.lane], e = h[3][c.lane];
                q0[2 * kp] = a.x, q0[2 * kp + 1] = a.y;
                q1[2 * kp] = b.x, q1[2 * kp + 1] = b.y;
                q2[2 * kp] = d.x, q2[2 * kp + 1] = d.y;
                q3[2 * kp] = e.x, q3[2 * kp + 1] = e.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double* h = &c.sm->hq[4 * N * cc + 4 * k][c.lane];
                q0[k] = h[0];
                q1[k] = h[32];
                q2[k] = h[64];
                q3[k] = h[96];
            }
        }
    }
    // Advance to the next row and prefetch the stream row D ahead into the
    // slot of the row just finished (RING = D + 1).
    __device__ __forceinline__ void begin(int) const {
        __syncwarp();  // every lane is done with the slot about to be refilled
        if (st.pf_left > 0) {
            issue_row(c, st.pf, st.cur);
            st.pf += (P + 2) * LS;
            --st.pf_left;
        } else if (next_qi != nullptr) {  // first row of the next group, with its halo columns
            issue_halo(c, next_qi);
            st.pf = next_qi + (C * c.j + 1) * LS;
            issue_row(c, st.pf, st.cur);
            st.pf += (P + 2) * LS;
            st.pf_left = ROWS - 1;
        }
        cp_commit();
        cp_wait<D>();
        __syncwarp();
        if constexpr ((RING & (RING - 1)) == 0) {
            st.cur = (st.cur + 1) & (RING - 1);
        } else {
            st.cur = (st.cur + 1 == RING) ? 0 : st.cur + 1;
        }
    }
    __device__ __forceinline__ void row(int, double (&q)[C][N]) const {
        if constexpr (V16) {
#pragma unroll
            for (int kp = 0; kp < N / 2; ++kp)
#pragma unroll
                for (int cc = 0; cc < C; ++cc) {
                    const double2 v = ring2(c, st.cur)[kp][cc][c.lane];
                    q[cc][2 * kp] = v.x, q[cc][2 * kp + 1] = v.y;
                }
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k)
#pragma unroll
                for (int cc = 0; cc < C; ++cc) q[cc][k] = c.sm->ring[st.cur][k][cc][c.lane];
        }
    }
    __device__ __forceinline__ void right(int, double (&q)[N]) const {  // first column of lane+1
        if constexpr (V16) {
#pragma unroll
            for (int kp = 0; kp < N / 2; ++kp) {
                const double2 v = ring2(c, st.cur)[kp][0][c.lane + 1];
                q[2 * kp] = v.x, q[2 * kp + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k) q[k] = c.sm->ring[st.cur][k][0][c.lane + 1];
        }
    }
};

template <int P, int C, int RING, int LS, int N>
struct DirectSrc {
    const Ctx<P, C, RING, LS, N>& c;
    __device__ __forceinline__ void halo(int cc, double (&q0)[N], double (&q1)[N], double (&q2)[N],
                                         double (&q3)[N]) const {
        const double* row = c.qi + (C * c.j + cc + 1) * (P + 2) * LS;
#pragma unroll
        for (int k = 0; k < N; ++k, row += c.sIn) {
            q0[k] = __ldg(row);
            q1[k] = __ldg(row + LS);
            q2[k] = __ldg(row + P * LS);
            q3[k] = __ldg(row + (P + 1) * LS);
        }
    }
    __device__ __forceinline__ void begin(int) const {}
    __device__ __forceinline__ void row(int r, double (&q)[C][N]) const {
        const double* p = c.qi + (r * (P + 2) + C * c.j + 1) * LS;
#pragma unroll
        for (int k = 0; k < N; ++k, p += c.sIn)
#pragma unroll
            for (int cc = 0; cc < C; ++cc) q[cc][k] = __ldg(p + cc * LS);
    }
    __device__ __forceinline__ void right(int r, double (&q)[N]) const {
        const double* p = c.qi + (r * (P + 2) + C * c.j + C + 1) * LS;
#pragma unroll
        for (int k = 0; k < N; ++k, p += c.sIn) q[k] = __ldg(p);
    }
};

// Faces and updates.  With R = double they are the reference's expressions
// (rusanov_face / rusanov_update, common.cuh).  With R = XReal (certified
// states, see Euler::fast_path_safe) the face is kept doubled,
//     H = (F_L + F_R) - w*(Q_R - Q_L)  = 2*G exactly,
// and the update uses 0.5*dt/h:  acc + (0.5*s)*(H_l - H_r)  is bit-identical to
// acc + s*(G_l - G_r) because every scaling by 2 or 1/2 involved is exact:
// certified states make all fluxes, states, wave speeds and their sums,
// differences and products zero or at least 2^-969 in magnitude (and far
// below 2^1023), and s = dt/h is range-checked on the host (StepArgs::fast).
// Saves the five multiplications by 0.5 of every face.
template <class R>
constexpr bool kFold = std::is_same<R, XReal>::value;

template <class R, int N>
__device__ __forceinline__ void face(const double (&qL)[N], const double (&qR)[N],
                                     const double (&fL)[N], const double (&fR)[N], double lamL,
                                     double lamR, double (&g)[N]) {
    if constexpr (kFold<R>) {
        const double w = py_max(lamL, lamR);
#pragma unroll
        for (int k = 0; k < N; ++k) g[k] = (fL[k] + fR[k]) - w * (qR[k] - qL[k]);
    } else {
        rusanov_face(qL, qR, fL, fR, lamL, lamR, g);
    }
}

template <class R, int P, int C, int RING, int LS, int N>
__device__ __forceinline__ void update(const Ctx<P, C, RING, LS, N>& c, double (&acc)[N],
                                       const double (&gl)[N], const double (&gr)[N]) {
    rusanov_update(acc, gl, gr, kFold<R> ? c.hscale : c.scale);
}

// x-faces of row Y (stream row r = Y+1) and the axis-0 update of this lane's cells.
// The face right of a lane's last column goes through the warp's xf exchange
// row; lane 0 of a patch reads its left face, lane L-1 its right face, from
// the boundary faces phase H parked there (index selects, no data selects).
template <class R, int P, int C, int RING, int LS, int N, class Src>
__device__ __forceinline__ void x_update(const Ctx<P, C, RING, LS, N>& c, const Src& src, int Y,
                                         const double (&q)[C][N], const double (&fx)[C][N],
                                         const double (&lx)[C], Row<C, N>& cur) {
    using Gm = Geo<P, C>;
    double qn[N], fxn[N], gR[N], gL[N];
    src.right(Y + 1, qn);
#pragma unroll
    for (int k = 0; k < N; ++k) fxn[k] = __shfl_down_sync(0xffffffffu, fx[0][k], 1);
    const double lxn = __shfl_down_sync(0xffffffffu, lx[0], 1);
    face<R>(q[C - 1], qn, fx[C - 1], fxn, lx[C - 1], lxn, gR);  // right of the last column
    __syncwarp();  // readers of the previous row's faces are done
#pragma unroll
    for (int k = 0; k < N; ++k) c.xf[k][c.lane] = gR[k];
    __syncwarp();
    const int h = c.hbase + Y;
    const int il = (c.j == 0) ? Gm::XL + h : c.lane - 1;
#pragma unroll
    for (int k = 0; k < N; ++k) gL[k] = c.xf[k][il];
    // the lane's own right face is still in gR; only a patch's last lane
    // replaces it by the boundary face (predicated loads: no data select,
    // and no shared-memory traffic for the other lanes)
    if (c.j == Gm::L - 1) {
#pragma unroll
        for (int k = 0; k < N; ++k) gR[k] = c.xf[k][Gm::XR + h];
    }
    // faces between this lane's own columns, then the updates left to right
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
        double gnext[N];
        if (cc + 1 < C) {
            face<R>(q[cc], q[cc + 1], fx[cc], fx[cc + 1], lx[cc], lx[cc + 1], gnext);
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k) gnext[k] = gR[k];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) cur.c[cc].acc[k] = q[cc][k];
        update<R>(c, cur.c[cc].acc, gL, gnext);
#pragma unroll
        for (int k = 0; k < N; ++k) gL[k] = gnext[k];
    }
}

// Finish row Y-1 (its upper y-faces just became known): store + reduce.
template <int P, int C, int RING, int RED, class R, int LS, class Eq, int N>
__device__ __forceinline__ void finish(const Ctx<P, C, RING, LS, N>& c, const Eq& eq, int Yprev,
                                       const Row<C, N>& prev, const double (&gy)[C][N], double& pred,
                                       LamFilter& lf, bool& bad) {
    double qn[C][N];
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
#pragma unroll
        for (int k = 0; k < N; ++k) qn[cc][k] = prev.c[cc].acc[k];
        update<R>(c, qn[cc], prev.c[cc].gy, gy[cc]);
    }
    // Full warps: a lane without a real patch runs the group's first patch
    // with the same column, sub-group and boundary faces as the lane that
    // owns it, so it stores the same bits to the same addresses -- no branch.
    if (Geo<P, C>::FULL || c.valid) {
        double* o = c.orow;  // == qo + (Yprev * P + C * j) * LS: rows finish in order
        if (LS == N && N % 2 == 0 && c.out16) {  // AoS: a cell's unknowns are contiguous
#pragma unroll
            for (int cc = 0; cc < C; ++cc)
#pragma unroll
                for (int kp = 0; kp < N / 2; ++kp)
                    __stcs(reinterpret_cast<double2*>(o + cc * LS + 2 * kp),
                           make_double2(qn[cc][2 * kp], qn[cc][2 * kp + 1]));
        } else {
#pragma unroll
            for (int k = 0; k < N; ++k, o += c.sOut) {
                if constexpr (C == 2 && LS == 1) {
                    __stcs(reinterpret_cast<double2*>(o), make_double2(qn[0][k], qn[1][k]));
                } else {
#pragma unroll
                    for (int cc = 0; cc < C; ++cc) __stcs(o + cc * LS, qn[cc][k]);
                }
            }
        }
    }
    c.orow += P * LS;
    if constexpr (RED == kReduceAll) {
#pragma unroll
        for (int cc = 0; cc < C; ++cc) running_max(pred, cell_lambda<R>(eq, qn[cc], bad));
    } else if constexpr (RED == kReduceFiltered) {  // warp-converged: every lane gets here
        bool need[C], any = false;
#pragma unroll
        // only lanes holding a real cell of the batch may feed tau (unused lanes of a
        // partly filled warp run on stand-in data)
        for (int cc = 0; cc < C; ++cc)
            any |= need[cc] = c.valid && !eq.lambda_below(qn[cc], lf.tau_lo);
        if (__any_sync(0xffffffffu, any)) {
#pragma unroll
            for (int cc = 0; cc < C; ++cc)
                if (need[cc]) running_max(pred, cell_lambda<R>(eq, qn[cc], bad));
            lf.raise(pred);
        }
    }
}

// Interior row Y >= 1: prev = row Y-1, cur <- row Y.
template <int P, int C, int RING, int RED, class R, class Src, int LS, class Eq, int N>
__device__ __forceinline__ void row_step(const Ctx<P, C, RING, LS, N>& c, const Src& src,
                                         const Eq& eq, int Y, const Row<C, N>& prev,
                                         Row<C, N>& cur, double& pred, LamFilter& lf, bool& bad) {
    src.begin(Y + 1);
    double q[C][N], fx[C][N], lx[C], gy[C][N];
    src.row(Y + 1, q);
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
        eval<R, true, true>(eq, q[cc], fx[cc], lx[cc], cur.c[cc].fy, cur.c[cc].ly, bad);
        face<R>(prev.c[cc].q, q[cc], prev.c[cc].fy, cur.c[cc].fy, prev.c[cc].ly, cur.c[cc].ly,
                gy[cc]);  // face at Y - 1/2
    }
    // the x-update of row Y is independent of finishing row Y-1: issuing it
    // first keeps both chains in one basic block (before the filter's vote)
    x_update<R>(c, src, Y, q, fx, lx, cur);
    finish<P, C, RING, RED, R>(c, eq, Y - 1, prev, gy, pred, lf, bad);
#pragma unroll
    for (int cc = 0; cc < C; ++cc)
#pragma unroll
        for (int k = 0; k < N; ++k) cur.c[cc].gy[k] = gy[cc][k], cur.c[cc].q[k] = q[cc][k];
}

// One patch group: phase H + the walk.  Returns this lane's max eigenvalue.
template <int P, int C, int RING, int RED, class R, class Src, int LS, class Eq, int N>
__device__ __forceinline__ double group(const Ctx<P, C, RING, LS, N>& c, const Src& src,
                                        const Eq& eq, LamFilter& lf, bool& bad) {
    c.orow = c.qo + C * c.j * LS;
    // ---- phase H: x-boundary faces of rows C*j .. C*j+C-1 ------------------
#pragma unroll
    for (int cc = 0; cc < C; ++cc) {
        double q0[N], q1[N], q2[N], q3[N], f0[N], f1[N], f2[N], f3[N], l0, l1, l2, l3, g[N], d[N], dl;
        src.halo(cc, q0, q1, q2, q3);
        eval<R, true, false>(eq, q0, f0, l0, d, dl, bad);
        eval<R, true, false>(eq, q1, f1, l1, d, dl, bad);
        eval<R, true, false>(eq, q2, f2, l2, d, dl, bad);
        eval<R, true, false>(eq, q3, f3, l3, d, dl, bad);
        const int h = c.hbase + C * c.j + cc;
        face<R>(q0, q1, f0, f1, l0, l1, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.xf[k][Geo<P, C>::XL + h] = g[k];
        face<R>(q2, q3, f2, f3, l2, l3, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.xf[k][Geo<P, C>::XR + h] = g[k];
    }
    __syncwarp();

    double pred = 0.0;
    Row<C, N> S0, S1;
    {  // row -1 (halo): y-flux only
        src.begin(0);
        double q[C][N];
        src.row(0, q);
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            double fx[N], lx;
            eval<R, false, true>(eq, q[cc], fx, lx, S0.c[cc].fy, S0.c[cc].ly, bad);
#pragma unroll
            for (int k = 0; k < N; ++k) S0.c[cc].q[k] = q[cc][k];
        }
    }
    {  // row 0: nothing to finish yet
        src.begin(1);
        double q[C][N], fx[C][N], lx[C];
        src.row(1, q);
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            eval<R, true, true>(eq, q[cc], fx[cc], lx[cc], S1.c[cc].fy, S1.c[cc].ly, bad);
            face<R>(S0.c[cc].q, q[cc], S0.c[cc].fy, S1.c[cc].fy, S0.c[cc].ly, S1.c[cc].ly,
                    S1.c[cc].gy);
#pragma unroll
            for (int k = 0; k < N; ++k) S1.c[cc].q[k] = q[cc][k];
        }
        x_update<R>(c, src, 0, q, fx, lx, S1);
    }
    int Y = 1;
#pragma unroll 1
    for (; Y + 1 < P; Y += 2) {  // two rows per trip through alternating Row sets
        row_step<P, C, RING, RED, R>(c, src, eq, Y, S1, S0, pred, lf, bad);
        row_step<P, C, RING, RED, R>(c, src, eq, Y + 1, S0, S1, pred, lf, bad);
    }
    if (Y < P) row_step<P, C, RING, RED, R>(c, src, eq, Y, S1, S0, pred, lf, bad);
    const Row<C, N>& last = (Y < P) ? S0 : S1;
    {  // row P (halo): y-flux, top faces, finish row P-1
        src.begin(P + 1);
        double q[C][N], gy[C][N];
        src.row(P + 1, q);
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            double fx[N], lx, fy[N], ly;
            eval<R, false, true>(eq, q[cc], fx, lx, fy, ly, bad);
            face<R>(last.c[cc].q, q[cc], last.c[cc].fy, fy, last.c[cc].ly, ly, gy[cc]);
        }
        finish<P, C, RING, RED, R>(c, eq, P - 1, last, gy, pred, lf, bad);
    }
    __syncwarp();  // boundary faces are rewritten by the next group
    return pred;
}

}  // namespace pencil

template <int P, int C, int RING, int N>
constexpr size_t pencil_smem_per_warp() {
    return sizeof(pencil::WarpSmem<P, C, RING, N>);
}

template <class Eq, int P, int C, int WARPS, int RED, int MINB, int RING, int LS, bool V16 = false>
__global__ void __launch_bounds__(WARPS * 32, MINB) fused2d_pencil_kernel(StepArgs a) {
    using namespace pencil;
    using Gm = Geo<P, C>;
    constexpr int L = Gm::L;
    constexpr int G = Gm::G;
    constexpr int N = Eq::kUnknowns;
    static_assert(Eq::kDim == 2, "the pencil walk is 2D");
    static_assert(P >= 2 && L <= 32, "pencil kernel covers p/C <= 32");
    static_assert(RING >= 2, "ring needs >= 2 slots");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto* smem = reinterpret_cast<WarpSmem<P, C, RING, N>*>(smem_raw);

    const int lane = threadIdx.x & 31;
    const int warp = WARPS == 1 ? 0 : (int)(threadIdx.x >> 5);  // WARPS == 1: the group loop is provably warp-uniform
    const int sub = lane / L;
    const bool lane_used = sub < G;
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const long long gstep = (long long)gridDim.x * WARPS;

    Ctx<P, C, RING, LS, N> c;
    c.sIn = a.in.k;
    c.sOut = a.out.k;
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);
    c.scale = scale;
    c.hscale = 0.5 * scale;
    c.lane = lane;
    c.j = lane - sub * L;
    c.hbase = sub * (P + 1);  // padded rows; unused lanes (sub == G) get slot G
    c.sm = &smem[warp];
    c.xf = smem[warp].xf;
    c.out16 = V16;  // the host picks V16 only for 16-byte aligned input AND output batches

    auto patch_of = [&](long long g) {
        const long long pt = t0 + g * G + (lane_used ? sub : 0);
        return (lane_used && pt < t1) ? pt : t0 + g * G;  // invalid lanes: a real patch, no stores
    };

    double red = 0.0;
    LamFilter lf;
    lf.init();
    long long g = (long long)blockIdx.x * WARPS + warp;
    Stream stream{};
    if (g < groups) {
        c.qi = in_base(a, patch_of(g));
        stream = RingSrc<P, C, RING, LS, N, V16>::prologue(c);
    }
    for (; g < groups; g += gstep) {
        const long long patch = patch_of(g);
        c.valid = lane_used && (t0 + g * G + sub) < t1;
        c.qi = in_base(a, patch);
        c.qo = out_base(a, patch);
        bool lane_fast = fast;
        if (a.dt_patch != nullptr) {  // local time stepping: this lane's patch's dt
            c.scale = patch_scale(a, scale, patch);
            c.hscale = 0.5 * c.scale;
            lane_fast = step_fast(a, c.scale);
        }
        const double* next_qi = (g + gstep < groups) ? in_base(a, patch_of(g + gstep)) : nullptr;

        bool bad = !lane_fast;  // run parameters outside the folded-face range: IEEE only
        const RingSrc<P, C, RING, LS, N, V16> ring{c, next_qi, stream};
        double pred;
        if constexpr (kHasFastPath<Eq>) {
            const LamFilter lf0 = lf;
            pred = group<P, C, RING, RED, XReal>(c, ring, eq, lf, bad);
            // Uncertified state in a real cell: IEEE redo.  Unused / out-of-range
            // lanes (stand-in patch, unwritten boundary slots) never feed a valid
            // lane, so their flags are ignored.
            if (__any_sync(0xffffffffu, bad && c.valid)) {
                bool unused = false;
                const DirectSrc<P, C, RING, LS, N> direct{c};
                lf = lf0;  // tau may have been raised from flagged states
                pred = group<P, C, RING, RED, double>(c, direct, eq, lf, unused);
            }
        } else {  // a policy without the fast-path hook: IEEE double throughout
            pred = group<P, C, RING, RED, double>(c, ring, eq, lf, bad);
        }

        if (!c.valid) pred = 0.0;
        running_max(red, pred);
        if (RED == kReduceAll && a.lam_patch != nullptr) {  // segmented max over the L lanes of a patch
            double v = pred;
#pragma unroll
            for (int off = 1; off < L; off <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, off);
                if (c.j + off < L) running_max(v, o);
            }
            if (c.valid && c.j == 0) a.lam_patch[patch] = v;
        }
    }
    cp_wait<0>();
    if (RED != kReduceNone && a.lam_bits != nullptr) reduce_epilogue<(WARPS > 1)>(a, red);
}

}  // namespace fvb
