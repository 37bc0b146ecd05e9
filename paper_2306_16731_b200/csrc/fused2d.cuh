// fused2d.cuh -- the nested-parallel ("patch-wise") flavour for 2D patches:
// one warp owns G = 32/P patches at a time, one lane per interior column.
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
//   * y-direction: lane x walks rows Y = -1..P, keeping the previous row's
//     state, y-flux, y-wave-speed, x-updated value and lower y-face in
//     registers (two alternating Row sets), so every y-face is computed once;
//   * x-direction: the x-face between columns x and x+1 uses the neighbour's
//     state (from the ring) and x-flux / wave speed (warp shuffles), and is
//     handed to lane x+1 by one more shuffle, so every interior x-face is
//     computed once; the two x-boundary faces of each row (halo column -1 | 0
//     and P-1 | halo P) are computed up front in "phase H" by lane r for row
//     r and parked in shared memory;
//   * update order is the reference's: Q + s*dX first (axis 0), then + s*dY;
//   * reduce: max_n lambda_n(Q_new) of every finished cell, shuffle max,
//     one 64-bit atomicMax per warp per launch.
//
// Arithmetic: the group is first computed with R = XReal (CUDA's fp64
// division / sqrt fast paths written out, reciprocal of rho shared, no
// branches); if any lane of the warp saw an operand outside the fast paths'
// range, the whole group is recomputed with R = double (plain IEEE, direct
// loads) and the stores are overwritten.  Either way every value is the
// reference's expression on the reference's operands, so output and
// eigenvalue are bit-identical to run_sequential (tests/test_gpu_parity.py).
#pragma once

#include "common.cuh"
#include "euler.cuh"

namespace fvb {

namespace pencil {

constexpr int N = 4;
constexpr int kLanePad = 33;  // ring rows hold lane 32 too, so lane 31 may read "lane+1"

struct Row {
    double q[N];    // state
    double fy[N];   // y-flux
    double ly;      // y-wave speed
    double acc[N];  // Q + s*dX (x-updated value)
    double gy[N];   // lower y-face G_{Y-1/2}
};

// With R = XReal the state must satisfy the domain's fast-path precondition;
// a violation marks the warp's group for the IEEE redo.
template <class R>
__device__ __forceinline__ void certify(const Euler<2>& eq, const R (&s)[N], bool& bad) {
    if constexpr (std::is_same<R, XReal>::value) bad |= !eq.fast_path_safe(s);
}

// Evaluate the microkernels of one state with scalar type R.
template <class R, bool X, bool Y>
__device__ __forceinline__ void eval(const Euler<2>& eq, const double (&q)[N], double (&fx)[N],
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

template <class R>
__device__ __forceinline__ double cell_lambda(const Euler<2>& eq, const double (&q)[N], bool& bad) {
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
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// Per-warp shared memory.
template <int RING>
struct WarpSmem {
    double ring[RING][N][kLanePad];  // streamed rows
    double hq[16][32];               // halo-column states of the group (phase H input)
    double gl[N * 48];               // x-face at -1/2 of each row (by hbase + row)
    double gr[N * 48];               // x-face at P-1/2 of each row
};

// Per-warp context of one patch group.
template <int P, int RING>
struct Ctx {
    const double* __restrict__ qi;  // this lane's patch, haloed input
    double* __restrict__ qo;        // this lane's patch, output
    long long sIn, sOut;            // SoA unknown strides
    double scale;
    int x, lane, hbase;             // column, lane, smem index of this patch's row 0
    bool valid;
    WarpSmem<RING>* sm;
};

// ---- row sources -------------------------------------------------------------
// RingSrc: rows of the current group come from the smem ring; begin(r) keeps
// the prefetch RING-1 rows ahead (continuing into the next group, whose halo
// columns ride along with its first row).  DirectSrc: plain loads (the IEEE
// redo path, which must not disturb the ring).
template <int P, int RING>
struct RingSrc {
    static constexpr int D = RING - 1;  // prefetch distance in rows
    static constexpr int ROWS = P + 2;  // rows per group: Y = -1..P
    const Ctx<P, RING>& c;
    const double* next_qi;              // next group's patch (this lane), or null
    int sbase;                          // stream index of this group's row 0

    __device__ __forceinline__ static void issue_row(const Ctx<P, RING>& c, const double* qi, int Y,
                                                     int slot) {
        const double* p = qi + (Y + 1) * (P + 2) + c.x + 1;
#pragma unroll
        for (int k = 0; k < N; ++k, p += c.sIn) cp_async8(&c.sm->ring[slot][k][c.lane], p);
    }
    __device__ __forceinline__ static void issue_halo(const Ctx<P, RING>& c, const double* qi) {
        const double* row = qi + (c.x + 1) * (P + 2);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            cp_async8(&c.sm->hq[4 * k + 0][c.lane], row + k * c.sIn);
            cp_async8(&c.sm->hq[4 * k + 1][c.lane], row + k * c.sIn + 1);
            cp_async8(&c.sm->hq[4 * k + 2][c.lane], row + k * c.sIn + P);
            cp_async8(&c.sm->hq[4 * k + 3][c.lane], row + k * c.sIn + P + 1);
        }
    }
    // Prologue for the first group of a warp: halo + rows r = 0..D-1, one commit group each.
    __device__ __forceinline__ static void prologue(const Ctx<P, RING>& c, int sbase) {
        issue_halo(c, c.qi);
#pragma unroll
        for (int r = 0; r < D; ++r) {
            issue_row(c, c.qi, r - 1, (sbase + r) % RING);
            cp_commit();
        }
    }
    __device__ __forceinline__ void halo(double (&q0)[N], double (&q1)[N], double (&q2)[N],
                                         double (&q3)[N]) const {
        cp_wait<D - 1>();  // the oldest pending group holds the halo + row 0
        __syncwarp();
#pragma unroll
        for (int k = 0; k < N; ++k) {
            q0[k] = c.sm->hq[4 * k + 0][c.lane];
            q1[k] = c.sm->hq[4 * k + 1][c.lane];
            q2[k] = c.sm->hq[4 * k + 2][c.lane];
            q3[k] = c.sm->hq[4 * k + 3][c.lane];
        }
    }
    // Make row r (Y = r-1) readable and prefetch row r + D of the stream.
    __device__ __forceinline__ void begin(int r) const {
        __syncwarp();  // every lane is done with the slot about to be refilled
        const int rr = r + D;
        if (rr < ROWS) {
            issue_row(c, c.qi, rr - 1, (sbase + rr) % RING);
        } else if (next_qi != nullptr) {
            const int r2 = rr - ROWS;
            if (r2 == 0) issue_halo(c, next_qi);
            issue_row(c, next_qi, r2 - 1, (sbase + rr) % RING);
        }
        cp_commit();
        cp_wait<D>();
        __syncwarp();
    }
    __device__ __forceinline__ void row(int r, double (&q)[N]) const {
        const int slot = (sbase + r) % RING;
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = c.sm->ring[slot][k][c.lane];
    }
    __device__ __forceinline__ void right(int r, double (&q)[N]) const {  // state of lane+1
        const int slot = (sbase + r) % RING;
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = c.sm->ring[slot][k][c.lane + 1];
    }
};

template <int P, int RING>
struct DirectSrc {
    const Ctx<P, RING>& c;
    __device__ __forceinline__ void halo(double (&q0)[N], double (&q1)[N], double (&q2)[N],
                                         double (&q3)[N]) const {
        const double* row = c.qi + (c.x + 1) * (P + 2);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            q0[k] = __ldg(row + k * c.sIn);
            q1[k] = __ldg(row + k * c.sIn + 1);
            q2[k] = __ldg(row + k * c.sIn + P);
            q3[k] = __ldg(row + k * c.sIn + P + 1);
        }
    }
    __device__ __forceinline__ void begin(int) const {}
    __device__ __forceinline__ void row(int r, double (&q)[N]) const {
        const double* p = c.qi + r * (P + 2) + c.x + 1;
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = __ldg(p + k * c.sIn);
    }
    __device__ __forceinline__ void right(int r, double (&q)[N]) const {
        const double* p = c.qi + r * (P + 2) + c.x + 2;
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = __ldg(p + k * c.sIn);
    }
};

// x-faces of row Y (stream row r = Y+1) and the axis-0 update of this lane's cell.
template <int P, int RING, class Src>
__device__ __forceinline__ void x_update(const Ctx<P, RING>& c, const Src& src, int Y,
                                         const double (&q)[N], const double (&fx)[N], double lx,
                                         double (&acc)[N]) {
    double qn[N], fxn[N], gr[N], gl[N];
    src.right(Y + 1, qn);
#pragma unroll
    for (int k = 0; k < N; ++k) fxn[k] = __shfl_down_sync(0xffffffffu, fx[k], 1);
    const double lxn = __shfl_down_sync(0xffffffffu, lx, 1);
    rusanov_face(q, qn, fx, fxn, lx, lxn, gr);  // face at x + 1/2
    // boundary faces from phase H: lane 0 needs the left one, lane P-1 the right one
    // (predicated loads straight into the face registers: no selects)
    if (c.x == P - 1) {
#pragma unroll
        for (int k = 0; k < N; ++k) gr[k] = c.sm->gr[k * 48 + c.hbase + Y];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) gl[k] = __shfl_up_sync(0xffffffffu, gr[k], 1);
    if (c.x == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) gl[k] = c.sm->gl[k * 48 + c.hbase + Y];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = q[k];
    rusanov_update(acc, gl, gr, c.scale);
}

// Finish row Y-1 (its upper y-face just became known): store + reduce.
template <int P, int RING, bool REDUCE, class R>
__device__ __forceinline__ void finish(const Ctx<P, RING>& c, const Euler<2>& eq, int Yprev,
                                       const Row& prev, const double (&gy)[N], double& pred,
                                       bool& bad) {
    double qn[N];
#pragma unroll
    for (int k = 0; k < N; ++k) qn[k] = prev.acc[k];
    rusanov_update(qn, prev.gy, gy, c.scale);
    if (c.valid) {
        double* o = c.qo + Yprev * P + c.x;
#pragma unroll
        for (int k = 0; k < N; ++k, o += c.sOut) __stcs(o, qn[k]);
    }
    if (REDUCE) running_max(pred, cell_lambda<R>(eq, qn, bad));
}

// Interior row Y >= 1: prev = row Y-1, cur <- row Y.
template <int P, int RING, bool REDUCE, class R, class Src>
__device__ __forceinline__ void row_step(const Ctx<P, RING>& c, const Src& src,
                                         const Euler<2>& eq, int Y, const Row& prev, Row& cur,
                                         double& pred, bool& bad) {
    src.begin(Y + 1);
    src.row(Y + 1, cur.q);
    double fx[N], lx, gy[N];
    eval<R, true, true>(eq, cur.q, fx, lx, cur.fy, cur.ly, bad);
    rusanov_face(prev.q, cur.q, prev.fy, cur.fy, prev.ly, cur.ly, gy);  // face at Y - 1/2
    finish<P, RING, REDUCE, R>(c, eq, Y - 1, prev, gy, pred, bad);
#pragma unroll
    for (int k = 0; k < N; ++k) cur.gy[k] = gy[k];
    x_update(c, src, Y, cur.q, fx, lx, cur.acc);
}

// One patch group: phase H + the walk.  Returns this lane's max eigenvalue.
template <int P, int RING, bool REDUCE, class R, class Src>
__device__ __forceinline__ double group(const Ctx<P, RING>& c, const Src& src, const Euler<2>& eq,
                                        bool& bad) {
    // ---- phase H: x-boundary faces of row r = x ---------------------------
    {
        double q0[N], q1[N], q2[N], q3[N], f0[N], f1[N], f2[N], f3[N], l0, l1, l2, l3, g[N], d[N], dl;
        src.halo(q0, q1, q2, q3);
        eval<R, true, false>(eq, q0, f0, l0, d, dl, bad);
        eval<R, true, false>(eq, q1, f1, l1, d, dl, bad);
        eval<R, true, false>(eq, q2, f2, l2, d, dl, bad);
        eval<R, true, false>(eq, q3, f3, l3, d, dl, bad);
        rusanov_face(q0, q1, f0, f1, l0, l1, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.sm->gl[k * 48 + c.hbase + c.x] = g[k];
        rusanov_face(q2, q3, f2, f3, l2, l3, g);
#pragma unroll
        for (int k = 0; k < N; ++k) c.sm->gr[k * 48 + c.hbase + c.x] = g[k];
    }
    __syncwarp();

    double pred = 0.0;
    Row S0, S1;
    {  // row -1 (halo): y-flux only
        src.begin(0);
        src.row(0, S0.q);
        double fx[N], lx;
        eval<R, false, true>(eq, S0.q, fx, lx, S0.fy, S0.ly, bad);
    }
    {  // row 0: nothing to finish yet
        src.begin(1);
        src.row(1, S1.q);
        double fx[N], lx;
        eval<R, true, true>(eq, S1.q, fx, lx, S1.fy, S1.ly, bad);
        rusanov_face(S0.q, S1.q, S0.fy, S1.fy, S0.ly, S1.ly, S1.gy);
        x_update(c, src, 0, S1.q, fx, lx, S1.acc);
    }
    int Y = 1;
#pragma unroll 1
    for (; Y + 1 < P; Y += 2) {  // two rows per trip through alternating Row sets
        row_step<P, RING, REDUCE, R>(c, src, eq, Y, S1, S0, pred, bad);
        row_step<P, RING, REDUCE, R>(c, src, eq, Y + 1, S0, S1, pred, bad);
    }
    if (Y < P) row_step<P, RING, REDUCE, R>(c, src, eq, Y, S1, S0, pred, bad);
    const Row& last = (Y < P) ? S0 : S1;
    {  // row P (halo): y-flux, top face, finish row P-1
        double q[N], fx[N], lx, fy[N], ly, gy[N];
        src.begin(P + 1);
        src.row(P + 1, q);
        eval<R, false, true>(eq, q, fx, lx, fy, ly, bad);
        rusanov_face(last.q, q, last.fy, fy, last.ly, ly, gy);
        finish<P, RING, REDUCE, R>(c, eq, P - 1, last, gy, pred, bad);
    }
    __syncwarp();  // boundary faces are rewritten by the next group
    return pred;
}

}  // namespace pencil

template <int P, int WARPS, bool REDUCE, int MINB, int RING = 4>
__global__ void __launch_bounds__(WARPS * 32, MINB) fused2d_pencil_kernel(StepArgs a) {
    using namespace pencil;
    constexpr int M = (P + 2) * (P + 2);
    constexpr int Mi = P * P;
    constexpr int G = 32 / P;  // patches per warp
    static_assert(P >= 2 && P <= 32, "pencil kernel covers 2 <= p <= 32");
    static_assert(G * (P + 1) <= 48, "boundary-face smem row too short");
    static_assert(RING >= 2, "ring needs >= 2 slots");
    const Euler<2> eq{a.gamma};

    __shared__ WarpSmem<RING> smem[WARPS];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int sub = lane / P;
    const bool lane_used = sub < G;
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const long long gstep = (long long)gridDim.x * WARPS;

    Ctx<P, RING> c;
    c.sIn = a.T * M;
    c.sOut = a.T * Mi;
    c.scale = a.scale;
    c.lane = lane;
    c.x = lane - sub * P;
    // padded rows (no bank conflict between patches); unused lanes (sub == G)
    // get their own slots: max index G*(P+1) + (32 - G*P) - 1 = G + 31 < 48
    c.hbase = sub * (P + 1);
    c.sm = &smem[warp];

    auto patch_of = [&](long long g) {
        const long long pt = t0 + g * G + (lane_used ? sub : 0);
        return (lane_used && pt < t1) ? pt : t0 + g * G;  // invalid lanes: a real patch, no stores
    };

    double red = 0.0;
    long long g = (long long)blockIdx.x * WARPS + warp;
    int sbase = 0;
    if (g < groups) {
        c.qi = a.q_in + patch_of(g) * M;
        RingSrc<P, RING>::prologue(c, sbase);
    }
    for (; g < groups; g += gstep) {
        const long long patch = patch_of(g);
        c.valid = lane_used && (t0 + g * G + sub) < t1;
        c.qi = a.q_in + patch * M;
        c.qo = a.q_out + patch * Mi;
        const double* next_qi = (g + gstep < groups) ? a.q_in + patch_of(g + gstep) * M : nullptr;

        bool bad = false;
        const RingSrc<P, RING> ring{c, next_qi, sbase};
        double pred = group<P, RING, REDUCE, XReal>(c, ring, eq, bad);
        if (__any_sync(0xffffffffu, bad)) {  // operand outside the fast paths: IEEE redo
            bool unused = false;
            const DirectSrc<P, RING> direct{c};
            pred = group<P, RING, REDUCE, double>(c, direct, eq, unused);
        }
        sbase = (sbase + P + 2) % RING;

        if (!c.valid) pred = 0.0;
        running_max(red, pred);
        if (REDUCE && a.lam_patch != nullptr) {  // segmented max over the P lanes of a patch
            double v = pred;
#pragma unroll
            for (int off = 1; off < P; off <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, off);
                if (c.x + off < P) running_max(v, o);
            }
            if (c.valid && c.x == 0) a.lam_patch[patch] = v;
        }
    }
    cp_wait<0>();
    if (REDUCE && a.lam_bits != nullptr) {
        red = warp_max(red);
        if (lane == 0) atomic_max_nonneg(a.lam_bits, red);
    }
}

}  // namespace fvb
