// fused3d.cuh -- the nested-parallel ("patch-wise") flavour for 3D patches:
// a plane walk along z with the haloed z-planes streamed into shared memory
// by TMA bulk copies.
//
// Reference realisation: run_patchwise (pkg/src/patchbench/executors.py:390-445)
// runs copy, flux_0..2, lambda_0..2, acc_0..2 and the reduce of one patch in
// one parallel region over the union range [-1,p]^3.  Here one "slot" of
// TH = roundup(p*p, 32) threads owns one patch at a time, thread t < p*p owns
// the interior column (x, y) = (t % p, t / p) and walks it along z:
//
//   * memory: the haloed patch is N*(p+2) contiguous z-planes of (p+2)^2
//     doubles per unknown (SoA, patchdata.py:163-165).  One elected thread
//     streams them through a RING-plane shared-memory ring with
//     cp.async.bulk (TMA, 1-D) completing on one mbarrier per ring slot,
//     RING-1 planes ahead of the compute and across patch boundaries; no
//     register staging, no per-thread address math for the loads;
//   * x / y: each thread evaluates flux_0, flux_1 (and flux_2) and the wave
//     speeds of its cell once and publishes the in-plane ones to shared
//     memory; the 4p halo cells of the plane (x = -1, p; y = -1, p) are
//     evaluated by threads t < 4p for their one axis.  Each thread then
//     computes the LEFT x-face and LEFT y-face of its cell (every interior
//     face once), the last 2p threads the right / top boundary faces, and
//     after one more slot barrier every thread reads its right faces;
//   * z: the thread keeps the previous plane's state, z-flux, z-wave speed,
//     x/y-updated value and lower z-face in registers, so every z-face is
//     computed once and cell (x, y, z-1) is finished (axis-2 update, store,
//     reduce) while plane z is processed;
//   * update order is the reference's: Q + s*dX, then + s*dY, then + s*dZ;
//   * reduce: max over axes of lambda(Q_new) of the finished cells, warp
//     shuffle max, one 64-bit atomicMax per warp per launch; per-patch maxima
//     (lam_patch) through a slot reduction.  Without per-patch maxima the
//     reduction is filtered (common.cuh LamFilter, Euler::lambda_below): a
//     warp evaluates the eigenvalues of a plane only if some lane's cell may
//     exceed the warp's running maximum -- a few planes per warp in a run.
//
// Arithmetic: as in fused2d.cuh -- each patch is first computed with
// R = XReal (CUDA's fp64 division / sqrt fast paths written out, the
// reciprocal of rho shared, doubled faces) on states the domain policy
// certifies with fast_path_safe(); if any thread of the slot met an
// uncertified state, the slot recomputes the patch in plain IEEE double
// (redo_cell, loads straight from global memory) and overwrites its stores.
// Either way output and eigenvalue are bit-identical to run_sequential.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "physics.cuh"

namespace fvb {

namespace slab {

template <int P>
struct Geo3 {
    static constexpr int E = P + 2;                        // haloed extent
    static constexpr int M2 = E * E;                       // haloed plane (doubles per unknown)
    static constexpr int M = E * E * E;                    // haloed patch
    static constexpr int Mi = P * P * P;                   // interior patch
    static constexpr int CELLS = P * P;                    // interior cells per plane
    static constexpr int HALO = 4 * P;                     // in-plane halo cells
    static constexpr int BF = 2 * P;                       // right / top boundary faces
    // threads per slot: enough for the cells and the halo duty; small p get
    // sub-warp slots (8 or 16 lanes: p = 2 / 3, 4 -- 2 or 4 patches per warp)
    static constexpr int NEED = CELLS > HALO ? CELLS : HALO;
    static constexpr int TH = NEED <= 8 ? 8 : NEED <= 16 ? 16 : ((NEED + 31) / 32) * 32;
    static_assert(HALO <= TH && BF <= TH, "slot too small for the halo work");
    // TMA bulk copies need 16-byte aligned, 16-byte sized planes: even p.
    // Odd p stream the same ring with per-thread cp.async arriving on the
    // same mbarriers (cp.async.mbarrier.arrive.noinc).
    static constexpr bool BULK = (M2 * 8) % 16 == 0;
};

// One streamed z-plane, [k][haloed in-plane lin]; 128-byte aligned slots so
// a tensor-map TMA copy may land in any of them.
template <int P, int N>
struct alignas(128) RingSlot {
    double v[N][Geo3<P>::M2];
};

template <int P, int RING, int N>
struct alignas(128) SlotSmem {
    using Gm = Geo3<P>;
    static constexpr int kN = N;
    static constexpr int NP = (N + 2) / 2 * 2;  // flux record length in doubles (even)
    RingSlot<P, N> ring[RING];     // streamed z-planes
    // per cell [flux_0..N-1, wave speed, pad]: a neighbour's whole record in
    // (N+1)/2 128-bit loads (put_rec / get_rec)
    double fxl[Gm::M2][NP];        // x-flux + x wave speed (interior + x-halo)
    double fyl[Gm::M2][NP];        // y-flux + y wave speed (interior + y-halo)
    double gx[N][Gm::M2];          // left x-face of cell (x, y), x in [0, P] (P: right boundary)
    double gy[N][Gm::M2];          // lower y-face of cell (x, y), y in [0, P] (P: top boundary)
    double red[Gm::TH >= 32 ? Gm::TH / 32 : 1];  // per-patch maximum (lam_patch, slots of whole warps)
    unsigned long long mbar[RING];
};

// ---- TMA bulk copy + mbarrier helpers ------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* m) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(m))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
// this thread's cp.async copies so far arrive on the mbarrier when complete
__device__ __forceinline__ void cp_async_arrive(unsigned long long* m) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void cp_async8_to(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void slot_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// 16-byte-aligned per-cell flux records: N flux components, the wave speed,
// padding to an even length (NP doubles).
template <int NP, int N>
__device__ __forceinline__ void put_rec(double* rec, const double (&f)[N], double l) {
    double v[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = k < N ? f[k] : (k == N ? l : 0.0);
    double2* r = reinterpret_cast<double2*>(rec);
#pragma unroll
    for (int i = 0; i < NP / 2; ++i) r[i] = make_double2(v[2 * i], v[2 * i + 1]);
}
template <int NP, int N>
__device__ __forceinline__ void get_rec(const double* rec, double (&f)[N], double& l) {
    const double2* r = reinterpret_cast<const double2*>(rec);
    double v[NP];
#pragma unroll
    for (int i = 0; i < NP / 2; ++i) {
        const double2 t = r[i];
        v[2 * i] = t.x;
        v[2 * i + 1] = t.y;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) f[k] = v[k];
    l = v[N];
}

// Max over the W-lane group of the calling lane (W a power of two <= 32),
// lanes `mask`; W = 32 is warp_max.
template <int W>
__device__ __forceinline__ double group_max(double v, unsigned mask) {
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(mask, v, off);
        running_max(v, o);
    }
    return v;
}

// bar.red.or over the slot's named barrier: true if any thread of the slot passed true
__device__ __forceinline__ bool slot_any(int id, int nthreads, bool v) {
    int r;
    asm volatile(
        "{\n"
        ".reg .pred P1, P2;\n"
        "setp.ne.u32 P1, %1, 0;\n"
        "bar.red.or.pred P2, %2, %3, P1;\n"
        "selp.u32 %0, 1, 0, P2;\n"
        "}\n"
        : "=r"(r)
        : "r"((int)v), "r"(id), "r"(nthreads)
        : "memory");
    return r != 0;
}

template <int P>
__device__ __forceinline__ int hlin(int x, int y) {  // haloed in-plane index of (x, y), x, y in [-1, P]
    return (x + 1) + Geo3<P>::E * (y + 1);
}

// Interior cell of slot thread t < p*p.  Every shared-memory array is indexed
// by the haloed in-plane index (row stride p+2).  64-bit accesses are served
// per half-warp, so for p = 8 (row stride 10 doubles = 20 banks) a half-warp
// takes rows y and y+4 (offset 40 doubles = 80 banks = 16 mod 32): its 16
// accesses hit 32 distinct banks for the cell, its x- and y-neighbours and
// its faces.  Other p: row-major.
template <int P>
__device__ __forceinline__ void cell_of(int t, int& x, int& y) {
    x = t % P;
    if constexpr (P == 8) {
        y = ((t >> 4) & 3) + 4 * ((t >> 3) & 1);
    } else {
        y = t / P;
    }
}

// One z-plane of the current patch, unknown k at haloed in-plane index lin:
// the ring slot (streamed) or global memory (the IEEE redo).
// LS: distance between cells (1, or N for AoS planes).
template <int LS>
struct Plane {
    const double* base;
    long long ks;  // distance between unknowns
    __device__ __forceinline__ double operator()(int k, int lin) const { return base[k * ks + lin * LS]; }
};

// With R = XReal the state must satisfy the domain's fast-path precondition;
// a violation marks the slot's patch for the IEEE redo.
template <class R, class Eq, int N>
__device__ __forceinline__ void certify(const Eq& eq, const R (&s)[N], bool& bad) {
    if constexpr (std::is_same<R, XReal>::value) bad |= !eq.fast_path_safe(s);
}

template <class R, int N>
__device__ __forceinline__ void to_r(const double (&q)[N], R (&s)[N]) {
#pragma unroll
    for (int k = 0; k < N; ++k) s[k] = q[k];
}

template <class R, class Eq, int N>
__device__ __forceinline__ void axis_eval(const Eq& eq, const R (&s)[N], int axis, double (&f)[N],
                                          double& l) {
    R fr[N];
    eq.flux(s, axis, fr);
    const R lr = eq.max_eigenvalue(s, axis);
#pragma unroll
    for (int k = 0; k < N; ++k) f[k] = val(fr[k]);
    l = val(lr);
}

template <class R, class Eq, int N>
__device__ __forceinline__ double cell_lambda(const Eq& eq, const double (&q)[N], bool& bad) {
    R s[N];
    to_r(q, s);
    certify(eq, s, bad);
    double v = val(eq.max_eigenvalue(s, 0));
    v = py_max(v, val(eq.max_eigenvalue(s, 1)));
    return py_max(v, val(eq.max_eigenvalue(s, 2)));
}

// Eigenvalue of a finished cell into the running maximum (see kReduce*).
// Converged over the vote group (every lane of the warp, or of a sub-warp
// slot: W lanes `mask`) -- every lane calls it (active = the lane finished
// a cell).
template <int RED, class R, int W = 32, class Eq, int N>
__device__ __forceinline__ void reduce_cell(const Eq& eq, const double (&qn)[N], bool active, double& pred,
                                            LamFilter& lf, bool& bad, unsigned mask = 0xffffffffu) {
    if constexpr (RED == kReduceAll) {
        if (active) running_max(pred, cell_lambda<R>(eq, qn, bad));
    } else if constexpr (RED == kReduceFiltered) {
        const bool need = active && !eq.lambda_below(qn, lf.tau_lo);
        if (__any_sync(mask, need)) {
            if (need) running_max(pred, cell_lambda<R>(eq, qn, bad));
            lf.raise_max(group_max<W>(pred, mask));
        }
    }
}

// Faces and updates: the reference's expressions (R = double), or on
// certified states the doubled face H = 2G with the update scaled by
// 0.5*dt/h, bit-identical (see fused2d.cuh, face()).
template <class R>
constexpr bool kFold = std::is_same<R, XReal>::value;

template <class R, int N>
__device__ __forceinline__ void face(const double (&qL)[N], const double (&qR)[N], const double (&fL)[N],
                                     const double (&fR)[N], double lamL, double lamR, double (&g)[N]) {
    if constexpr (kFold<R>) {
        const double w = py_max(lamL, lamR);
#pragma unroll
        for (int k = 0; k < N; ++k) g[k] = (fL[k] + fR[k]) - w * (qR[k] - qL[k]);
    } else {
        rusanov_face(qL, qR, fL, fR, lamL, lamR, g);
    }
}

// Per-slot constants.
template <int P, int RING, int LS, int N_>
struct SlabCtx {
    static constexpr int N = N_;
    SlotSmem<P, RING, N>* S;
    const double* q_in;
    double* q_out;
    const double* const* in_tab;  // SHARED mode: per-patch arrays (see StepArgs)
    double* const* out_tab;
    long long sIn, sOut, pIn, pOut, first, stride, njobs;  // unknown / patch strides
    double scale, hscale;
    int t, bar;
    unsigned mask;  // the slot's lanes of the warp (sub-warp slots)
    // this thread's interior column, halo cell and boundary face
    bool real, halo, bface, bx;  // real: owns a cell (else a stand-in duplicate of one)
    bool bulk;                   // plane copies by TMA bulk copy (bulk_ok), else cp.async
    int lc, ci, hl, haxis, bl, bstep;  // ci: interior in-plane index x + p*y
    // Every slot thread walks a column: threads beyond p*p walk a duplicate
    // of a real column (identical values, no stores), so the plane phases are
    // branch-free for every p -- a per-thread guard made ptxas spill.
    __device__ __forceinline__ constexpr bool cell() const { return true; }
    // Slot-wide barrier / vote: named barriers for slots of whole warps,
    // warp primitives under the slot's lane mask for sub-warp slots.
    static constexpr int TH = Geo3<P>::TH;
    static constexpr int VW = TH < 32 ? TH : 32;  // vote / max group width
    __device__ __forceinline__ void sync() const {
        if constexpr (TH >= 32) slot_sync(bar, TH);
        else __syncwarp(mask);
    }
    __device__ __forceinline__ bool any(bool v) const {
        if constexpr (TH >= 32) return slot_any(bar, TH, v);
        else return __any_sync(mask, v);
    }
    __device__ __forceinline__ const double* in_base(long long patch) const {
        return in_tab != nullptr ? in_tab[patch] : q_in + patch * pIn;
    }
    __device__ __forceinline__ double* out_base(long long patch) const {
        return out_tab != nullptr ? out_tab[patch] : q_out + patch * pOut;
    }
};

// Bulk copies need 16-byte aligned sources: even p (whole planes are 16-byte
// multiples) and a batch whose base and strides are 16-byte aligned.  Else
// (odd p, or e.g. a sub-view starting 8 bytes into an allocation) the slot
// threads copy the plane with 8-byte cp.async.
// SoA / AoSoA (LS = 1) copy one plane per unknown: unknown and patch strides
// even.  AoS (LS = N) copies the whole interleaved plane from the patch base:
// only the patch stride N*(p+2)^3 (even for even p) matters.  Per-patch
// pointer tables (SHARED mode, host-mapped arrays) always use cp.async.
template <int P, int LS>
__device__ __forceinline__ bool bulk_ok(const StepArgs& a) {
    if (a.in_tab != nullptr) return false;
    return Geo3<P>::BULK && (reinterpret_cast<unsigned long long>(a.q_in) % 16 == 0) &&
           (LS != 1 || a.in.k % 2 == 0) && (a.in.p % 2 == 0);
}

// Threads arriving on a ring slot's mbarrier per job: the elected issuer
// (TMA, expect_tx) or every slot thread (cp.async).
template <int P>
__device__ __forceinline__ unsigned ring_arrivals(bool bulk) {
    return bulk ? 1u : (unsigned)Geo3<P>::TH;
}

// Plane job j (patch first + (j / (P+2))*stride, plane j % (P+2)) into ring
// slot j % RING, completing on that slot's mbarrier.  Every slot thread calls
// it: with bulk copies thread 0 issues TMA bulk copies, else every thread
// copies its share of the plane with cp.async and arrives asynchronously.
template <int P, int RING, int LS, int N>
__device__ __forceinline__ void issue_job(const SlabCtx<P, RING, LS, N>& c, long long j) {
    using Gm = Geo3<P>;
    constexpr unsigned PLANE_BYTES = Gm::M2 * 8;
    const long long patch = c.first + (j / (P + 2)) * c.stride;
    const int plane = (int)(j % (P + 2));
    const int r = (int)(j % RING);
    const double* src = c.in_base(patch) + (long long)plane * Gm::M2 * LS;
    if (Gm::BULK && c.bulk) {
        if (c.t != 0) return;
        mbar_expect_tx(&c.S->mbar[r], N * PLANE_BYTES);
        if constexpr (LS == 1) {  // SoA / AoSoA: one contiguous plane per unknown
#pragma unroll
            for (int k = 0; k < N; ++k)
                bulk_g2s(&c.S->ring[r].v[k][0], src + k * c.sIn, PLANE_BYTES, &c.S->mbar[r]);
        } else {  // AoS: the plane's N unknowns interleaved, one copy, kept [cell][k] in the slot
            bulk_g2s(&c.S->ring[r].v[0][0], src, N * PLANE_BYTES, &c.S->mbar[r]);
        }
    } else {
        double* dst = &c.S->ring[r].v[0][0];
        for (int e = c.t; e < N * Gm::M2; e += Gm::TH) {
            if constexpr (LS == 1) {
                const int k = e / Gm::M2, lin = e - k * Gm::M2;
                cp_async8_to(dst + e, src + k * c.sIn + lin);
            } else {
                cp_async8_to(dst + e, src + e);  // AoS plane: N * M2 contiguous
            }
        }
        cp_async_arrive(&c.S->mbar[r]);
    }
}

// Carried along z for one column: the previous plane's state, z-flux,
// z-wave speed, x/y-updated value and lower z-face.
template <int N>
struct Carry {
    double q[N], fz[N], lz, acc[N], gz[N];
};

// The TMA ring of one slot: plane job j lives in ring slot j % RING; the
// next job is issued into a slot as soon as every thread is done with it.
template <int P, int RING, int LS, int N>
struct PlaneWalk {
    const SlabCtx<P, RING, LS, N>& c;
    long long& j;

    __device__ __forceinline__ Plane<LS> acquire() const {
        const int r = (int)(j % RING);
        mbar_wait(&c.S->mbar[r], (unsigned)((j / RING) & 1));
        return Plane<LS>{&c.S->ring[r].v[0][0], LS == 1 ? Geo3<P>::M2 : 1};
    }
    // every read of the current plane's ring slot is done (call after a slot barrier)
    __device__ __forceinline__ void release() const {
        if (j + RING < c.njobs) {
            // no proxy fence: the slot's generic reads are ordered before the
            // async-proxy refill by the slot barrier (CUTLASS TMA-pipeline convention)
            issue_job(c, j + RING);
        }
        ++j;
    }
};

// Interior plane z.  Phase 1 evaluates the microkernels of the plane's
// cells (publishing the in-plane fluxes) and of the halo cells, then the
// z-face below and finishes cell (x, y, z-1) -- so the previous plane's
// values die before the first barrier.  Phase 2: left x/y-faces and the
// boundary faces.  Phase 3: right faces and the x/y update.
template <int P, int RING, int RED, class R, class W, int LS, class Eq, int N>
__device__ __forceinline__ void interior_plane(const SlabCtx<P, RING, LS, N>& c, const W& w, const Eq& eq,
                                               int z, const Carry<N>& prev, Carry<N>& cur, double* qo,
                                               double& pred, LamFilter& lf, bool& bad) {
    using Gm = Geo3<P>;
    constexpr int E = Gm::E, M2 = Gm::M2, TH = Gm::TH, CELLS = Gm::CELLS;
    constexpr int NP = SlotSmem<P, RING, N>::NP;
    SlotSmem<P, RING, N>& S = *c.S;
    const double s = kFold<R> ? c.hscale : c.scale;
    const auto pl = w.acquire();
    const int lc = c.lc;

    // ---- phase 1 -----------------------------------------------------------
    double fx[N], lx = 0.0, fy[N], ly = 0.0;
    if (c.cell()) {
#pragma unroll
        for (int k = 0; k < N; ++k) cur.q[k] = pl(k, lc);
        R sr[N];
        to_r(cur.q, sr);
        certify(eq, sr, bad);
        axis_eval(eq, sr, 0, fx, lx);
        axis_eval(eq, sr, 1, fy, ly);
        axis_eval(eq, sr, 2, cur.fz, cur.lz);
        put_rec<NP>(S.fxl[lc], fx, lx);
        put_rec<NP>(S.fyl[lc], fy, ly);
    }
    if (c.halo) {
        double h[N], f[N], l;
#pragma unroll
        for (int k = 0; k < N; ++k) h[k] = pl(k, c.hl);
        R sr[N];
        to_r(h, sr);
        certify(eq, sr, bad);
        if (c.haxis == 0) {
            axis_eval(eq, sr, 0, f, l);
            put_rec<NP>(S.fxl[c.hl], f, l);
        } else {
            axis_eval(eq, sr, 1, f, l);
            put_rec<NP>(S.fyl[c.hl], f, l);
        }
    }
    if (z >= 1) {  // finish (x, y, z-1)
        double qn[N];
        if (c.cell()) {
            face<R>(prev.q, cur.q, prev.fz, cur.fz, prev.lz, cur.lz, cur.gz);  // face at z - 1/2
#pragma unroll
            for (int k = 0; k < N; ++k) qn[k] = prev.acc[k];
            rusanov_update(qn, prev.gz, cur.gz, s);
            if (Geo3<P>::CELLS == Geo3<P>::TH || c.real)
#pragma unroll
                for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + (z - 1) * CELLS * LS, qn[k]);
        }
        reduce_cell<RED, R, SlabCtx<P, RING, LS, N>::VW>(eq, qn, c.cell(), pred, lf, bad, c.mask);
    } else if (c.cell()) {
        face<R>(prev.q, cur.q, prev.fz, cur.fz, prev.lz, cur.lz, cur.gz);
    }
    c.sync();

    // ---- phase 2 -----------------------------------------------------------
    double gxl[N], gyl[N];
    if (c.cell()) {
        double qn[N], fn[N], ln;
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = pl(k, lc - 1);
        get_rec<NP>(S.fxl[lc - 1], fn, ln);
        face<R>(qn, cur.q, fn, fx, ln, lx, gxl);
#pragma unroll
        for (int k = 0; k < N; ++k) qn[k] = pl(k, lc - E);
        get_rec<NP>(S.fyl[lc - E], fn, ln);
        face<R>(qn, cur.q, fn, fy, ln, ly, gyl);
#pragma unroll
        for (int k = 0; k < N; ++k) S.gx[k][lc] = gxl[k], S.gy[k][lc] = gyl[k];
    }
    if (c.bface) {
        double qL[N], qR[N], fL[N], fR[N], g[N], lL, lR;
        const double(*F)[NP] = c.bx ? S.fxl : S.fyl;
        double(*G)[M2] = c.bx ? S.gx : S.gy;
        const int bl = c.bl, br = c.bl + c.bstep;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            qL[k] = pl(k, bl);
            qR[k] = pl(k, br);
        }
        get_rec<NP>(F[bl], fL, lL);
        get_rec<NP>(F[br], fR, lR);
        face<R>(qL, qR, fL, fR, lL, lR, g);
#pragma unroll
        for (int k = 0; k < N; ++k) G[k][br] = g[k];
    }
    c.sync();  // faces published; this plane's ring slot no longer read
    w.release();

    // ---- phase 3 -----------------------------------------------------------
    if (c.cell()) {
#pragma unroll
        for (int k = 0; k < N; ++k) cur.acc[k] = cur.q[k];
        double gr[N];
#pragma unroll
        for (int k = 0; k < N; ++k) gr[k] = S.gx[k][lc + 1];
        rusanov_update(cur.acc, gxl, gr, s);
#pragma unroll
        for (int k = 0; k < N; ++k) gr[k] = S.gy[k][lc + E];
        rusanov_update(cur.acc, gyl, gr, s);
    }
}

// One patch: the plane walk, two interior planes per trip through
// alternating carry sets (no register copies; odd p: one more plane).  Returns this thread's max
// eigenvalue of the patch's finished cells.
template <int P, int RING, int RED, class R, int LS, class Eq, int N>
__device__ __forceinline__ double slab_patch(const SlabCtx<P, RING, LS, N>& c, const Eq& eq, long long patch,
                                             long long& j, LamFilter& lf, bool& bad) {
    using Gm = Geo3<P>;
    constexpr int TH = Gm::TH, CELLS = Gm::CELLS;
    const double s = kFold<R> ? c.hscale : c.scale;
    double* qo = c.out_base(patch) + c.ci * LS;
    const PlaneWalk<P, RING, LS, N> w{c, j};
    double pred = 0.0;
    Carry<N> A, B;

    {  // z = -1 (halo plane): z-flux only
        const auto pl = w.acquire();
        if (c.cell()) {
#pragma unroll
            for (int k = 0; k < N; ++k) A.q[k] = pl(k, c.lc);
            R sr[N];
            to_r(A.q, sr);
            certify(eq, sr, bad);
            axis_eval(eq, sr, 2, A.fz, A.lz);
        }
        c.sync();
        w.release();
    }
#pragma unroll 1
    for (int z = 0; z + 1 < P; z += 2) {
        interior_plane<P, RING, RED, R>(c, w, eq, z, A, B, qo, pred, lf, bad);
        interior_plane<P, RING, RED, R>(c, w, eq, z + 1, B, A, qo, pred, lf, bad);
    }
    if constexpr (P % 2 == 1) interior_plane<P, RING, RED, R>(c, w, eq, P - 1, A, B, qo, pred, lf, bad);
    const Carry<N>& L = (P % 2 == 1) ? B : A;  // the carry of plane P-1
    {  // z = P (halo plane): top z-face, finish z = P-1
        const auto pl = w.acquire();
        double qn[N];
        if (c.cell()) {
            double q[N], fz[N], lz, gz[N];
#pragma unroll
            for (int k = 0; k < N; ++k) q[k] = pl(k, c.lc);
            R sr[N];
            to_r(q, sr);
            certify(eq, sr, bad);
            axis_eval(eq, sr, 2, fz, lz);
            face<R>(L.q, q, L.fz, fz, L.lz, lz, gz);
#pragma unroll
            for (int k = 0; k < N; ++k) qn[k] = L.acc[k];
            rusanov_update(qn, L.gz, gz, s);
            if (Geo3<P>::CELLS == Geo3<P>::TH || c.real)
#pragma unroll
                for (int k = 0; k < N; ++k) __stcs(qo + k * c.sOut + (P - 1) * CELLS * LS, qn[k]);
        }
        reduce_cell<RED, R, SlabCtx<P, RING, LS, N>::VW>(eq, qn, c.cell(), pred, lf, bad, c.mask);
        c.sync();
        w.release();
    }
    return pred;
}

// The IEEE redo of one cell (x, y, z): the reference's accumulate sequence
// (acc = Q; + s*(F_l - F_r) per axis in order) straight from global memory,
// both faces of every axis recomputed from the neighbour states.  Rare, so
// it is written for a small register footprint, not for speed; the faces
// are the same pure expressions of the same operands as in the plane walk,
// so its bits are the IEEE bits of run_sequential.
template <int P, int LS, class Eq, int N>
__device__ __forceinline__ void redo_cell(const Eq& eq, const double* qi, long long sIn, int x, int y,
                                          int z, double scale, double (&acc)[N]) {
    constexpr int E = Geo3<P>::E;
    const int lin = (x + 1) + E * (y + 1) + E * E * (z + 1);
    double q[N];
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = q[k] = qi[k * sIn + lin * LS];
#pragma unroll 1
    for (int axis = 0; axis < 3; ++axis) {
        const int st = axis == 0 ? 1 : axis == 1 ? E : E * E;
        double f[N], gl[N], gr[N];
        eq.flux(q, axis, f);
        const double l = eq.max_eigenvalue(q, axis);
        {
            double qn[N], fn[N];
#pragma unroll
            for (int k = 0; k < N; ++k) qn[k] = qi[k * sIn + (lin - st) * LS];
            eq.flux(qn, axis, fn);
            rusanov_face(qn, q, fn, f, eq.max_eigenvalue(qn, axis), l, gl);
        }
        {
            double qn[N], fn[N];
#pragma unroll
            for (int k = 0; k < N; ++k) qn[k] = qi[k * sIn + (lin + st) * LS];
            eq.flux(qn, axis, fn);
            rusanov_face(q, qn, f, fn, l, eq.max_eigenvalue(qn, axis), gr);
        }
        rusanov_update(acc, gl, gr, scale);
    }
}

}  // namespace slab

template <int P, int RING, int N>
constexpr size_t slab_smem_per_slot() {
    return sizeof(slab::SlotSmem<P, RING, N>);
}

template <class Eq, int P, int SLOTS, int RING, int RED, int MINB, int LS>
__global__ void __launch_bounds__(SLOTS* slab::Geo3<P>::TH, MINB) fused3d_slab_kernel(StepArgs a) {
    using namespace slab;
    using Gm = Geo3<P>;
    constexpr int E = Gm::E, TH = Gm::TH;
    constexpr int N = Eq::kUnknowns;
    static_assert(Eq::kDim == 3, "the plane walk is 3D");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int slot = threadIdx.x / TH;
    SlabCtx<P, RING, LS, N> c;
    c.t = threadIdx.x - slot * TH;
    c.S = reinterpret_cast<SlotSmem<P, RING, N>*>(smem_raw) + slot;
    c.bar = 1 + slot;  // named barrier of this slot (0 is __syncthreads)
    c.mask = TH >= 32 ? 0xffffffffu : ((1u << (TH & 31)) - 1u) << ((threadIdx.x & 31) & ~(TH - 1));
    c.q_in = a.q_in;
    c.q_out = a.q_out;
    c.in_tab = a.in_tab;
    c.out_tab = a.out_tab;
    c.sIn = a.in.k;
    c.sOut = a.out.k;
    c.pIn = a.in.p;
    c.pOut = a.out.p;
    // Sub-warp slots stream with per-thread cp.async.  A bulk copy is a
    // warp-level (uniform-datapath) instruction; two slots of one warp
    // issuing them independently is correct (each completes on its slot's
    // mbarrier) but compute-sanitizer's racecheck attributes the copies to
    // lane 0 and reports thousands of warp-level warnings; with cp.async it
    // is clean.  Cost: p = 4 at 34.7% instead of 40.2% of the roofline
    // (p = 2 is 3% faster).
    c.bulk = TH >= 32 && bulk_ok<P, LS>(a);
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);
    c.scale = scale;
    c.hscale = 0.5 * scale;
    c.first = a.t0 + (long long)blockIdx.x * SLOTS + slot;
    c.stride = (long long)gridDim.x * SLOTS;
    const long long npatch = c.first < a.t1 ? (a.t1 - c.first + c.stride - 1) / c.stride : 0;
    c.njobs = npatch * (P + 2);  // job = (patch, plane), streamed in order

    const int t = c.t;
    c.real = t < Gm::CELLS;
    int cx = 0, cy = 0;
    cell_of<P>(c.real ? t : t % Gm::CELLS, cx, cy);
    c.lc = hlin<P>(cx, cy);
    c.ci = cx + P * cy;
    c.halo = t < Gm::HALO;
    c.hl = 0, c.haxis = 0;
    if (c.halo) {
        const int side = t / P, i = t % P;
        const int hx = side == 0 ? -1 : side == 1 ? P : i;
        const int hy = side == 2 ? -1 : side == 3 ? P : i;
        c.hl = hlin<P>(hx, hy);
        c.haxis = side < 2 ? 0 : 1;
    }
    const int b = t - (TH - Gm::BF);  // boundary-face duty: b in [0, P) x-face, [P, 2P) y-face
    c.bface = b >= 0;
    c.bx = b < P;
    const int bi = c.bx ? b : b - P;
    c.bl = c.bface ? (c.bx ? hlin<P>(P - 1, bi) : hlin<P>(bi, P - 1)) : 0;  // left / lower cell
    c.bstep = c.bx ? 1 : E;  // the face is stored at the right / upper cell's index

    if (t == 0) {
#pragma unroll
        for (int r = 0; r < RING; ++r) mbar_init(&c.S->mbar[r], ring_arrivals<P>(c.bulk));
        fence_mbar_init();
    }
    c.sync();
    for (long long j = 0; j < RING && j < c.njobs; ++j) issue_job(c, j);

    double red = 0.0;
    long long j = 0;
    LamFilter lf;
    lf.init();
    for (long long ip = 0; ip < npatch; ++ip) {
        const long long patch = c.first + ip * c.stride;
        bool patch_fast = fast;
        if (a.dt_patch != nullptr) {  // local time stepping: this patch's dt
            c.scale = patch_scale(a, scale, patch);
            c.hscale = 0.5 * c.scale;
            patch_fast = step_fast(a, c.scale);
        }
        bool bad = !patch_fast;  // run parameters outside the folded-face range: IEEE only
        const LamFilter lf0 = lf;
        double pred;
        bool redo = false;
        if constexpr (kHasFastPath<Eq>) {
            pred = slab_patch<P, RING, RED, XReal>(c, eq, patch, j, lf, bad);
            redo = c.any(bad);  // an uncertified state in this patch
        } else {  // a policy without the fast-path hook: IEEE double throughout
            pred = slab_patch<P, RING, RED, double>(c, eq, patch, j, lf, bad);
        }
        if (redo) {  // IEEE redo
            pred = 0.0;
            if (c.real) {
                const double* qi = in_base(a, patch);
                double* qo = out_base(a, patch) + c.ci * LS;
#pragma unroll 1
                for (int z = 0; z < P; ++z) {
                    double qn[N];
                    redo_cell<P, LS>(eq, qi, c.sIn, cx, cy, z, c.scale, qn);
#pragma unroll
                    for (int k = 0; k < N; ++k) qo[k * c.sOut + z * Gm::CELLS * LS] = qn[k];
                    if (RED != kReduceNone) running_max(pred, cell_max_eigenvalue(eq, qn));
                }
            }
            if (RED == kReduceFiltered) {  // the fast pass may have raised tau from flagged states
                lf = lf0;
                lf.raise_max(group_max<SlabCtx<P, RING, LS, N>::VW>(pred, c.mask));
            }
        }
        running_max(red, pred);
        if (RED == kReduceAll && a.lam_patch != nullptr) {  // slot-wide max of this patch
            if constexpr (TH < 32) {
                const double w = group_max<TH>(pred, c.mask);
                if (t == 0) a.lam_patch[patch] = w;
            } else {
                const double w = warp_max(pred);
                if ((t & 31) == 0) c.S->red[t >> 5] = w;
                c.sync();
                if (t == 0) {
                    double v = c.S->red[0];
#pragma unroll
                    for (int i = 1; i < TH / 32; ++i) running_max(v, c.S->red[i]);
                    a.lam_patch[patch] = v;
                }
                c.sync();
            }
        }
    }
    if (RED != kReduceNone && a.lam_bits != nullptr) reduce_epilogue<(SLOTS * slab::Geo3<P>::TH > 32)>(a, red);
}

}  // namespace fvb
