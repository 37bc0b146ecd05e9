// fused2d_tma.cuh -- the 2D pencil kernel (fused2d.cuh) with its rows and
// halo columns streamed by tensor-map TMA copies instead of per-lane cp.async.
//
// One warp still owns G = 32/p patches (one column per lane) and walks rows
// Y = -1..P; the arithmetic, faces, exchange row, filter and IEEE redo are
// fused2d.cuh's (group<>() is shared).  What changes is the source of rows:
//   * the input batch is described by two 4-D tensor maps, dimensions
//     ordered by stride -- [col][row][patch][k] (SoA) or [col][row][k][patch]
//     (AoSoA): a ROWS box {p+2, RS, G, N} (RS = 2 whole haloed rows of the
//     warp's G patches, every unknown -- TMA wants the box to start 16-byte
//     aligned, so the halo columns ride along) and a HALO box {2, p, G, N}
//     (the column pair -1, 0 or p-1, p of rows 0..p-1);
//   * lane 0 issues ONE copy per two rows (plus two per group for the halo
//     columns) into a RING-slot shared-memory ring, RING-1 slots ahead and
//     across groups, completing on one mbarrier per slot -- no per-lane
//     address arithmetic, LDGSTS or L1 allocation for the stream;
//   * the smem image of a slot follows the map ([k][patch][row][p+2 cols]
//     for SoA): lane (s, j) reads column j+1 of patch s and its right
//     neighbour j+2.
// Groups are aligned to the batch end (the last group starts at t1 - G), so
// every lane holds a real patch; a patch covered by two groups is computed
// twice with identical bits.  SoA / AoSoA batches of >= G patches; AoS and
// the rest take the cp.async kernel.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "fused2d.cuh"
#include "fused3d.cuh"  // mbarrier helpers

namespace fvb {

namespace pencil {

template <int P, int RS_, int N>
struct TmaGeo {
    static constexpr int G = 32 / P;
    static_assert(G * P == 32, "the TMA pencil needs p | 32 (one column per lane, full warps)");
    static constexpr int E = P + 2;                       // haloed row length
    static constexpr int RS = RS_;                        // rows per ring slot (one copy)
    static_assert((P + 2) % RS == 0, "a group's rows must fill whole slots");
    static constexpr int PAIRS = (P + 2) / RS;            // slots per group
    static constexpr int KS = G * RS * E;                 // doubles per unknown of one slot
    static constexpr int SLOT = (N * KS + 15) / 16 * 16;  // 128-byte ring slots
    static constexpr int HALF = N * G * P * 2;            // doubles of one halo box
    static constexpr unsigned SLOT_BYTES = N * KS * 8;
    static constexpr unsigned HALO_BYTES = 2 * HALF * 8;  // both column pairs
};

template <int P, int RING, int RS, int N>
struct alignas(128) TmaWarpSmem {
    using Tg = TmaGeo<P, RS, N>;
    double ring[RING][Tg::SLOT];             // [k][patch][row][col] (+ pad)
    double hl[Tg::HALF], hr[Tg::HALF];       // halo column pairs (see TmaSrc)
    double xf[N][Geo<P, 1>::XSP];            // x-face exchange + boundary faces (fused2d.cuh)
    unsigned long long mbar[RING];
};

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                     unsigned long long* m) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(slab::smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"(slab::smem_u32(m))
        : "memory");
}

// Consumer state of a warp's ring, persistent across groups.  The producer
// needs none: the slot to refill is always the one just consumed, and which
// (group, pair) goes into it follows from the consumer's row (TmaSrc::begin).
struct TmaStream {
    int cur;         // ring slot of the current row pair
    unsigned phase;  // bit r: parity of the next completion of slot r
};

// The ring holds RS haloed rows per slot, one tensor-map copy each; the
// first slot of a group also carries its two halo-column boxes.  No proxy
// fence before refilling a slot: its generic reads are ordered by the
// __syncwarp (the CUTLASS TMA-pipeline convention for consumer release).
// PM: patch-major batch (AoSoA, map [col][row][k][patch]): a slot is
// [patch][k][row][col] and a halo box [patch][k][row][2]; else (SoA, map
// [col][row][patch][k]) [k][patch][row][col] and [k][patch][row][2].
template <int P, int RING, int RS, bool PM, int N>
struct TmaSrc {
    static constexpr int D = RING - 1;  // prefetch distance in slots
    using Tg = TmaGeo<P, RS, N>;
    static_assert(D <= Tg::PAIRS, "the prefetch may not run more than one group ahead");
    static constexpr int SK = PM ? RS * Tg::E : Tg::KS;                // slot: unknown stride
    static constexpr int SS = PM ? N * RS * Tg::E : RS * Tg::E;        // slot: patch stride
    static constexpr int HK = PM ? 2 * P : 2 * 32;                     // halo: unknown stride
    static constexpr int HS = PM ? 2 * N * P : 2 * P;                  // halo: patch stride
    using Smem = TmaWarpSmem<P, RING, RS, N>;
    using Cx = Ctx<P, 1, RING, 1, N>;
    const Cx& c;
    Smem* S;
    const CUtensorMap* map_rows;
    const CUtensorMap* map_halo;
    TmaStream& st;
    int cur_patch;   // first patch of the current group
    int next_patch;  // first patch of the warp's next group, or -1

    // pair m of the group starting at patch `patch` into ring slot r (lane 0)
    __device__ __forceinline__ static void issue(const Cx& c, Smem* S, const CUtensorMap* rows,
                                                 const CUtensorMap* halo, int r, int patch, int m) {
        if (c.lane == 0) {
            const int c2 = PM ? 0 : patch, c3 = PM ? patch : 0;
            if (m == 0) {
                slab::mbar_expect_tx(&S->mbar[r], Tg::SLOT_BYTES + Tg::HALO_BYTES);
                tma4(S->hl, halo, 0, 1, c2, c3, &S->mbar[r]);
                tma4(S->hr, halo, P, 1, c2, c3, &S->mbar[r]);
            } else {
                slab::mbar_expect_tx(&S->mbar[r], Tg::SLOT_BYTES);
            }
            tma4(&S->ring[r][0], rows, 0, RS * m, c2, c3, &S->mbar[r]);
        }
    }
    // the first D pairs of the warp's first group into slots 0..D-1
    __device__ __forceinline__ static TmaStream prologue(const Cx& c, Smem* S, const CUtensorMap* rows,
                                                         const CUtensorMap* halo, int first_patch) {
        if (first_patch >= 0) {
#pragma unroll
            for (int m = 0; m < D; ++m) issue(c, S, rows, halo, m, first_patch, m);
        }
        return TmaStream{RING - 1, 0u};
    }
    __device__ __forceinline__ void halo(int, double (&q0)[N], double (&q1)[N], double (&q2)[N],
                                         double (&q3)[N]) const {
        // the halo columns complete with the group's first slot
        const int s0 = (st.cur + 1 == RING) ? 0 : st.cur + 1;
        slab::mbar_wait(&S->mbar[s0], (st.phase >> s0) & 1u);  // no phase flip: begin(0) consumes it
        const int i = (c.lane / P) * HS + 2 * c.j;  // lane (patch s, row j)
#pragma unroll
        for (int k = 0; k < N; ++k) {
            q0[k] = S->hl[k * HK + i];
            q1[k] = S->hl[k * HK + i + 1];
            q2[k] = S->hr[k * HK + i];
            q3[k] = S->hr[k * HK + i + 1];
        }
    }
    // haloed row r: a new slot every RS rows.  Refill the slot just finished
    // (st.cur) with pair r/RS + D: of this group, or of the warp's next one.
    __device__ __forceinline__ void begin(int r) const {
        if (r % RS == 0) {
            __syncwarp();  // every lane is done with the slot about to be refilled
            const int m = r / RS + D;
            if (m < Tg::PAIRS) {
                issue(c, S, map_rows, map_halo, st.cur, cur_patch, m);
            } else if (next_patch >= 0) {
                issue(c, S, map_rows, map_halo, st.cur, next_patch, m - Tg::PAIRS);
            }
            st.cur = (st.cur + 1 == RING) ? 0 : st.cur + 1;
            slab::mbar_wait(&S->mbar[st.cur], (st.phase >> st.cur) & 1u);
            st.phase ^= 1u << st.cur;
        }
    }
    // lane (s, j), row rr of the slot: s*SS + rr*E + j + 1
    __device__ __forceinline__ const double* at(int r) const {
        const int s = c.lane / P;
        return &S->ring[st.cur][s * SS + (r % RS) * Tg::E + c.j + 1];
    }
    __device__ __forceinline__ void row(int r, double (&q)[1][N]) const {
        const double* p = at(r);
#pragma unroll
        for (int k = 0; k < N; ++k) q[0][k] = p[k * SK];
    }
    __device__ __forceinline__ void right(int r, double (&q)[N]) const {
        const double* p = at(r) + 1;
#pragma unroll
        for (int k = 0; k < N; ++k) q[k] = p[k * SK];
    }
};

}  // namespace pencil

template <int P, int RING, int RS, int N>
constexpr size_t pencil_tma_smem() {
    return sizeof(pencil::TmaWarpSmem<P, RING, RS, N>);
}

// One warp per CTA; groups g = blockIdx.x, + gridDim.x, ...; group g covers
// patches min(t0 + g*G, t1 - G) + [0, G).
template <class Eq, int P, int RED, int MINB, int RING, int RS, bool PM>
__global__ void __launch_bounds__(32, MINB)
    fused2d_pencil_tma_kernel(StepArgs a, const __grid_constant__ CUtensorMap rows,
                              const __grid_constant__ CUtensorMap halo) {
    using namespace pencil;
    using Gm = Geo<P, 1>;
    constexpr int L = Gm::L, G = Gm::G;
    constexpr int N = Eq::kUnknowns;
    static_assert(Gm::FULL, "full warps only");
    static_assert(Eq::kDim == 2, "the pencil walk is 2D");
    static_assert(RED != kReduceFiltered || kHasLambdaBelow<Eq>, "filtered reduction needs lambda_below");
    const Eq eq(a.gamma);

    extern __shared__ __align__(128) unsigned char smem_raw[];
    auto* S = reinterpret_cast<TmaWarpSmem<P, RING, RS, N>*>(smem_raw);

    const int lane = threadIdx.x;
    const int sub = lane / L;
    const long long t0 = a.t0, t1 = a.t1;
    const long long groups = (t1 - t0 + G - 1) / G;
    const long long t_last = t1 - G;
    const long long gstep = gridDim.x;

    Ctx<P, 1, RING, 1, N> c;
    c.sIn = a.in.k;
    c.sOut = a.out.k;
    const double scale = step_scale(a);
    const bool fast = step_fast(a, scale);
    c.scale = scale;
    c.hscale = 0.5 * scale;
    c.lane = lane;
    c.j = lane - sub * L;
    c.hbase = sub * (P + 1);
    c.valid = true;
    c.out16 = false;
    c.sm = nullptr;  // no cp.async ring
    c.xf = S->xf;

    auto first_of = [&](long long g) {
        const long long f = t0 + g * G;
        return f < t_last ? f : t_last;
    };

    if (lane == 0) {
#pragma unroll
        for (int r = 0; r < RING; ++r) slab::mbar_init(&S->mbar[r], 1);
        slab::fence_mbar_init();
    }
    __syncwarp();

    double red = 0.0;
    LamFilter lf;
    lf.init();
    long long g = blockIdx.x;
    TmaStream stream =
        TmaSrc<P, RING, RS, PM, N>::prologue(c, S, &rows, &halo, g < groups ? (int)first_of(g) : -1);
    for (; g < groups; g += gstep) {
        const long long patch = first_of(g) + sub;
        c.qi = a.q_in + patch * a.in.p;
        c.qo = a.q_out + patch * a.out.p;
        bool lane_fast = fast;
        if (a.dt_patch != nullptr) {  // local time stepping: this lane's patch's dt
            c.scale = patch_scale(a, scale, patch);
            c.hscale = 0.5 * c.scale;
            lane_fast = step_fast(a, c.scale);
        }
        bool bad = !lane_fast;
        const TmaSrc<P, RING, RS, PM, N> src{c, S, &rows, &halo, stream, (int)first_of(g),
                                             g + gstep < groups ? (int)first_of(g + gstep) : -1};
        double pred;
        if constexpr (kHasFastPath<Eq>) {
            const LamFilter lf0 = lf;
            pred = group<P, 1, RING, RED, XReal>(c, src, eq, lf, bad);
            if (__any_sync(0xffffffffu, bad)) {  // IEEE redo from global memory
                bool unused = false;
                const DirectSrc<P, 1, RING, 1, N> direct{c};
                lf = lf0;
                pred = group<P, 1, RING, RED, double>(c, direct, eq, lf, unused);
            }
        } else {  // a policy without the fast-path hook: IEEE double throughout
            pred = group<P, 1, RING, RED, double>(c, src, eq, lf, bad);
        }
        running_max(red, pred);
        if (RED == kReduceAll && a.lam_patch != nullptr) {  // segmented max over the L lanes of a patch
            double v = pred;
#pragma unroll
            for (int off = 1; off < L; off <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, off);
                if (c.j + off < L) running_max(v, o);
            }
            if (c.j == 0) a.lam_patch[patch] = v;
        }
    }
    if (RED != kReduceNone && a.lam_bits != nullptr) reduce_epilogue<false>(a, red);
}

}  // namespace fvb
