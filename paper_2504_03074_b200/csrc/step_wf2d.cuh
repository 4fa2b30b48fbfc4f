// 2D wavefront temporal blocking: T leapfrog steps per pass over HBM (sm_100a).
//
// A CTA = 1 producer warp + NW consumer warps.  The producer streams rows of
// W^s, W^{s-1}, f and acc into a ring of STAGES shared-memory row stages with
// cp.async.bulk (completion on "full" mbarriers; a stage is refilled once all
// consumer warps arrived on its "empty" mbarrier).  Each consumer warp owns a
// 64-column strip (lane = 2 adjacent columns) and marches it down the rows
// with a software wavefront: at input row r it advances time level t at row
// r - t for t = 1..T, keeping three rows of every level in registers
// (x-neighbours by warp shuffles).  Strips overlap by 2T columns so each warp
// is self-contained (no __syncthreads in the loop); a warp's output is the
// 64 - 2T columns in the middle of its strip.  The filter accumulation of a
// row collects c_{s+t} W^{s+t} from each level as the wavefront passes (same
// order as the reference), so only W^{s+T-1}, W^{s+T} and acc are written:
//
//     HBM per point and pass: read W^s, W^{s-1}, f, acc; write W^{s+T-1}, W^{s+T}, acc
//     = 56 B per T updates (T = 4: 14 B/update vs 48 B for one step per pass).
//
// Every value is produced by the same explicitly rounded operations in the
// same order as the reference (bitwise parity); Dirichlet and out-of-domain
// points of every intermediate level are forced to exactly 0.
#pragma once

namespace wf2d {

using bulk::bulk_g2s;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::smem_u32;
using bulk::update_point;

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// row-segment padding in the stages (elements; bulk copies need 16-B aligned destinations)
#ifndef WHB_WF_PAD
#define WHB_WF_PAD 16
#endif

template <int T, int NW>
struct Lay {
    static constexpr int OW = 64 - 2 * T;          // output columns per warp
    static constexpr int CW = NW * OW;             // output columns per CTA
    static constexpr int SEG = CW + 2 * T;         // staged columns per row (start at c0 - T)
    static constexpr int SEGP = (SEG + WHB_WF_PAD - 1) / WHB_WF_PAD * WHB_WF_PAD;
    static constexpr int CWP = (CW + WHB_WF_PAD - 1) / WHB_WF_PAD * WHB_WF_PAD;
    static constexpr int STAGE = 3 * SEGP + CWP;   // W^s | W^{s-1} | f | acc
    static constexpr int THREADS = 32 * (NW + 1);
};

template <int T, int NW, int ST>
constexpr size_t wf_smem_bytes() {
    return (size_t)ST * Lay<T, NW>::STAGE * sizeof(double) + 2 * ST * sizeof(uint64_t);
}

// Per-pass scalars of a single-member launch, passed as kernel parameters: the update chain
// reads them straight from the constant bank instead of holding ~28 registers per thread.
struct WfScal {
    double h[5], cs[5], ca[5];  // level t = 1..T: dt^2 factor, forcing cos factor, filter weight
    double acc0, osc;
};
// Batched launches: one WfScal per member of the launch (blockIdx.z), also as kernel parameters
// (8.7 KB; CUDA 12.1+ allows 32 KB): CTA-uniform, so they stay in the constant bank / uniform
// registers instead of ~30 per-thread registers loaded from the member table.
constexpr int WF_TAB = 64;
template <int N>
struct WfTab {
    WfScal m[N];
};

// K1: kind of the first step of the pass (FIRST when s == 0); K2: kind of the last (LAST ends the solve).
// PS: one member per launch (scalars in ps.m[0]); otherwise up to WF_TAB members, scalars of member
// blockIdx.z in ps.m[blockIdx.z].
// GM: geometry mode -- 0 generic; 1 square cells (both axes carry bitwise-equal taps): one centre
// product per point; 2 square cells and c^2 == 1 (no c^2 product: a dependent fp64 multiply and two
// selects less per update).
template <int T, int NW, int ST, int K1, int K2, bool ZF, bool PS = false, int GM = 0>
// steady-state row-loop unroll (measured: 3, the period of the level queues, is within noise
// of 2 -- 321.4 vs 322.3 Gpts/s on config 2, 302.9 vs 299.9 on config 5; the queue shifts are
// renames either way)
#ifndef WHB_WF_UNROLL
#define WHB_WF_UNROLL 2
#endif
#define WF_PRAGMA_(x) _Pragma(#x)
#define WF_UNROLL_(n) WF_PRAGMA_(unroll n)
#define WF_UNROLL(n) WF_UNROLL_(n)
// WHB_WF_CLEAN=1: in batched launches (scalars from the member table), rows whose levels are all
// interior (and strips wholly interior in x) run a row body without the zeroing selects.
// Measured: batched config 5 296 -> 306 Gpts/s; single-member config 2 343 -> 329, so the
// single-member (PS) kernels keep one row body.
#ifndef WHB_WF_CLEAN
#define WHB_WF_CLEAN 1
#endif
// WHB_WF_WARMSKIP=0: compute every level on every input row (the pre-cone rows too)
#ifndef WHB_WF_WARMSKIP
#define WHB_WF_WARMSKIP 1
#endif
#ifndef WHB_WF_MINB
#define WHB_WF_MINB 3
#endif
__global__ void __launch_bounds__(Lay<T, NW>::THREADS, WHB_WF_MINB)
    wf2d_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin, int i_end,
                int chunk_len, int part_off, const WfTab<PS ? 1 : WF_TAB> ps) {
    using L = Lay<T, NW>;
    constexpr bool SQ = GM >= 1;
    constexpr int C2M = GM == 2 ? 0 : -1;
    constexpr bool USE_CLEAN = WHB_WF_CLEAN && !PS;
    constexpr int DL = T;  // output row lag: level t of input row r is computed at row r - t
    static_assert(T % 2 == 0 && T >= 2 && T <= 12, "T even (pair-aligned output columns)");
    static_assert(ST >= DL + 2, "stages must cover rows r-DL .. r plus one in flight");
    extern __shared__ __align__(128) double smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)ST * L::STAGE);
    uint64_t *empty = full + ST;

    const Member m = members[member_off + blockIdx.z];
    // warp index via a shuffle: provably warp-uniform, so the role branch below is not divergent
    // and the wavefront shuffles need no convergence barriers
    const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int c0 = blockIdx.x * L::CW;  // first output column of this CTA
    const int i0 = i_begin + blockIdx.y * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    const bool fpi_last = (K2 == K_LAST && m.out_mode == WHB_OUT_FPI);
    if (i0 >= i1) {
        if (fpi_last && threadIdx.x == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    const double *wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *wA = level_ptr(m, s + T - 1);  // second-to-last level written
    double *wB = level_ptr(m, s + T);      // last level written
    const long long S0 = g.S0;
    constexpr bool LOAD_PA = (K1 != K_FIRST);
    constexpr uint32_t stage_bytes = (uint32_t)((L::SEG + (LOAD_PA ? L::SEG : 0) + (ZF ? 0 : L::SEG) +
                                                 (LOAD_PA ? L::CW : 0)) * 8);
    // rows r = i0-T .. i1+T-1 enter the wavefront (planes; out-of-allocation rows are clamped:
    // their values only feed out-of-domain rows, which are forced to 0)
    const int r0 = i0 - T;
    const int nrows = i1 - i0 + T + DL;

    if (threadIdx.x == 0) {
        for (int q = 0; q < ST; ++q) {
            mbar_init(full + q, 1);
            mbar_init(empty + q, NW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double rsum = 0.0;
    if (warp == NW) {
        // ---------------- producer warp: one elected lane streams the rows
        if (lane == 0) {
            for (int idx = 0; idx < nrows; ++idx) {
                const int slot = idx % ST;
                if (idx >= ST) mbar_wait(empty + slot, ((idx / ST) - 1) & 1);
                int plane = r0 + idx;
                plane = max(0, min(plane, g.i_hi));  // stays inside the allocated planes
                double *st = smem + (size_t)slot * L::STAGE;
                const long long off = (long long)plane * S0 + (c0 - T);
                mbar_expect_tx(full + slot, stage_bytes);
                bulk_g2s(st, wcur + off, L::SEG * 8, full + slot);
                if (LOAD_PA) bulk_g2s(st + L::SEGP, wprv + off, L::SEG * 8, full + slot);
                if (!ZF) bulk_g2s(st + 2 * L::SEGP, m.f + off, L::SEG * 8, full + slot);
                if (LOAD_PA) bulk_g2s(st + 3 * L::SEGP, m.acc + (long long)plane * S0 + c0, L::CW * 8, full + slot);
            }
        }
        __syncwarp();
    } else {
        // ---------------- consumer warp
        const int xs = warp * L::OW;          // strip start inside the staged segment
        const int col = c0 - T + xs + 2 * lane;  // global column of this lane's first point
        const bool own = (2 * lane >= T) && (2 * lane < 64 - T);
        const bool okc0 = own && col >= 1 && col < g.n2 - 1;
        const bool okc1 = own && col + 1 >= 1 && col + 1 < g.n2 - 1;
        const bool in0 = col >= 1 && col < g.n2 - 1;          // interior column (any level)
        const bool in1 = col + 1 >= 1 && col + 1 < g.n2 - 1;
        // every lane of this warp interior in x: then only the (warp-uniform) row test remains
        const bool warp_in = __all_sync(0xffffffffu, in0 && in1);
        // per-level scalars: level t (1..T) is produced by step s+t-1
        double hcoef[T + 1], cosl[T + 1], cacc[T + 1];
        const WfScal &sc = ps.m[PS ? 0 : blockIdx.z];
#pragma unroll
        for (int t = 1; t <= T; ++t) {
            hcoef[t] = sc.h[t];
            cosl[t] = sc.cs[t];
            cacc[t] = sc.ca[t];
        }
        const double acc0 = sc.acc0;
        const double oscale = sc.osc;
        // a strip wholly past the last interior column (the ragged right edge of the grid) has
        // nothing to write: it only keeps the stage barriers' arrival counts, so the issue slots go
        // to the SM's other warps
        const bool idle = __all_sync(0xffffffffu, !(okc0 || okc1));
        if (idle) {
            for (int idx = 0; idx < nrows; ++idx) {
                mbar_wait(full + (idx % ST), (idx / ST) & 1);
                __syncwarp();
                if (idx >= T && lane == 0) mbar_arrive(empty + ((idx - T) % ST));
            }
            if (lane == 0)
                for (int idx = max(0, nrows - T); idx < nrows; ++idx) mbar_arrive(empty + (idx % ST));
            __syncwarp();
        } else {
        // level queues: Q[t][0..2] = level t at rows (r-t-2, r-t-1, r-t); Q[0] = W^s
            double2 Q[T + 1][3];
            double2 A[T];  // A[t-1] = partial filter sum of row r-t
    #pragma unroll
            for (int t = 0; t <= T; ++t)
    #pragma unroll
                for (int u = 0; u < 3; ++u) Q[t][u] = make_double2(0.0, 0.0);
    #pragma unroll
            for (int t = 0; t < T; ++t) A[t] = make_double2(0.0, 0.0);
    
            // last pass: v (W^0, needed for the residual / x - W(x,0)) of the row finishing in the
            // NEXT iteration is loaded one iteration ahead so its HBM latency hides behind a row
            constexpr bool NEED_V = (K2 == K_LAST);
            const bool want_v = NEED_V && m.out_mode != WHB_OUT_PLAIN && own;
            auto vload = [&](int orow) -> double2 {
                if (!want_v || orow < i0 || orow >= i1) return make_double2(0.0, 0.0);
                return *reinterpret_cast<const double2 *>(m.v + (long long)orow * S0 + col);
            };
            double2 vcur = vload(r0 - T);
            // one input row of the wavefront (its stage already waited for)
            // WARM (input rows idx < 2T): level t at row r - t is only needed (by the outputs
            // [i0, i1) through the stencil cone) from row i0 - (T - t) on, i.e. for idx >= 2t; the
            // earlier rows of each level are skipped (left 0) instead of computed.
            // CLEAN: every lane interior in x (warp_in) and the rows r-T .. r-1 of this input row's
            // levels all interior: no zeroing selects
            auto row_step = [&](const int idx, auto warm_tag, auto clean_tag) {
                constexpr bool WARM = decltype(warm_tag)::value;
                constexpr bool CLEAN = decltype(clean_tag)::value;
                const int r = r0 + idx;
                const int slot = idx % ST;
                const double2 vnext = vload(r + 1 - T);
                const double *st = smem + (size_t)slot * L::STAGE;
                // W^s row r into the level-0 queue
                Q[0][0] = Q[0][1];
                Q[0][1] = Q[0][2];
                Q[0][2] = *reinterpret_cast<const double2 *>(st + xs + 2 * lane);
                double2 nw[T + 1];  // newest value of each level this row
    #pragma unroll
                for (int t = 1; t <= T; ++t) {
                    const int row = r - t;  // plane of level t computed now
                    if (WARM && idx < 2 * t) {  // warp-uniform: row below the cone of the outputs
                        nw[t] = make_double2(0.0, 0.0);
                    } else {
                    // stage holding row `row` (rows r-T..r are resident)
                    const double *sr = smem + (size_t)((idx - t + ST) % ST) * L::STAGE;
                    const double2 cm = Q[t - 1][0], cc = Q[t - 1][1], cp = Q[t - 1][2];
                    // x neighbours of the centre row of level t-1
                    const double xl = __shfl_up_sync(0xffffffffu, cc.y, 1);
                    const double xh = __shfl_down_sync(0xffffffffu, cc.x, 1);
                    double2 fv = make_double2(0.0, 0.0);
                    if (!ZF) fv = *reinterpret_cast<const double2 *>(sr + 2 * L::SEGP + xs + 2 * lane);
                    double2 pv;  // level t-2 at this row (W^{s-1} for t = 1)
                    if (t == 1) {
                        pv = LOAD_PA ? *reinterpret_cast<const double2 *>(sr + L::SEGP + xs + 2 * lane)
                                     : make_double2(0.0, 0.0);
                    } else {
                        pv = (t == 2) ? Q[0][0] : Q[t - 2][0];
                    }
                    const bool firstk = (K1 == K_FIRST) && (t == 1);
                    double a, b;
                    if (firstk) {
                        a = update_point<K_FIRST, ZF, false, SQ, C2M>(g, cm.x, cc.x, cp.x, 0.0, 0.0, xl, cc.y, fv.x, 0.0,
                                                             hcoef[t], cosl[t]);
                        b = update_point<K_FIRST, ZF, false, SQ, C2M>(g, cm.y, cc.y, cp.y, 0.0, 0.0, cc.x, xh, fv.y, 0.0,
                                                             hcoef[t], cosl[t]);
                    } else {
                        a = update_point<K_MID, ZF, false, SQ, C2M>(g, cm.x, cc.x, cp.x, 0.0, 0.0, xl, cc.y, fv.x, pv.x,
                                                           hcoef[t], cosl[t]);
                        b = update_point<K_MID, ZF, false, SQ, C2M>(g, cm.y, cc.y, cp.y, 0.0, 0.0, cc.x, xh, fv.y, pv.y,
                                                           hcoef[t], cosl[t]);
                    }
                    if (CLEAN) {
                        nw[t] = make_double2(a, b);
                    } else {
                        const bool rin = (row >= g.i_lo) && (row < g.i_hi);
                        if (rin && warp_in) nw[t] = make_double2(a, b);  // uniform: no per-lane selects
                        else nw[t] = make_double2((rin && in0) ? a : 0.0, (rin && in1) ? b : 0.0);
                    }
                    }
                    Q[t][0] = Q[t][1];
                    Q[t][1] = Q[t][2];
                    Q[t][2] = nw[t];
                }
                // filter sums: row r-t gets c_{s+t} * level t (levels in increasing order per row)
    #pragma unroll
                for (int t = T; t >= 2; --t) {
                    A[t - 1].x = whb_add(A[t - 2].x, whb_mul(cacc[t], nw[t].x));
                    A[t - 1].y = whb_add(A[t - 2].y, whb_mul(cacc[t], nw[t].y));
                }
                {
                    double2 init;
                    if (K1 == K_FIRST) {  // c0 * W^0 (timestep.py:284), W^0 = level 0 at row r-1
                        init = make_double2(whb_mul(acc0, Q[0][1].x), whb_mul(acc0, Q[0][1].y));
                    } else {
                        const double *sr1 = smem + (size_t)((idx - 1 + ST) % ST) * L::STAGE;
                        const int ao = xs + 2 * lane - T;  // acc segment starts at c0 (= strip offset T)
                        init = (ao >= 0 && ao + 1 < L::CW) ? *reinterpret_cast<const double2 *>(sr1 + 3 * L::SEGP + ao)
                                                           : make_double2(0.0, 0.0);
                    }
                    A[0].x = whb_add(init.x, whb_mul(cacc[1], nw[1].x));
                    A[0].y = whb_add(init.y, whb_mul(cacc[1], nw[1].y));
                }
                // finished row r-T: write W^{s+T-1}, W^{s+T}, acc (or the pass output)
                const int orow = r - T;
                if (orow >= i0 && orow < i1) {
                    const long long p = (long long)orow * S0 + col;
                    const double2 wa2 = Q[T - 1][1];
                    const double2 wb2 = nw[T];
                    const double2 ac = A[T - 1];
                    if (K2 == K_MID) {
                        if (okc0 && okc1) {
                            *reinterpret_cast<double2 *>(wA + p) = wa2;
                            *reinterpret_cast<double2 *>(wB + p) = wb2;
                            *reinterpret_cast<double2 *>(m.acc + p) = ac;
                        } else {
                            if (okc0) { wA[p] = wa2.x; wB[p] = wb2.x; m.acc[p] = ac.x; }
                            if (okc1) { wA[p + 1] = wa2.y; wB[p + 1] = wb2.y; m.acc[p + 1] = ac.y; }
                        }
                    } else {
                        const double o0 = whb_mul(oscale, ac.x);
                        const double o1 = whb_mul(oscale, ac.y);
                        if (m.out_mode == WHB_OUT_FPI) {
                            if (okc0) { const double d = o0 - vcur.x; rsum += d * d; m.v[p] = o0; }
                            if (okc1) { const double d = o1 - vcur.y; rsum += d * d; m.v[p + 1] = o1; }
                        } else if (m.out_mode == WHB_OUT_AV) {
                            if (okc0) m.dst[p] = whb_sub(vcur.x, o0);
                            if (okc1) m.dst[p + 1] = whb_sub(vcur.y, o1);
                        } else {
                            if (okc0) m.dst[p] = o0;
                            if (okc1) m.dst[p + 1] = o1;
                        }
                    }
                }
                vcur = vnext;
                // the stage of row r-T is no longer needed by this warp
                __syncwarp();
                if (idx >= T && lane == 0) mbar_arrive(empty + ((idx - T) % ST));
            };
            const int nwarm = WHB_WF_WARMSKIP ? min(nrows, 2 * T) : 0;
            int idx = 0;
            for (; idx < nwarm; ++idx) {
                mbar_wait(full + (idx % ST), (idx / ST) & 1);
                row_step(idx, std::true_type{}, std::false_type{});
            }
            WF_UNROLL(WHB_WF_UNROLL)
            for (; idx < nrows; ++idx) {
                mbar_wait(full + (idx % ST), (idx / ST) & 1);
                if constexpr (USE_CLEAN) {
                    const int r = r0 + idx;
                    if (warp_in && r - T >= g.i_lo && r - 1 < g.i_hi) row_step(idx, std::false_type{}, std::true_type{});
                    else row_step(idx, std::false_type{}, std::false_type{});
                } else {
                    row_step(idx, std::false_type{}, std::false_type{});
                }
            }
            // release the stages still held (rows nrows-T .. nrows-1) so the producer never blocks
            if (lane == 0)
                for (int idx = max(0, nrows - T); idx < nrows; ++idx) mbar_arrive(empty + (idx % ST));
            __syncwarp();
        }
    }
    if (fpi_last) {
        const double tsum = block_sum(rsum);
        if (threadIdx.x == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = tsum;
    }
}

}  // namespace wf2d
