// Fused leapfrog + filter step, TMA bulk-copy pipelined (sm_100a).
//
// One CTA owns a tile of BY rows (axis 1; 1 in 2D) x TX columns (axis 2,
// contiguous) and marches it through a chunk of axis-0 planes.  For every
// plane p it needs W^n at planes p-1, p, p+1 (with a 1-cell halo in axes 1
// and 2 at plane p) and W^{n-1}, f, acc at plane p.  Those rows are moved
// HBM -> shared memory by the bulk-copy (TMA) engine (`cp.async.bulk`, one
// instruction per row segment) into a ring of STAGES plane-stages, each
// completing on its own mbarrier with a transaction-byte count; so only one
// thread issues loads and up to STAGES-3 planes are in flight per CTA while
// the other threads compute.  Results (W^{n+1}, acc) are written with 16-byte
// vector stores straight from registers (each point is written exactly once).
//
// Every thread updates two adjacent points (k, k+1).  Arithmetic is the
// reference order with explicitly rounded __dadd_rn/__dmul_rn (bitwise parity).
#pragma once

namespace bulk {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WHB_WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WHB_WAIT%=;\n}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// TMA tensor load of a 3D box (coordinates innermost first; out-of-bounds elements read as 0).
__device__ __forceinline__ void tma_load_3d(void *sdst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(sdst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int TX, int BY, bool A1>
struct Layout {
    static constexpr int WX = TX + 4;                 // w row segment: columns k0-2 .. k0+TX+1
    static constexpr int WR = A1 ? BY + 2 : 1;        // w rows: j0-1 .. j0+BY (3D) or the row (2D)
    static constexpr int W_ELEMS = WR * WX;
    static constexpr int W_PAD = (W_ELEMS + 15) / 16 * 16;  // keep every sub-buffer 128-B aligned (TMA)
    static constexpr int T_ELEMS = BY * TX;           // prev / f / acc tile
    static constexpr int STAGE_ELEMS = W_PAD + 3 * T_ELEMS;
    static constexpr int THREADS = TX * BY / 2;
};

template <int TX, int BY, int STAGES, bool A1>
constexpr size_t bulk_smem_bytes() {
    return (size_t)STAGES * Layout<TX, BY, A1>::STAGE_ELEMS * sizeof(double) + STAGES * sizeof(uint64_t);
}

// One point of the fused update, reference order (grid.py:357-366, timestep.py:137-140, 284-300).
// SQ: every axis carries the same taps (square / cubic cells, clo_a and cmid_a bitwise equal):
// the centre product cmid*wc is formed once and added per axis — the same values, in the same
// order, as the reference's per-axis products.
// C2: -1 = multiply by c^2 when g.use_c2 (runtime), 0 = never (c^2 == 1: x * 1.0 == x, so skipping
// the product is bitwise neutral), 1 = always.
template <int KIND, bool ZF, bool A1, bool SQ = false, int C2 = -1>
__device__ __forceinline__ double update_point(const Geom &g, double wm, double wc, double wp, double yl,
                                               double yh, double xl, double xh, double fv, double wpv,
                                               double h, double cosn) {
    // The reference sums into np.zeros (0.0 + first product); that add only turns a -0.0 first
    // product into +0.0, and it is dropped here because the returned update cannot see it: the
    // sums differ only when EVERY product is -0.0, which includes cmid*wc (cmid < 0), so wc == +0.0;
    // then 2*wc - wpv (or wc itself on the first step) is +0.0 or nonzero, never -0.0, and adding
    // h*d = +-0.0 to it gives the same bits either way.
    double lap;
    if constexpr (SQ) {
        const double mc = whb_mul(g.cmid0, wc);
        lap = whb_mul(g.clo0, wm);
        lap = whb_add(lap, mc);
        lap = whb_add(lap, whb_mul(g.clo0, wp));
        if (A1) {
            lap = whb_add(lap, whb_mul(g.clo0, yl));
            lap = whb_add(lap, mc);
            lap = whb_add(lap, whb_mul(g.clo0, yh));
        }
        lap = whb_add(lap, whb_mul(g.clo0, xl));
        lap = whb_add(lap, mc);
        lap = whb_add(lap, whb_mul(g.clo0, xh));
    } else {
        lap = whb_mul(g.clo0, wm);
        lap = whb_add(lap, whb_mul(g.cmid0, wc));
        lap = whb_add(lap, whb_mul(g.clo0, wp));
        if (A1) {
            lap = whb_add(lap, whb_mul(g.clo1, yl));
            lap = whb_add(lap, whb_mul(g.cmid1, wc));
            lap = whb_add(lap, whb_mul(g.clo1, yh));
        }
        lap = whb_add(lap, whb_mul(g.clo2, xl));
        lap = whb_add(lap, whb_mul(g.cmid2, wc));
        lap = whb_add(lap, whb_mul(g.clo2, xh));
    }
    if (C2 < 0 ? g.use_c2 != 0 : C2 != 0) lap = whb_mul(lap, g.c2);
    if (KIND == K_FIRST) {
        const double d = ZF ? lap : whb_sub(lap, fv);
        return whb_add(wc, whb_mul(h, d));
    }
    const double d = ZF ? lap : whb_sub(lap, whb_mul(fv, cosn));
    return whb_add(whb_sub(whb_mul(2.0, wc), wpv), whb_mul(h, d));
}

// TENSOR = false: one cp.async.bulk per row segment (any member table, 2D rows);
// TENSOR = true : one cp.async.bulk.tensor.3d box per array and plane (3D, member 0's
//                 tensor maps passed as __grid_constant__ parameters).
template <int TX, int BY, int STAGES, bool A1, int KIND, bool ZF, bool TENSOR>
__global__ void __launch_bounds__(Layout<TX, BY, A1>::THREADS)
    step_bulk_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin,
                     int i_end, int chunk_len, int JT, int part_off, const __grid_constant__ CUtensorMap tm_w,
                     const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
                     const __grid_constant__ CUtensorMap tm_a) {
    using L = Layout<TX, BY, A1>;
    static_assert(STAGES >= 4, "need >= 4 stages (3 live planes + 1 in flight)");
    extern __shared__ __align__(128) double smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)STAGES * L::STAGE_ELEMS);

    const Member m = members[member_off + blockIdx.z];
    const int tid = threadIdx.x;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = blockIdx.x * TX;
    const int j0 = A1 ? jt * BY : 0;
    const int i0 = i_begin + ch * chunk_len;
    const int i1 = min(i_end, i0 + chunk_len);
    if (i0 >= i1) {  // empty chunk (uniform per CTA): keep its residual slot at zero
        if (KIND == K_LAST && m.out_mode == WHB_OUT_FPI && threadIdx.x == 0)
            m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }

    const double *wcur = level_ptr(m, s);
    const double *wprv = level_ptr(m, s - 1);
    double *wnxt = level_ptr(m, s + 1);
    const double cosn = (KIND == K_FIRST) ? 1.0 : m.cos_f[s];
    const double h = (KIND == K_FIRST) ? m.half_dt2 : m.dt2;
    const double acc0 = m.acc_c[0];
    const double accn = m.acc_c[s + 1];
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr bool LOAD_PA = (KIND != K_FIRST);
    const uint32_t stage_bytes = (uint32_t)(L::W_ELEMS * 8 + (LOAD_PA ? 2 * L::T_ELEMS * 8 : 0) +
                                            (ZF ? 0 : L::T_ELEMS * 8));
    // planes i0-1 .. i1 are staged; local stage t <-> plane i0-1+t
    const int n_stages_total = i1 - i0 + 2;

    auto issue = [&](int t) {
        const int slot = t % STAGES;
        double *st = smem + (size_t)slot * L::STAGE_ELEMS;
        const long long pl = (long long)(i0 - 1 + t) * S0;
        uint64_t *bar = bars + slot;
        mbar_expect_tx(bar, stage_bytes);
        if constexpr (TENSOR) {
            const int plane = i0 - 1 + t;
            double *tp = st + L::W_PAD;
            tma_load_3d(st, &tm_w, k0 - 2, j0 - 1, plane, bar);
            if (LOAD_PA) {
                tma_load_3d(tp, &tm_p, k0, j0, plane, bar);
                tma_load_3d(tp + 2 * L::T_ELEMS, &tm_a, k0, j0, plane, bar);
            }
            if (!ZF) tma_load_3d(tp + L::T_ELEMS, &tm_f, k0, j0, plane, bar);
            return;
        }
        if constexpr (!TENSOR) {
#pragma unroll 1
        for (int r = 0; r < L::WR; ++r) {
            const int j = A1 ? j0 - 1 + r : 0;
            bulk_g2s(st + r * L::WX, wcur + pl + (long long)j * P + (k0 - 2), L::WX * 8, bar);
        }
        double *tp = st + L::W_PAD;
#pragma unroll 1
        for (int r = 0; r < BY; ++r) {
            const long long off = pl + (long long)(j0 + r) * P + k0;
            if (LOAD_PA) {
                bulk_g2s(tp + r * TX, wprv + off, TX * 8, bar);
                bulk_g2s(tp + 2 * L::T_ELEMS + r * TX, m.acc + off, TX * 8, bar);
            }
            if (!ZF) bulk_g2s(tp + L::T_ELEMS + r * TX, m.f + off, TX * 8, bar);
        }
        }
    };

    if (tid == 0) {
        for (int t = 0; t < STAGES; ++t) mbar_init(bars + t, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        const int pro = min(n_stages_total, STAGES);
        for (int t = 0; t < pro; ++t) issue(t);
    }
    __syncthreads();

    // thread -> (row ty, column pair)
    const int ty = A1 ? tid / (TX / 2) : 0;
    const int tx2 = A1 ? tid % (TX / 2) : tid;
    const int kl = 2 * tx2;          // local column of the first point
    const int k = k0 + kl;
    const int j = j0 + ty;
    const bool row_ok = !A1 || (j >= g.j_lo && j < g.j_hi);
    const bool ok0 = row_ok && (k >= 1) && (k < g.n2 - 1);
    const bool ok1 = row_ok && (k + 1 < g.n2 - 1);
    const int wr = A1 ? ty + 1 : 0;  // center row inside the w segment
    const int wc = kl + 2;           // center column inside the w segment
    double rsum = 0.0;
    // last step: v of the next plane is loaded one plane ahead (hides its HBM latency)
    const bool want_v = (KIND == K_LAST) && m.out_mode != WHB_OUT_PLAIN && row_ok && (ok0 || ok1);
    const long long pbase = (long long)j * P + k;
    double2 vcur = want_v ? *reinterpret_cast<const double2 *>(m.v + (long long)i0 * S0 + pbase) : make_double2(0.0, 0.0);

    for (int i = i0; i < i1; ++i) {
        const int t = i - i0 + 1;  // stage of plane i
        const double2 vnext = (want_v && i + 1 < i1)
                                  ? *reinterpret_cast<const double2 *>(m.v + (long long)(i + 1) * S0 + pbase)
                                  : make_double2(0.0, 0.0);
        if (i > i0) {
            __syncthreads();  // everyone is done with plane i-1: stage of plane i-2 is free
            if (tid == 0) {
                const int tn = t + STAGES - 2;  // = (stage of plane i-2) + STAGES
                if (tn < n_stages_total) {
                    fence_proxy_async();
                    issue(tn);
                }
            }
        }
        if (i == i0) {
            mbar_wait(bars + ((t - 1) % STAGES), ((t - 1) / STAGES) & 1);
            mbar_wait(bars + (t % STAGES), (t / STAGES) & 1);
        }
        mbar_wait(bars + ((t + 1) % STAGES), ((t + 1) / STAGES) & 1);

        const double *sm_m = smem + (size_t)((t - 1) % STAGES) * L::STAGE_ELEMS;
        const double *sm_c = smem + (size_t)(t % STAGES) * L::STAGE_ELEMS;
        const double *sm_p = smem + (size_t)((t + 1) % STAGES) * L::STAGE_ELEMS;
        const double *tpc = sm_c + L::W_PAD;

        const double2 c2 = *reinterpret_cast<const double2 *>(sm_c + wr * L::WX + wc);
        const double xl = sm_c[wr * L::WX + wc - 1];
        const double xh = sm_c[wr * L::WX + wc + 2];
        const double2 m2 = *reinterpret_cast<const double2 *>(sm_m + wr * L::WX + wc);
        const double2 p2 = *reinterpret_cast<const double2 *>(sm_p + wr * L::WX + wc);
        double2 yl2 = make_double2(0.0, 0.0), yh2 = make_double2(0.0, 0.0);
        if (A1) {
            yl2 = *reinterpret_cast<const double2 *>(sm_c + (wr - 1) * L::WX + wc);
            yh2 = *reinterpret_cast<const double2 *>(sm_c + (wr + 1) * L::WX + wc);
        }
        double2 f2 = make_double2(0.0, 0.0), pv2 = make_double2(0.0, 0.0), a2 = make_double2(0.0, 0.0);
        if (!ZF) f2 = *reinterpret_cast<const double2 *>(tpc + L::T_ELEMS + ty * TX + kl);
        if (LOAD_PA) {
            pv2 = *reinterpret_cast<const double2 *>(tpc + ty * TX + kl);
            a2 = *reinterpret_cast<const double2 *>(tpc + 2 * L::T_ELEMS + ty * TX + kl);
        }
        const double n0 = update_point<KIND, ZF, A1>(g, m2.x, c2.x, p2.x, yl2.x, yh2.x, xl, c2.y, f2.x, pv2.x, h, cosn);
        const double n1 = update_point<KIND, ZF, A1>(g, m2.y, c2.y, p2.y, yl2.y, yh2.y, c2.x, xh, f2.y, pv2.y, h, cosn);

        const long long p = (long long)i * S0 + (long long)j * P + k;
        if (KIND == K_FIRST || KIND == K_MID) {
            double a0, a1;
            if (KIND == K_FIRST) {
                a0 = whb_add(whb_mul(acc0, c2.x), whb_mul(accn, n0));
                a1 = whb_add(whb_mul(acc0, c2.y), whb_mul(accn, n1));
            } else {
                a0 = whb_add(a2.x, whb_mul(accn, n0));
                a1 = whb_add(a2.y, whb_mul(accn, n1));
            }
            if (ok0 && ok1) {
                *reinterpret_cast<double2 *>(wnxt + p) = make_double2(n0, n1);
                *reinterpret_cast<double2 *>(m.acc + p) = make_double2(a0, a1);
            } else {
                if (ok0) { wnxt[p] = n0; m.acc[p] = a0; }
                if (ok1) { wnxt[p + 1] = n1; m.acc[p + 1] = a1; }
            }
        } else {
            const double o0 = whb_mul(m.out_scale, whb_add(a2.x, whb_mul(accn, n0)));
            const double o1 = whb_mul(m.out_scale, whb_add(a2.y, whb_mul(accn, n1)));
            if (m.out_mode == WHB_OUT_FPI) {
                if (ok0) {
                    const double d0 = o0 - vcur.x;
                    rsum += d0 * d0;
                    m.v[p] = o0;
                }
                if (ok1) {
                    const double d1 = o1 - vcur.y;
                    rsum += d1 * d1;
                    m.v[p + 1] = o1;
                }
            } else if (m.out_mode == WHB_OUT_AV) {
                if (ok0) m.dst[p] = whb_sub(vcur.x, o0);
                if (ok1) m.dst[p + 1] = whb_sub(vcur.y, o1);
            } else {
                if (ok0) m.dst[p] = o0;
                if (ok1) m.dst[p + 1] = o1;
            }
        }
        vcur = vnext;
    }
    if (KIND == K_LAST && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (tid == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace bulk
