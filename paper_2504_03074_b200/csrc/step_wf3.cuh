// Three leapfrog steps per pass over HBM (3D temporal blocking), TMA pipelined, sm_100a.
//
// A CTA owns a BY x 64 tile (axes 1 x 2) and marches it through a chunk of
// axis-0 planes as a wavefront in time: when plane i of W^s arrives it computes
//     level 1 (W^{s+1}) at plane i-1 on the tile + a 2-cell ring,
//     level 2 (W^{s+2}) at plane i-2 on the tile + a 1-cell ring,
//     level 3 (W^{s+3}) at plane i-3 on the tile,
// each level from three planes of the level below kept in shared-memory rings.
// Per point and pass HBM sees: read W^s, W^{s-1}, f, acc; write W^{s+2},
// W^{s+3}, acc — 56 B per 3 updates (18.7 B/update against 28 for the two-step
// kernel and 48 for one step), plus halo re-reads served mostly by L2.
// Redundant arithmetic: levels 1 and 2 on their rings (21 % at BY = 12).
//
// Inputs per plane land by TMA (cp.async.bulk.tensor.3d) in a ring of NST
// stages (W^s with a 3-cell halo, W^{s-1} with 2, acc on the tile) and an f
// ring of NF planes (f of a plane serves all three levels, over three
// iterations).  Time levels live in a 6-slot global ring (level_ptr): the pass
// reads s, s-1 and writes s+2, s+3, which never alias with 6 slots.
// Every value is formed by the reference's operations in the reference's order
// (update_point, bitwise parity); Dirichlet and out-of-domain points of every
// intermediate level are exactly 0.
#pragma once

namespace wf3 {

using bulk::fence_proxy_async;
using bulk::mbar_expect_tx;
using bulk::mbar_init;
using bulk::mbar_wait;
using bulk::tma_load_3d;
using bulk::update_point;

constexpr int pad16(int x) { return (x + 15) / 16 * 16; }
constexpr int TX = 64;
constexpr int NST = 5;  // W^s / W^{s-1} / acc stages: planes i-2 .. i live, i+1 and i+2 in flight
constexpr int NF = 6;   // f planes: i-3 .. i live (used by levels 3 .. 1), i+1, i+2 in flight

template <int BY>
struct Lay {
    static constexpr int R0 = BY + 6, C0 = TX + 8;  // W^s box: rows j0-3 .., columns k0-4 .. (16-B aligned start)
    static constexpr int R1 = BY + 4, C1 = TX + 4;  // level 1 region, W^{s-1} and f boxes
    static constexpr int R2 = BY + 2, C2 = TX + 2;  // level 2 region
    static constexpr int C2S = TX + 4;              // its row stride; column ex at ex + 1 (tile pairs 16-B aligned)
    static constexpr int N0 = pad16(R0 * C0), N1 = pad16(R1 * C1), N2 = pad16(R2 * C2S), NA = BY * TX;
    static constexpr int STAGE = N0 + N1 + NA;      // W^s | W^{s-1} | acc
    static constexpr int THREADS = TX * BY / 2;
};

template <int BY>
constexpr size_t smem_bytes() {
    using L = Lay<BY>;
    return (size_t)(NST * L::STAGE + NF * L::N1 + 3 * L::N1 + 3 * L::N2) * sizeof(double) + NST * sizeof(uint64_t);
}

template <int BY, int K1, int K2, bool ZF>
__global__ void __launch_bounds__(Lay<BY>::THREADS)
    wf3_kernel(Geom g, const Member *__restrict__ members, int member_off, int s, int i_begin, int i_end,
               int chunk_len, int JT, int part_off, const __grid_constant__ CUtensorMap tm_w,
               const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_f,
               const __grid_constant__ CUtensorMap tm_a) {
    using L = Lay<BY>;
    extern __shared__ __align__(128) double smem[];
    double *stg = smem;                    // NST x STAGE
    double *fr = stg + NST * L::STAGE;     // NF x N1
    double *l1 = fr + NF * L::N1;          // 3 x N1
    double *l2 = l1 + 3 * L::N1;           // 3 x N2
    uint64_t *bars = reinterpret_cast<uint64_t *>(l2 + 3 * L::N2);

    const Member m = members[member_off + blockIdx.z];
    const int tid = threadIdx.x;
    const int jt = blockIdx.y % JT;
    const int ch = blockIdx.y / JT;
    const int k0 = blockIdx.x * TX;
    const int j0 = jt * BY;
    const int o0 = i_begin + ch * chunk_len;  // output planes [o0, o1)
    const int o1 = min(i_end, o0 + chunk_len);
    constexpr bool FPI_CAN = (K2 == K_LAST);
    if (o0 >= o1) {
        if (FPI_CAN && m.out_mode == WHB_OUT_FPI && tid == 0)
            m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    double *w2g = level_ptr(m, s + 2);
    double *w3g = level_ptr(m, s + 3);
    // per-level scalars: level t is produced by step s+t-1 (timestep.py:137-140, 284-300)
    constexpr bool FIRST = (K1 == K_FIRST);
    const double h1 = FIRST ? m.half_dt2 : m.dt2;
    const double cs1 = FIRST ? 1.0 : m.cos_f[s];
    const double h2 = m.dt2, cs2 = m.cos_f[s + 1];
    const double h3 = m.dt2, cs3 = m.cos_f[s + 2];
    const double c1 = m.acc_c[s + 1], c2 = m.acc_c[s + 2], c3 = m.acc_c[s + 3];
    const double acc0 = m.acc_c[0];
    const long long S0 = g.S0;
    const int P = g.P;

    constexpr bool LOAD_P = !FIRST, LOAD_A = !FIRST;
    constexpr uint32_t bytes = (uint32_t)((L::R0 * L::C0 + (LOAD_P ? L::R1 * L::C1 : 0) + (ZF ? 0 : L::R1 * L::C1) +
                                           (LOAD_A ? L::NA : 0)) * 8);
    const int ifirst = o0 - 3;
    const int nq = (o1 - o0) + 6;  // iterations: planes ifirst .. o1+2 enter

    auto issue = [&](int q) {
        const int p = ifirst + q;
        double *st = stg + (size_t)(q % NST) * L::STAGE;
        uint64_t *bar = bars + (q % NST);
        mbar_expect_tx(bar, bytes);
        tma_load_3d(st, &tm_w, k0 - 4, j0 - 3, p, bar);
        if (LOAD_P) tma_load_3d(st + L::N0, &tm_p, k0 - 2, j0 - 2, p, bar);
        if (LOAD_A) tma_load_3d(st + L::N0 + L::N1, &tm_a, k0, j0, p, bar);
        if (!ZF) tma_load_3d(fr + (size_t)(q % NF) * L::N1, &tm_f, k0 - 2, j0 - 2, p, bar);
    };

    if (tid == 0) {
        for (int t = 0; t < NST; ++t) mbar_init(bars + t, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        issue(0);
        if (nq > 1) issue(1);
    }
    __syncthreads();

    // main pair of this thread on the tile (level 3, outputs, filter sums)
    const int ty = tid / (TX / 2);
    const int kl = 2 * (tid % (TX / 2));
    const int j = j0 + ty;
    const int k = k0 + kl;
    const bool row_ok = (j >= g.j_lo && j < g.j_hi);
    const bool ok0 = row_ok && (k >= 1) && (k < g.n2 - 1);
    const bool ok1 = row_ok && (k + 1 < g.n2 - 1);
    const long long pbase = (long long)j * P + k;
    double2 A0 = make_double2(0.0, 0.0), A1 = A0, A2 = A0;  // filter sums of planes i-1, i-2, i-3
    double rsum = 0.0;

    for (int q = 0; q < nq; ++q) {
        const int i = ifirst + q;
        if (tid == 0 && q + 2 < nq) {
            fence_proxy_async();  // stage/f slots of plane i+2 were last read in iteration q-1
            issue(q + 2);
        }
        mbar_wait(bars + (q % NST), (q / NST) & 1);

        // ---- level 1 (step s) at plane p1 = i-1, region (BY+4) x (TX+4) from origin (j0-2, k0-2)
        const int p1 = i - 1;
        const bool do1 = q >= 2;  // p1 >= o0 - 2 (p1 <= o1 + 1 since q < nq)
        if (do1) {
            const double *Sm = stg + (size_t)((q - 2) % NST) * L::STAGE;  // W^s plane i-2
            const double *Sc = stg + (size_t)((q - 1) % NST) * L::STAGE;  // W^s plane i-1 (+ W^{s-1}, acc)
            const double *Sp = stg + (size_t)(q % NST) * L::STAGE;        // W^s plane i
            const double *Pv = Sc + L::N0;
            const double *Fv = fr + (size_t)((q - 1) % NF) * L::N1;
            double *D = l1 + (size_t)((p1 - (o0 - 2)) % 3) * L::N1;
            const bool pin = (p1 >= g.i_lo) && (p1 < g.i_hi);
            for (int idx = tid; idx < L::R1 * L::C1; idx += L::THREADS) {
                const int ey = idx / L::C1, ex = idx - (idx / L::C1) * L::C1;
                const int r0 = (ey + 1) * L::C0 + ex + 2;  // W^s at (j0-2+ey, k0-2+ex)
                const double wc = Sc[r0];
                const double fv = ZF ? 0.0 : Fv[idx];
                const double pv = LOAD_P ? Pv[idx] : 0.0;
                const double w = update_point<FIRST ? K_FIRST : K_MID, ZF, true>(
                    g, Sm[r0], wc, Sp[r0], Sc[r0 - L::C0], Sc[r0 + L::C0], Sc[r0 - 1], Sc[r0 + 1], fv, pv, h1, cs1);
                const int jj = j0 - 2 + ey, kk = k0 - 2 + ex;
                const bool in = pin && jj >= g.j_lo && jj < g.j_hi && kk >= 1 && kk < g.n2 - 1;
                D[idx] = in ? w : 0.0;
            }
        }
        __syncthreads();
        if (do1) {
            // filter sum of plane p1 starts: (acc or c0*W^0) + c1*W^{s+1}   (timestep.py:284, 298)
            const double *Sc = stg + (size_t)((q - 1) % NST) * L::STAGE;
            const double *D = l1 + (size_t)((p1 - (o0 - 2)) % 3) * L::N1;
            const double2 w1 = *reinterpret_cast<const double2 *>(D + (ty + 2) * L::C1 + kl + 2);
            double2 init;
            if (FIRST) {
                const double *W0 = Sc + (ty + 3) * L::C0 + kl + 4;
                init = make_double2(whb_mul(acc0, W0[0]), whb_mul(acc0, W0[1]));
            } else {
                init = *reinterpret_cast<const double2 *>(Sc + L::N0 + L::N1 + ty * TX + kl);
            }
            A0 = make_double2(whb_add(init.x, whb_mul(c1, w1.x)), whb_add(init.y, whb_mul(c1, w1.y)));
        }

        // ---- level 2 (step s+1) at plane p2 = i-2, region (BY+2) x (TX+2) from origin (j0-1, k0-1)
        const int p2 = i - 2;
        const bool do2 = q >= 4;  // p2 >= o0 - 1 (p2 <= o1 since q < nq)
        if (do2) {
            const double *Em = l1 + (size_t)((p2 - 1 - (o0 - 2)) % 3) * L::N1;
            const double *Ec = l1 + (size_t)((p2 - (o0 - 2)) % 3) * L::N1;
            const double *Ep = l1 + (size_t)((p2 + 1 - (o0 - 2)) % 3) * L::N1;
            const double *Ws = stg + (size_t)((q - 2) % NST) * L::STAGE;  // W^s plane p2 (prev of step s+1)
            const double *Fv = fr + (size_t)((q - 2) % NF) * L::N1;
            double *D = l2 + (size_t)((p2 - (o0 - 1)) % 3) * L::N2;
            const bool pin = (p2 >= g.i_lo) && (p2 < g.i_hi);
            for (int idx = tid; idx < L::R2 * L::C2; idx += L::THREADS) {
                const int ey = idx / L::C2, ex = idx - (idx / L::C2) * L::C2;
                const int r1 = (ey + 1) * L::C1 + ex + 1;
                const double fv = ZF ? 0.0 : Fv[r1];
                const double w = update_point<K_MID, ZF, true>(g, Em[r1], Ec[r1], Ep[r1], Ec[r1 - L::C1],
                                                               Ec[r1 + L::C1], Ec[r1 - 1], Ec[r1 + 1], fv,
                                                               Ws[(ey + 2) * L::C0 + ex + 3], h2, cs2);
                const int jj = j0 - 1 + ey, kk = k0 - 1 + ex;
                const bool in = pin && jj >= g.j_lo && jj < g.j_hi && kk >= 1 && kk < g.n2 - 1;
                D[ey * L::C2S + ex + 1] = in ? w : 0.0;
            }
        }
        __syncthreads();
        if (do2) {
            const double *D = l2 + (size_t)((p2 - (o0 - 1)) % 3) * L::N2;
            const double2 w2 = *reinterpret_cast<const double2 *>(D + (ty + 1) * L::C2S + kl + 2);
            A1 = make_double2(whb_add(A1.x, whb_mul(c2, w2.x)), whb_add(A1.y, whb_mul(c2, w2.y)));
        }

        // ---- level 3 (step s+2) at plane p3 = i-3 on the tile: the pass output
        const int p3 = i - 3;
        if (q >= 6) {  // p3 >= o0 (and p3 < o1 since q < nq)
            const double *Em = l2 + (size_t)((p3 - 1 - (o0 - 1)) % 3) * L::N2;
            const double *Ec = l2 + (size_t)((p3 - (o0 - 1)) % 3) * L::N2;
            const double *Ep = l2 + (size_t)((p3 + 1 - (o0 - 1)) % 3) * L::N2;
            const double *E1 = l1 + (size_t)((p3 - (o0 - 2)) % 3) * L::N1;  // W^{s+1} at p3 (prev)
            const double *Fv = fr + (size_t)((q - 3) % NF) * L::N1;
            const int r2 = (ty + 1) * L::C2S + kl + 2;
            const int r1 = (ty + 2) * L::C1 + kl + 2;
            const double2 e_c = *reinterpret_cast<const double2 *>(Ec + r2);
            const double2 e_m = *reinterpret_cast<const double2 *>(Em + r2);
            const double2 e_p = *reinterpret_cast<const double2 *>(Ep + r2);
            const double2 e_yl = *reinterpret_cast<const double2 *>(Ec + r2 - L::C2S);
            const double2 e_yh = *reinterpret_cast<const double2 *>(Ec + r2 + L::C2S);
            const double e_xl = Ec[r2 - 1], e_xh = Ec[r2 + 2];
            const double2 pv = *reinterpret_cast<const double2 *>(E1 + r1);
            const double2 fv = ZF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2 *>(Fv + r1);
            const double n0 = update_point<K_MID, ZF, true>(g, e_m.x, e_c.x, e_p.x, e_yl.x, e_yh.x, e_xl, e_c.y,
                                                           fv.x, pv.x, h3, cs3);
            const double n1 = update_point<K_MID, ZF, true>(g, e_m.y, e_c.y, e_p.y, e_yl.y, e_yh.y, e_c.x, e_xh,
                                                           fv.y, pv.y, h3, cs3);
            const double a0 = whb_add(A2.x, whb_mul(c3, n0));
            const double a1 = whb_add(A2.y, whb_mul(c3, n1));
            const long long p = (long long)p3 * S0 + pbase;
            if (K2 == K_MID) {
                if (ok0 && ok1) {
                    *reinterpret_cast<double2 *>(w2g + p) = e_c;
                    *reinterpret_cast<double2 *>(w3g + p) = make_double2(n0, n1);
                    *reinterpret_cast<double2 *>(m.acc + p) = make_double2(a0, a1);
                } else {
                    if (ok0) { w2g[p] = e_c.x; w3g[p] = n0; m.acc[p] = a0; }
                    if (ok1) { w2g[p + 1] = e_c.y; w3g[p + 1] = n1; m.acc[p + 1] = a1; }
                }
            } else {
                const double u0 = whb_mul(m.out_scale, a0);
                const double u1 = whb_mul(m.out_scale, a1);
                if (m.out_mode == WHB_OUT_FPI) {
                    if (ok0) { const double d = u0 - m.v[p]; rsum += d * d; m.v[p] = u0; }
                    if (ok1) { const double d = u1 - m.v[p + 1]; rsum += d * d; m.v[p + 1] = u1; }
                } else if (m.out_mode == WHB_OUT_AV) {
                    if (ok0) m.dst[p] = whb_sub(m.v[p], u0);
                    if (ok1) m.dst[p + 1] = whb_sub(m.v[p + 1], u1);
                } else {
                    if (ok0) m.dst[p] = u0;
                    if (ok1) m.dst[p + 1] = u1;
                }
            }
        }
        A2 = A1;
        A1 = A0;
        __syncthreads();  // every read of this iteration's stage / ring slots is done
    }
    if (FPI_CAN && m.out_mode == WHB_OUT_FPI) {
        const double t = block_sum(rsum);
        if (tid == 0) m.partials[part_off + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

}  // namespace wf3
