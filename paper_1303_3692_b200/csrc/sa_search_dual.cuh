// sa_search_dual.cuh -- k_match with TWO reads per thread, advanced in lock step (A/B: SA_MATCH_DUAL).
//
// Why: the C4 search is bound by the number of random DRAM accesses in flight.  A pointer chase over
// 16 GiB with the kernel's thread count (148 x 1280, one access outstanding per thread) reaches 33.9 G
// accesses/s, the rate k_match's DRAM lines run at; with 606 k threads the same chase reaches 43.4 G/s
// (profiles/r02/r02h/rand_mlp.json).  Occupancy cannot grow (48 registers: 40 spill and run slower,
// r01-3), so this kernel gives each thread two reads -- slots t and t + ceil(Q/2) of the ordered batch,
// two independent dependency chains -- and issues both reads' probe loads before either compare: up to
// two outstanding accesses per thread.  Each read follows exactly search_read's steps (the same bracket,
// pivots, split and bounds, written as the phase machine of sa_search_long.cuh), so results are equal.
#pragma once

#include "sa_search_long.cuh"

namespace sa_search {

template <int QW>
struct DualRead {
    QueryWords<QW> P;
    uint64_t q;       // the read (its result goes to out[q])
    uint32_t m;
    uint32_t phase;   // PH_* of sa_search_long.cuh
    uint32_t Lp1, R, lcpL, lcpR, hLp1, hR, hlcpL, hlcpR, lo, hi;
};

// bracket of search_read (m == 0, m < k, m >= k; no sub-tables, no trees) -> the first phase
template <int QW>
__device__ __forceinline__ void dual_start(const MatchArgs &a, DualRead<QW> &r) {
    const uint32_t k = a.k, m = r.m;
    auto clamp = [&](uint32_t v) { return min(max(v, a.clo), a.chi); };
    r.lcpL = r.lcpR = 0;
    if (m == 0) {
        r.lo = a.clo;
        r.hi = a.chi;
        r.phase = PH_DONE;
    } else if (m < k) {
        const bool rt = m < a.route_bases;
        const uint32_t kk = rt ? a.route_bases : k;
        const uint32_t *T = rt ? a.route : a.table;
        const uint64_t x = r.P.first() >> (64 - 2 * m);
        const uint32_t Ta = ld_u32(T + (x << (2 * (kk - m))));
        const uint32_t Tb = ld_u32(T + ((x + 1) << (2 * (kk - m))));
        r.Lp1 = clamp(Ta > kk ? Ta - kk : 0);
        r.R = clamp(Ta);
        r.hLp1 = clamp(Tb > kk ? Tb - kk : 0);
        r.hR = clamp(Tb);
        r.phase = PH_SLO;
    } else {
        const uint64_t x = r.P.first() >> (64 - 2 * k);
        uint32_t L1, R1;
        table_pair(a.table, x, L1, R1);
        r.Lp1 = clamp(L1);
        r.R = clamp(R1);
        r.phase = PH_DESC;
    }
}

// transitions at an empty interval (as k_match_long)
template <int QW>
__device__ __forceinline__ void dual_settle(DualRead<QW> &r) {
    while (r.phase != PH_DONE && r.R <= r.Lp1) {
        if (r.phase == PH_DESC) { r.lo = r.hi = r.R; r.phase = PH_DONE; }
        else if (r.phase == PH_LO) { r.lo = r.R; r.Lp1 = r.hLp1; r.R = r.hR; r.lcpL = r.hlcpL; r.lcpR = r.hlcpR; r.phase = PH_HI; }
        else if (r.phase == PH_SLO) { r.lo = r.R; r.Lp1 = r.hLp1; r.R = r.hR; r.lcpL = r.lcpR = 0; r.phase = PH_SHI; }
        else { r.hi = r.R; r.phase = PH_DONE; }
    }
}

template <int QW>
__device__ __forceinline__ void dual_apply(DualRead<QW> &r, uint32_t p, int sign, uint32_t lcp) {
    if (r.phase == PH_DESC) {
        if (sign == 0) {
            r.hLp1 = p + 1; r.hR = r.R; r.hlcpL = lcp; r.hlcpR = r.lcpR;
            r.R = p; r.lcpR = lcp;
            r.phase = PH_LO;
        } else if (sign < 0) { r.R = p; r.lcpR = lcp; } else { r.Lp1 = p + 1; r.lcpL = lcp; }
    } else {
        const bool lower = r.phase == PH_LO || r.phase == PH_SLO;
        if (sign < 0 || (lower && sign == 0)) { r.R = p; r.lcpR = lcp; } else { r.Lp1 = p + 1; r.lcpL = lcp; }
    }
}

template <int QW, int L>
#ifndef SA_DUAL_MINB
#define SA_DUAL_MINB 4
#endif
__global__ void __launch_bounds__(256, SA_DUAL_MINB) k_match_dual(const MatchArgs a, uint64_t half) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= half) return;
    DualRead<QW> r0, r1;
    const bool v1 = t + half < a.Q;
    {
        const uint64_t s0 = t, s1 = t + half;
        r0.q = a.order ? (uint64_t)__ldg(a.order + s0) : s0;
        r0.m = read_len(a, a.rows_ordered ? s0 : r0.q);
        load_read<QW>(a, a.rows_ordered ? s0 : r0.q, r0.m, r0.P);
        if (v1) {
            r1.q = a.order ? (uint64_t)__ldg(a.order + s1) : s1;
            r1.m = read_len(a, a.rows_ordered ? s1 : r1.q);
            load_read<QW>(a, a.rows_ordered ? s1 : r1.q, r1.m, r1.P);
        } else {
            r1.m = 0;
        }
    }
    dual_start(a, r0);
    if (v1) dual_start(a, r1); else r1.phase = PH_DONE;
    while (true) {
        dual_settle(r0);
        dual_settle(r1);
        const bool a0 = r0.phase != PH_DONE, a1 = r1.phase != PH_DONE;
        if (!a0 && !a1) break;
        // both probes' loads before either compare: two independent accesses in flight
        Probe<L> p0r, p1r;
        uint32_t p0 = 0, p1 = 0;
        if (a0) { p0 = (uint32_t)(((uint64_t)r0.Lp1 - 1 + r0.R) >> 1); p0r.load(a, p0); }
        if (a1) { p1 = (uint32_t)(((uint64_t)r1.Lp1 - 1 + r1.R) >> 1); p1r.load(a, p1); }
        uint32_t texts = 0;
        if (a0) {
            int sign;
            uint32_t lcp;
            const bool inb = r0.phase == PH_DESC || r0.phase == PH_LO || r0.phase == PH_HI;
            compare_probe(a, p0r, r0.P, r0.m, min(r0.lcpL, r0.lcpR), inb, sign, lcp, texts);
            dual_apply(r0, p0, sign, lcp);
        }
        if (a1) {
            int sign;
            uint32_t lcp;
            const bool inb = r1.phase == PH_DESC || r1.phase == PH_LO || r1.phase == PH_HI;
            compare_probe(a, p1r, r1.P, r1.m, min(r1.lcpL, r1.lcpR), inb, sign, lcp, texts);
            dual_apply(r1, p1, sign, lcp);
        }
    }
    reinterpret_cast<uint2 *>(a.out)[r0.q] = make_uint2(r0.lo, r0.hi);
    if (v1) reinterpret_cast<uint2 *>(a.out)[r1.q] = make_uint2(r1.lo, r1.hi);
}

}  // namespace sa_search
