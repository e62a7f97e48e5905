// coeff.cuh — a4 + a5 arithmetic shared by the stand-alone epilogue (epilogue.cu) and the fused
// epilogue of the tcgen05 kernel (contract_tf32.cu): one output coefficient from the real
// quadrant products P of a clip (Prop. 3).
//   interior (Eq. Fkl, alpha case 4):  S(m,+n) = (Pcc - Pss) - i (Psc + Pcs)
//                                                S(m,-n) = (Pcc + Pss) - i (Psc - Pcs)
//                                                F[m,n]  = -S / (4 pi^2 m n)
//   axes (Eqs. Fk0/F0l P:835-842, alpha cases 2-3): S(m,0) = P[c_m, y] - i P[s_m, y]
//                                                F[m,0]  = i S / (2 pi m T)   (and F[0,n] likewise)
//   DC (Eq. Fdc, Step 1): F[0,0] = area / T^2 from the exact int64 area.
//   mirror: F[-m,-n] = conj F[m,n], computed as the bitwise conjugate of the (m,n) value.
#pragma once
#include "common.cuh"

namespace fcfs {

// getP(px, tx, py, ty): P at logical quadrant rows (pair px, t = 0 cos / 1 sin) x (py, ty)
template <class GetP>
__device__ __forceinline__ double2 coeff_from_P(const GetP &getP, const SidePlan &X, const SidePlan &Y, int32_t T,
                                                int m, int n, double dc) {
    const double pi = 3.141592653589793238462643383279502884;
    if (m == 0 && n == 0) return make_double2(dc, 0.0);
    const bool neg = (m < 0) || (m == 0 && n < 0);
    if (neg) { m = -m; n = -n; }
    double re, im;
    if (n == 0) {
        const int pm = m - X.f0, pa = Y.nf;
        const double sre = getP(pm, 0, pa, 0), sim = -getP(pm, 1, pa, 0);
        const double d = 2.0 * pi * (double)m * (double)T;
        re = -sim / d; im = sre / d;
    } else if (m == 0) {
        const int pa = X.nf, pn = n - Y.f0;
        const double sre = getP(pa, 0, pn, 0), sim = -getP(pa, 0, pn, 1);
        const double d = 2.0 * pi * (double)n * (double)T;
        re = -sim / d; im = sre / d;
    } else {
        const int an = n < 0 ? -n : n;
        const int pm = m - X.f0, pn = an - Y.f0;
        const double pcc = getP(pm, 0, pn, 0), pcs = getP(pm, 0, pn, 1);
        const double psc = getP(pm, 1, pn, 0), pss = getP(pm, 1, pn, 1);
        double sre, sim;
        if (n > 0) { sre = pcc - pss; sim = -(psc + pcs); }
        else { sre = pcc + pss; sim = -(psc - pcs); }
        const double d = -4.0 * pi * pi * (double)m * (double)n;
        re = sre / d; im = sim / d;
    }
    if (neg) im = -im;
    return make_double2(re, im);
}

// largest n >= 0 with m^2 + n^2 <= r2 (the same double comparison as the definition), -1 if none
__host__ __device__ inline int pupil_nmax(int m, double r2, int N) {
    const double mm = (double)m * (double)m;
    if (mm > r2) return -1;
    int n = (int)floor(sqrt(r2 - mm));
    while (n + 1 <= N && mm + (double)(n + 1) * (double)(n + 1) <= r2) ++n;
    while (n >= 0 && mm + (double)n * (double)n > r2) --n;
    return n < N ? n : N;
}

__device__ __forceinline__ void store_out(void *F, int64_t o, double2 v, int out_f32) {
    if (out_f32) ((float2 *)F)[o] = make_float2((float)v.x, (float)v.y);
    else ((double2 *)F)[o] = v;
}

// an output (m, n) of a single-clip ROWS epilogue: to F at the shard-relative index o_rel, or — the peer
// mode — to every peer buffer at the full DENSE-window index (the all_gather of the rows done by the
// epilogue's own stores over NVLink; the caller orders the peers' reads after this kernel)
__device__ __forceinline__ void store_row_out(const EpiArgs &ea, void *F, int64_t o_rel, int m, int n, double2 v) {
    if (ea.peer_n == 0) {
        store_out(F, o_rel, v, ea.out_f32);
        return;
    }
    const int64_t o = (int64_t)(m + ea.M) * (2 * ea.N + 1) + (n + ea.N);
    for (int p = 0; p < ea.peer_n; ++p) store_out(ea.peer[p], o, v, ea.out_f32);
}

}  // namespace fcfs
