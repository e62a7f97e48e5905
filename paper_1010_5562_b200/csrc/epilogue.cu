// epilogue.cu — a4 + a5: axes, DC, quadrant recombination, scaling, mirror, window/pupil.
//
// From the real quadrant products P (contract_fp64.cu / contract_tf32.cu) of one clip:
//   interior (Eq. Fkl, alpha case 4):  S(m,+n) = (Pcc - Pss) - i (Psc + Pcs)
//                                                S(m,-n) = (Pcc + Pss) - i (Psc - Pcs)
//                                                F[m,n]  = -S / (4 pi^2 m n)
//   axes (Eqs. Fk0/F0l P:835-842, alpha cases 2-3): S(m,0) = P[c_m, y] - i P[s_m, y]
//                                                F[m,0]  = i S / (2 pi m T)   (and F[0,n] likewise)
//   DC (Eq. Fdc, Step 1): F[0,0] = area / T^2 from the exact int64 area.
//   mirror: F[-m,-n] = conj F[m,n], written as a bitwise conjugate of the computed value.
// The window is the signed low-pass box |m|<=M, |n|<=N (reading A3), optionally masked or
// packed to the pupil disk m^2+n^2 <= r2 (reading A11).  P of a clip is the
// fixed-order sum of its split-K partial tiles (deterministic).
#include "coeff.cuh"

namespace fcfs {

// P at logical quadrant rows (px, tx) x (py, ty): pair index p, t = 0 cos / 1 sin (axis: p = nf, t = 0)
__device__ __forceinline__ double getP(const double *P_ws, const GemmPlan &pl, int64_t clip, int px, int tx, int py,
                                       int ty) {
    const int ix = phys_row(px, tx, pl.phys), iy = phys_row(py, ty, pl.phys);
    const int tix = ix / kTile, tiy = iy / kTile;
    const int64_t base = ((clip * pl.tiles_x + tix) * pl.tiles_y + tiy) * pl.splits;
    const int64_t off = (int64_t)(ix - tix * kTile) * kTile + (iy - tiy * kTile);
    double s = 0.0;
    for (int sp = 0; sp < pl.splits; ++sp) s += P_ws[(base + sp) * (kTile * kTile) + off];
    return s;
}

__device__ double2 coeff(const double *P_ws, const GemmPlan &pl, const EpiArgs &ea, int64_t clip, int m, int n,
                         double dc) {
    auto get = [&](int px, int tx, int py, int ty) { return getP(P_ws, pl, clip, px, tx, py, ty); };
    return coeff_from_P(get, pl.X, pl.Y, ea.T, m, n, dc);
}

// grid: (output rows, clips, grid-stride over clips beyond 65535); block loops over n
__global__ void k_epilogue(const double *__restrict__ P_ws, GemmPlan pl, EpiArgs ea, void *F) {
    const int m = ea.m_lo + (int)blockIdx.x;
    if (m > ea.m_hi) return;
    for (int64_t clip = blockIdx.y; clip < pl.B; clip += gridDim.y) {
        const int64_t area = ea.area_dev ? ea.area_dev[clip] : ea.area_host;
        const double dc = (double)area / ((double)ea.T * (double)ea.T);
        int64_t off;
        int nlo, nhi;
        if (ea.layout == FCFS_LAYOUT_PUPIL) {
            off = 0;
            for (int mm = -ea.M; mm < m; ++mm) {
                int c = pupil_nmax(mm, ea.r2, ea.N);
                off += c < 0 ? 0 : 2 * c + 1;
            }
            int c = pupil_nmax(m, ea.r2, ea.N);
            if (c < 0) return;
            nlo = -c; nhi = c;
        } else {
            off = (int64_t)(m - ea.m_lo) * (2 * ea.N + 1);
            nlo = -ea.N; nhi = ea.N;
        }
        off += clip * ea.out_per_clip;
        for (int n = nlo + (int)threadIdx.x; n <= nhi; n += blockDim.x) {
            double2 v;
            bool keep = true;
            if (ea.layout == FCFS_LAYOUT_DENSE && ea.r2 >= 0.0)
                keep = (double)m * (double)m + (double)n * (double)n <= ea.r2;
            v = keep ? coeff(P_ws, pl, ea, clip, m, n, dc) : make_double2(0.0, 0.0);
            store_row_out(ea, F, off + (n - nlo), m, n, v);
        }
    }
    if (ea.peer_n) __threadfence_system();   // peer stores performed before the kernel's completion is seen
}

fcfs_status launch_epilogue(const GemmPlan &plan, const double *P_ws, const EpiArgs &ea, void *F, cudaStream_t s) {
    const int rows = ea.m_hi - ea.m_lo + 1;
    if (rows <= 0 || plan.B <= 0) return FCFS_OK;
    dim3 grid((unsigned)rows, (unsigned)(plan.B < 65535 ? plan.B : 65535));
    k_epilogue<<<grid, 128, 0, s>>>(P_ws, plan, ea, F);
    FCFS_CHECK_LAUNCH("k_epilogue");
    return FCFS_OK;
}

}  // namespace fcfs
