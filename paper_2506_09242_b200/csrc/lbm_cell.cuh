// Cell-local lattice Boltzmann dynamics on the device.
//
// Each function restates its reference counterpart with the SAME sequence of
// non-trivial IEEE operations, so that with -fmad=false the results are
// bit-identical to the reference CPU solver (verified against the oracle):
//   D3Q19 tables ....... proj/include/dolb/descriptor.hpp:13-46
//   compute_rho_u ...... descriptor.hpp:64-76
//   equilibrium2/4 ..... descriptor.hpp:79-121
//   bgk/trt/rr ......... proj/include/dolb/collision.hpp:46-164
//   smagorinsky ........ collision.hpp:169-183
//   boundaries ......... proj/include/dolb/boundaries.hpp:10-133
//   ChainRecipe::apply . proj/include/dolb/chain.hpp:104-144
// The reference multiplies by lattice constants c in {-1,0,1} (T(c)*f). Here
// the loops are unrolled at compile time: c = +-1 becomes +-f (exact) and
// c = 0 terms are dropped (they only add a signed zero, which never changes
// a value). Everything else keeps the reference association order.
#pragma once

#include <cstdint>
#include <utility>

namespace dlb {

// ---------------------------------------------------------------------------
// Velocity sets. D3Q27 (no reference) follows SURVEY.md A.8: 0-18 identical to
// the frozen D3Q19 table, corners appended as adjacent opposite pairs.
template <int Q>
struct Lat;

template <>
struct Lat<19> {
    static constexpr int q = 19;
    static constexpr int c[19][3] = {
        {0, 0, 0},
        {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
        {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0},
        {-1, 0, -1}, {1, 0, 1}, {-1, 0, 1}, {1, 0, -1},
        {0, -1, -1}, {0, 1, 1}, {0, -1, 1}, {0, 1, -1}};
    static constexpr double w[19] = {
        1.0 / 3.0,
        1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0, 1.0 / 18.0,
        1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0,
        1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0, 1.0 / 36.0};
};

template <>
struct Lat<27> {
    static constexpr int q = 27;
    static constexpr int c[27][3] = {
        {0, 0, 0},
        {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
        {-1, -1, 0}, {1, 1, 0}, {-1, 1, 0}, {1, -1, 0},
        {-1, 0, -1}, {1, 0, 1}, {-1, 0, 1}, {1, 0, -1},
        {0, -1, -1}, {0, 1, 1}, {0, -1, 1}, {0, 1, -1},
        {-1, -1, -1}, {1, 1, 1}, {-1, -1, 1}, {1, 1, -1},
        {-1, 1, -1}, {1, -1, 1}, {1, -1, -1}, {-1, 1, 1}};
    static constexpr double w[27] = {
        8.0 / 27.0,
        2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0, 2.0 / 27.0,
        1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0,
        1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0, 1.0 / 54.0,
        1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0,
        1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0, 1.0 / 216.0};
};

// opposite(i) = i +- 1 for i >= 1 in both sets (descriptor.hpp:41-45).
__host__ __device__ constexpr int opp_of(int i) { return i == 0 ? 0 : ((i & 1) ? i + 1 : i - 1); }

// Compile-time loop: f(std::integral_constant<int, I>) for I in [0, N).
template <typename F, int... I>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, I...>) {
    (f(std::integral_constant<int, I>{}), ...);
}
template <int N, typename F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, N>{});
}

// Signed accumulation helper: s (+|-)= v with the first term initialising s.
// Equivalent in value to the reference's `s = 0; s += T(c) * v` sequence.
template <typename T>
struct Acc {
    T s;
    bool any = false;
    __device__ __forceinline__ void add(int sign, T v) {
        if (!any) {
            s = sign > 0 ? v : -v;
            any = true;
        } else {
            s = sign > 0 ? s + v : s - v;
        }
    }
    __device__ __forceinline__ T get() const { return any ? s : T(0); }
};

// Device image of ChainRecipe<T> (chain.hpp:86-102); parameters cast to T on
// the host as compile_chain<T> does (chain.hpp:150-156).
enum : int32_t { KIND_NODYN = 0, KIND_BB = 1, KIND_MBB = 2, KIND_COLLIDE = 3 };
enum : int32_t { BASE_BGK = 0, BASE_TRT = 1, BASE_RR = 2 };

template <typename T>
struct DevRecipe {
    int32_t kind, base, has_reg, reg_is_pressure, reg_axis, reg_orient, has_les, pad;
    T omega;
    T omega_minus;  // T(derive_omega_minus(double(omega), double(lambda))) when !has_les
    T lambda, smagorinsky_c, omega_bulk_ho, target_rho;
    T wall_velocity[3];
};

// Kind mask: compile-time subset of dynamics a kernel instantiation contains
// (the paper's hand-picked dispatch set).
enum : unsigned {
    KM_NODYN = 1u, KM_BB = 2u, KM_MBB = 4u, KM_BGK = 8u, KM_TRT = 16u, KM_RR = 32u,
    KM_LES = 64u, KM_REGV = 128u, KM_REGP = 256u,
    KM_ALL = 511u,
    KM_SKIP = 512u,  // variant flag: NoDynamics cells skipped (no loads / stores)
    KM_KE = 1024u,   // variant flag: also write the new state's per-cell kinetic energy (fused reduce input)
    KM_XREC = 2048u, // variant flag: recipe table in global memory (registries beyond kMaxSlots instances)
};

template <typename T, int Q>
struct Cell {
    using L = Lat<Q>;

    // descriptor.hpp:64-76
    static __device__ __forceinline__ void rho_u(const T (&f)[Q], T& rho, T (&u)[3]) {
        T drho = f[0];
        Acc<T> j[3];
        sfor<Q - 1>([&](auto I0) {
            constexpr int i = decltype(I0)::value + 1;
            drho = drho + f[i];
            sfor<3>([&](auto A) {
                constexpr int c = L::c[i][decltype(A)::value];
                if constexpr (c != 0) j[decltype(A)::value].add(c, f[i]);
            });
        });
        rho = T(1) + drho;
        u[0] = j[0].get() / rho;
        u[1] = j[1].get() / rho;
        u[2] = j[2].get() / rho;
    }

    // c_i . u with the reference's left-to-right component order.
    template <int i>
    static __device__ __forceinline__ T cdot(const T (&u)[3]) {
        Acc<T> a;
        sfor<3>([&](auto A) {
            constexpr int c = L::c[i][decltype(A)::value];
            if constexpr (c != 0) a.add(c, u[decltype(A)::value]);
        });
        return a.get();
    }

    static __device__ __forceinline__ T usqr_of(const T (&u)[3]) {
        return u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    }

    // descriptor.hpp:79-92 (one direction)
    template <int i>
    static __device__ __forceinline__ T eq2(T rho, const T (&u)[3], T usqr) {
        constexpr double wd = L::w[i];
        const T wi = T(wd);
        const T cu = cdot<i>(u);
        const T series = T(3) * cu + T(4.5) * cu * cu - T(1.5) * usqr;
        return wi * (rho - T(1)) + wi * rho * series;
    }

    // Hermite coefficient c_a^2 - cs2 with cs2 = T(1)/T(3) (descriptor.hpp:101,111-113)
    template <int ca>
    static __device__ __forceinline__ T herm() {
        const T cs2 = T(1) / T(3);
        if constexpr (ca != 0) return T(1) - cs2;
        else return -cs2;
    }

    // descriptor.hpp:98-121 (one direction)
    template <int i>
    static __device__ __forceinline__ T eq4(T rho, const T (&u)[3], T usqr) {
        constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
        constexpr double wd = L::w[i];
        const T wi = T(wd);
        const T cu = cdot<i>(u);
        const T hxx = herm<cx>(), hyy = herm<cy>(), hzz = herm<cz>();
        Acc<T> third;
        // cy*hxx*u0*u0*u1 + cz*hxx*u0*u0*u2 + cx*hyy*u1*u1*u0 + cz*hyy*u1*u1*u2
        // + cx*hzz*u2*u2*u0 + cy*hzz*u2*u2*u1, each evaluated left to right.
        if constexpr (cy != 0) third.add(cy, hxx * u[0] * u[0] * u[1]);
        if constexpr (cz != 0) third.add(cz, hxx * u[0] * u[0] * u[2]);
        if constexpr (cx != 0) third.add(cx, hyy * u[1] * u[1] * u[0]);
        if constexpr (cz != 0) third.add(cz, hyy * u[1] * u[1] * u[2]);
        if constexpr (cx != 0) third.add(cx, hzz * u[2] * u[2] * u[0]);
        if constexpr (cy != 0) third.add(cy, hzz * u[2] * u[2] * u[1]);
        T series = T(3) * cu + T(4.5) * cu * cu - T(1.5) * usqr;
        if (third.any) series = series + T(13.5) * third.s;
        return wi * (rho - T(1)) + wi * rho * series;
    }

    // Second-moment accumulation sum_i c_a c_b v_i (descriptor.hpp:130-141),
    // components xx, xy, xz, yy, yz, zz.
    static __device__ __forceinline__ void second_moment(const T (&v)[Q], T (&p)[6]) {
        Acc<T> a[6];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            if constexpr (cx * cx != 0) a[0].add(1, v[i]);
            if constexpr (cx * cy != 0) a[1].add(cx * cy, v[i]);
            if constexpr (cx * cz != 0) a[2].add(cx * cz, v[i]);
            if constexpr (cy * cy != 0) a[3].add(1, v[i]);
            if constexpr (cy * cz != 0) a[4].add(cy * cz, v[i]);
            if constexpr (cz * cz != 0) a[5].add(1, v[i]);
        });
        for (int k = 0; k < 6; ++k) p[k] = a[k].get();
    }

    // H2 : P for direction i: (cx^2-cs2)P0 + (cy^2-cs2)P3 + (cz^2-cs2)P5
    //                         + 2 (cx cy P1 + cx cz P2 + cy cz P4)
    template <int i>
    static __device__ __forceinline__ T h2_contract(const T (&p)[6]) {
        constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
        T s = herm<cx>() * p[0] + herm<cy>() * p[3] + herm<cz>() * p[5];
        Acc<T> in;
        if constexpr (cx * cy != 0) in.add(cx * cy, p[1]);
        if constexpr (cx * cz != 0) in.add(cx * cz, p[2]);
        if constexpr (cy * cz != 0) in.add(cy * cz, p[4]);
        if (in.any) s = s + T(2) * in.s;
        return s;
    }

    // collision.hpp:46-81 — unrolled BGK, pairwise over opposite directions.
    static __device__ __forceinline__ void bgk(T (&f)[Q], T omega) {
        T drho = f[0];
        Acc<T> j[3];
        sfor<Q - 1>([&](auto I0) {
            constexpr int i = decltype(I0)::value + 1;
            drho = drho + f[i];
            sfor<3>([&](auto A) {
                constexpr int c = L::c[i][decltype(A)::value];
                if constexpr (c != 0) j[decltype(A)::value].add(c, f[i]);
            });
        });
        const T rho = T(1) + drho;
        const T inv_rho = T(1) / rho;
        const T u[3] = {j[0].get() * inv_rho, j[1].get() * inv_rho, j[2].get() * inv_rho};
        const T usqr = T(1.5) * (u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        const T om1 = T(1) - omega;
        constexpr double wd0 = L::w[0];
        const T w0 = T(wd0);
        f[0] = om1 * f[0] + omega * (w0 * (rho - T(1)) - w0 * rho * usqr);
        sfor<(Q - 1) / 2>([&](auto P) {
            constexpr int i = 2 * decltype(P)::value + 1;  // i, i+1 opposite; cu along i+1
            const T cu = cdot<i + 1>(u);
            constexpr double wd = L::w[i];
            const T w = T(wd);
            const T wr = rho * w;
            const T sym = wr * (T(4.5) * cu * cu - usqr);
            const T asym = wr * T(3) * cu;
            const T base = w * (rho - T(1));
            f[i] = om1 * f[i] + omega * (base + sym - asym);
            f[i + 1] = om1 * f[i + 1] + omega * (base + sym + asym);
        });
    }

    // equilibrium2 of an opposite pair (i, i+1) sharing the terms that are
    // exactly equal: cu_i = -cu_{i+1}, so 3 cu_i = -(3 cu_{i+1}) and
    // (4.5 cu_i) cu_i = (4.5 cu_{i+1}) cu_{i+1} bit for bit; the series are then
    // formed with the reference's association ((3cu + q) - 1.5 usqr).
    template <int i>
    static __device__ __forceinline__ void eq2_pair(T rho, const T (&u)[3], T u15, T& ei, T& ej) {
        constexpr double wd = L::w[i];
        const T w = T(wd);
        const T cu = cdot<i + 1>(u);
        const T t3 = T(3) * cu;
        const T q = T(4.5) * cu * cu;
        const T base = w * (rho - T(1));
        const T wr = w * rho;
        ej = base + wr * ((t3 + q) - u15);
        ei = base + wr * ((q - t3) - u15);
    }

    // collision.hpp:85-101, evaluated per opposite pair: the j member uses
    // fm_j = -fm_i and em_j = -em_i, which is exact in IEEE arithmetic.
    static __device__ __forceinline__ void trt(T (&f)[Q], T omega, T omega_minus) {
        T rho, u[3];
        rho_u(f, rho, u);
        const T usqr = usqr_of(u);
        const T u15 = T(1.5) * usqr;
        {
            constexpr double wd0 = L::w[0];
            const T w0 = T(wd0);
            const T e0 = w0 * (rho - T(1)) + w0 * rho * (-u15);
            const T fp = (f[0] + f[0]) * T(0.5);
            const T fm = (f[0] - f[0]) * T(0.5);
            const T ep = (e0 + e0) * T(0.5);
            const T em = (e0 - e0) * T(0.5);
            f[0] = f[0] - omega * (fp - ep) - omega_minus * (fm - em);
        }
        sfor<(Q - 1) / 2>([&](auto P) {
            constexpr int i = 2 * decltype(P)::value + 1;
            T ei, ej;
            eq2_pair<i>(rho, u, u15, ei, ej);
            const T fi = f[i], fj = f[i + 1];
            const T fp = (fi + fj) * T(0.5);
            const T fm = (fi - fj) * T(0.5);
            const T ep = (ei + ej) * T(0.5);
            const T em = (ei - ej) * T(0.5);
            const T even = omega * (fp - ep);
            const T odd = omega_minus * (fm - em);
            f[i] = fi - even - odd;
            f[i + 1] = fj - even + odd;
        });
    }

    // collision.hpp:108-164. f is overwritten by feq4 as soon as f_i - feq_i
    // has entered the second moment (same per-component accumulation order),
    // so only one q-array is live.
    static __device__ __forceinline__ void rr(T (&f)[Q], T omega, T omega_bulk_ho) {
        T rho, u[3];
        rho_u(f, rho, u);
        const T usqr = usqr_of(u);
        Acc<T> acc[6];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            const T feq = eq4<i>(rho, u, usqr);
            const T fn = f[i] - feq;
            if constexpr (cx * cx != 0) acc[0].add(1, fn);
            if constexpr (cx * cy != 0) acc[1].add(cx * cy, fn);
            if constexpr (cx * cz != 0) acc[2].add(cx * cz, fn);
            if constexpr (cy * cy != 0) acc[3].add(1, fn);
            if constexpr (cy * cz != 0) acc[4].add(cy * cz, fn);
            if constexpr (cz * cz != 0) acc[5].add(1, fn);
            f[i] = feq;
        });
        T a2[6];
        for (int k = 0; k < 6; ++k) a2[k] = acc[k].get();
        const T trace3 = (a2[0] + a2[3] + a2[5]) / T(3);
        const T gdev = T(1) - omega;
        const T ghob = T(1) - omega_bulk_ho;
        T a2r[6];
        a2r[0] = gdev * (a2[0] - trace3) + ghob * trace3;
        a2r[1] = gdev * a2[1];
        a2r[2] = gdev * a2[2];
        a2r[3] = gdev * (a2[3] - trace3) + ghob * trace3;
        a2r[4] = gdev * a2[4];
        a2r[5] = gdev * (a2[5] - trace3) + ghob * trace3;
        const T a3_xxy = ghob * (T(2) * u[0] * a2[1] + u[1] * a2[0]);
        const T a3_xxz = ghob * (T(2) * u[0] * a2[2] + u[2] * a2[0]);
        const T a3_yyx = ghob * (T(2) * u[1] * a2[1] + u[0] * a2[3]);
        const T a3_yyz = ghob * (T(2) * u[1] * a2[4] + u[2] * a2[3]);
        const T a3_zzx = ghob * (T(2) * u[2] * a2[2] + u[0] * a2[5]);
        const T a3_zzy = ghob * (T(2) * u[2] * a2[4] + u[1] * a2[5]);
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int cx = L::c[i][0], cy = L::c[i][1], cz = L::c[i][2];
            constexpr double wd = L::w[i];
            const T wi = T(wd);
            const T hxx = herm<cx>(), hyy = herm<cy>(), hzz = herm<cz>();
            const T second = h2_contract<i>(a2r);
            Acc<T> third;
            if constexpr (cy != 0) third.add(cy, hxx * a3_xxy);
            if constexpr (cz != 0) third.add(cz, hxx * a3_xxz);
            if constexpr (cx != 0) third.add(cx, hyy * a3_yyx);
            if constexpr (cz != 0) third.add(cz, hyy * a3_yyz);
            if constexpr (cx != 0) third.add(cx, hzz * a3_zzx);
            if constexpr (cy != 0) third.add(cy, hzz * a3_zzy);
            T inner = T(4.5) * second;
            if (third.any) inner = inner + T(13.5) * third.s;
            f[i] = f[i] + wi * inner;
        });
    }

    // collision.hpp:169-183 (pi_neq from descriptor.hpp:126-143)
    static __device__ __forceinline__ T smagorinsky_omega(const T (&f)[Q], T omega, T smago_c) {
        const T cs4 = T(1) / T(9);
        T rho, u[3];
        rho_u(f, rho, u);
        const T usqr = usqr_of(u);
        T fn[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            fn[i] = f[i] - eq2<i>(rho, u, usqr);
        });
        T pi[6];
        second_moment(fn, pi);
        const T pi_sq = pi[0] * pi[0] + pi[3] * pi[3] + pi[5] * pi[5] +
                        T(2) * (pi[1] * pi[1] + pi[2] * pi[2] + pi[4] * pi[4]);
        const T q_norm = sqrt(T(2) * pi_sq);
        const T tau0 = T(1) / omega;
        const T tau_eff =
            T(0.5) * (tau0 + sqrt(tau0 * tau0 + T(2) * smago_c * smago_c * q_norm / (rho * cs4)));
        return T(1) / tau_eff;
    }

    // boundaries.hpp:10-17
    static __device__ __forceinline__ void bounce_back(T (&f)[Q]) {
        sfor<(Q - 1) / 2>([&](auto P) {
            constexpr int i = 2 * decltype(P)::value + 1;
            const T t = f[i];
            f[i] = f[i + 1];
            f[i + 1] = t;
        });
    }

    // boundaries.hpp:23-31
    static __device__ __forceinline__ void moving_bounce_back(T (&f)[Q], const T (&uw)[3]) {
        bounce_back(f);
        sfor<Q - 1>([&](auto I0) {
            constexpr int i = decltype(I0)::value + 1;
            const T cu = cdot<i>(uw);
            constexpr double wd = L::w[i];
            f[i] = f[i] + T(2) * T(wd) * T(3) * cu;
        });
    }

    // boundaries.hpp:45-59 + 71-90 + 95-133, for a compile-time (axis, orient).
    template <int AX, int OR>
    static __device__ __forceinline__ void regularized(T (&f)[Q], bool pressure, T target_rho,
                                                       const T (&uw)[3]) {
        Acc<T> s_zero, s_out;
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr int ca = L::c[i][AX] * OR;
            constexpr double wd = L::w[i];
            const T raw = f[i] + T(wd);
            if constexpr (ca == 0) s_zero.add(1, raw);
            else if constexpr (ca < 0) s_out.add(1, raw);
        });
        T rho, u[3];
        if (!pressure) {
            const T un = OR > 0 ? uw[AX] : -uw[AX];
            rho = (s_zero.get() + T(2) * s_out.get()) / (T(1) - un);
            u[0] = uw[0];
            u[1] = uw[1];
            u[2] = uw[2];
        } else {
            rho = target_rho;
            const T un = T(1) - (s_zero.get() + T(2) * s_out.get()) / rho;
            u[0] = T(0);
            u[1] = T(0);
            u[2] = T(0);
            u[AX] = OR > 0 ? un : -un;
        }
        const T usqr = usqr_of(u);
        T feq[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            feq[i] = eq2<i>(rho, u, usqr);
        });
        T fneq[Q];
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            if constexpr (L::c[i][AX] * OR > 0) fneq[i] = f[opp_of(i)] - feq[opp_of(i)];
            else fneq[i] = f[i] - feq[i];
        });
        T pi[6];
        second_moment(fneq, pi);
        sfor<Q>([&](auto I) {
            constexpr int i = decltype(I)::value;
            constexpr double wd = L::w[i];
        const T wi = T(wd);
            f[i] = feq[i] + wi * T(4.5) * h2_contract<i>(pi);
        });
    }

    static __device__ __forceinline__ void regularized_any(T (&f)[Q], const DevRecipe<T>& r) {
        const bool p = r.reg_is_pressure != 0;
        const T (&uw)[3] = r.wall_velocity;
        const int key = r.reg_axis * 2 + (r.reg_orient > 0 ? 0 : 1);
        switch (key) {
            case 0: regularized<0, 1>(f, p, r.target_rho, uw); break;
            case 1: regularized<0, -1>(f, p, r.target_rho, uw); break;
            case 2: regularized<1, 1>(f, p, r.target_rho, uw); break;
            case 3: regularized<1, -1>(f, p, r.target_rho, uw); break;
            case 4: regularized<2, 1>(f, p, r.target_rho, uw); break;
            default: regularized<2, -1>(f, p, r.target_rho, uw); break;
        }
    }

    // chain.hpp:104-144, restricted at compile time to the kinds in KM.
    template <unsigned KM>
    static __device__ __forceinline__ void apply(T (&f)[Q], const DevRecipe<T>& r) {
        if constexpr ((KM & KM_NODYN) != 0) {
            if (r.kind == KIND_NODYN) return;
        }
        if constexpr ((KM & KM_BB) != 0) {
            if (r.kind == KIND_BB) {
                bounce_back(f);
                return;
            }
        }
        if constexpr ((KM & KM_MBB) != 0) {
            if (r.kind == KIND_MBB) {
                moving_bounce_back(f, r.wall_velocity);
                return;
            }
        }
        if constexpr ((KM & (KM_REGV | KM_REGP)) != 0) {
            if (r.has_reg) regularized_any(f, r);
        }
        T om = r.omega;
        T om_minus = r.omega_minus;
        if constexpr ((KM & KM_LES) != 0) {
            if (r.has_les) {
                om = smagorinsky_omega(f, om, r.smagorinsky_c);
                const double hm = double(r.lambda) / (1.0 / double(om) - 0.5);
                om_minus = T(1.0 / (hm + 0.5));
            }
        }
        constexpr unsigned bases = KM & (KM_BGK | KM_TRT | KM_RR);
        if constexpr (bases == KM_BGK) {
            bgk(f, om);
        } else if constexpr (bases == KM_TRT) {
            trt(f, om, om_minus);
        } else if constexpr (bases == KM_RR) {
            rr(f, om, r.omega_bulk_ho);
        } else {
            if constexpr ((KM & KM_BGK) != 0) {
                if (r.base == BASE_BGK) {
                    bgk(f, om);
                    return;
                }
            }
            if constexpr ((KM & KM_TRT) != 0) {
                if (r.base == BASE_TRT) {
                    trt(f, om, om_minus);
                    return;
                }
            }
            if constexpr ((KM & KM_RR) != 0) {
                if (r.base == BASE_RR) rr(f, om, r.omega_bulk_ho);
            }
        }
    }
};

}  // namespace dlb
