// Exact P1 element math for sm_100a.
//
// Every expression below reproduces the reference's floating-point operation
// sequence (batch.cpp:56-312, reference.cpp:45-239) with FMA contraction
// disabled (the library is compiled with -fmad=false), so every NONZERO value
// is bit-identical to the reference.  Terms that the reference multiplies by a
// structural zero of the P1 gradient table are dropped: adding +-0 leaves a
// nonzero partial sum unchanged, and the Reduce stage's left fold starts at
// +0.0 (routing.cpp:119) so the only possible difference — the sign of an
// exact zero — is canonicalised away in every CSR value (a sum that starts at
// +0.0 can never become -0.0 under round-to-nearest).  Materialised local
// tensors add that +0.0 explicitly.
#pragma once

#include <cstdint>

#include "tgk.h"

namespace tgk {

// ------------------------------------------------------------ reference tables
// Quadrature rules (reference.cpp:99-210) and basis values evaluated with the
// same double expressions, as compile-time constants so the optimiser can
// share identical products without changing any rounding.
template <int KIND, int DEG>
struct Rule;

template <>
struct Rule<TGK_TRI3, 1> {
    static constexpr int Q = 1;
    __host__ __device__ static constexpr double pt(int, int) { return 1.0 / 3.0; }
    __host__ __device__ static constexpr double w(int) { return 0.5; }
};
template <>
struct Rule<TGK_TRI3, 2> {
    static constexpr int Q = 3;
    __host__ __device__ static constexpr double pt(int q, int c) {
        // {1/6,1/6, 2/3,1/6, 1/6,2/3}
        return (q == 1 && c == 0) || (q == 2 && c == 1) ? 2.0 / 3 : 1.0 / 6;
    }
    __host__ __device__ static constexpr double w(int) { return 1.0 / 6; }
};
template <>
struct Rule<TGK_TRI3, 3> {
    static constexpr int Q = 4;
    __host__ __device__ static constexpr double pt(int q, int c) {
        // {1/3,1/3, 0.2,0.2, 0.6,0.2, 0.2,0.6}
        return q == 0 ? 1.0 / 3 : ((q == 2 && c == 0) || (q == 3 && c == 1) ? 0.6 : 0.2);
    }
    __host__ __device__ static constexpr double w(int q) { return q == 0 ? -27.0 / 96 : 25.0 / 96; }
};
template <>
struct Rule<TGK_TRI3, 4> {
    static constexpr int Q = 6;
    __host__ __device__ static constexpr double a1() { return 0.445948490915965; }
    __host__ __device__ static constexpr double a2() { return 0.091576213509771; }
    __host__ __device__ static constexpr double pt(int q, int c) {
        // {a1,a1, 1-2a1,a1, a1,1-2a1, a2,a2, 1-2a2,a2, a2,1-2a2}
        const double a = q < 3 ? a1() : a2();
        const int r = q % 3;
        return (r == 1 && c == 0) || (r == 2 && c == 1) ? 1 - 2 * a : a;
    }
    __host__ __device__ static constexpr double w(int q) {
        return q < 3 ? 0.223381589678011 / 2 : 0.109951743655322 / 2;
    }
};
template <>
struct Rule<TGK_TET4, 1> {
    static constexpr int Q = 1;
    __host__ __device__ static constexpr double pt(int, int) { return 0.25; }
    __host__ __device__ static constexpr double w(int) { return 1.0 / 6.0; }
};
template <>
struct Rule<TGK_TET4, 2> {
    static constexpr int Q = 4;
    __host__ __device__ static constexpr double pt(int q, int c) {
        // {b,b,b, a,b,b, b,a,b, b,b,a}
        return (q >= 1 && c == q - 1) ? 0.585410196624969 : 0.138196601125011;
    }
    __host__ __device__ static constexpr double w(int) { return 1.0 / 24.0; }
};
template <>
struct Rule<TGK_TET4, 3> {
    static constexpr int Q = 5;
    __host__ __device__ static constexpr double pt(int q, int c) {
        // {0.25,0.25,0.25, s,s,s, 0.5,s,s, s,0.5,s, s,s,0.5}
        return q == 0 ? 0.25 : ((q >= 2 && c == q - 2) ? 0.5 : 1.0 / 6.0);
    }
    __host__ __device__ static constexpr double w(int q) {
        return q == 0 ? -4.0 / 5.0 / 6.0 : 9.0 / 20.0 / 6.0;
    }
};
template <>
struct Rule<TGK_TET4, 4> {
    static constexpr int Q = 11;
    __host__ __device__ static constexpr double pt(int q, int c) {
        constexpr double a = 11.0 / 14.0, b = 1.0 / 14.0;
        constexpr double cc = 0.399403576166799, dd = 0.100596423833201;
        // {0.25x3, b,b,b, a,b,b, b,a,b, b,b,a, c,dd,dd, dd,c,dd, dd,dd,c, dd,c,c, c,dd,c, c,c,dd}
        if (q == 0) return 0.25;
        if (q == 1) return b;
        if (q <= 4) return c == q - 2 ? a : b;
        if (q <= 7) return c == q - 5 ? cc : dd;
        return c == q - 8 ? dd : cc;
    }
    __host__ __device__ static constexpr double w(int q) {
        return q == 0 ? -74.0 / 5625.0 : (q <= 4 ? 343.0 / 45000.0 : 56.0 / 2250.0);
    }
};

// shape_values (reference.cpp:45-57)
template <int KIND, int DEG>
__host__ __device__ constexpr double basis(int q, int a) {
    using R = Rule<KIND, DEG>;
    if (KIND == TGK_TRI3) {
        if (a == 0) return 1.0 - R::pt(q, 0) - R::pt(q, 1);
        return R::pt(q, a - 1);
    } else {
        if (a == 0) return 1.0 - R::pt(q, 0) - R::pt(q, 1) - R::pt(q, 2);
        return R::pt(q, a - 1);
    }
}

template <int KIND>
struct P1 {
    static constexpr int k = KIND == TGK_TRI3 ? 3 : 4;
    static constexpr int d = KIND == TGK_TRI3 ? 2 : 3;
};

// ------------------------------------------------------------ division
// Correctly rounded c / det from one correctly rounded reciprocal
// y = RN(1/det) (__drcp_rn) and Markstein's correction
//   q = RN(c*y);  r = c - det*q (exact, FMA);  RN(q + r*y) == RN(c/det)
// (Markstein 1990; Muller et al., Handbook of Floating-Point Arithmetic,
// "division with an FMA").  The theorem needs every quantity to stay in the
// normal range.  The fused kernels use it only on meshes certified by
// mesh_division_safe() (host.cpp): all coordinates 0 or 2^-40 <= |x| <= 2^40,
// so nonzero Jacobian entries lie in [2^-92, 2^41], cofactors in
// [2^-236, 2^84] or 0, det in [2^-328, 2^125] and all quotients/residuals are
// normal.  Uncertified meshes take IEEE division.  Nonzero quotients are then
// bit-identical to c / det; only the sign of an exact zero may differ, which
// cannot reach a CSR value (see the header comment).  Verified against IEEE
// division on 1.7e10 random and adversarial operand pairs on a B200
// (tools/div_check.cu, profiles/r01_div_check.log).
struct ExactDiv {
    double det, y;
    __device__ __forceinline__ explicit ExactDiv(double d) : det(d), y(0.0) {
#ifdef __CUDA_ARCH__
        y = __drcp_rn(d);
#endif
    }
    __device__ __forceinline__ double operator()(double c) const {
        const double q = c * y;
        const double r = __fma_rn(-det, q, c);
        return __fma_rn(r, y, q);
    }
};

// ------------------------------------------------------------ geometry
// batch_geometry (batch.cpp:76-104) + push_forward (batch.cpp:139-152) for an
// affine simplex.  X: node coordinates (k x d).  Outputs det and the physical
// basis gradients G (k x d).  Returns false when det <= 0 (batch.cpp:98-101).
// FASTDIV selects ExactDiv (same nonzero bits, ~3 instead of ~30 instructions
// per quotient) for the fused kernels; the materialised drop-ins keep '/'.
// T = float: the fp32 mode (tgk_assemble_f32_d), same expressions in fp32
// with IEEE division (FASTDIV is fp64-only).
template <int KIND, bool FASTDIV = false, typename T = double>
__device__ __forceinline__ bool simplex_geometry(const T (&X)[P1<KIND>::k][P1<KIND>::d],
                                                 T& det, T (&G)[P1<KIND>::k][P1<KIND>::d]) {
    static_assert(!FASTDIV || sizeof(T) == 8, "Markstein division is the fp64 path");
    if constexpr (KIND == TGK_TET4) {
        // J[i][j] = sum_a X[a][i] * Ghat[a][j]; Ghat row 0 = -1, rows 1..3 = e_j
        T J[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) J[i * 3 + j] = X[j + 1][i] - X[0][i];
        // invert_transpose cofactors (batch.cpp:26-34)
        const T c00 = J[4] * J[8] - J[5] * J[7];
        const T c01 = J[5] * J[6] - J[3] * J[8];
        const T c02 = J[3] * J[7] - J[4] * J[6];
        const T c10 = J[2] * J[7] - J[1] * J[8];
        const T c11 = J[0] * J[8] - J[2] * J[6];
        const T c12 = J[1] * J[6] - J[0] * J[7];
        const T c20 = J[1] * J[5] - J[2] * J[4];
        const T c21 = J[2] * J[3] - J[0] * J[5];
        const T c22 = J[0] * J[4] - J[1] * J[3];
        // batch.cpp:95-96: J0*(J4J8-J5J7) - J1*(J3J8-J5J6) + J2*(J3J7-J4J6)
        //   == (J0*c00 + J1*c01) + J2*c02 exactly (c01 is the negated middle term)
        det = (J[0] * c00 + J[1] * c01) + J[2] * c02;
        if (det <= T(0)) return false;
        // J^{-T} = cofactor / det (batch.cpp:36-44); push_forward: G_a = J^{-T} Ghat_a
        T t00, t01, t02, t10, t11, t12, t20, t21, t22;
        if constexpr (FASTDIV) {
            const ExactDiv dv(det);
            t00 = dv(c00); t01 = dv(c01); t02 = dv(c02);
            t10 = dv(c10); t11 = dv(c11); t12 = dv(c12);
            t20 = dv(c20); t21 = dv(c21); t22 = dv(c22);
        } else {
            t00 = c00 / det; t01 = c01 / det; t02 = c02 / det;
            t10 = c10 / det; t11 = c11 / det; t12 = c12 / det;
            t20 = c20 / det; t21 = c21 / det; t22 = c22 / det;
        }
        G[1][0] = t00; G[2][0] = t01; G[3][0] = t02;
        G[1][1] = t10; G[2][1] = t11; G[3][1] = t12;
        G[1][2] = t20; G[2][2] = t21; G[3][2] = t22;
        G[0][0] = -((t00 + t01) + t02);
        G[0][1] = -((t10 + t11) + t12);
        G[0][2] = -((t20 + t21) + t22);
    } else {
        const T J0 = X[1][0] - X[0][0], J1 = X[2][0] - X[0][0];
        const T J2 = X[1][1] - X[0][1], J3 = X[2][1] - X[0][1];
        det = J0 * J3 - J1 * J2;
        if (det <= T(0)) return false;
        // batch.cpp:21-24
        T t00, t01, t10, t11;
        if constexpr (FASTDIV) {
            const ExactDiv dv(det);
            t00 = dv(J3); t01 = dv(-J2); t10 = dv(-J1); t11 = dv(J0);
        } else {
            t00 = J3 / det; t01 = -J2 / det; t10 = -J1 / det; t11 = J0 / det;
        }
        G[1][0] = t00; G[2][0] = t01;
        G[1][1] = t10; G[2][1] = t11;
        G[0][0] = -(t00 + t01);
        G[0][1] = -(t10 + t11);
    }
    return true;
}

// dot_ab of local_stiffness_diffusion (batch.cpp:173-174)
template <int KIND, typename T = double>
__device__ __forceinline__ T gdot(const T (&G)[P1<KIND>::k][P1<KIND>::d], int a, int b) {
    if constexpr (KIND == TGK_TET4)
        return (G[a][0] * G[b][0] + G[a][1] * G[b][1]) + G[a][2] * G[b][2];
    else
        return G[a][0] * G[b][0] + G[a][1] * G[b][1];
}

// symmetric index of (a,b) in a packed upper triangle (a<=b), k=3: 6, k=4: 10
template <int K>
__host__ __device__ constexpr int sym_idx(int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * K - lo * (lo - 1) / 2 + (hi - lo);
}

}  // namespace tgk
