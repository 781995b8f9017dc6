// Register butterflies shared by the FFT passes (k_fft.cu) and the fused
// H-stage + FFT pass (k_p2fa.cu): radix 2, 3, 4, 8, 16 on double2 values,
// forward (INV = false) or inverse sign.
#pragma once

#include "common.cuh"

namespace mnb {
namespace {

template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {  // a * (-i) forward, a * (+i) inverse
    return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
    const double2 t = a;
    a = c_add(t, b);
    b = c_sub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
    const double2 t0 = c_add(x0, x2), t1 = c_sub(x0, x2);
    const double2 t2 = c_add(x1, x3), t3 = mul_mi<INV>(c_sub(x1, x3));
    x0 = c_add(t0, t2);
    x2 = c_sub(t0, t2);
    x1 = c_add(t1, t3);
    x3 = c_sub(t1, t3);
}

template <bool INV>
__device__ __forceinline__ void dft3(double2& x0, double2& x1, double2& x2) {
    constexpr double h = 0.86602540378443864676;  // sqrt(3)/2
    const double2 t1 = c_add(x1, x2);
    const double2 t2 = make_double2(x0.x - 0.5 * t1.x, x0.y - 0.5 * t1.y);
    const double2 d = c_sub(x1, x2);
    const double2 t3 = mul_mi<INV>(make_double2(h * d.x, h * d.y));
    x0 = c_add(x0, t1);
    x1 = c_add(t2, t3);
    x2 = c_sub(t2, t3);
}

template <bool INV>
__device__ __forceinline__ double2 w8mul(double2 a, int k) {  // a * w8^k, k in {1,2,3}
    constexpr double r = 0.70710678118654752440;
    if (k == 2) return mul_mi<INV>(a);
    // w8^1 = (1 - i)/sqrt2 (fwd), w8^3 = (-1 - i)/sqrt2 (fwd)
    const double2 m = mul_mi<INV>(a);  // a*(-i)
    if (k == 1) return make_double2(r * (a.x + m.x), r * (a.y + m.y));
    return make_double2(r * (m.x - a.x), r * (m.y - a.y));
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* x) {
    // even/odd split: E = DFT4(x0,x2,x4,x6), O = DFT4(x1,x3,x5,x7)
    dft4<INV>(x[0], x[2], x[4], x[6]);
    dft4<INV>(x[1], x[3], x[5], x[7]);
    double2 o1 = w8mul<INV>(x[3], 1), o2 = w8mul<INV>(x[5], 2), o3 = w8mul<INV>(x[7], 3);
    const double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6], o0 = x[1];
    x[0] = c_add(e0, o0); x[4] = c_sub(e0, o0);
    x[1] = c_add(e1, o1); x[5] = c_sub(e1, o1);
    x[2] = c_add(e2, o2); x[6] = c_sub(e2, o2);
    x[3] = c_add(e3, o3); x[7] = c_sub(e3, o3);
}

template <bool INV>
__device__ __forceinline__ void dft16(double2* x) {
    // n = n2 + 4 n1, k = k1 + 4 k2:  y[k1+4k2] = sum_n2 w4^{n2 k2} w16^{n2 k1} sum_n1 w4^{n1 k1} x[n2+4n1]
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(x[n2], x[n2 + 4], x[n2 + 8], x[n2 + 12]);
    // after: x[n2 + 4 k1] = A[n2][k1]; twiddle by w16^{n2 k1}
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, r = 0.70710678118654752440;
    const double sg = INV ? 1.0 : -1.0;
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) {
            const int e = n2 * k1;  // 1..9
            double wc, ws;
            switch (e) {
                case 1: wc = c1; ws = s1; break;
                case 2: wc = r; ws = r; break;
                case 3: wc = s1; ws = c1; break;
                case 4: wc = 0.0; ws = 1.0; break;
                case 6: wc = -r; ws = r; break;
                case 9: wc = -c1; ws = -s1; break;
                default: wc = 1.0; ws = 0.0; break;
            }
            const double2 w = make_double2(wc, sg * ws);
            x[n2 + 4 * k1] = c_mul(x[n2 + 4 * k1], w);
        }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(x[4 * k1], x[4 * k1 + 1], x[4 * k1 + 2], x[4 * k1 + 3]);
    // now x[4 k1 + k2] = y[k1 + 4 k2]: transpose 4x4 in registers
    double2 t[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) t[i] = x[i];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) x[k1 + 4 * k2] = t[4 * k1 + k2];
}

// dft16 without the closing register transpose: output frequency q is left in
// x[4*(q%4) + q/4] (callers index it at compile time, no register moves).
template <bool INV>
__device__ __forceinline__ void dft16_np(double2* x) {
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) dft4<INV>(x[n2], x[n2 + 4], x[n2 + 8], x[n2 + 12]);
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, r = 0.70710678118654752440;
    const double sg = INV ? 1.0 : -1.0;
#pragma unroll
    for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < 4; ++k1) {
            const int e = n2 * k1;
            double wc, ws;
            switch (e) {
                case 1: wc = c1; ws = s1; break;
                case 2: wc = r; ws = r; break;
                case 3: wc = s1; ws = c1; break;
                case 4: wc = 0.0; ws = 1.0; break;
                case 6: wc = -r; ws = r; break;
                case 9: wc = -c1; ws = -s1; break;
                default: wc = 1.0; ws = 0.0; break;
            }
            x[n2 + 4 * k1] = c_mul(x[n2 + 4 * k1], make_double2(wc, sg * ws));
        }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<INV>(x[4 * k1], x[4 * k1 + 1], x[4 * k1 + 2], x[4 * k1 + 3]);
}
__host__ __device__ constexpr int d16(int q) { return 4 * (q % 4) + q / 4; }

}  // namespace
}  // namespace mnb
