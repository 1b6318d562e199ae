// Register-resident FFT engine for the AIMx grid passes (sm_100a).
//
// A line of length L = R1 * R2 is transformed by T = min(R1, R2) threads of
// one warp (T <= 32), each holding E = L / T complex values in registers:
//   input distribution  D(R1,R2): v[a R2 + n2] = x[t + T a + R1 n2],  a < R1/T
//   step 1: DFT_R2 over n2 for each n1 = t + T a   (in registers)
//   twiddle Y[n1][k2] *= W_L^(n1 k2)               (shared-memory table)
//   exchange through a per-line shared buffer [k2][n1] (row stride R1 + 1),
//            one block barrier (all threads of the CTA call fft2 uniformly)
//   step 3: DFT_R1 over n1 for each k2 = t + T c  (in registers)
//   output distribution D(R2,R1): v[c R1 + k1] = X[t + T c + R2 k1]
// This is the four-step factorisation X[k2 + R2 k1] = sum_n1 W_L^(n1 k2)
// W_R1^(n1 k1) sum_n2 x[n1 + R1 n2] W_R2^(n2 k2).  Because D(R2,R1) is the
// input distribution of a transform with the factors swapped, a forward
// (R1,R2) transform followed by an inverse (R2,R1) one returns to D(R1,R2)
// with no extra data movement: loads and stores go straight between
// registers and global memory.  The small DFTs (2, 4, 8, 16, 32) are fully
// unrolled with twiddles from a constant-bank table (free FFMA operands).
#pragma once

#include "fft.cuh"

namespace aimx {

// W_32^m = exp(-2 pi i m / 32), exactly symmetric
static __constant__ double2 c_w32d[32] = {
    {1.0, -0.0},
    {0.9807852804032304, -0.19509032201612825},
    {0.9238795325112867, -0.3826834323650898},
    {0.8314696123025452, -0.5555702330196022},
    {0.7071067811865476, -0.7071067811865475},
    {0.5555702330196022, -0.8314696123025452},
    {0.3826834323650898, -0.9238795325112867},
    {0.19509032201612825, -0.9807852804032304},
    {-0.0, -1.0},
    {-0.19509032201612825, -0.9807852804032304},
    {-0.3826834323650898, -0.9238795325112867},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.7071067811865475, -0.7071067811865476},
    {-0.8314696123025452, -0.5555702330196022},
    {-0.9238795325112867, -0.3826834323650898},
    {-0.9807852804032304, -0.19509032201612825},
    {-1.0, 0.0},
    {-0.9807852804032304, 0.19509032201612825},
    {-0.9238795325112867, 0.3826834323650898},
    {-0.8314696123025452, 0.5555702330196022},
    {-0.7071067811865476, 0.7071067811865475},
    {-0.5555702330196022, 0.8314696123025452},
    {-0.3826834323650898, 0.9238795325112867},
    {-0.19509032201612825, 0.9807852804032304},
    {0.0, 1.0},
    {0.19509032201612825, 0.9807852804032304},
    {0.3826834323650898, 0.9238795325112867},
    {0.5555702330196022, 0.8314696123025452},
    {0.7071067811865475, 0.7071067811865476},
    {0.8314696123025452, 0.5555702330196022},
    {0.9238795325112867, 0.3826834323650898},
    {0.9807852804032304, 0.19509032201612825}};
static __constant__ float2 c_w32f[32] = {
    {1.0, -0.0},
    {0.9807852804032304, -0.19509032201612825},
    {0.9238795325112867, -0.3826834323650898},
    {0.8314696123025452, -0.5555702330196022},
    {0.7071067811865476, -0.7071067811865475},
    {0.5555702330196022, -0.8314696123025452},
    {0.3826834323650898, -0.9238795325112867},
    {0.19509032201612825, -0.9807852804032304},
    {-0.0, -1.0},
    {-0.19509032201612825, -0.9807852804032304},
    {-0.3826834323650898, -0.9238795325112867},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.7071067811865475, -0.7071067811865476},
    {-0.8314696123025452, -0.5555702330196022},
    {-0.9238795325112867, -0.3826834323650898},
    {-0.9807852804032304, -0.19509032201612825},
    {-1.0, 0.0},
    {-0.9807852804032304, 0.19509032201612825},
    {-0.9238795325112867, 0.3826834323650898},
    {-0.8314696123025452, 0.5555702330196022},
    {-0.7071067811865476, 0.7071067811865475},
    {-0.5555702330196022, 0.8314696123025452},
    {-0.3826834323650898, 0.9238795325112867},
    {-0.19509032201612825, 0.9807852804032304},
    {0.0, 1.0},
    {0.19509032201612825, 0.9807852804032304},
    {0.3826834323650898, 0.9238795325112867},
    {0.5555702330196022, 0.8314696123025452},
    {0.7071067811865475, 0.7071067811865476},
    {0.8314696123025452, 0.5555702330196022},
    {0.9238795325112867, 0.3826834323650898},
    {0.9807852804032304, 0.19509032201612825}};

template <typename T2> __device__ __forceinline__ T2 w32(int m);
template <> __device__ __forceinline__ float2 w32<float2>(int m) { return c_w32f[m & 31]; }
template <> __device__ __forceinline__ double2 w32<double2>(int m) { return c_w32d[m & 31]; }

template <typename T2, bool INV> __device__ __forceinline__ T2 twmul(T2 v, T2 w) {
  if (INV) w.y = -w.y;
  return cmul(v, w);
}

// DFT of length 16 (4 x 4), natural order in and out.
template <typename T2, bool INV> __device__ __forceinline__ void dft16(T2* v) {
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) dft4<T2, INV>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
    for (int k2 = 1; k2 < 4; ++k2) v[n1 + 4 * k2] = twmul<T2, INV>(v[n1 + 4 * k2], w32<T2>(2 * n1 * k2));
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) dft4<T2, INV>(v[4 * k2], v[4 * k2 + 1], v[4 * k2 + 2], v[4 * k2 + 3]);
  // X[k2 + 4 k1] sits at v[4 k2 + k1]
  T2 t[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) t[k] = v[4 * (k & 3) + (k >> 2)];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = t[k];
}

// DFT of length 32 (4 x 8), natural order in and out.
template <typename T2, bool INV> __device__ __forceinline__ void dft32(T2* v) {
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {
    T2 u[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) u[n2] = v[n1 + 4 * n2];
    dft8<T2, INV>(u);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) v[n1 + 4 * k2] = (n1 == 0 || k2 == 0) ? u[k2] : twmul<T2, INV>(u[k2], w32<T2>(n1 * k2));
  }
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) dft4<T2, INV>(v[4 * k2], v[4 * k2 + 1], v[4 * k2 + 2], v[4 * k2 + 3]);
  // X[k2 + 8 k1] sits at v[4 k2 + k1]
  T2 t[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) t[k] = v[4 * (k & 7) + (k >> 3)];
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = t[k];
}


// W_24^m = exp(-2 pi i m / 24) (the radix-3 lengths 48, 96, 192 = 3 * 2^k)
static __constant__ double2 c_w24d[24] = {
    {1.0, 0.0},
    {0.9659258262890683, -0.25881904510252074},
    {0.8660254037844387, -0.49999999999999994},
    {0.7071067811865476, -0.7071067811865475},
    {0.5000000000000001, -0.8660254037844386},
    {0.25881904510252074, -0.9659258262890683},
    {0.0, -1.0},
    {-0.25881904510252063, -0.9659258262890683},
    {-0.4999999999999998, -0.8660254037844387},
    {-0.7071067811865475, -0.7071067811865476},
    {-0.8660254037844387, -0.49999999999999994},
    {-0.9659258262890682, -0.258819045102521},
    {-1.0, 0.0},
    {-0.9659258262890683, 0.2588190451025208},
    {-0.8660254037844388, 0.4999999999999997},
    {-0.7071067811865479, 0.7071067811865471},
    {-0.5000000000000004, 0.8660254037844384},
    {-0.25881904510252063, 0.9659258262890683},
    {0.0, 1.0},
    {0.2588190451025203, 0.9659258262890684},
    {0.5000000000000001, 0.8660254037844386},
    {0.7071067811865474, 0.7071067811865477},
    {0.8660254037844384, 0.5000000000000004},
    {0.9659258262890681, 0.25881904510252157}};
static __constant__ float2 c_w24f[24] = {
    {1.0f, 0.0f},
    {0.9659258262890683f, -0.25881904510252074f},
    {0.8660254037844387f, -0.49999999999999994f},
    {0.7071067811865476f, -0.7071067811865475f},
    {0.5000000000000001f, -0.8660254037844386f},
    {0.25881904510252074f, -0.9659258262890683f},
    {0.0f, -1.0f},
    {-0.25881904510252063f, -0.9659258262890683f},
    {-0.4999999999999998f, -0.8660254037844387f},
    {-0.7071067811865475f, -0.7071067811865476f},
    {-0.8660254037844387f, -0.49999999999999994f},
    {-0.9659258262890682f, -0.258819045102521f},
    {-1.0f, 0.0f},
    {-0.9659258262890683f, 0.2588190451025208f},
    {-0.8660254037844388f, 0.4999999999999997f},
    {-0.7071067811865479f, 0.7071067811865471f},
    {-0.5000000000000004f, 0.8660254037844384f},
    {-0.25881904510252063f, 0.9659258262890683f},
    {0.0f, 1.0f},
    {0.2588190451025203f, 0.9659258262890684f},
    {0.5000000000000001f, 0.8660254037844386f},
    {0.7071067811865474f, 0.7071067811865477f},
    {0.8660254037844384f, 0.5000000000000004f},
    {0.9659258262890681f, 0.25881904510252157f}};

template <typename T2> __device__ __forceinline__ T2 w24(int m);
template <> __device__ __forceinline__ float2 w24<float2>(int m) { return c_w24f[m % 24]; }
template <> __device__ __forceinline__ double2 w24<double2>(int m) { return c_w24d[m % 24]; }

// DFT of length 3: X1, X2 = a - (b + c)/2 -+ j (sqrt3/2)(b - c) (forward; +- inverse)
template <typename T2, bool INV> __device__ __forceinline__ void dft3(T2& a, T2& b, T2& c) {
  using R = decltype(T2::x);
  const R h = (R)0.86602540378443864676;   // sin(2 pi / 3)
  const T2 t1 = cadd(b, c), t2 = csub(b, c);
  const T2 m = mk<T2>(a.x - (R)0.5 * t1.x, a.y - (R)0.5 * t1.y);
  a = cadd(a, t1);
  // -j h t2 = h (t2.y, -t2.x)
  const T2 jt = INV ? mk<T2>(-h * t2.y, h * t2.x) : mk<T2>(h * t2.y, -h * t2.x);
  b = cadd(m, jt);
  c = csub(m, jt);
}

// DFT of length 24 (3 x 8), natural order in and out.
template <typename T2, bool INV> __device__ __forceinline__ void dft24(T2* v) {
#pragma unroll
  for (int n1 = 0; n1 < 3; ++n1) {
    T2 u[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) u[n2] = v[n1 + 3 * n2];
    dft8<T2, INV>(u);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) v[n1 + 3 * k2] = (n1 == 0 || k2 == 0) ? u[k2] : twmul<T2, INV>(u[k2], w24<T2>(n1 * k2));
  }
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) dft3<T2, INV>(v[3 * k2], v[3 * k2 + 1], v[3 * k2 + 2]);
  // X[k2 + 8 k1] sits at v[3 k2 + k1]
  T2 t[24];
#pragma unroll
  for (int k = 0; k < 24; ++k) t[k] = v[3 * (k & 7) + (k >> 3)];
#pragma unroll
  for (int k = 0; k < 24; ++k) v[k] = t[k];
}

template <typename T2, int R, bool INV> __device__ __forceinline__ void dftr(T2* v) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) dft2<T2, INV>(v);
  else if constexpr (R == 4) dft4<T2, INV>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<T2, INV>(v);
  else if constexpr (R == 16) dft16<T2, INV>(v);
  else if constexpr (R == 24) dft24<T2, INV>(v);
  else dft32<T2, INV>(v);
}

// Factorisation of each supported length.
template <int L> struct Fac;
template <> struct Fac<8> { static constexpr int R1 = 1, R2 = 8; };
template <> struct Fac<16> { static constexpr int R1 = 1, R2 = 16; };
template <> struct Fac<32> { static constexpr int R1 = 4, R2 = 8; };
template <> struct Fac<64> { static constexpr int R1 = 8, R2 = 8; };
template <> struct Fac<128> { static constexpr int R1 = 8, R2 = 16; };
template <> struct Fac<256> { static constexpr int R1 = 16, R2 = 16; };
template <> struct Fac<512> { static constexpr int R1 = 16, R2 = 32; };
template <> struct Fac<1024> { static constexpr int R1 = 32, R2 = 32; };
// radix-3 lengths (cfg4's 96^3 grid pads to 192): R2 = 24 = 3 x 8, T = R1 threads
template <> struct Fac<48> { static constexpr int R1 = 2, R2 = 24; };
template <> struct Fac<96> { static constexpr int R1 = 4, R2 = 24; };
template <> struct Fac<192> { static constexpr int R1 = 8, R2 = 24; };

template <int R1, int R2> struct TwoLevel {
  static constexpr int L = R1 * R2;
  static constexpr int T = R1 < R2 ? R1 : R2;   // threads per line
  static constexpr int E = L / T;               // complex values per thread
  static constexpr int XB = R2 * (R1 + 1);   // exchange elements: [k2 < R2][n1 < R1], row stride R1 + 1
  // element index held in slot i under the input distribution D(R1,R2)
  static __device__ __forceinline__ int in_index(int t, int i) {
    return t + T * (i / R2) + R1 * (i % R2);
  }
  // ... and under the output distribution D(R2,R1)
  static __device__ __forceinline__ int out_index(int t, int i) {
    return t + T * (i / R1) + R2 * (i % R1);
  }
};

// v: E registers in D(R1,R2) -> D(R2,R1).  xb: this line's exchange buffer,
// tw: W_L table (shared), t: thread index within the line.
template <typename T2, int R1, int R2, bool INV>
__device__ __forceinline__ void fft2(T2* v, T2* xb, const T2* tw, int t) {
  using TL = TwoLevel<R1, R2>;
  constexpr int T = TL::T, A = R1 / T, C = R2 / T;
  if constexpr (R2 == 1) {   // one thread holds the whole line in natural order
    dftr<T2, R1, INV>(v);
    return;
  }
#pragma unroll
  for (int a = 0; a < A; ++a) dftr<T2, R2, INV>(v + a * R2);
  if constexpr (R1 > 1) {
#pragma unroll
    for (int a = 0; a < A; ++a) {
      const int n1 = t + T * a;
#pragma unroll
      for (int k2 = 1; k2 < R2; ++k2) v[a * R2 + k2] = twmul<T2, INV>(v[a * R2 + k2], tw[n1 * k2]);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < A; ++a)
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) xb[k2 * (R1 + 1) + t + T * a] = v[a * R2 + k2];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) v[c * R1 + n1] = xb[(t + T * c) * (R1 + 1) + n1];
#pragma unroll
    for (int c = 0; c < C; ++c) dftr<T2, R1, INV>(v + c * R1);
  }
}

}  // namespace aimx
