// Generic-length FFT pass (non-power-of-two axes): the reference's
// Kernel1d MixedRadix and Bluestein paths (kernels.hpp:143-216, 283-293)
// for lengths the radix-8 Stockham pass does not cover.
//
// Same lane addressing and store epilogue (fused exchange, normalize, lane
// kinds) as the main pass; the transform itself runs in shared memory:
//   * smooth lengths (largest prime factor <= 13): self-sorting mixed-radix
//     Stockham, radices 8/4/2 then 3, 5, 7, 11, 13, ping-pong buffers;
//   * other lengths: Bluestein / chirp-z with a power-of-two convolution of
//     length m = bit_ceil(2n - 1), chirp and kernel spectrum precomputed on
//     the host in double (kernels.hpp:179-216 semantics).
// Twiddles come from sincospi in the working precision's double path.
#pragma once

#include "fft_pass.cuh"

namespace dfftb {

constexpr int kMaxStages = 24;

struct GenParams {
  PassParams p;
  int n;          // transform length
  int L;          // working length: n (mixed radix) or m (Bluestein)
  int W;          // lanes per CTA
  int nrad;
  int rad[kMaxStages];
  int bluestein;
  const void* chirp;  // n complex: exp(-i pi j^2 / n)
  const void* kfft;   // m complex: FFT_m(conj chirp, wrapped) / m
};

template <typename T>
__device__ __forceinline__ Cpx<T> unit_root(int k, int M) {
  // exp(-2 pi i k / M)
  double s, c;
  sincospi(-2.0 * (double)k / (double)M, &s, &c);
  return Cpx<T>{(T)c, (T)s};
}

// One mixed-radix Stockham stage over W lanes of length L in shared memory:
// out[(j/ns)*ns*R + j%ns + r*ns] = DFT_R( in[j + r*L/R] * w^(r*(j%ns)) )
template <typename T>
__device__ void generic_stage(const Cpx<T>* in, Cpx<T>* out, int L, int W, int R, int ns) {
  using C = Cpx<T>;
  const int nb = L / R;
  for (int b = threadIdx.x; b < W * nb; b += blockDim.x) {
    const int w = b / nb;
    const int j = b - w * nb;
    const C* li = in + (size_t)w * L;
    C* lo = out + (size_t)w * L;
    C x[16];
    const int pp = j % ns;
    for (int r = 0; r < R; ++r) {
      C v = li[j + r * nb];
      if (r && pp) v = cmul(v, unit_root<T>(r * pp, ns * R));
      x[r] = v;
    }
    C y[16];
    if (R == 2) {
      y[0] = cadd(x[0], x[1]);
      y[1] = csub(x[0], x[1]);
    } else if (R == 4) {
      y[0] = x[0]; y[1] = x[1]; y[2] = x[2]; y[3] = x[3];
      dft4<C, T>(y[0], y[1], y[2], y[3]);
    } else if (R == 8) {
      for (int r = 0; r < 8; ++r) y[r] = x[r];
      dft8<C, T>(y);
    } else {
      // odd prime radix: direct DFT with the R roots of unity
      C root[16];
      for (int m = 0; m < R; ++m) root[m] = unit_root<T>(m, R);
      for (int t = 0; t < R; ++t) {
        C acc = x[0];
        for (int jj = 1; jj < R; ++jj) acc = cadd(acc, cmul(x[jj], root[(jj * t) % R]));
        y[t] = acc;
      }
    }
    const int base = (j - pp) * R + pp;
    for (int r = 0; r < R; ++r) lo[base + r * ns] = y[r];
  }
  __syncthreads();
}

// forward DFT of W lanes of length L held in a; result lands in a or b,
// returned pointer says which
template <typename T>
__device__ Cpx<T>* generic_fft(Cpx<T>* a, Cpx<T>* b, const GenParams& g) {
  int ns = 1;
  for (int s = 0; s < g.nrad; ++s) {
    generic_stage<T>(a, b, g.L, g.W, g.rad[s], ns);
    ns *= g.rad[s];
    Cpx<T>* t = a;
    a = b;
    b = t;
  }
  return a;
}

template <typename T>
__global__ void __launch_bounds__(256) fft_generic_kernel(const __grid_constant__ GenParams g) {
  using C = Cpx<T>;
  const PassParams& p = g.p;
  extern __shared__ __align__(16) unsigned char smem_gen[];
  C* a = reinterpret_cast<C*>(smem_gen);
  C* b = a + (size_t)g.W * g.L;
  const int n = g.n, L = g.L, W = g.W;
  const int tiles_b = (p.B + W - 1) / W;
  const int alpha = blockIdx.x / tiles_b;
  const int beta0 = (blockIdx.x - alpha * tiles_b) * W;
  const bool adj = p.in_si != 1;
  const int lane_len = p.in_mode == kInHermitian ? n / 2 + 1 : n;
  double lmax = 0.0, limag = 0.0;

  // ---- load (lane semantics as in the Stockham pass), coalesced mapping
  for (int e = threadIdx.x; e < W * n; e += blockDim.x) {
    const int w = adj ? e % W : e / n;
    const int i = adj ? e / W : e % n;
    const int beta = beta0 + w;
    C x = C{T(0), T(0)};
    if (beta < p.B) {
      const int64_t lane = in_alpha_off(p, alpha) + (int64_t)beta * p.in_sb;
      if (p.in_mode == kInComplex) {
        x = reinterpret_cast<const C*>(p.in)[lane + (int64_t)i * p.in_si];
      } else if (p.in_mode == kInReal) {
        x.x = reinterpret_cast<const T*>(p.in)[lane + (int64_t)i * p.in_si];
      } else {
        const bool lo = i <= n / 2;
        x = reinterpret_cast<const C*>(p.in)[lane + (int64_t)(lo ? i : n - i) * p.in_si];
        if (lo) {
          const double m = hypot((double)x.x, (double)x.y);
          lmax = m > lmax ? m : lmax;
        }
        if (i == 0 || (n % 2 == 0 && i == n / 2)) {
          limag = fabs((double)x.y) > limag ? fabs((double)x.y) : limag;
          x.y = T(0);
        }
        if (!lo) x.y = -x.y;  // Hermitian mirror
      }
    }
    if (p.inverse) x.y = -x.y;
    if (g.bluestein) x = cmul(x, reinterpret_cast<const C*>(g.chirp)[i]);
    a[(size_t)w * L + i] = x;
  }
  (void)lane_len;
  if (g.bluestein) {
    for (int e = threadIdx.x; e < W * (L - n); e += blockDim.x) {
      const int w = e / (L - n);
      a[(size_t)w * L + n + (e - w * (L - n))] = C{T(0), T(0)};
    }
  }
  __syncthreads();
  if (p.in_mode == kInHermitian) herm_reduce(p.herm, lmax, limag);

  C* r = generic_fft<T>(a, b, g);
  if (g.bluestein) {
    // pointwise with the kernel spectrum, then the inverse length-m DFT as
    // conj(F(conj .)), then the output chirp (run_bluestein, kernels.hpp:283-293)
    const C* kf = reinterpret_cast<const C*>(g.kfft);
    for (int e = threadIdx.x; e < W * L; e += blockDim.x) {
      C v = cmul(r[e], kf[e % L]);
      r[e] = C{v.x, -v.y};
    }
    __syncthreads();
    C* other = r == a ? b : a;
    r = generic_fft<T>(r, other, g);
    const C* ch = reinterpret_cast<const C*>(g.chirp);
    for (int e = threadIdx.x; e < W * n; e += blockDim.x) {
      const int w = e / n, k = e - w * n;
      C v = r[(size_t)w * L + k];
      v.y = -v.y;
      r[(size_t)w * L + k] = cmul(v, ch[k]);
    }
    __syncthreads();
  }

  // ---- store: coalesced along whichever of (k, lane) is contiguous in dest
  const T sc = static_cast<T>(p.scale);
  const bool k_contig = p.dest[0].sk == 1;
  for (int e = threadIdx.x; e < W * p.n_out; e += blockDim.x) {
    const int w = k_contig ? e / p.n_out : e % W;
    const int k = k_contig ? e - w * p.n_out : e / W;
    const int beta = beta0 + w;
    if (beta >= p.B) continue;
    const int q = p.ndest > 1 ? (int)(k / p.oblk) : 0;
    const int kk = k - (int)(q * p.oblk);
    const Dest& d = p.dest[q];
    const int64_t off = d.base + dst_alpha_off(p, d, alpha) + (int64_t)beta * d.sb + (int64_t)kk * d.sk;
    C v = r[(size_t)w * L + k];
    if (p.inverse) v.y = -v.y;
    if (p.out_real) {
      reinterpret_cast<T*>(d.ptr)[off] = v.x * sc;
    } else {
      reinterpret_cast<C*>(d.ptr)[off] = C{v.x * sc, v.y * sc};
    }
  }
}

}  // namespace dfftb
