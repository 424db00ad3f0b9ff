// Single-launch batch norm (K5-support of DESIGN.md): statistics, finalisation and the
// elementwise pass of a BN layer in ONE persistent cooperative kernel.
//
//   forward : pass 1 per-channel sum / sum-of-squares of the CTA's rows -> partials
//             grid barrier -> channel finalisation (mean, rstd, running stats)
//             grid barrier -> pass 2 y = act(gamma*(x-mean)*rstd + beta [+ res])
//   backward: pass 1 dz = dy * relu-mask, partials of sum(dz) and sum(dz*xhat) [dz stored]
//             grid barrier -> dbeta/dgamma
//             grid barrier -> pass 2 dx = gamma*rstd*(dz - dbeta/M - xhat*dgamma/M)
//
// Why one launch: the three-kernel form (partial / finalize / apply) paid two launch tails
// and a serial finalize per layer, and its apply pass re-read the tensors from HBM after the
// L2 had been flushed by other CTAs.  Here each CTA re-reads exactly the rows it reduced in
// pass 1 (L2-hot for all but the largest tensors).  Every reduction is fixed-order (thread ->
// smem in row-lane order -> partial per CTA -> channel sum over CTAs in index order), so
// results are bit-identical run to run and identical to the three-kernel numerics up to the
// summation tree.
//
// Co-residency for the grid barrier is guaranteed by a cooperative launch (capturable into
// CUDA graphs); the barrier is a generation counter in global memory that returns to zero.
#include "cvb_common.cuh"
#include <cuda_bf16.h>
#include <math.h>

namespace {

typedef __nv_bfloat16 bf16;
constexpr int THREADS = 512;
constexpr int MAX_OCC = 2;        // CTAs per SM (partials workspace = grid * 2 * C floats)
constexpr int UNROLL = 4;

__device__ __forceinline__ void ld8(const bf16* p, float v[8]) {
  uint4 u = __ldcg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
// L2 residency between the two passes: pass-1 loads mark lines evict_last, pass-2 loads
// evict_first, and pass 2 walks each CTA's rows last-to-first (the lines pass 1 touched last
// are the ones still in L2).  hint == 0: plain __ldcg, forward order (A/B knob CVB_BN_L2HINT=0).
__device__ __forceinline__ uint4 ldv_pol(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t pol_keep() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t pol_drop() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldv(const void* p, bool hint, uint64_t pol) {
  return hint ? ldv_pol(p, pol) : __ldcg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ unsigned ldg_u8(const unsigned char* p, bool hint, uint64_t pol) {
  if (!hint) return __ldcg(p);
  unsigned short r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void unpack8(const uint4& u, float v[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) { float2 f = __bfloat1622float2(h[i]); v[2 * i] = f.x; v[2 * i + 1] = f.y; }
}
__device__ __forceinline__ void ld8h(const bf16* p, float v[8], bool hint, uint64_t pol) { unpack8(ldv(p, hint, pol), v); }

__device__ __forceinline__ void st8(bf16* p, const float v[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; i++) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}

// All CTAs are co-resident (cooperative launch): two-level grid barrier (cvb_common.cuh).
__device__ __forceinline__ void grid_sync(unsigned* bar) { cvb_grid_barrier(bar); }

__device__ __forceinline__ void bn_trace(long long* tr, int k) {
  if (tr && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[blockIdx.x * 8 + k] = t;
  }
}

// Fixed-order block reduction of per-thread (s[8], q[8]) for channel group g, row lane rl
// into the channel-major partials part[2][C][grid] (this CTA's column).  The staging layout
// sh[k][rl][g] is conflict-free for both the writes (consecutive threads = consecutive g) and
// the column sums (consecutive threads = consecutive g of one k); the row-major [rl][g][16]
// layout it replaces was 16-way bank-conflicted (1.8 us per launch, traced).
__device__ __forceinline__ void block_partials(const float s[8], const float q[8], int G, int RL, int g, int rl,
                                               int C, float* __restrict__ part, float* sh) {
  const int RG = RL * G;
  if (rl < RL) {
#pragma unroll
    for (int i = 0; i < 8; i++) { sh[i * RG + rl * G + g] = s[i]; sh[(8 + i) * RG + rl * G + g] = q[i]; }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < G * 16; idx += THREADS) {
    const int k = idx / G, gg = idx - k * G;
    float acc = 0.f;
    for (int l = 0; l < RL; l++) acc += sh[k * RG + l * G + gg];
    part[((int64_t)(k >> 3) * C + gg * 8 + (k & 7)) * gridDim.x + blockIdx.x] = acc;
  }
}

// Channel c's totals over all CTAs' partials, fixed order (lane-strided, then a warp tree),
// computed by ONE warp reading the channel's contiguous partial row (coalesced); no block
// barrier, so a CTA finalises up to 16 channels at once.  Result valid in lane 0.
__device__ __forceinline__ void channel_total_warp(const float* __restrict__ part, int C, int c, double& s,
                                                   double& q) {
  const int l = threadIdx.x & 31, P = (int)gridDim.x;
  const float* ps = part + (int64_t)c * P;
  const float* pq = part + ((int64_t)C + c) * P;
  double a = 0, b = 0;
  for (int k = l; k < P; k += 32) { a += __ldcg(ps + k); b += __ldcg(pq + k); }
#pragma unroll
  for (int o = 16; o; o >>= 1) { a += __shfl_down_sync(0xffffffffu, a, o); b += __shfl_down_sync(0xffffffffu, b, o); }
  s = a;
  q = b;
}

struct FwdArgs {
  const bf16* x; int64_t rows; int C, xcs;
  float* part; unsigned* bar;
  float* mean; float* rstd; float eps; float* run_mean; float* run_var; float momentum;
  const float* gamma; const float* beta; const bf16* res; int rcs; int relu;
  bf16* y; int ycs, ycoff;   // y == nullptr: statistics only
  int four_rows;             // pass 2 without residual: 4 rows in flight (CVB_BN_FWD_TWO_ROWS=1: off)
  long long* trace;          // CVB_BN_TRACE: per-CTA phase timestamps (globaltimer ns), debug only
  int hint;                  // L2 residency hints + reversed pass 2 (see ldv)
  int st_off, st_C;          // st_C > 0: statistics of channels [st_off, st_off + st_C) only (the
                             // others' mean/rstd are given); pass 2 normalises all C channels
  unsigned char* mask;       // optional ReLU mask out: byte [row][C/8], bit k = (bf16 y of channel 8g+k > 0)
};

// bf16 round-to-nearest-even of a non-negative fp32 value is > 0 iff the value exceeds 2^-134
// (half the smallest bf16 subnormal; the tie rounds to 0): the mask bit equals (bf16(o) > 0)
__device__ __forceinline__ unsigned relu_bits(const float o[8]) {
  const float lim = __int_as_float(0x00008000);   // 2^-134
  unsigned b = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) b |= (o[k] > lim ? 1u : 0u) << k;
  return b;
}

// OCC = 2: two 512-thread CTAs per SM (<= 64 registers) -- more loads in flight for the
// latency-bound wide-channel layers; OCC = 1 keeps 86 registers (measured better at C <= 64)
template <int OCC>
__global__ void __launch_bounds__(THREADS, OCC) bn_fwd_fused(const FwdArgs a) {
  extern __shared__ float sh[];
  __shared__ float s_scale[2048], s_shift[2048];
  const int C = a.C, G = C / 8, RL = THREADS / G;
  const int g = threadIdx.x % G, rl = threadIdx.x / G;
  const int64_t per = (a.rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(a.rows, r0 + per);
  bn_trace(a.trace, 0);
  // ---- pass 1: partial statistics (of the statistics channel range) ----
  const int C1 = a.st_C ? a.st_C : C, G1 = C1 / 8, RL1 = THREADS / G1;
  const int g1 = threadIdx.x % G1, rl1 = threadIdx.x / G1;
  const bf16* x1 = a.x + (a.st_C ? a.st_off : 0);
  const bool hint = a.hint != 0;
  const uint64_t pk = hint ? pol_keep() : 0, pd = hint ? pol_drop() : 0;
  float s[8] = {0}, q[8] = {0};
  if (rl1 < RL1) {
    int64_t r = r0 + rl1;
    for (; r + (UNROLL - 1) * RL1 < r1; r += UNROLL * RL1) {
      float v[UNROLL][8];
#pragma unroll
      for (int u = 0; u < UNROLL; u++) ld8h(x1 + (r + u * RL1) * a.xcs + g1 * 8, v[u], hint, pk);
#pragma unroll
      for (int u = 0; u < UNROLL; u++)
#pragma unroll
        for (int i = 0; i < 8; i++) { s[i] += v[u][i]; q[i] += v[u][i] * v[u][i]; }
    }
    for (; r < r1; r += RL1) {
      float v[8];
      ld8h(x1 + r * a.xcs + g1 * 8, v, hint, pk);
#pragma unroll
      for (int i = 0; i < 8; i++) { s[i] += v[i]; q[i] += v[i] * v[i]; }
    }
  }
  bn_trace(a.trace, 1);
  block_partials(s, q, G1, RL1, g1, rl1, C1, a.part, sh);
  bn_trace(a.trace, 2);
  grid_sync(a.bar);
  bn_trace(a.trace, 3);
  // ---- finalisation: warp w of CTA b owns channel b + w * grid ----
  {
    const int c = blockIdx.x + (threadIdx.x >> 5) * gridDim.x;
    if (c < C1) {
      double ts, tq;
      channel_total_warp(a.part, C1, c, ts, tq);
      if ((threadIdx.x & 31) == 0) {
        const double cnt = (double)a.rows;
        const double m = ts / cnt;
        double var = tq / cnt - m * m;
        if (var < 0) var = 0;
        const int co = c + (a.st_C ? a.st_off : 0);
        a.mean[co] = (float)m;
        a.rstd[co] = (float)(1.0 / sqrt(var + (double)a.eps));
        if (a.run_mean) {
          const double unb = cnt > 1 ? var * cnt / (cnt - 1) : var;
          a.run_mean[c] = (float)((1.0 - a.momentum) * a.run_mean[c] + a.momentum * m);
          a.run_var[c] = (float)((1.0 - a.momentum) * a.run_var[c] + a.momentum * unb);
        }
      }
    }
  }
  bn_trace(a.trace, 4);
  if (!a.y) return;
  grid_sync(a.bar);
  bn_trace(a.trace, 5);
  // ---- pass 2: normalise the same rows ----
  for (int c = threadIdx.x; c < C; c += THREADS) {
    s_scale[c] = a.gamma[c] * __ldcg(a.rstd + c);
    s_shift[c] = __ldcg(a.mean + c);
  }
  __syncthreads();
  if (rl >= RL) return;
  float sc[8], mu[8], be[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { sc[k] = s_scale[g * 8 + k]; mu[k] = s_shift[g * 8 + k]; be[k] = a.beta[g * 8 + k]; }
  int64_t r = r0 + rl;
  // pass 2 row order: reversed with the hints (R maps a forward row index to the row visited)
#define R(x) (hint ? r0 + r1 - 1 - (x) : (x))
  if (!a.res && a.four_rows) {   // four rows' raw 16-byte loads in flight per thread
    for (; r + 3 * RL < r1; r += 4 * RL) {
      uint4 u[4];
#pragma unroll
      for (int j = 0; j < 4; j++) u[j] = ldv(a.x + R(r + j * RL) * a.xcs + g * 8, hint, pd);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[j]);
        float o[8];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const float2 f = __bfloat1622float2(h[i]);
          const float z0 = (f.x - mu[2 * i]) * sc[2 * i] + be[2 * i];
          const float z1 = (f.y - mu[2 * i + 1]) * sc[2 * i + 1] + be[2 * i + 1];
          o[2 * i] = a.relu ? fmaxf(z0, 0.f) : z0;
          o[2 * i + 1] = a.relu ? fmaxf(z1, 0.f) : z1;
        }
        st8(a.y + R(r + j * RL) * a.ycs + a.ycoff + g * 8, o);
      }
    }
  }
  if (!a.res) {   // two rows in flight per thread
    for (; r + RL < r1; r += 2 * RL) {
      float v0[8], v1[8], o[8];
      ld8h(a.x + R(r) * a.xcs + g * 8, v0, hint, pd);
      ld8h(a.x + R(r + RL) * a.xcs + g * 8, v1, hint, pd);
#pragma unroll
      for (int k = 0; k < 8; k++) { const float z = (v0[k] - mu[k]) * sc[k] + be[k]; o[k] = a.relu ? fmaxf(z, 0.f) : z; }
      st8(a.y + R(r) * a.ycs + a.ycoff + g * 8, o);
#pragma unroll
      for (int k = 0; k < 8; k++) { const float z = (v1[k] - mu[k]) * sc[k] + be[k]; o[k] = a.relu ? fmaxf(z, 0.f) : z; }
      st8(a.y + R(r + RL) * a.ycs + a.ycoff + g * 8, o);
    }
  }
  if (a.res) {   // residual: two rows' x and res loads in flight per thread
    for (; r + RL < r1; r += 2 * RL) {
      const uint4 ux0 = ldv(a.x + R(r) * a.xcs + g * 8, hint, pd);
      const uint4 ur0 = ldv(a.res + R(r) * a.rcs + g * 8, false, 0);
      const uint4 ux1 = ldv(a.x + R(r + RL) * a.xcs + g * 8, hint, pd);
      const uint4 ur1 = ldv(a.res + R(r + RL) * a.rcs + g * 8, false, 0);
#pragma unroll
      for (int j = 0; j < 2; j++) {
        float v[8], rv[8], o[8];
        unpack8(j ? ux1 : ux0, v);
        unpack8(j ? ur1 : ur0, rv);
#pragma unroll
        for (int k = 0; k < 8; k++) {
          float z = (v[k] - mu[k]) * sc[k] + be[k];
          z += rv[k];
          o[k] = a.relu ? fmaxf(z, 0.f) : z;
        }
        const int64_t rr = R(r + j * RL);
        st8(a.y + rr * a.ycs + a.ycoff + g * 8, o);
        if (a.mask) a.mask[rr * G + g] = (unsigned char)relu_bits(o);
      }
    }
  }
  for (; r < r1; r += RL) {
    float v[8], o[8], rv[8];
    ld8h(a.x + R(r) * a.xcs + g * 8, v, hint, pd);
    if (a.res) ld8(a.res + R(r) * a.rcs + g * 8, rv);
#pragma unroll
    for (int k = 0; k < 8; k++) {
      float z = (v[k] - mu[k]) * sc[k] + be[k];
      if (a.res) z += rv[k];
      o[k] = a.relu ? fmaxf(z, 0.f) : z;
    }
    st8(a.y + R(r) * a.ycs + a.ycoff + g * 8, o);
    if (a.mask) a.mask[R(r) * G + g] = (unsigned char)relu_bits(o);
  }
#undef R
  bn_trace(a.trace, 6);
}

struct BwdArgs {
  const bf16* dy; int dycs; const bf16* x; int xcs; const bf16* y; int ycs;
  int64_t rows; int C;
  const float* mean; const float* rstd; const float* gamma; const float* beta; int relu;
  float* part; unsigned* bar; float* dgamma; float* dbeta;
  bf16* dx; int dxcs; float* dx32; int accum32; bf16* dz_out;
  int two_rows;              // pass 2: two rows' raw loads in flight (CVB_BN_BWD_ONE_ROW=1: off)
  long long* trace;          // CVB_BN_TRACE: per-CTA phase timestamps (globaltimer ns), debug only
  int hint;                  // L2 residency hints + reversed pass 2 (see ldv)
  const unsigned char* mask; // optional ReLU mask (cvb_bn_forward_mask's), read instead of y
};

// Per-channel constants live in shared memory (8 consecutive floats per channel group, two
// 16-byte LDS each): keeps the kernel under 64 registers so two 512-thread CTAs fit per SM
// (twice the loads in flight of the register-resident form, no spills).
struct ChanSmem {
  float mu[2048], rs[2048], ga[2048], be[2048];
};

__device__ __forceinline__ void lds8(const float* p, float v[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// dz = dy * relu-mask and xhat for one row (8 channels of group g)
__device__ __forceinline__ void bwd_load(const BwdArgs& a, int64_t r, int g, const ChanSmem& cs, float d[8],
                                         float xh[8], bool hint = false, uint64_t pol = 0) {
  float xv[8];
  ld8h(a.dy + r * a.dycs + g * 8, d, hint, pol);
  ld8h(a.x + r * a.xcs + g * 8, xv, hint, pol);
  float mu[8], rs[8];
  lds8(cs.mu + g * 8, mu);
  lds8(cs.rs + g * 8, rs);
  // explicit rounding / FMA steps (no compiler-chosen contraction): DenseNet's deferred gather
  // (bn_gather_dx) repeats this arithmetic and must reproduce it bit for bit
#pragma unroll
  for (int k = 0; k < 8; k++) xh[k] = __fmul_rn(__fsub_rn(xv[k], mu[k]), rs[k]);
  if (a.relu) {
    if (a.mask) {
      const unsigned b = ldg_u8(a.mask + r * (a.C / 8) + g, hint, pol);
#pragma unroll
      for (int k = 0; k < 8; k++) if (!((b >> k) & 1u)) d[k] = 0.f;
    } else if (a.y) {
      float yv[8];
      ld8h(a.y + r * a.ycs + g * 8, yv, hint, pol);
#pragma unroll
      for (int k = 0; k < 8; k++) if (!(yv[k] > 0.f)) d[k] = 0.f;
    } else {
      float ga[8], be[8];
      lds8(cs.ga + g * 8, ga);
      lds8(cs.be + g * 8, be);
#pragma unroll
      for (int k = 0; k < 8; k++) if (!(__fmaf_rn(xh[k], ga[k], be[k]) > 0.f)) d[k] = 0.f;
    }
  }
}

// pass-1 body for one row from raw loads (mask recomputed from x): the bwd_load arithmetic,
// accumulated into s = sum(dz), q = sum(dz * xhat) in the same order (bit-identical)
__device__ __forceinline__ void bwd_stats_raw(const BwdArgs& a, const ChanSmem& cs, int g, const uint4& ud,
                                              const uint4& ux, float s[8], float q[8]) {
  // one bf16 pair at a time, per-channel constants read as scalars: few live registers (the
  // two-CTA instantiation's 64-register cap otherwise spilled s / q every iteration)
  const uint32_t* hd = reinterpret_cast<const uint32_t*>(&ud);
  const uint32_t* hx = reinterpret_cast<const uint32_t*>(&ux);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float2 fd = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hd[i]));
    const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hx[i]));
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const int k = 2 * i + j, c = g * 8 + k;
      float d = j ? fd.y : fd.x;
      const float xh = __fmul_rn(__fsub_rn(j ? fx.y : fx.x, cs.mu[c]), cs.rs[c]);
      if (a.relu && !(__fmaf_rn(xh, cs.ga[c], cs.be[c]) > 0.f)) d = 0.f;
      s[k] += d;
      q[k] += d * xh;
    }
  }
}

// pass-1 body with the forward's ReLU mask bits (residual layers): dz = dy * mask stored to
// dz_out (the residual branch's gradient), statistics as bwd_stats_raw
__device__ __forceinline__ void bwd_stats_mask(const ChanSmem& cs, int g, const uint4& ud, const uint4& ux,
                                               unsigned mb, float s[8], float q[8], bf16* dz_dst) {
  const uint32_t* hd = reinterpret_cast<const uint32_t*>(&ud);
  const uint32_t* hx = reinterpret_cast<const uint32_t*>(&ux);
  float dz[8];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float2 fd = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hd[i]));
    const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hx[i]));
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const int k = 2 * i + j, c = g * 8 + k;
      const float d = ((mb >> k) & 1u) ? (j ? fd.y : fd.x) : 0.f;
      const float xh = __fmul_rn(__fsub_rn(j ? fx.y : fx.x, cs.mu[c]), cs.rs[c]);
      s[k] += d;
      q[k] += d * xh;
      dz[k] = d;
    }
  }
  if (dz_dst) st8(dz_dst, dz);
}

// pass-2 body for one row from raw loads: dz = dy * relu-mask(x), dx = gamma*rstd*(dz - mean(dz)
// - xhat*mean(dz*xhat)) (same arithmetic as bwd_load + the generic loop)
__device__ __forceinline__ void bwd_apply_raw(const BwdArgs& a, const ChanSmem& cs, const float* sh, int C, int g,
                                              const uint4& ud, const uint4& ux, bf16* dst) {
  float d[8], xv[8], mu[8], rs[8];
  const __nv_bfloat162* hd = reinterpret_cast<const __nv_bfloat162*>(&ud);
  const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&ux);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float2 fd = __bfloat1622float2(hd[i]), fx = __bfloat1622float2(hx[i]);
    d[2 * i] = fd.x; d[2 * i + 1] = fd.y; xv[2 * i] = fx.x; xv[2 * i + 1] = fx.y;
  }
  lds8(cs.mu + g * 8, mu);
  lds8(cs.rs + g * 8, rs);
  float xh[8];
#pragma unroll
  for (int k = 0; k < 8; k++) xh[k] = (xv[k] - mu[k]) * rs[k];
  if (a.relu) {
    float ga[8], be[8];
    lds8(cs.ga + g * 8, ga);
    lds8(cs.be + g * 8, be);
#pragma unroll
    for (int k = 0; k < 8; k++) if (!(xh[k] * ga[k] + be[k] > 0.f)) d[k] = 0.f;
  }
  float kk[8], kb[8], kg[8], o[8];
  lds8(sh + g * 8, kk);
  lds8(sh + C + g * 8, kb);
  lds8(sh + 2 * C + g * 8, kg);
#pragma unroll
  for (int k = 0; k < 8; k++) o[k] = kk[k] * (d[k] - kb[k] - xh[k] * kg[k]);
  st8(dst, o);
}

// pass-2 body from the stored dz (already masked): dx = gamma*rstd*(dz - mean(dz) - xhat*mean(dz*xhat))
__device__ __forceinline__ void bwd_apply_dz(const ChanSmem& cs, const float* sh, int C, int g, const uint4& uz,
                                             const uint4& ux, bf16* dst) {
  float d[8], xv[8], mu[8], rs[8], kk[8], kb[8], kg[8], o[8];
  const __nv_bfloat162* hz = reinterpret_cast<const __nv_bfloat162*>(&uz);
  const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&ux);
#pragma unroll
  for (int i = 0; i < 4; i++) {
    const float2 fz = __bfloat1622float2(hz[i]), fx = __bfloat1622float2(hx[i]);
    d[2 * i] = fz.x; d[2 * i + 1] = fz.y; xv[2 * i] = fx.x; xv[2 * i + 1] = fx.y;
  }
  lds8(cs.mu + g * 8, mu);
  lds8(cs.rs + g * 8, rs);
  lds8(sh + g * 8, kk);
  lds8(sh + C + g * 8, kb);
  lds8(sh + 2 * C + g * 8, kg);
#pragma unroll
  for (int k = 0; k < 8; k++) o[k] = kk[k] * (d[k] - kb[k] - (xv[k] - mu[k]) * rs[k] * kg[k]);
  st8(dst, o);
}

// OCC = 2: two 512-thread CTAs per SM at <= 64 registers (the large layers); OCC = 1: one CTA per
// SM with room for every per-row value in registers (no spills; fewer CTAs in the grid
// barriers) for the small, latency-bound layers
template <int OCC>
__global__ void __launch_bounds__(THREADS, OCC) bn_bwd_fused(const BwdArgs a) {
  extern __shared__ float sh[];
  __shared__ ChanSmem cs;
  const int C = a.C, G = C / 8, RL = THREADS / G;
  const int g = threadIdx.x % G, rl = threadIdx.x / G;
  const int64_t per = (a.rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(a.rows, r0 + per);
  for (int c = threadIdx.x; c < C; c += THREADS) {
    cs.mu[c] = a.mean[c]; cs.rs[c] = a.rstd[c]; cs.ga[c] = a.gamma[c]; cs.be[c] = a.beta[c];
  }
  __syncthreads();
  bn_trace(a.trace, 0);
  // ---- pass 1: sum(dz), sum(dz * xhat) ----
  const bool hint = a.hint != 0;
  const uint64_t pk = hint ? pol_keep() : 0, pd = hint ? pol_drop() : 0;
  float s[8] = {0}, q[8] = {0};
  if (rl < RL) {
    int64_t r = r0 + rl;
    if (!a.y && !a.mask && !a.dz_out) {
      // raw 16-byte loads of two (one CTA per SM: four) rows in flight, converted one row at a
      // time
      if (OCC == 1)
        for (; r + 3 * RL < r1; r += 4 * RL) {
          uint4 ud[4], ux[4];
#pragma unroll
          for (int j = 0; j < 4; j++) {
            ud[j] = ldv(a.dy + (r + j * RL) * a.dycs + g * 8, hint, pk);
            ux[j] = ldv(a.x + (r + j * RL) * a.xcs + g * 8, hint, pk);
          }
#pragma unroll
          for (int j = 0; j < 4; j++) bwd_stats_raw(a, cs, g, ud[j], ux[j], s, q);
        }
      for (; r + RL < r1; r += 2 * RL) {
        const uint4 ud0 = ldv(a.dy + r * a.dycs + g * 8, hint, pk), ux0 = ldv(a.x + r * a.xcs + g * 8, hint, pk);
        const uint4 ud1 = ldv(a.dy + (r + RL) * a.dycs + g * 8, hint, pk);
        const uint4 ux1 = ldv(a.x + (r + RL) * a.xcs + g * 8, hint, pk);
        bwd_stats_raw(a, cs, g, ud0, ux0, s, q);
        bwd_stats_raw(a, cs, g, ud1, ux1, s, q);
      }
    }
    if (OCC == 1 && a.mask && a.relu && !a.y) {   // residual layers: the forward's mask bits
      const int Gm = C / 8;
      for (; r + 3 * RL < r1; r += 4 * RL) {
        uint4 ud[4], ux[4];
        unsigned mb[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          ud[j] = ldv(a.dy + (r + j * RL) * a.dycs + g * 8, hint, pk);
          ux[j] = ldv(a.x + (r + j * RL) * a.xcs + g * 8, hint, pk);
          mb[j] = ldg_u8(a.mask + (r + j * RL) * Gm + g, hint, pk);
        }
#pragma unroll
        for (int j = 0; j < 4; j++)
          bwd_stats_mask(cs, g, ud[j], ux[j], mb[j], s, q, a.dz_out ? a.dz_out + (r + j * RL) * C + g * 8 : nullptr);
      }
    }
    for (; r + RL < r1; r += 2 * RL) {
      float d0[8], x0[8], d1[8], x1[8];
      bwd_load(a, r, g, cs, d0, x0, hint, pk);
      bwd_load(a, r + RL, g, cs, d1, x1, hint, pk);
#pragma unroll
      for (int k = 0; k < 8; k++) { s[k] += d0[k]; q[k] += d0[k] * x0[k]; }
#pragma unroll
      for (int k = 0; k < 8; k++) { s[k] += d1[k]; q[k] += d1[k] * x1[k]; }
      if (a.dz_out) { st8(a.dz_out + r * C + g * 8, d0); st8(a.dz_out + (r + RL) * C + g * 8, d1); }
    }
    for (; r < r1; r += RL) {
      float d[8], xh[8];
      bwd_load(a, r, g, cs, d, xh, hint, pk);
#pragma unroll
      for (int k = 0; k < 8; k++) { s[k] += d[k]; q[k] += d[k] * xh[k]; }
      if (a.dz_out) st8(a.dz_out + r * C + g * 8, d);
    }
  }
  bn_trace(a.trace, 1);
  block_partials(s, q, G, RL, g, rl, C, a.part, sh);
  bn_trace(a.trace, 2);
  grid_sync(a.bar);
  bn_trace(a.trace, 3);
  {
    const int c = blockIdx.x + (threadIdx.x >> 5) * gridDim.x;   // warp w of CTA b: channel b + w * grid
    if (c < C) {
      double ts, tq;
      channel_total_warp(a.part, C, c, ts, tq);
      if ((threadIdx.x & 31) == 0) { a.dbeta[c] = (float)ts; a.dgamma[c] = (float)tq; }
    }
  }
  bn_trace(a.trace, 4);
  if (!a.dx && !a.dx32) return;
  grid_sync(a.bar);
  bn_trace(a.trace, 5);
  // ---- pass 2: dx over the same rows; its per-channel factors go to the (now free)
  // partial-reduction smem: sh[0:C) = gamma*rstd, sh[C:2C) = mean(dz), sh[2C:3C) = mean(dz*xhat)
  const float invM = 1.0f / (float)a.rows;
  for (int c = threadIdx.x; c < C; c += THREADS) {
    sh[c] = cs.ga[c] * cs.rs[c];
    sh[C + c] = __ldcg(a.dbeta + c) * invM;
    sh[2 * C + c] = __ldcg(a.dgamma + c) * invM;
  }
  __syncthreads();
  if (rl >= RL) return;
  int64_t r = r0 + rl;
#define R(x) (hint ? r0 + r1 - 1 - (x) : (x))
  if (a.dz_out && !a.dx32) {
    // pass 1 stored dz = dy * mask (the residual branch's gradient): pass 2 reads it instead of
    // dy and y -- two tensors per row instead of three -- two (one CTA per SM: four) rows' loads
    // in flight
    if (OCC == 1)
      for (; r + 3 * RL < r1; r += 4 * RL) {
        uint4 uz[4], ux[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          uz[j] = ldv(a.dz_out + R(r + j * RL) * C + g * 8, hint, pd);
          ux[j] = ldv(a.x + R(r + j * RL) * a.xcs + g * 8, hint, pd);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) bwd_apply_dz(cs, sh, C, g, uz[j], ux[j], a.dx + R(r + j * RL) * a.dxcs + g * 8);
      }
    for (; r + RL < r1; r += 2 * RL) {
      const uint4 uz0 = ldv(a.dz_out + R(r) * C + g * 8, hint, pd);
      const uint4 ux0 = ldv(a.x + R(r) * a.xcs + g * 8, hint, pd);
      const uint4 uz1 = ldv(a.dz_out + R(r + RL) * C + g * 8, hint, pd);
      const uint4 ux1 = ldv(a.x + R(r + RL) * a.xcs + g * 8, hint, pd);
      bwd_apply_dz(cs, sh, C, g, uz0, ux0, a.dx + R(r) * a.dxcs + g * 8);
      bwd_apply_dz(cs, sh, C, g, uz1, ux1, a.dx + R(r + RL) * a.dxcs + g * 8);
    }
    if (r < r1) {
      const uint4 uz0 = ldv(a.dz_out + R(r) * C + g * 8, hint, pd);
      const uint4 ux0 = ldv(a.x + R(r) * a.xcs + g * 8, hint, pd);
      bwd_apply_dz(cs, sh, C, g, uz0, ux0, a.dx + R(r) * a.dxcs + g * 8);
    }
    bn_trace(a.trace, 6);
    return;
  }
  if (a.two_rows && !a.dx32 && !a.y && !a.mask) {
    // bf16 dx, mask recomputed from x: two (one CTA per SM: four) rows' raw 16-byte loads in
    // flight per thread (the pass is load-latency bound), converted one row at a time
    if (OCC == 1)
      for (; r + 3 * RL < r1; r += 4 * RL) {
        uint4 ud[4], ux[4];
#pragma unroll
        for (int j = 0; j < 4; j++) {
          ud[j] = ldv(a.dy + R(r + j * RL) * a.dycs + g * 8, hint, pd);
          ux[j] = ldv(a.x + R(r + j * RL) * a.xcs + g * 8, hint, pd);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) bwd_apply_raw(a, cs, sh, C, g, ud[j], ux[j], a.dx + R(r + j * RL) * a.dxcs + g * 8);
      }
    for (; r + RL < r1; r += 2 * RL) {
      const uint4 ud0 = ldv(a.dy + R(r) * a.dycs + g * 8, hint, pd);
      const uint4 ux0 = ldv(a.x + R(r) * a.xcs + g * 8, hint, pd);
      const uint4 ud1 = ldv(a.dy + R(r + RL) * a.dycs + g * 8, hint, pd);
      const uint4 ux1 = ldv(a.x + R(r + RL) * a.xcs + g * 8, hint, pd);
      bwd_apply_raw(a, cs, sh, C, g, ud0, ux0, a.dx + R(r) * a.dxcs + g * 8);
      bwd_apply_raw(a, cs, sh, C, g, ud1, ux1, a.dx + R(r + RL) * a.dxcs + g * 8);
    }
  }
  for (; r < r1; r += RL) {
    float d[8], xh[8], o[8], kk[8], kb[8], kg[8];
    bwd_load(a, R(r), g, cs, d, xh, hint, pd);
    lds8(sh + g * 8, kk);
    lds8(sh + C + g * 8, kb);
    lds8(sh + 2 * C + g * 8, kg);
#pragma unroll
    for (int k = 0; k < 8; k++) o[k] = __fmul_rn(kk[k], __fmaf_rn(-xh[k], kg[k], __fsub_rn(d[k], kb[k])));
    if (a.dx32) {
      float4* p4 = reinterpret_cast<float4*>(a.dx32 + R(r) * a.dxcs + g * 8);
      if (a.accum32) {
        float4 u = p4[0], w = p4[1];
        o[0] = __fadd_rn(u.x, o[0]); o[1] = __fadd_rn(u.y, o[1]); o[2] = __fadd_rn(u.z, o[2]);
        o[3] = __fadd_rn(u.w, o[3]); o[4] = __fadd_rn(w.x, o[4]); o[5] = __fadd_rn(w.y, o[5]);
        o[6] = __fadd_rn(w.z, o[6]); o[7] = __fadd_rn(w.w, o[7]);
      }
      p4[0] = make_float4(o[0], o[1], o[2], o[3]);
      p4[1] = make_float4(o[4], o[5], o[6], o[7]);
    } else {
      st8(a.dx + R(r) * a.dxcs + g * 8, o);
    }
  }
  bn_trace(a.trace, 6);
#undef R
}

unsigned* g_bar[64] = {nullptr};
long long* g_trace = nullptr;   // CVB_BN_TRACE: [grid][8] phase timestamps of the last launch

long long* trace_buf() {
  static int on = -1;
  if (on < 0) on = getenv("CVB_BN_TRACE") ? 1 : 0;
  if (!on) return nullptr;
  if (!g_trace) cudaMalloc(&g_trace, sizeof(long long) * 8 * 4096);
  return g_trace;
}
int g_grid[64] = {0}, g_grid_f[64] = {0}, g_grid_f2[64] = {0};

// *grid: the backward kernel's co-resident grid; *grid_f: the forward kernel's (it needs
// fewer registers, so more CTAs fit).  The partials workspace covers the larger.
int fused_setup(int C, unsigned** bar, int* grid, int* grid_f = nullptr) {
  int dev = 0;
  CVB_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) { cvb_set_error("bn fused: device index"); return CVB_EINVAL; }
  if (!g_bar[dev]) {
    CVB_CUDA(cudaMalloc(&g_bar[dev], CVB_GRID_BAR_WORDS * sizeof(unsigned)));
    CVB_CUDA(cudaMemset(g_bar[dev], 0, CVB_GRID_BAR_WORDS * sizeof(unsigned)));
    CVB_CUDA(cudaDeviceSynchronize());
    const size_t smem = (size_t)THREADS * 16 * sizeof(float);
    CVB_CUDA(cudaFuncSetAttribute(bn_fwd_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CVB_CUDA(cudaFuncSetAttribute(bn_fwd_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CVB_CUDA(cudaFuncSetAttribute(bn_bwd_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CVB_CUDA(cudaFuncSetAttribute(bn_bwd_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ_f = 0, occ_b = 0, occ_f2 = 0;
    CVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f, bn_fwd_fused<1>, THREADS, smem));
    CVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_f2, bn_fwd_fused<2>, THREADS, smem));
    if (occ_f2 > MAX_OCC) occ_f2 = MAX_OCC;
    g_grid_f2[dev] = (occ_f2 < 1 ? 1 : occ_f2) * cvb_num_sms();
    CVB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, bn_bwd_fused<2>, THREADS, smem));
    if (occ_f > MAX_OCC) occ_f = MAX_OCC;
    if (occ_b > MAX_OCC) occ_b = MAX_OCC;
    if (occ_f < 1 || occ_b < 1) { cvb_set_error("bn fused: kernel does not fit on an SM"); return CVB_EINVAL; }
    g_grid[dev] = occ_b * cvb_num_sms();
    g_grid_f[dev] = occ_f * cvb_num_sms();
  }
  *bar = g_bar[dev];
  *grid = g_grid[dev];
  if (grid_f) *grid_f = g_grid_f[dev];
  (void)C;
  return CVB_OK;
}

// Experiment knob (CVB_BN_MIN_ELEMS): fewer CTAs for small tensors.  Measured on B200: no gain
// (the fixed cost is per phase, not per CTA) -- off by default.
int size_grid(int grid, int64_t rows, int C) {
  static int env = -1;
  if (env < 0) { const char* e = getenv("CVB_BN_MIN_ELEMS"); env = e ? atoi(e) : 0; }   // measured: no gain, off
  if (env <= 0) return grid;
  const int64_t want = (rows * C + env - 1) / env;
  return (int)(want < grid ? (want < 8 ? 8 : want) : grid);
}

int l2hint_knob() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("CVB_BN_L2HINT"); v = e ? atoi(e) : 1; }
  return v;
}

int two_rows_knob() {
  static int v = -1;
  if (v < 0) v = getenv("CVB_BN_BWD_ONE_ROW") ? 0 : 1;
  return v;
}

template <class Args>
int launch_coop(void (*kern)(Args), const Args& a, int grid, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = (size_t)THREADS * 16 * sizeof(float);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CVB_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return CVB_OK;
}

}  // namespace

// Floats of partials workspace the fused BN kernels need for C channels.
CVB_API int64_t cvb_bn_fused_workspace_floats(int C) {
  unsigned* bar;
  int grid = 0, grid_f = 0;
  if (fused_setup(C, &bar, &grid, &grid_f)) return -1;
  int dev = 0;
  cudaGetDevice(&dev);
  int P = grid > grid_f ? grid : grid_f;
  if (g_grid_f2[dev] > P) P = g_grid_f2[dev];   // the two-CTA forward's grid
  return (int64_t)P * 2 * C;
}

// Batch-norm forward in one launch: statistics of x ([rows][C], stride xcs) -> mean/rstd
// (+ running stats), then y = act(gamma*(x-mean)*rstd + beta [+ res]) written at channel
// offset ycoff of y (stride ycs).  y == NULL: statistics only.
CVB_API int cvb_bn_forward_range(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd,
                                 float eps, float* run_mean, float* run_var, float momentum, const float* gamma,
                                 const float* beta, const void* res, int rcs, int relu, void* y, int ycs, int ycoff,
                                 int st_off, int st_C, void* stream);
CVB_API int cvb_bn_forward(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                           float* run_mean, float* run_var, float momentum, const float* gamma, const float* beta,
                           const void* res, int rcs, int relu, void* y, int ycs, int ycoff, void* stream) {
  return cvb_bn_forward_range(x, rows, C, xcs, ws, mean, rstd, eps, run_mean, run_var, momentum, gamma, beta, res, rcs,
                              relu, y, ycs, ycoff, 0, 0, stream);
}

// As cvb_bn_forward, but the batch statistics are computed only for channels [st_off,
// st_off + st_C) (st_C > 0; multiple of 8); mean/rstd of the other channels are inputs.  DenseNet:
// the statistics of the newest concat slice and the normalisation of the whole prefix in one
// launch (no running statistics are updated for a partial range).
namespace {
int bn_forward_impl(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd, float eps,
                    float* run_mean, float* run_var, float momentum, const float* gamma, const float* beta,
                    const void* res, int rcs, int relu, void* y, int ycs, int ycoff, int st_off, int st_C,
                    void* mask, void* stream) {
  if (st_C && (st_C % 8 || st_off % 8 || st_off < 0 || st_off + st_C > C || run_mean)) {
    cvb_set_error("bn_forward_range: bad statistics range");
    return CVB_EINVAL;
  }
  if (C % 8 || C > 2048 || C / 8 > THREADS) { cvb_set_error("bn_forward: C must be a multiple of 8, <= 2048"); return CVB_EINVAL; }
  unsigned* bar;
  int grid_b, grid;
  int rc = fused_setup(C, &bar, &grid_b, &grid);
  if (rc) return rc;
  FwdArgs a{(const bf16*)x, rows, C, xcs, ws, bar, mean, rstd, eps, run_mean, run_var, momentum, gamma, beta,
            (const bf16*)res, rcs, relu, (bf16*)y, ycs, ycoff, getenv("CVB_BN_FWD_TWO_ROWS") ? 0 : 1, trace_buf(),
            l2hint_knob(), st_off, st_C, (unsigned char*)mask};
  if (mask && !y) { cvb_set_error("bn_forward: a ReLU mask needs y"); return CVB_EINVAL; }
  // two CTAs per SM for large statistics passes (>= 12M elements: ResNet-18's stage-1..3
  // layers, +1.1% per step at 24M, +0.2% more at 12M); smaller ones measured better at one CTA
  // (fewer CTAs in the grid barriers).  Decided by the STATISTICS extent: the grid fixes the row partition of the
  // fixed-order reduction, so a slice's statistics come out bit-identical whether computed alone
  // or inside cvb_bn_forward_range.
  static long long occ2_min = -1;
  if (occ2_min < 0) { const char* e = getenv("CVB_BN_FWD_OCC2_MIN_ELEMS"); occ2_min = e ? atoll(e) : 12000000ll; }
  int dev = 0;
  CVB_CUDA(cudaGetDevice(&dev));
  const bool two = rows * (int64_t)(st_C ? st_C : C) >= occ2_min && g_grid_f2[dev] > 0;
  const int gf = size_grid(two ? g_grid_f2[dev] : grid, rows, C);
  if (C > 16 * gf) { cvb_set_error("bn_forward: more channels than finalising warps"); return CVB_EINVAL; }
  return two ? launch_coop(bn_fwd_fused<2>, a, gf, (cudaStream_t)stream)
             : launch_coop(bn_fwd_fused<1>, a, gf, (cudaStream_t)stream);
}
}  // namespace

CVB_API int cvb_bn_forward_range(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd,
                                 float eps, float* run_mean, float* run_var, float momentum, const float* gamma,
                                 const float* beta, const void* res, int rcs, int relu, void* y, int ycs, int ycoff,
                                 int st_off, int st_C, void* stream) {
  return bn_forward_impl(x, rows, C, xcs, ws, mean, rstd, eps, run_mean, run_var, momentum, gamma, beta, res, rcs,
                         relu, y, ycs, ycoff, st_off, st_C, nullptr, stream);
}

// cvb_bn_forward that also writes the ReLU mask of y: mask[row][C/8] bytes, bit k of byte g =
// (y[row][8g + k] > 0).  Read back by cvb_bn_backward_fused_mask instead of y: 1/16 of the bytes.
CVB_API int cvb_bn_forward_mask(const void* x, int64_t rows, int C, int xcs, float* ws, float* mean, float* rstd,
                                float eps, float* run_mean, float* run_var, float momentum, const float* gamma,
                                const float* beta, const void* res, int rcs, int relu, void* y, int ycs, int ycoff,
                                void* mask, void* stream) {
  return bn_forward_impl(x, rows, C, xcs, ws, mean, rstd, eps, run_mean, run_var, momentum, gamma, beta, res, rcs,
                         relu, y, ycs, ycoff, 0, 0, mask, stream);
}

// Batch-norm (+ReLU) backward in one launch (same contract as cvb_bn_backward).
namespace {
int bn_backward_impl(const void* dy, int dycs, const void* x, int xcs, const void* y, int ycs, int64_t rows, int C,
                     const float* mean, const float* rstd, const float* gamma, const float* beta, int relu, float* ws,
                     float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32, int accum32, void* dz_out,
                     const void* mask, void* stream) {
  if (C % 8 || C / 8 > THREADS) { cvb_set_error("bn_backward: bad C"); return CVB_EINVAL; }
  unsigned* bar;
  int grid;
  int rc = fused_setup(C, &bar, &grid);
  if (rc) return rc;
  BwdArgs a{(const bf16*)dy, dycs, (const bf16*)x, xcs, (const bf16*)y, ycs, rows, C, mean, rstd, gamma, beta, relu,
            ws, bar, dgamma, dbeta, (bf16*)dx, dxcs, dx32, accum32, (bf16*)dz_out, two_rows_knob(), trace_buf(),
            l2hint_knob(), (const unsigned char*)mask};
  // one CTA per SM (116+ registers, no spills; pass 1 with four rows' raw loads in flight).  The
  // two-CTA instantiation (64 registers) spilled its statistics accumulators inside the pass-1
  // loop; with pass 1 reworked, one CTA per SM at every size measured best (ResNet-18 +0.6% over
  // two CTAs above 12M elements, same-box).  CVB_BN_BWD_OCC1_MAX_ELEMS: two CTAs from that size.
  // (The grid is fixed by (rows, C): DenseNet's statistics-only and full passes of a layer
  // partition alike.)
  static long long one_max = -1;
  if (one_max < 0) { const char* e = getenv("CVB_BN_BWD_OCC1_MAX_ELEMS"); one_max = e ? atoll(e) : (1ll << 62); }
  const bool one = rows * (int64_t)C < one_max;
  const int gb = size_grid(one ? cvb_num_sms() : grid, rows, C);
  if (C > 16 * gb) { cvb_set_error("bn_backward: more channels than finalising warps"); return CVB_EINVAL; }
  return one ? launch_coop(bn_bwd_fused<1>, a, gb, (cudaStream_t)stream)
             : launch_coop(bn_bwd_fused<2>, a, gb, (cudaStream_t)stream);
}
}  // namespace

CVB_API int cvb_bn_backward_fused(const void* dy, int dycs, const void* x, int xcs, const void* y, int ycs, int64_t rows,
                                  int C, const float* mean, const float* rstd, const float* gamma, const float* beta,
                                  int relu, float* ws, float* dgamma, float* dbeta, void* dx, int dxcs, float* dx32,
                                  int accum32, void* dz_out, void* stream) {
  return bn_backward_impl(dy, dycs, x, xcs, y, ycs, rows, C, mean, rstd, gamma, beta, relu, ws, dgamma, dbeta, dx,
                          dxcs, dx32, accum32, dz_out, nullptr, stream);
}

// cvb_bn_backward_fused with the ReLU mask written by cvb_bn_forward_mask in place of y
CVB_API int cvb_bn_backward_fused_mask(const void* dy, int dycs, const void* x, int xcs, const void* mask,
                                       int64_t rows, int C, const float* mean, const float* rstd, const float* gamma,
                                       const float* beta, int relu, float* ws, float* dgamma, float* dbeta, void* dx,
                                       int dxcs, float* dx32, int accum32, void* dz_out, void* stream) {
  if (!mask) { cvb_set_error("bn_backward_mask: mask is NULL"); return CVB_EINVAL; }
  return bn_backward_impl(dy, dycs, x, xcs, nullptr, 0, rows, C, mean, rstd, gamma, beta, relu, ws, dgamma, dbeta,
                          dx, dxcs, dx32, accum32, dz_out, mask, stream);
}

// ---- DenseNet: deferred input gradient of the BNs over a concat prefix ------------------
// Every BN over the concat buffer of a dense block normalises the same channels with the same
// batch statistics (mean, rstd shared); only gamma/beta differ per layer.  Instead of each
// layer's backward adding its dx into an fp32 concat gradient (pass 2 re-reading dy and x and
// read-modify-writing 4 bytes per element per layer), the layers run the statistics pass only
// (dbeta = sum dz, dgamma = sum dz*xhat) and keep their dY.  The gradient of a channel range is
// then formed ONCE, when it is needed, from every later layer's dY slice:
//   out = base + sum_l  k_l * (dz_l - dbeta_l/M - xhat * dgamma_l/M),
//   dz_l = dy_l * [gamma_l * xhat + beta_l > 0],  k_l = gamma_l * rstd,  xhat = (x - mean) * rstd
// with the layers summed in the order given (the backward order) -- the same fp32 arithmetic,
// in the same order, as the accumulating per-layer form (bit-identical).
namespace {
constexpr int GATHER_MAX_LAYERS = 32;
struct GatherArgs {
  const bf16* x; int xcs; int64_t rows; int nc;
  const float* mean; const float* rstd;
  const float* base; int bcs;            // fp32 base gradient (channel 0 of the range), may be null
  int nl;
  const bf16* dy[GATHER_MAX_LAYERS];     // layer l's dY at channel 0 of the range (stride dycs[l])
  int dycs[GATHER_MAX_LAYERS];
  const float* gamma[GATHER_MAX_LAYERS];
  const float* beta[GATHER_MAX_LAYERS];
  const float* dgamma[GATHER_MAX_LAYERS];   // raw sums from the statistics pass
  const float* dbeta[GATHER_MAX_LAYERS];
  void* out; int ocs; int out_f32;
};

constexpr int GATHER_THREADS = 256, GATHER_CH = 64;   // a CTA: 64 channels (8 groups) x 32 row lanes

// one gather term: dz = dy * mask, acc += k * (dz - kb - xhat * kg)
__device__ __forceinline__ void gather_term(const uint4& u, const float* cfl, int g, const float xh[8], float acc[8]) {
  float d[8], kk[8], kb[8], kg[8], ga[8], be[8];
  unpack8(u, d);
  lds8(cfl + 0 * GATHER_CH + g * 8, kk);
  lds8(cfl + 1 * GATHER_CH + g * 8, kb);
  lds8(cfl + 2 * GATHER_CH + g * 8, kg);
  lds8(cfl + 3 * GATHER_CH + g * 8, ga);
  lds8(cfl + 4 * GATHER_CH + g * 8, be);
#pragma unroll
  for (int k = 0; k < 8; k++) {   // bwd_load + the accumulating pass-2 loop, same roundings
    if (!(__fmaf_rn(xh[k], ga[k], be[k]) > 0.f)) d[k] = 0.f;
    const float o = __fmul_rn(kk[k], __fmaf_rn(-xh[k], kg[k], __fsub_rn(d[k], kb[k])));
    acc[k] = __fadd_rn(acc[k], o);
  }
}

// Latency-bound (ncu: long-scoreboard stalls, 16 warps per SM at 110 registers): every load of a
// row -- x, the fp32 base and the first GATHER_BATCH layers' dY -- is issued before any is used,
// and three CTAs fit per SM.
// the same term with the coefficients read per element (fewer live registers: 3 CTAs per SM)
__device__ __forceinline__ void gather_term_s(const uint4& u, const float* cfl, int g, const float xh[8], float acc[8]) {
  float d[8];
  unpack8(u, d);
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const float* c = cfl + g * 8 + k;
    if (!(__fmaf_rn(xh[k], c[3 * GATHER_CH], c[4 * GATHER_CH]) > 0.f)) d[k] = 0.f;
    const float o = __fmul_rn(c[0], __fmaf_rn(-xh[k], c[2 * GATHER_CH], __fsub_rn(d[k], c[GATHER_CH])));
    acc[k] = __fadd_rn(acc[k], o);
  }
}

constexpr int GATHER_BATCH = 8;
template <int OCC>
__global__ void __launch_bounds__(GATHER_THREADS, OCC) bn_gather_dx(const __grid_constant__ GatherArgs a) {
  __shared__ __align__(16) float cf[GATHER_MAX_LAYERS][5][GATHER_CH];   // kk, kb, kg, gamma, beta
  __shared__ __align__(16) float cm[2][GATHER_CH];                      // mean, rstd
  CVB_PDL_PROLOGUE();
  const int cbase = blockIdx.y * GATHER_CH, nch = min(GATHER_CH, a.nc - cbase);
  const float invM = 1.0f / (float)a.rows;
  for (int i = threadIdx.x; i < a.nl * GATHER_CH; i += GATHER_THREADS) {
    const int l = i / GATHER_CH, c = i % GATHER_CH;
    if (c < nch) {
      const float ga = a.gamma[l][cbase + c], rs = a.rstd[cbase + c];
      cf[l][0][c] = ga * rs;
      cf[l][1][c] = a.dbeta[l][cbase + c] * invM;
      cf[l][2][c] = a.dgamma[l][cbase + c] * invM;
      cf[l][3][c] = ga;
      cf[l][4][c] = a.beta[l][cbase + c];
    }
  }
  for (int c = threadIdx.x; c < nch; c += GATHER_THREADS) { cm[0][c] = a.mean[cbase + c]; cm[1][c] = a.rstd[cbase + c]; }
  __syncthreads();
  // G channel groups of 8 x (256 / G) row lanes: every thread busy for 32-channel slices too
  const int G = nch / 8, g = threadIdx.x % G, rl = threadIdx.x / G, RL = GATHER_THREADS / G;
  if (rl >= RL) return;
  const int cg = cbase + g * 8;
  const int nb = a.nl < GATHER_BATCH ? a.nl : GATHER_BATCH;
  for (int64_t r = (int64_t)blockIdx.x * RL + rl; r < a.rows; r += (int64_t)gridDim.x * RL) {
    const uint4 ux = __ldcg(reinterpret_cast<const uint4*>(a.x + r * a.xcs + cg));
    float4 b0 = make_float4(0.f, 0.f, 0.f, 0.f), b1 = b0;
    if (a.base) {
      const float4* b4 = reinterpret_cast<const float4*>(a.base + r * a.bcs + cg);
      b0 = __ldcg(b4);
      b1 = __ldcg(b4 + 1);
    }
    uint4 u[GATHER_BATCH];
#pragma unroll
    for (int j = 0; j < GATHER_BATCH; j++)
      if (j < nb) u[j] = __ldcg(reinterpret_cast<const uint4*>(a.dy[j] + r * a.dycs[j] + cg));
    float xh[8], acc[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    {
      float xv[8];
      unpack8(ux, xv);
#pragma unroll
      for (int k = 0; k < 8; k++) xh[k] = __fmul_rn(__fsub_rn(xv[k], cm[0][g * 8 + k]), cm[1][g * 8 + k]);
    }
#pragma unroll
    for (int j = 0; j < GATHER_BATCH; j++)
      if (j < nb) {
        if (OCC >= 3) gather_term_s(u[j], &cf[j][0][0], g, xh, acc);
        else gather_term(u[j], &cf[j][0][0], g, xh, acc);
      }
    for (int l0 = GATHER_BATCH; l0 < a.nl; l0 += GATHER_BATCH) {   // later layers, a batch in flight
#pragma unroll
      for (int j = 0; j < GATHER_BATCH; j++)
        if (l0 + j < a.nl) u[j] = __ldcg(reinterpret_cast<const uint4*>(a.dy[l0 + j] + r * a.dycs[l0 + j] + cg));
#pragma unroll
      for (int j = 0; j < GATHER_BATCH; j++)
        if (l0 + j < a.nl) {
          if (OCC >= 3) gather_term_s(u[j], &cf[l0 + j][0][0], g, xh, acc);
          else gather_term(u[j], &cf[l0 + j][0][0], g, xh, acc);
        }
    }
    if (a.out_f32) {
      float4* o4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + r * a.ocs + cg);
      o4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      o4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
      st8(reinterpret_cast<bf16*>(a.out) + r * a.ocs + cg, acc);
    }
  }
}

}  // namespace

// DenseNet deferred BN input gradient over channels [0, nc) of a concat range (see
// bn_gather_dx).  Pointer arrays are host arrays of nl (<= 32) entries, each already offset to
// the range's first channel; layers are summed in array order.  out may alias base (fp32).
CVB_API int cvb_bn_gather_dx(const void* x, int xcs, int64_t rows, int nc, const float* mean, const float* rstd,
                             const float* base, int bcs, int nl, const void* const* dy, const int* dycs,
                             const float* const* gamma, const float* const* beta, const float* const* dgamma,
                             const float* const* dbeta, void* out, int ocs, int out_f32, void* stream) {
  if (nc % 8 || nl < 0 || nl > GATHER_MAX_LAYERS || !out) { cvb_set_error("bn_gather_dx: bad arguments"); return CVB_EINVAL; }
  GatherArgs a;
  memset(&a, 0, sizeof(a));
  a.x = (const bf16*)x; a.xcs = xcs; a.rows = rows; a.nc = nc; a.mean = mean; a.rstd = rstd;
  a.base = base; a.bcs = bcs; a.nl = nl;
  for (int l = 0; l < nl; l++) {
    a.dy[l] = (const bf16*)dy[l]; a.dycs[l] = dycs[l];
    a.gamma[l] = gamma[l]; a.beta[l] = beta[l]; a.dgamma[l] = dgamma[l]; a.dbeta[l] = dbeta[l];
  }
  a.out = out; a.ocs = ocs; a.out_f32 = out_f32;
  const int chunks = (nc + GATHER_CH - 1) / GATHER_CH;
  const int rl_per_cta = GATHER_THREADS / ((nc < GATHER_CH ? nc : GATHER_CH) / 8);
  const int64_t rblocks = (rows + rl_per_cta - 1) / rl_per_cta;
  int64_t bx = (int64_t)cvb_num_sms() * 8 / chunks;
  if (bx < 1) bx = 1;
  if (bx > rblocks) bx = rblocks;
  static int occ = -1;
  if (occ < 0) { const char* e = getenv("CVB_GATHER_OCC"); occ = e ? atoi(e) : 2; }
  if (occ >= 3)
    cvb_launch(bn_gather_dx<3>, dim3((unsigned)bx, (unsigned)chunks), dim3(GATHER_THREADS), 0, (cudaStream_t)stream, a);
  else
    cvb_launch(bn_gather_dx<2>, dim3((unsigned)bx, (unsigned)chunks), dim3(GATHER_THREADS), 0, (cudaStream_t)stream, a);
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}


// Debug: copy the last traced BN launch's per-CTA phase timestamps ([n][8] globaltimer ns).
CVB_API int cvb_bn_debug_trace(long long* out, int n) {
  if (!g_trace) { cvb_set_error("bn trace: run with CVB_BN_TRACE=1"); return CVB_EINVAL; }
  CVB_CUDA(cudaDeviceSynchronize());
  CVB_CUDA(cudaMemcpy(out, g_trace, sizeof(long long) * 8 * (size_t)n, cudaMemcpyDeviceToHost));
  return CVB_OK;
}
