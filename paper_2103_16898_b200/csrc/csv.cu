// Bit-exact CSV -> binary64 dataset parse on the GPU.
//
// Replaces covault.workload.parse_dataset (/root/reference/pkg/src/covault/workload.py:24-41)
// for ASCII text: str.splitlines() line breaks, strip(), blank and '#' lines skipped, split(","),
// the last field is the label, and every field converted like Python's float() -- which is
// correctly rounded (round-half-even) decimal -> binary64, so the result must be bit-identical.
//
// Pipeline (all device work; the host only reads a handful of counters):
//   1. index:  per 4 KB chunk count line breaks and field delimiters (',' + breaks), scan the
//      chunk counts, then write every break / delimiter position (block-level scans).
//   2. lines:  one thread per line: blank / comment / data, field count; an exclusive scan of the
//      data flags gives each data line its row index.
//   3. fill:   one thread per field: locate its line (binary search over the break delimiter
//      indices), parse the number and store it straight into X[row][col] or y[row].
// Number conversion (per field, no host fallback):
//   * Python float() grammar: sign, digits with PEP-515 underscores, '.', exponent, inf /
//     infinity / nan (case-insensitive), surrounding whitespace;
//   * <= 19 significant digits: Clinger's exact fast path when it applies, else the
//     Eisel-Lemire 128-bit product (Lemire 2021; always correct for a 64-bit significand,
//     Mushtak & Lemire 2023);
//   * more digits: Eisel-Lemire on the truncated significand w and w+1; when they differ, an
//     exact big-integer comparison of the full decimal string with the halfway point.
// Errors are reported, not repaired: the first (line, column) that is a too-short row or an
// invalid number wins, exactly the row order in which the reference raises.
#include "cvb_common.cuh"
#include "pow5_table.cuh"
#include <vector>

namespace {

constexpr int CT = 256;                 // threads per CTA in the byte passes
constexpr int CB = 16;                  // bytes per thread
constexpr int CHUNK = CT * CB;          // 4 KB per CTA

__device__ __forceinline__ bool is_break(const uint8_t* t, size_t i, size_t len) {
  const uint8_t c = t[i];
  if (c == '\n') return !(i > 0 && t[i - 1] == '\r');   // "\r\n" breaks once, at the '\r'
  return c == '\r' || c == 0x0b || c == 0x0c || c == 0x1c || c == 0x1d || c == 0x1e;
}

__device__ __forceinline__ int break_len(const uint8_t* t, size_t i, size_t len) {
  return (t[i] == '\r' && i + 1 < len && t[i + 1] == '\n') ? 2 : 1;
}

__device__ __forceinline__ bool is_ws(uint8_t c) {   // whitespace that can occur inside a line
  return c == ' ' || c == '\t' || c == 0x1f;
}

// per-thread counts of breaks and delimiters over its CB bytes
__device__ __forceinline__ void count16(const uint8_t* t, size_t len, size_t i0, int* nb, int* nd) {
  int b = 0, d = 0;
  for (int k = 0; k < CB; k++) {
    const size_t i = i0 + k;
    if (i >= len) break;
    const bool br = is_break(t, i, len);
    b += br;
    d += br || t[i] == ',';
  }
  *nb = b;
  *nd = d;
}

__global__ void csv_count(const uint8_t* __restrict__ t, size_t len, int2* __restrict__ counts) {
  __shared__ int sb[CT], sd[CT];
  const size_t i0 = (size_t)blockIdx.x * CHUNK + (size_t)threadIdx.x * CB;
  int b, d;
  count16(t, len, i0, &b, &d);
  sb[threadIdx.x] = b;
  sd[threadIdx.x] = d;
  __syncthreads();
  for (int s = CT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) { sb[threadIdx.x] += sb[threadIdx.x + s]; sd[threadIdx.x] += sd[threadIdx.x + s]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[blockIdx.x] = make_int2(sb[0], sd[0]);
}

// exclusive scan of n int2 counts in place (one CTA of 1024 threads, sequential tiles); the
// totals land in tot[0..1]
__global__ void scan_int2(int2* __restrict__ c, int64_t n, long long* __restrict__ tot,
                          long long* __restrict__ base) {
  __shared__ long long sa[1024], sb2[1024];
  long long carry_a = 0, carry_b = 0;
  for (int64_t t0 = 0; t0 < n; t0 += 1024) {
    const int64_t i = t0 + threadIdx.x;
    const int2 v = i < n ? c[i] : make_int2(0, 0);
    sa[threadIdx.x] = v.x;
    sb2[threadIdx.x] = v.y;
    __syncthreads();
    for (int s = 1; s < 1024; s <<= 1) {   // Hillis-Steele inclusive scan
      long long a = threadIdx.x >= s ? sa[threadIdx.x - s] : 0, b = threadIdx.x >= s ? sb2[threadIdx.x - s] : 0;
      __syncthreads();
      sa[threadIdx.x] += a;
      sb2[threadIdx.x] += b;
      __syncthreads();
    }
    if (i < n) {
      base[2 * i] = carry_a + sa[threadIdx.x] - v.x;
      base[2 * i + 1] = carry_b + sb2[threadIdx.x] - v.y;
    }
    carry_a += sa[1023];
    carry_b += sb2[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) { tot[0] = carry_a; tot[1] = carry_b; }
}

// break k: brk_pos[k] (position), brk_next[k] (start of the next line), brk_didx[k] (its
// index among the delimiters); delimiter j: dl_pos[j], dl_next[j]
__global__ void csv_mark(const uint8_t* __restrict__ t, size_t len, const long long* __restrict__ base,
                         int64_t* __restrict__ brk_pos, int64_t* __restrict__ brk_next, int64_t* __restrict__ brk_didx,
                         int64_t* __restrict__ dl_pos, int64_t* __restrict__ dl_next) {
  __shared__ int sb[CT], sd[CT];
  const size_t i0 = (size_t)blockIdx.x * CHUNK + (size_t)threadIdx.x * CB;
  int b, d;
  count16(t, len, i0, &b, &d);
  sb[threadIdx.x] = b;
  sd[threadIdx.x] = d;
  __syncthreads();
  for (int s = 1; s < CT; s <<= 1) {
    const int xb = threadIdx.x >= s ? sb[threadIdx.x - s] : 0, xd = threadIdx.x >= s ? sd[threadIdx.x - s] : 0;
    __syncthreads();
    sb[threadIdx.x] += xb;
    sd[threadIdx.x] += xd;
    __syncthreads();
  }
  long long kb = base[2 * blockIdx.x] + sb[threadIdx.x] - b, kd = base[2 * blockIdx.x + 1] + sd[threadIdx.x] - d;
  for (int k = 0; k < CB; k++) {
    const size_t i = i0 + k;
    if (i >= len) break;
    const bool br = is_break(t, i, len);
    if (br || t[i] == ',') {
      const int64_t nxt = (int64_t)i + (br ? break_len(t, i, len) : 1);
      dl_pos[kd] = (int64_t)i;
      dl_next[kd] = nxt;
      if (br) {
        brk_pos[kb] = (int64_t)i;
        brk_next[kb] = nxt;
        brk_didx[kb] = kd;
        kb++;
      }
      kd++;
    }
  }
}

// one thread per line: data flag (1) and field count; atomics collect min/max field counts of
// data lines
__global__ void csv_lines(const uint8_t* __restrict__ t, int64_t nlines, const int64_t* __restrict__ brk_pos,
                          const int64_t* __restrict__ brk_next, const int64_t* __restrict__ brk_didx,
                          int* __restrict__ is_data, long long* __restrict__ stats) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nlines) return;
  const int64_t s = k ? brk_next[k - 1] : 0, e = brk_pos[k];
  int64_t p = s;
  while (p < e && is_ws(t[p])) p++;
  const bool data = p < e && t[p] != '#';
  is_data[k] = data ? 1 : 0;
  if (data) {
    const long long nf = brk_didx[k] - (k ? brk_didx[k - 1] : -1);
    atomicMin(&stats[0], nf);
    atomicMax(&stats[1], nf);
  }
}

// exclusive scan of int flags -> int64 rows, multi-CTA (1024 per tile): tile sums, then offsets
__global__ void tile_sums(const int* __restrict__ f, int64_t n, long long* __restrict__ sums) {
  __shared__ int s[1024];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  s[threadIdx.x] = i < n ? f[i] : 0;
  __syncthreads();
  for (int k = 512; k > 0; k >>= 1) {
    if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[blockIdx.x] = s[0];
}

__global__ void tile_scan_serial(long long* __restrict__ sums, int64_t ntiles, long long* __restrict__ total) {
  if (threadIdx.x || blockIdx.x) return;
  long long acc = 0;
  for (int64_t i = 0; i < ntiles; i++) { const long long v = sums[i]; sums[i] = acc; acc += v; }
  *total = acc;
}

__global__ void tile_apply(const int* __restrict__ f, int64_t n, const long long* __restrict__ sums,
                           int64_t* __restrict__ rows) {
  __shared__ int s[1024];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int v = i < n ? f[i] : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int k = 1; k < 1024; k <<= 1) {
    const int x = threadIdx.x >= k ? s[threadIdx.x - k] : 0;
    __syncthreads();
    s[threadIdx.x] += x;
    __syncthreads();
  }
  if (i < n) rows[i] = v ? sums[blockIdx.x] + s[threadIdx.x] - v : -1;
}

// ---- decimal -> binary64 ----------------------------------------------------------------
struct AM { uint64_t mantissa; int32_t power2; };

__device__ __forceinline__ AM compute_float(int64_t q, uint64_t w) {
  // Eisel-Lemire for binary64 (mantissa_explicit_bits 52, minimum_exponent -1023)
  AM a;
  if (w == 0 || q < CVB_POW5_MIN_Q) { a.mantissa = 0; a.power2 = 0; return a; }
  if (q > CVB_POW5_MAX_Q) { a.mantissa = 0; a.power2 = 0x7FF; return a; }
  const int lz = __clzll(w);
  w <<= lz;
  const int idx = 2 * (int)(q - CVB_POW5_MIN_Q);
  const uint64_t t0 = __ldg(reinterpret_cast<const unsigned long long*>(cvb_pow5_128) + idx);
  const uint64_t t1 = __ldg(reinterpret_cast<const unsigned long long*>(cvb_pow5_128) + idx + 1);
  uint64_t hi = __umul64hi(w, t0), lo = w * t0;
  const uint64_t precision_mask = 0xFFFFFFFFFFFFFFFFull >> 55;
  if ((hi & precision_mask) == precision_mask) {
    const uint64_t shi = __umul64hi(w, t1);
    const uint64_t nlo = lo + shi;
    if (shi > nlo) hi++;
    lo = nlo;
  }
  const int upperbit = (int)(hi >> 63);
  const int shift = upperbit + 64 - 52 - 3;
  a.mantissa = hi >> shift;
  a.power2 = (int32_t)(((((152170 + 65536) * (int32_t)q) >> 16) + 63) + upperbit - lz - (-1023));
  if (a.power2 <= 0) {
    if (-a.power2 + 1 >= 64) { a.mantissa = 0; a.power2 = 0; return a; }
    a.mantissa >>= -a.power2 + 1;
    a.mantissa += (a.mantissa & 1);
    a.mantissa >>= 1;
    a.power2 = (a.mantissa < (1ull << 52)) ? 0 : 1;
    return a;
  }
  if (lo <= 1 && q >= -4 && q <= 23 && (a.mantissa & 3) == 1) {
    if ((a.mantissa << shift) == hi) a.mantissa &= ~1ull;
  }
  a.mantissa += (a.mantissa & 1);
  a.mantissa >>= 1;
  if (a.mantissa >= (2ull << 52)) { a.mantissa = 1ull << 52; a.power2++; }
  a.mantissa &= ~(1ull << 52);
  if (a.power2 >= 0x7FF) { a.power2 = 0x7FF; a.mantissa = 0; }
  return a;
}

__device__ __forceinline__ uint64_t am_bits(AM a) { return ((uint64_t)a.power2 << 52) | a.mantissa; }

// ---- big integers for the rare > 19-digit ambiguous case ---------------------------------
constexpr int BL = 168;   // 32-bit limbs (5376 bits)
struct Big { uint32_t d[BL]; int n; };

__device__ void big_set(Big& b, uint64_t v) {
  b.n = 0;
  while (v) { b.d[b.n++] = (uint32_t)v; v >>= 32; }
}
__device__ void big_muladd(Big& b, uint32_t m, uint32_t add) {
  uint64_t c = add;
  for (int i = 0; i < b.n; i++) {
    const uint64_t p = (uint64_t)b.d[i] * m + c;
    b.d[i] = (uint32_t)p;
    c = p >> 32;
  }
  if (c && b.n < BL) b.d[b.n++] = (uint32_t)c;
}
__device__ void big_pow5(Big& b, int64_t e) {
  while (e >= 13) { big_muladd(b, 1220703125u, 0); e -= 13; }
  uint32_t m = 1;
  while (e-- > 0) m *= 5;
  if (m != 1) big_muladd(b, m, 0);
}
__device__ void big_shl(Big& b, int64_t s) {
  const int w = (int)(s / 32), r = (int)(s % 32);
  if (b.n == 0) return;
  int n = b.n + w + 1;
  if (n > BL) n = BL;
  for (int i = n - 1; i >= 0; i--) {
    const int src = i - w;
    uint32_t v = 0;
    if (src >= 0 && src < b.n) v = b.d[src] << r;
    if (r && src - 1 >= 0 && src - 1 < b.n) v |= b.d[src - 1] >> (32 - r);
    b.d[i] = v;
  }
  b.n = n;
  while (b.n && !b.d[b.n - 1]) b.n--;
}
__device__ int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; i--)
    if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
  return 0;
}

// exact decision between candidate `bits` and the next double: compare the decimal digits
// D x 10^e10 (digits ds[0..nd), sticky = non-zero digits dropped beyond them) with the halfway
// point of the candidate
__device__ uint64_t slow_round(uint64_t bits, const uint8_t* ds, int nd, int64_t e10, bool sticky, Big* A, Big* B) {
  const int e = (int)(bits >> 52) & 0x7FF;
  const uint64_t m = e ? ((bits & ((1ull << 52) - 1)) | (1ull << 52)) : (bits & ((1ull << 52) - 1));
  const int64_t e2 = e ? (int64_t)e - 1075 : -1074;
  big_set(*A, 0);
  for (int i = 0; i < nd;) {        // A = D, nine digits at a time
    uint32_t chunk = 0, mul = 1;
    for (int k = 0; k < 9 && i < nd; k++, i++) { chunk = chunk * 10 + ds[i]; mul *= 10; }
    if (A->n == 0) big_set(*A, chunk);
    else big_muladd(*A, mul, chunk);
  }
  big_set(*B, 2 * m + 1);
  int64_t a2 = e10, b2 = e2 - 1;
  if (e10 >= 0) big_pow5(*A, e10);
  else big_pow5(*B, -e10);
  if (a2 > b2) big_shl(*A, a2 - b2);
  else if (b2 > a2) big_shl(*B, b2 - a2);
  const int c = big_cmp(*A, *B);
  const bool up = c > 0 || (c == 0 && (sticky || (m & 1)));
  return up ? bits + 1 : bits;
}

__constant__ double c_p10[23] = {1e0, 1e1, 1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8, 1e9, 1e10, 1e11,
                                 1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};

__device__ __forceinline__ uint8_t lower(uint8_t c) { return (c >= 'A' && c <= 'Z') ? (uint8_t)(c + 32) : c; }

__device__ bool match_ci(const uint8_t* p, int64_t n, const char* word) {
  int64_t i = 0;
  for (; word[i]; i++)
    if (i >= n || lower(p[i]) != (uint8_t)word[i]) return false;
  return i == n;
}

// Python float() of bytes [s, e).  Returns false for text float() rejects.
constexpr int MAXD = 800;   // digits kept for the exact comparison (binary64 needs <= 768)
__device__ bool parse_double(const uint8_t* t, int64_t s, int64_t e, double* out) {
  while (s < e && is_ws(t[s])) s++;
  while (e > s && is_ws(t[e - 1])) e--;
  if (s >= e) return false;
  bool neg = false;
  if (t[s] == '+' || t[s] == '-') { neg = t[s] == '-'; s++; }
  if (s >= e) return false;
  const uint8_t c0 = lower(t[s]);
  if (c0 == 'i' || c0 == 'n') {
    unsigned long long b;
    if (match_ci(t + s, e - s, "inf") || match_ci(t + s, e - s, "infinity")) b = 0x7FF0000000000000ull;
    else if (match_ci(t + s, e - s, "nan")) b = 0x7FF8000000000000ull;
    else return false;
    *out = __longlong_as_double((long long)(b | (neg ? 1ull << 63 : 0ull)));   // sign as a bit (NaN too)
    return true;
  }
  // mantissa digits (underscores only between two digits), optional '.', optional exponent
  uint64_t w = 0;
  int nsig = 0;            // significant digits seen (after leading zeros)
  int64_t dexp = 0;        // decimal exponent adjustment of w
  bool truncated = false, any_digit = false, seen_dot = false;
  int64_t p = s;
  int64_t first_sig = -1;  // position of the first significant digit (for the slow path)
  for (; p < e; p++) {
    const uint8_t c = t[p];
    if (c >= '0' && c <= '9') {
      any_digit = true;
      if (nsig == 0 && c == '0') { if (seen_dot) dexp--; continue; }
      if (nsig == 0) first_sig = p;
      if (nsig < 19) { w = w * 10 + (c - '0'); if (seen_dot) dexp--; }
      else { if (c != '0') truncated = true; if (!seen_dot) dexp++; }
      nsig++;
    } else if (c == '_') {
      if (p == s || p + 1 >= e || !(t[p - 1] >= '0' && t[p - 1] <= '9') || !(t[p + 1] >= '0' && t[p + 1] <= '9'))
        return false;
    } else if (c == '.' && !seen_dot) {
      seen_dot = true;
    } else {
      break;
    }
  }
  if (!any_digit) return false;
  int64_t ex = 0;
  if (p < e) {
    if (t[p] != 'e' && t[p] != 'E') return false;
    p++;
    bool eneg = false;
    if (p < e && (t[p] == '+' || t[p] == '-')) { eneg = t[p] == '-'; p++; }
    if (p >= e || !(t[p] >= '0' && t[p] <= '9')) return false;
    for (; p < e; p++) {
      const uint8_t c = t[p];
      if (c >= '0' && c <= '9') { if (ex < 100000000) ex = ex * 10 + (c - '0'); }
      else if (c == '_') {
        if (p + 1 >= e || !(t[p - 1] >= '0' && t[p - 1] <= '9') || !(t[p + 1] >= '0' && t[p + 1] <= '9')) return false;
      } else return false;
    }
    if (eneg) ex = -ex;
  }
  const int64_t q = dexp + ex;
  uint64_t bits;
  if (w == 0) {
    bits = 0;
  } else if (!truncated && q >= -22 && q <= 22 && w <= (1ull << 53)) {
    const double dw = (double)w;
    const double v = q >= 0 ? __dmul_rn(dw, c_p10[q]) : __ddiv_rn(dw, c_p10[-q]);
    bits = (uint64_t)__double_as_longlong(v);
  } else {
    const AM a1 = compute_float(q, w);
    bits = am_bits(a1);
    if (truncated) {
      const AM a2 = compute_float(q, w + 1);
      if (am_bits(a2) != bits) {
        // exact comparison over the full significant digit string
        uint8_t ds[MAXD];
        int nd = 0;
        bool sticky = false, dot = false;
        int64_t fracpos = 0, frac_at_last = 0, int_dropped = 0;
        for (int64_t k = s; k < e; k++) {
          const uint8_t c = t[k];
          if (c == '.') { dot = true; continue; }
          if (c == '_') continue;
          if (c < '0' || c > '9') break;
          if (dot) fracpos++;
          if (k < first_sig) continue;                 // leading zeros
          if (nd < MAXD) { ds[nd++] = (uint8_t)(c - '0'); frac_at_last = dot ? fracpos : 0; }
          else { if (c != '0') sticky = true; if (!dot) int_dropped++; }
        }
        // value = D x 10^e10 (+ sticky): D = the kept digits
        const int64_t e10 = ex + int_dropped - frac_at_last;
        Big A, B;
        bits = slow_round(bits, ds, nd, e10, sticky, &A, &B);
      }
    }
  }
  *out = __longlong_as_double((long long)(bits | (neg ? 1ull << 63 : 0ull)));
  return true;
}

// one thread per field (delimiter index j = the field that ends at delimiter j)
__global__ void csv_fill(const uint8_t* __restrict__ t, int64_t nfields, int64_t nlines,
                         const int64_t* __restrict__ dl_pos, const int64_t* __restrict__ dl_next,
                         const int64_t* __restrict__ brk_didx, const int64_t* __restrict__ rows, int64_t F,
                         double* __restrict__ X, double* __restrict__ y, unsigned long long* __restrict__ err) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nfields) return;
  // line k = first break whose delimiter index >= j
  int64_t lo = 0, hi = nlines - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (brk_didx[mid] >= j) hi = mid; else lo = mid + 1;
  }
  const int64_t k = lo;
  const int64_t row = rows[k];
  if (row < 0) return;                                   // blank or comment line
  const int64_t first = k ? brk_didx[k - 1] + 1 : 0;
  const int64_t nf = brk_didx[k] - first + 1, col = j - first;
  const unsigned long long key = ((unsigned long long)k << 24) | (unsigned long long)min(col, (int64_t)0xFFFFFF);
  if (nf < 2) {                                          // "bad dataset row" (workload.py:32-33)
    if (col == 0) atomicMin(err, (unsigned long long)k << 24);
    return;
  }
  const int64_t s = j ? dl_next[j - 1] : 0, e = dl_pos[j];
  double v;
  if (!parse_double(t, s, e, &v)) { atomicMin(err, key); return; }
  if (nf != F + 1) return;                               // ragged: reported by the field-count check
  if (col < F) X[row * F + col] = v;
  else y[row] = v;
}

}  // namespace

// ---- C ABI -------------------------------------------------------------------------------
struct cvb_csv {
  const uint8_t* text;
  size_t len;
  int64_t nlines, nfields, rows, F;
  long long nf_min, nf_max;
  int64_t *brk_pos, *brk_next, *brk_didx, *dl_pos, *dl_next, *rows_of_line;
  int* is_data;
  unsigned long long* err;
  cudaStream_t s;
};

static void csv_release(cvb_csv* c) {
  if (!c) return;
  for (void* p : {(void*)c->brk_pos, (void*)c->brk_next, (void*)c->brk_didx, (void*)c->dl_pos, (void*)c->dl_next,
                  (void*)c->rows_of_line, (void*)c->is_data, (void*)c->err})
    if (p) cudaFreeAsync(p, c->s);
  cudaStreamSynchronize(c->s);
  free(c);
}

// Pass 1 (index).  text_dev: the ASCII text, which must END WITH a line break (the host appends
// one).  On return info[0..5] = {rows (data lines), F (fields of the first data line - 1),
// nf_min, nf_max (field counts over data lines), lines, fields}.  Synchronises `stream`.
CVB_API int cvb_csv_index(const uint8_t* text_dev, size_t len, int64_t info[6], cvb_csv** out, void* stream) {
  if (!text_dev || !len || !info || !out) { cvb_set_error("csv_index: bad arguments"); return CVB_EINVAL; }
  cvb_csv* c = (cvb_csv*)calloc(1, sizeof(cvb_csv));
  if (!c) return CVB_ENOMEM;
  c->text = text_dev; c->len = len; c->s = (cudaStream_t)stream;
  cudaStream_t s = c->s;
  const int64_t nch = (int64_t)((len + CHUNK - 1) / CHUNK);
  int2* counts = nullptr;
  long long *base = nullptr, *tot = nullptr, *stats = nullptr, *tsum = nullptr;
  long long h_tot[2] = {0, 0}, h_stats[2] = {0, 0};
  int rc = CVB_OK;
  cudaError_t e = cudaMallocAsync((void**)&counts, sizeof(int2) * nch, s);
  if (!e) e = cudaMallocAsync((void**)&base, sizeof(long long) * 2 * nch, s);
  if (!e) e = cudaMallocAsync((void**)&tot, sizeof(long long) * 4, s);
  if (!e) { csv_count<<<(unsigned)nch, CT, 0, s>>>(text_dev, len, counts); e = cudaGetLastError(); }
  if (!e) { scan_int2<<<1, 1024, 0, s>>>(counts, nch, tot, base); e = cudaGetLastError(); }
  if (!e) e = cudaMemcpyAsync(h_tot, tot, sizeof(h_tot), cudaMemcpyDeviceToHost, s);
  if (!e) e = cudaStreamSynchronize(s);
  c->nlines = h_tot[0]; c->nfields = h_tot[1];
  if (!e && c->nlines == 0) { cvb_set_error("csv_index: text must end with a line break"); rc = CVB_EINVAL; }
  const size_t L8 = sizeof(int64_t) * (size_t)(c->nlines > 0 ? c->nlines : 1);
  const size_t F8 = sizeof(int64_t) * (size_t)(c->nfields > 0 ? c->nfields : 1);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->brk_pos, L8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->brk_next, L8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->brk_didx, L8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->rows_of_line, L8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->is_data, sizeof(int) * (size_t)c->nlines, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->dl_pos, F8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->dl_next, F8, s);
  if (!e && !rc) e = cudaMallocAsync((void**)&c->err, sizeof(unsigned long long), s);
  if (!e && !rc) {
    csv_mark<<<(unsigned)nch, CT, 0, s>>>(text_dev, len, base, c->brk_pos, c->brk_next, c->brk_didx, c->dl_pos,
                                          c->dl_next);
    stats = tot + 2;
    const long long init[2] = {0x7FFFFFFFFFFFFFFFll, 0};
    cudaMemcpyAsync(stats, init, sizeof(init), cudaMemcpyHostToDevice, s);
    csv_lines<<<(unsigned)((c->nlines + 255) / 256), 256, 0, s>>>(text_dev, c->nlines, c->brk_pos, c->brk_next,
                                                                   c->brk_didx, c->is_data, stats);
    const int64_t nt = (c->nlines + 1023) / 1024;
    e = cudaMallocAsync((void**)&tsum, sizeof(long long) * (size_t)(nt + 1), s);
    if (!e) {
      tile_sums<<<(unsigned)nt, 1024, 0, s>>>(c->is_data, c->nlines, tsum);
      tile_scan_serial<<<1, 32, 0, s>>>(tsum, nt, tsum + nt);
      tile_apply<<<(unsigned)nt, 1024, 0, s>>>(c->is_data, c->nlines, tsum, c->rows_of_line);
      const unsigned long long none = ~0ull;
      cudaMemcpyAsync(c->err, &none, sizeof(none), cudaMemcpyHostToDevice, s);
      long long h_rows = 0;
      cudaMemcpyAsync(&h_rows, tsum + nt, sizeof(long long), cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(h_stats, stats, sizeof(h_stats), cudaMemcpyDeviceToHost, s);
      e = cudaGetLastError();
      if (!e) e = cudaStreamSynchronize(s);
      c->rows = h_rows;
    }
  }
  if (counts) cudaFreeAsync(counts, s);
  if (base) cudaFreeAsync(base, s);
  if (tot) cudaFreeAsync(tot, s);
  if (tsum) cudaFreeAsync(tsum, s);
  if (e) { cvb_set_error("csv_index: %s", cudaGetErrorString(e)); rc = CVB_ECUDA; }
  if (rc) { csv_release(c); return rc; }
  c->nf_min = c->rows ? h_stats[0] : 0;
  c->nf_max = c->rows ? h_stats[1] : 0;
  // F = fields of the FIRST data line - 1 (the reference's feature count is set by row 0)
  c->F = 0;
  if (c->rows) {
    int64_t first = -1;
    std::vector<int> flags(1024);
    for (int64_t k0 = 0; k0 < c->nlines && first < 0; k0 += 1024) {
      const int64_t m = c->nlines - k0 < 1024 ? c->nlines - k0 : 1024;
      cudaMemcpy(flags.data(), c->is_data + k0, sizeof(int) * m, cudaMemcpyDeviceToHost);
      for (int64_t i = 0; i < m; i++) if (flags[i]) { first = k0 + i; break; }
    }
    int64_t d[2] = {-1, -1};
    if (first > 0) cudaMemcpy(d, c->brk_didx + first - 1, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost);
    else cudaMemcpy(d + 1, c->brk_didx, sizeof(int64_t), cudaMemcpyDeviceToHost);
    c->F = d[1] - d[0] - 1;
  }
  info[0] = c->rows; info[1] = c->F; info[2] = c->nf_min; info[3] = c->nf_max; info[4] = c->nlines;
  info[5] = c->nfields;
  *out = c;
  return CVB_OK;
}

// Pass 2 (fill): X_dev rows x F binary64 (row-major), y_dev rows labels; written only when every
// data line has F+1 fields.  err_out[0..3] = {line of the first error or -1, its column,
// line start byte, line end byte}.  Synchronises `stream`.
CVB_API int cvb_csv_fill(cvb_csv* c, double* X_dev, double* y_dev, int64_t err_out[4]) {
  if (!c || !err_out || (c->rows && c->F > 0 && (!X_dev || !y_dev))) { cvb_set_error("csv_fill: bad arguments"); return CVB_EINVAL; }
  cudaStream_t s = c->s;
  if (c->nfields)
    csv_fill<<<(unsigned)((c->nfields + 127) / 128), 128, 0, s>>>(c->text, c->nfields, c->nlines, c->dl_pos, c->dl_next,
                                                                   c->brk_didx, c->rows_of_line, c->F, X_dev, y_dev,
                                                                   c->err);
  unsigned long long key = ~0ull;
  CVB_CUDA(cudaGetLastError());
  CVB_CUDA(cudaMemcpyAsync(&key, c->err, sizeof(key), cudaMemcpyDeviceToHost, s));
  CVB_CUDA(cudaStreamSynchronize(s));
  err_out[0] = err_out[1] = err_out[2] = err_out[3] = -1;
  if (key != ~0ull) {
    const int64_t k = (int64_t)(key >> 24);
    err_out[0] = k;
    err_out[1] = (int64_t)(key & 0xFFFFFF);
    int64_t b[2] = {0, 0};
    if (k > 0) CVB_CUDA(cudaMemcpy(b, c->brk_next + k - 1, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CVB_CUDA(cudaMemcpy(b + 1, c->brk_pos + k, sizeof(int64_t), cudaMemcpyDeviceToHost));
    err_out[2] = b[0];
    err_out[3] = b[1];
  }
  return CVB_OK;
}

CVB_API void cvb_csv_free(cvb_csv* c) { csv_release(c); }
