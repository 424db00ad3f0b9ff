// tcgen05 implicit-GEMM engine for conv / dense layers (K5 of DESIGN.md).
//
// No reference code exists for this layer type (the reference trainer is a logistic toy,
// pkg/src/covault/workload.py:48-71); the CNN is defined from the paper's prose
// -- see DESIGN.md.
//
// One persistent, warp-specialised kernel serves every GEMM of a training step:
//   warp 0      TMA producer: per K-block, G boxes per operand, loaded straight from the
//               NHWC activation (4-D tensor map; conv padding = TMA out-of-bounds zero
//               fill) or from 2-D weight / dense maps, into a multi-stage smem ring.
//   warp 1      TMEM allocator + tcgen05.mma issuer (kind::f16, bf16 in, fp32 accumulate in
//               TMEM, 128 x BN tile, 4 MMAs of K=16 per 64-wide K-block), double-buffered
//               accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> bias -> bf16/fp32 -> global (NHWC rows,
//               dense rows or fp32 split-K partials).
// All per-K-block box coordinates and all UMMA smem descriptors are precomputed on the host
// (box table + descriptor templates in the parameter bank), so the single-thread issue
// loops are a handful of uniform instructions per TMA / MMA (measured: without this the
// issue loops, not the tensor core, bounded the kernel).
// Modes:
//   FWD   A = gathered activation (K-major, K = taps x Cin), B = weights [Cout][K] (K-major).
//         Used for conv forward and for dgrad (input dY or its zero-upsampled copy, weights
//         flipped/transposed).  Stride-2 convs read the input through 4 parity views.
//   WGRAD A = dY (MN-major, M = Cout), B = gathered input (MN-major, N = taps x Cin),
//         K = output pixels in 64-pixel boxes, split over CTAs, fp32 partials.
//   DENSE 2-D operands, each K-major or MN-major (FC fwd/dgrad/wgrad).
#include "cvb_common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdlib.h>

namespace {

enum { MODE_FWD = 0, MODE_WGRAD = 1, MODE_DENSE = 2, MODE_HALO = 3 };
// MODE_HALO (stride-1 conv, 8x16 output tiles): a K-block is one channel group of the input
// *halo* tile ((8+KW-1) x (16+KH-1) pixels), loaded once as 8-channel no-swizzle planes; each
// tap is just a different UMMA descriptor start row into the same smem (core matrices are 8
// consecutive pixels = 128 contiguous bytes, 8-row groups one halo row apart).  9x fewer L2
// reads and TMA issues than one box per tap; the weights stay resident in smem.
enum { OUT_NHWC = 0, OUT_ROWS = 1, OUT_PARTIAL = 2 };

constexpr int BM = 128;          // UMMA M (cta_group::1)
constexpr int BK = 64;           // K elements per pipeline stage
constexpr int NUM_THREADS = 320; // up to 10 warps: producer, MMA, 4 or 8 epilogue warps
constexpr int MAX_BOXES = 512;   // box-table entries

// n / d for 0 <= n < 2^31 by multiply-high (host-precomputed magic; no runtime divide in
// the per-tile bookkeeping of the role loops).
struct FastDiv {
  uint32_t d, mul, shift;
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return (uint32_t)(((uint64_t)__umulhi(n, mul) + n) >> shift);
  }
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t s = 0;
  while ((1ull << s) < d) s++;
  f.shift = s;
  f.mul = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  return f;
}

struct GemmParams {
  CUtensorMap mapA[4];
  CUtensorMap mapB[4];
  uint64_t adesc[8], bdesc[8];   // UMMA descriptor templates, start address relative to the stage
  int kr, ksteps;                // K rows per stage of MN-major operands (64 / 128), MMAs per stage
  int mode;
  int a_major, b_major;     // 0 = K-major, 1 = MN-major
  int a_cel, b_cel;         // elements per box row (8,16,32,64)
  int ga, gb;               // boxes per stage (A, B)
  uint32_t a_box_stride, b_box_stride;   // smem bytes between boxes
  int BN;
  int M, N;                 // logical GEMM extents (rows, cols)
  int m_tiles, n_tiles, splits;
  int num_kb;               // total K-blocks of the full K range
  int kb_per_split;
  uint32_t tx_bytes;
  uint32_t a_box_bytes;     // bytes TMA writes per A box (WGRAD: per-tile A box count varies)
  uint32_t a_stage_bytes;   // smem bytes of the A part of one pipeline stage
  uint32_t b_stage_bytes;   // smem bytes of the B part of one stage (0: BN * kr * 2)
  int w_halo;               // WGRAD halo: one (bw+KW-1)-wide box per K-block carries every kw tap
  int w_groups;             // WGRAD halo over cin = 64 * w_groups: N tile t = (kh t / G, channel group t % G)
  int w_cin;                // ... its input channels (output column = kh*KW*cin + kw*cin + g*64 + ci)
  int w_pair;               // WGRAD halo, Cout = 64: an N tile holds TWO kh rows (M rows 0-63: kh 2t+1, 64-127: kh 2t)
  int w_kh;                 // kernel height (w_pair: which M halves are real)
  int b_res;                // 1: the whole B operand (one N tile, all K) is loaded once per CTA
  uint32_t b_res_bytes;     // size of the resident B region
  int b_slabs;              // 64-wide K slabs of the resident B
  uint32_t idesc;
  int stages;
  // conv geometry
  int tw, th, tn;           // pixel-box extents (FWD: the M tile; WGRAD: the K chunk)
  int ptiles_w, ptiles_h;   // tile counts along w, h of the pixel space
  int OH, OW, NIMG;         // pixel space (FWD: output; WGRAD: dY)
  // epilogue
  int out_mode, out_f32;
  void* out;
  int64_t ldc;              // row stride of the output in elements
  int col_off;
  const float* bias;
  int part_rows;            // OUT_PARTIAL: rows per split slab
  int accum;                // add into the existing output
  // TMA-store epilogue (st_tma): each epilogue warp stages its 32 rows x st_ch columns in a
  // swizzled smem buffer and issues one bulk tensor store (reduce-add when accumulating)
  int st_tma;
  int st_ch;                // columns per store chunk (divides BN); st_ch * elem = 32/64/128 B
  uint32_t st_swz;          // swizzle mask of the chunk rows (7: 128B, 3: 64B, 1: 32B)
  uint32_t stg_off;         // smem offset of the 4 x 2 staging buffers (4 KB each)
  int st_bw, st_bh, st_bn;  // the warp's box in pixel space (NHWC); dense/partial: 32,1,1
  FastDiv fd_m, fd_n, fd_mn, fd_pw, fd_ph;   // m_tiles, n_tiles, m_tiles*n_tiles, ptiles_w, ptiles_h
  int n_epi;                // epilogue warps: 4, or 8 (two per TMEM lane quarter, column halves)
  int epi_alt;              // n_epi == 8: the two warp groups take alternate tiles (all columns)
  int nacc_log2;            // TMEM accumulator buffers: 1 << nacc_log2 (2 or 4)
  int two_cta;              // launched with two CTAs per SM (half the shared memory each)
  uint32_t stg_warp;        // staging bytes per epilogue warp (two buffers)
  int st_rows;              // valid rows of an M tile (multiple of 32); warps past it store nothing
  int out_par;              // 1: NHWC output is the parity sub-grid (out_ph, out_pw) of an out_H x out_W image;
                            // 2: rows out_ph::2 only (every column) of an out_H x out_W image
  int out_ph, out_pw, out_H, out_W;
  CUtensorMap mapC;
  int dbg;                  // profiling knobs: 1 = skip MMA, 2 = skip TMA (results invalid)
  int kb_pair;              // MMA warp issues two 4-MMA K-blocks per batch (FWD / DENSE / WGRAD, ksteps 4)
  int pair;                 // CTA pair (cta_group::2, M = 256): FWD with streamed weights; B split by rank
  int hs;                   // HALO with streamed weights (wide stride-1 3x3 convs): A = kw-box halo per
                            // 64-channel group (ring `stages`), B = one tap's weight box (ring `stages_b`)
  int stages_b;
  uint32_t b_tap_bytes;     // bytes of one tap's weight box in this CTA
  const void* b_ptr;        // FWD weights [b_rows][b_ld] (host-side: the pair plan re-encodes mapB)
  int64_t b_rows, b_cols, b_ld;
  long long* trace;         // debug: clock64 timeline of CTA 0 (5 x 4096 slots) or null
  int nbox;
  // MODE_HALO geometry
  int h_cin, h_cg, h_planes, h_pitch, h_pad, h_kh, h_kw;
  int h_rows;                   // 1: the halo is ONE SW128 box of 64-channel (128-byte) pixel rows
  int h_kwbox;                  // 1: one 8-pixel-wide SW128 box per kw tap (planes = KW): every tap's
                                //    A start is 1024-byte aligned (row-shifted SW128 starts issue at
                                //    ~99 cycles per MMA, aligned ones at 44-64: scripts/mma_rate.py)
  int no_epi_alt;               // planning: keep the column-split epilogue (smaller staging)
  int h_rowpad;                 // 1: 32-channel input (cin == 32) loaded as 128-byte SW128 rows whose
                                //    upper half is TMA zero fill (SW64 operand reads run at half rate)
  int h_mps;                    // MMAs per stage (taps * cg/16)
  uint32_t h_plane_stride;      // bytes between 8-channel planes (>= halo pixels * 16, 128-aligned)
  uint32_t h_box_bytes;         // bytes TMA writes per plane
  uint32_t boxtab[MAX_BOXES];   // packed (map, channel, dw, dh) per gathered box
};

#define TRACE(type, idx)                                                                        \
  do {                                                                                          \
    if (p.trace && blockIdx.x == 0 && (idx) < 4096) p.trace[(type) * 4096 + (idx)] = clock64(); \
  } while (0)

__host__ __device__ inline uint32_t pack_box(int mi, int cc, int dw, int dh) {
  return (uint32_t)mi | ((uint32_t)cc << 2) | ((uint32_t)(dw + 64) << 18) | ((uint32_t)(dh + 64) << 25);
}

// ---------------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Long waits (the epilogue's accumulator-full wait spans a whole tile): one lane polls with a
// back-off, so idle warps do not keep the shared-memory pipe (the MMA operand path) busy.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_lazy(uint64_t* bar, uint32_t parity, bool lazy) {
  if (!lazy) { mbar_wait(bar, parity); return; }
  if ((threadIdx.x & 31) == 0)
    while (!mbar_test(bar, parity)) __nanosleep(128);
  __syncwarp();
  mbar_wait(bar, parity);   // every lane observes the completed phase (memory ordering)
}
__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint32_t dst, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "+r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
// Issued by the whole (converged) warp; only the elected lane's instruction executes, so the
// descriptor arithmetic stays on the uniform datapath (no R2UR moves per MMA).
__device__ __forceinline__ void umma_bf16_el(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc,
                                             uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(leader) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---- CTA pair (cta_group::2): one 256 x N MMA over the two SMs of a TPC ------------------
// The leader (cluster rank 0) issues every MMA; each CTA holds its own 128 rows of A and N/2
// rows of B at the same smem offsets, and its 128 accumulator rows in its own TMEM.  Both
// CTAs' TMA loads complete on the LEADER's full barrier; the MMA commits arrive on the same
// barrier offset in both CTAs (multicast); both epilogues release the leader's accumulator.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in cluster rank 0
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* map, uint32_t dst, uint32_t bar_c, int c0, int c1,
                                                 int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_c), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t dst, uint32_t bar_c, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_c), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void umma_bf16_pair_el(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t acc, uint32_t leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(leader) : "memory");
}
// commit to the same barrier offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(smem_u32(bar)), "h"((uint16_t)3) : "memory");
}
template <int PAIR>
__device__ __forceinline__ void umma_t(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc,
                                       uint32_t leader) {
  if (PAIR) umma_bf16_pair_el(tmem_d, adesc, bdesc, idesc, acc, leader);
  else umma_bf16_el(tmem_d, adesc, bdesc, idesc, acc, leader);
}
template <int PAIR>
__device__ __forceinline__ void commit_t(uint64_t* bar) {
  if (PAIR) umma_commit_pair(bar);
  else umma_commit(bar);
}
// 32 consecutive fp32 columns of this thread's TMEM lane; caller waits with tmem_wait()
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void tma_red_add_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               ::"l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// ---------------------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------------------
// Store 16 fp32 accumulator values of one output row (bias / accumulate / bf16 pack).
__device__ __forceinline__ void store16(const GemmParams& p, int64_t off, int col, const uint32_t* r, bool has_k) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; j++) v[j] = has_k ? __uint_as_float(r[j]) : 0.f;
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] += (col + j < p.N) ? __ldg(p.bias + col + j) : 0.f;
  }
  const bool full = col + 16 <= p.N;
  if (p.accum) {
#pragma unroll
    for (int j = 0; j < 16; j++)
      if (full || col + j < p.N)
        v[j] += p.out_f32 ? reinterpret_cast<const float*>(p.out)[off + j]
                          : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.out)[off + j]);
  }
  if (full) {
    if (p.out_f32) {
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + off);
#pragma unroll
      for (int j = 0; j < 4; j++) d[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    } else {
      uint32_t pk[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
        pk[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      uint4* d = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + off);
      d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; j++) {
      if (col + j < p.N) {
        if (p.out_f32) reinterpret_cast<float*>(p.out)[off + j] = v[j];
        else reinterpret_cast<__nv_bfloat16*>(p.out)[off + j] = __float2bfloat16_rn(v[j]);
      }
    }
  }
}

// Loop-invariant epilogue parameters, copied once into registers through opaque movs: left to
// the compiler they are re-loaded from the kernel-parameter constant bank for every chunk, and
// those loads miss the constant cache behind the producer / MMA warps' descriptor and box-table
// reads (traced: ~900 cycles per 64-column chunk of a short-K tile).
struct EpiK {
  const float* bias;
  int st_ch, swz, f32, N, accum, col_off;
};
__device__ __forceinline__ int pin(int v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
__device__ __forceinline__ uint32_t pinu(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
__device__ __forceinline__ const float* pinp(const float* v) {
  uint64_t u = reinterpret_cast<uint64_t>(v);
  asm volatile("mov.b64 %0, %0;" : "+l"(u));
  return reinterpret_cast<const float*>(u);
}

// Stage 16 fp32 accumulator values (columns [cc, cc+16) of the chunk) of row r into the
// chunk buffer: bias, bf16/fp32 pack, 16-byte pieces at swizzled offsets (bank-conflict-free).
__device__ __forceinline__ void stage16(const EpiK& p, uint32_t buf, int r, int cc, int col, const uint32_t* rr,
                                        bool has_k) {
  float v[16];
#pragma unroll
  for (int j = 0; j < 16; j++) v[j] = has_k ? __uint_as_float(rr[j]) : 0.f;
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 16; j++) v[j] += (col + j < p.N) ? __ldg(p.bias + col + j) : 0.f;
  }
  const uint32_t rowbytes = (uint32_t)p.st_ch * (p.f32 ? 4u : 2u);
  if (p.f32) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t off = r * rowbytes + (uint32_t)(cc + 4 * q) * 4u;
      const uint32_t ph = off ^ (((off >> 7) & p.swz) << 4);
      st_shared_v4(buf + ph, __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]), __float_as_uint(v[4 * q + 2]),
                   __float_as_uint(v[4 * q + 3]));
    }
  } else {
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
      pk[j] = *reinterpret_cast<uint32_t*>(&h);
    }
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const uint32_t off = r * rowbytes + (uint32_t)(cc + 8 * q) * 2u;
      const uint32_t ph = off ^ (((off >> 7) & p.swz) << 4);
      st_shared_v4(buf + ph, pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
    }
  }
}

// Halo-mode MMA issue for one K-block (channel group kb) with the tap geometry known at
// compile time: every A/B descriptor offset folds to a constant or one uniform add per tap,
// so the issue loop is a few uniform instructions per MMA (the generic loop needed ~18 and
// starved the tensor core: 96 cycles per N=32 MMA against a 40-cycle floor).
template <int KH, int KW, int NJ, int PAIR = 0>
__device__ __forceinline__ void halo_issue(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc, uint32_t acc_flag,
                                           uint32_t leader, int kb, uint32_t cin16, uint32_t slab16) {
  constexpr uint32_t pitch = 8 + KW - 1;
  constexpr uint32_t plane2 = 2u * ((((pitch * (16 + KH - 1) * 16) + 127) / 128 * 128) >> 4);
  uint32_t qt = (uint32_t)kb * NJ;
#pragma unroll
  for (int kh = 0; kh < KH; kh++) {
#pragma unroll
    for (int kw = 0; kw < KW; kw++) {
      // NJ consecutive 16-element K units starting at qt never cross a 64-wide slab when
      // NJ divides 4 and qt is a multiple of NJ
      const uint64_t bt = b0 + (uint64_t)((qt >> 2) * slab16 + ((qt & 3u) << 1));
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        umma_t<PAIR>(tmem_d, a0 + (uint32_t)(kh * pitch + kw) + (uint32_t)j * plane2, bt + 2u * j, idesc, acc_flag, leader);
        acc_flag = 1u;
      }
      qt += cin16;
    }
  }
}

// Halo mode, 64-channel groups as SW128 pixel rows (one 128-byte TMA row per halo pixel
// instead of eight 16-byte plane rows): tap (kh, kw) = start row kh*pitch + kw (8 x 16-byte
// units per row), 16-channel step j = +32 bytes inside the swizzled row.  UMMA derives the
// swizzle from absolute smem address bits, so row-shifted starts read the TMA layout exactly.
template <int KH, int KW, int NJ, int RU, int PITCH = 8 + KW - 1, int PAIR = 0>
__device__ __forceinline__ void halo_rows_issue_t(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                uint32_t acc_flag, uint32_t leader, int kb, uint32_t cin16,
                                                uint32_t slab16) {
  constexpr uint32_t pitch = PITCH;   // RU: 16-byte units per smem pixel row (>= 2*NJ)
  uint32_t qt = (uint32_t)kb * NJ;
#pragma unroll
  for (int kh = 0; kh < KH; kh++) {
#pragma unroll
    for (int kw = 0; kw < KW; kw++) {
      const uint64_t bt = b0 + (uint64_t)((qt >> 2) * slab16 + ((qt & 3u) << 1));
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        umma_t<PAIR>(tmem_d, a0 + (uint32_t)((kh * pitch + kw) * RU + 2 * j), bt + 2u * j, idesc, acc_flag, leader);
        acc_flag = 1u;
      }
      qt += cin16;
    }
  }
}

// kw-box halo: box kw holds the 8 x (16+KH-1) pixels the kw taps read, so tap (kh, kw) starts
// kh*8 rows (kh KB) into box kw -- an aligned SW128 start (SBO = 1024 B)
template <int KH, int KW, int NJ, int PAIR = 0>
__device__ __forceinline__ void halo_kw_issue(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t idesc,
                                              uint32_t acc_flag, uint32_t leader, int kb, uint32_t cin16,
                                              uint32_t slab16, uint32_t box16) {
  uint32_t qt = (uint32_t)kb * NJ;
#pragma unroll
  for (int kh = 0; kh < KH; kh++) {
#pragma unroll
    for (int kw = 0; kw < KW; kw++) {
      const uint64_t bt = b0 + (uint64_t)((qt >> 2) * slab16 + ((qt & 3u) << 1));
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        umma_t<PAIR>(tmem_d, a0 + (uint32_t)kw * box16 + (uint32_t)(kh * 64 + 2 * j), bt + 2u * j, idesc, acc_flag,
                     leader);
        acc_flag = 1u;
      }
      qt += cin16;
    }
  }
}

// Halo mode with 8 input channels (the padded RGB / grey stem): one 16-wide MMA K step
// covers TWO taps.  The second K half of a no-swizzle K-major operand sits LBO bytes after
// the first, so LBO = 16 B (the next pixel = the next kw tap, a0) or (pitch - KW + 1) * 16 B
// (the next tap wraps to the next halo row, a1).  Flattened K = tap * 8 + ci matches the
// natural [cout][kh][kw][8] weights; the odd last tap pairs with K >= KH*KW*8, which the
// weight map zero-fills (its A half reads the extra halo column, finite data).
template <int KH, int KW, int PAIR = 0>
__device__ __forceinline__ void halo8_issue(uint32_t tmem_d, uint64_t a0, uint64_t a1, uint64_t b0, uint32_t idesc,
                                            uint32_t leader, uint32_t slab16) {
  constexpr int T = KH * KW, PITCH = 8 + KW;
#pragma unroll
  for (int q = 0; q < (T + 1) / 2; q++) {
    const int t0 = 2 * q, kh = t0 / KW, kw = t0 % KW;
    const bool wraps = (t0 + 1 < T) && ((t0 + 1) / KW != kh);
    umma_t<PAIR>(tmem_d, (wraps ? a1 : a0) + (uint32_t)(kh * PITCH + kw),
                 b0 + (uint64_t)((q >> 2) * slab16 + ((q & 3) << 1)), idesc, q > 0 ? 1u : 0u, leader);
  }
}

// One K-block's MMAs from descriptor templates held in registers: the MMA asm carries a
// "memory" clobber, so descriptors read from the parameter bank inside the loop would be
// re-loaded (LDC -> UTCHMMA dependency chains, ~100 cycles per MMA measured) before every MMA.
template <int KS, int PAIR = 0>
__device__ __forceinline__ void issue_ksteps(const uint64_t (&ad)[8], const uint64_t (&bd)[8], uint32_t idesc,
                                             uint32_t tmem_d, uint64_t sa, uint64_t sb, bool acc, bool leader) {
#pragma unroll
  for (int k = 0; k < KS; k++)
    umma_t<PAIR>(tmem_d, ad[k] + sa, bd[k] + sb, idesc, (acc || k > 0) ? 1u : 0u, leader);
}

template <int PAIR>
__device__ __forceinline__ void release_acc_t(uint32_t tempty0, int acc) {
  if (PAIR) mbar_arrive_remote(tempty0 + 8u * (uint32_t)acc);
  else asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8u * (uint32_t)acc) : "memory");
}
#define release_acc(t0, a) release_acc_t<PAIR>(t0, a)

// PAIR = 1: CTA-pair instantiation (MODE_FWD with streamed weights only; see the cta_group::2
// helpers above).  Every tcgen05 instruction of a kernel must use one cta_group, hence the
// separate instantiation.
// MODE: the kernel is instantiated per GEMM mode (code of the other modes is dead and dropped):
// the single all-mode kernel was ~150 KB of SASS and its epilogue / issue loops stalled on
// instruction fetch (ncu: "no instruction" stalls; ~1,800 cycles per short-K tile epilogue).
#define PMODE (MODE)
template <int PAIR, int MODE>
__global__ void __launch_bounds__(NUM_THREADS, 1) umma_gemm_kernel(const __grid_constant__ GemmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_stage = p.a_stage_bytes;         // 16 KB (halo mode: planes * plane stride)
  const uint32_t b_stage = (p.b_res || (PMODE == MODE_HALO && p.hs)) ? 0u : (p.b_stage_bytes ? p.b_stage_bytes : p.BN * p.kr * 2);
  const uint32_t stage_bytes = a_stage + b_stage;
  const uint32_t b_kb_bytes = p.BN * BK * 2;        // resident B: one K-block slab
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * stage_bytes + p.b_res_bytes +
                                               (p.st_tma ? (uint32_t)p.n_epi * p.stg_warp : 0u));
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;       // [nacc <= 4]
  uint64_t* tempty = tfull + 4;             // [nacc <= 4]
  uint64_t* bres_full = tempty + 4;         // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres_full + 1);
  uint64_t* full_b = bres_full + 2;           // HS: weight-tap ring [stages_b]
  uint64_t* empty_b = full_b + 16;            // [stages_b <= 16]

  // shfl: lets the compiler prove the role index warp-uniform (keeps the issue loops on the
  // uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nacc = 1 << p.nacc_log2, acc_cols = nacc * p.BN;
  const int tmem_cols = acc_cols <= 32 ? 32 : acc_cols <= 64 ? 64 : acc_cols <= 128 ? 128 : acc_cols <= 256 ? 256 : 512;

  // CTA pair: rank 1's tiles are the odd M tiles of each unit; only rank 0 issues MMAs
  const int rank = PAIR ? (int)cluster_rank() : 0;
  const int cl = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;      // scheduling slot
  const int ncl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int mtu = PAIR ? p.m_tiles >> 1 : p.m_tiles;                   // M units (tile pairs)
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 4; i++) { prefetch_map(&p.mapA[i]); prefetch_map(&p.mapB[i]); }
    if (p.st_tma) prefetch_map(&p.mapC);
    for (int i = 0; i < p.stages; i++) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < nacc; i++) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], (p.epi_alt ? 4 : p.n_epi) * (PAIR ? 2 : 1));
    }
    mbar_init(bres_full, 1);
    for (int i = 0; i < p.stages_b; i++) { mbar_init(&full_b[i], 1); mbar_init(&empty_b[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)), "r"(tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // the peer's barriers exist before any multicast commit / TMA
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem0 = smem_u32(smem);
  CVB_PDL_PROLOGUE();   // barrier init / TMEM alloc / descriptor prefetch overlap the previous kernel

  const int units = mtu * p.n_tiles * p.splits;

  // Role loops run on whole, converged warps; only the issuing instructions are predicated on
  // one elected lane.  Stage / phase counters are incremental (no divisions in the loops).
  const uint32_t bres = smem0 + p.stages * stage_bytes;   // resident B region (if any)
  if (warp == 0) {
    const bool leader = elect_one();
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    int sb_i = 0;        // HS weight-tap ring
    uint32_t phb = 0;
    if (p.b_res && leader && cl < units) {
      // whole B operand (single N tile): b_slabs slabs of BN x 64, loaded once per CTA (pair:
      // this CTA's BN/2 rows, completing on the leader's barrier)
      if constexpr (PAIR) {
        const uint32_t bar_c = mapa_rank0(smem_u32(bres_full));
        const int half = p.BN >> 1;
        if (rank == 0) mbar_expect_tx(bres_full, 2u * p.b_slabs * p.gb * half * p.b_cel * 2);
        for (int kb = 0; kb < p.b_slabs; kb++)
          for (int g = 0; g < p.gb; g++)
            tma_load_2d_pair(&p.mapB[0], bres + kb * (half * BK * 2) + g * p.b_box_stride, bar_c, kb * BK + g * p.b_cel,
                             rank * half);
      } else {
        mbar_expect_tx(bres_full, p.b_slabs * p.gb * p.BN * p.b_cel * 2);
        for (int kb = 0; kb < p.b_slabs; kb++)
          for (int g = 0; g < p.gb; g++)
            tma_load_2d(&p.mapB[0], bres + kb * b_kb_bytes + g * p.b_box_stride, bres_full, kb * BK + g * p.b_cel, 0);
      }
    }
    __syncwarp();
    for (int u = cl; u < units; u += ncl) {
      const int rest = (int)p.fd_m.div((uint32_t)u), mt = (u - rest * mtu) * (PAIR ? 2 : 1) + rank;
      const int sp = (int)p.fd_n.div((uint32_t)rest), nt = rest - sp * p.n_tiles;
      const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      int tw0 = 0, th0 = 0, tn0 = 0;
      if (PMODE == MODE_FWD || PMODE == MODE_HALO) {
        const int r2 = (int)p.fd_pw.div((uint32_t)mt), r3 = (int)p.fd_ph.div((uint32_t)r2);
        tw0 = (mt - r2 * p.ptiles_w) * p.tw;
        th0 = (r2 - r3 * p.ptiles_h) * p.th;
        tn0 = r3 * p.tn;
      }
      // WGRAD: K-block kb is a pixel box; walk it incrementally
      int pw = 0, ph0 = 0, pn = 0;
      if (PMODE == MODE_WGRAD) {
        pw = (kb0 % p.ptiles_w) * p.tw;
        const int r2 = kb0 / p.ptiles_w;
        ph0 = (r2 % p.ptiles_h) * p.th;
        pn = (r2 / p.ptiles_h) * p.tn;
      }
      const int m0 = mt * BM, n0 = nt * p.BN;
      if ((PMODE == MODE_HALO && p.hs)) {   // per channel group: the halo (3 kw boxes), then the 9 taps' weight boxes
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_lazy(&empty[s], ph ^ 1, false);
          if (leader) {
            const uint32_t sa = smem0 + s * stage_bytes;
            if constexpr (PAIR) {
              const uint32_t bar_c = mapa_rank0(smem_u32(&full[s]));
              if (rank == 0) mbar_expect_tx(&full[s], 2u * p.tx_bytes);
              for (int j = 0; j < p.h_planes; j++)
                tma_load_4d_pair(&p.mapA[0], sa + j * p.h_plane_stride, bar_c, kb * 64, tw0 - p.h_pad + j,
                                 th0 - p.h_pad, tn0);
            } else {
              mbar_expect_tx(&full[s], p.tx_bytes);
              for (int j = 0; j < p.h_planes; j++)
                tma_load_4d(&p.mapA[0], sa + j * p.h_plane_stride, &full[s], kb * 64, tw0 - p.h_pad + j,
                            th0 - p.h_pad, tn0);
            }
          }
          __syncwarp();
          if (++s == p.stages) { s = 0; ph ^= 1; }
          for (int t = 0; t < p.h_kh * p.h_kw; t++) {
            mbar_wait_lazy(&empty_b[sb_i], phb ^ 1, false);
            if (leader) {
              const uint32_t dst = bres + sb_i * p.b_tap_bytes;
              const int col = t * p.h_cin + kb * 64;
              if constexpr (PAIR) {
                const uint32_t bar_c = mapa_rank0(smem_u32(&full_b[sb_i]));
                if (rank == 0) mbar_expect_tx(&full_b[sb_i], 2u * p.b_tap_bytes);
                tma_load_2d_pair(&p.mapB[0], dst, bar_c, col, n0 + rank * (p.BN >> 1));
              } else {
                mbar_expect_tx(&full_b[sb_i], p.b_tap_bytes);
                tma_load_2d(&p.mapB[0], dst, &full_b[sb_i], col, n0);
              }
            }
            __syncwarp();
            if (++sb_i == p.stages_b) { sb_i = 0; phb ^= 1; }
          }
        }
        continue;
      }
      // WGRAD: A boxes past M (Cout) would be all zero fill -- skip them; their accumulator
      // rows are never stored.
      int ga_eff = p.ga;
      uint32_t tx = p.tx_bytes;
      if (PMODE == MODE_WGRAD) {
        ga_eff = min(p.ga, (p.M - m0 + p.a_cel - 1) / p.a_cel);
        tx = p.tx_bytes - (uint32_t)(p.ga - ga_eff) * p.a_box_bytes;
        if ((PMODE == MODE_WGRAD ? p.w_pair : 0)) { ga_eff = (PMODE == MODE_WGRAD ? p.w_pair : 0) == 2 ? 2 : 1; tx = p.tx_bytes; }   // kh-paired / kh-quad dY boxes
      }
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        mbar_wait_lazy(&empty[s], ph ^ 1, (p.dbg & 256) != 0);
        if (leader) {
          if (!(p.dbg & 32)) TRACE(0, it);
          const uint32_t sa = smem0 + s * stage_bytes, sb = sa + a_stage;
          if constexpr (PAIR) {
            // both CTAs' boxes complete on the leader's barrier; the leader expects both halves
            const uint32_t bar_c = mapa_rank0(smem_u32(&full[s]));
            if (rank == 0) mbar_expect_tx(&full[s], 2u * tx);
            if (PMODE == MODE_WGRAD) {   // own 128 Cout rows of dY, this CTA's half of the input boxes
              for (int b = 0; b < p.ga; b++)
                tma_load_4d_pair(&p.mapA[0], sa + b * p.a_box_stride, bar_c, m0 + b * p.a_cel, pw, ph0, pn);
              const int gh = p.gb >> 1;
              const uint32_t* tab = p.boxtab + nt * p.gb + rank * gh;
              for (int j = 0; j < gh; j++) {
                const uint32_t e = tab[j];
                tma_load_4d_pair(&p.mapB[e & 3], sb + j * p.b_box_stride, bar_c, (int)((e >> 2) & 0xFFFF),
                                 pw + (int)((e >> 18) & 127) - 64, ph0 + (int)(e >> 25) - 64, pn);
              }
            } else if (PMODE == MODE_HALO) {   // this CTA's halo tile (weights are resident)
              for (int j = 0; j < p.h_planes; j++) {
                if ((PMODE == MODE_HALO && p.h_kwbox))
                  tma_load_4d_pair(&p.mapA[0], sa + j * p.h_plane_stride, bar_c, kb * p.h_cg, tw0 - p.h_pad + j,
                                   th0 - p.h_pad, tn0);
                else
                  tma_load_4d_pair(&p.mapA[0], sa + j * p.h_plane_stride, bar_c, kb * p.h_cg + 8 * j, tw0 - p.h_pad,
                                   th0 - p.h_pad, tn0);
              }
            } else {
            const uint32_t* tab = p.boxtab + kb * p.ga;
            for (int g = 0; g < p.ga; g++) {
              const uint32_t e = tab[g];
              tma_load_4d_pair(&p.mapA[e & 3], sa + g * p.a_box_stride, bar_c, (int)((e >> 2) & 0xFFFF),
                               tw0 + (int)((e >> 18) & 127) - 64, th0 + (int)(e >> 25) - 64, tn0);
            }
            for (int g = 0; g < p.gb; g++)
              tma_load_2d_pair(&p.mapB[0], sb + g * p.b_box_stride, bar_c, kb * BK + g * p.b_cel,
                               n0 + rank * (p.BN >> 1));
            }
          } else if (p.dbg & 2) {
            mbar_arrive(&full[s]);
          } else {
            mbar_expect_tx(&full[s], tx);
            if (PMODE == MODE_HALO) {
              if ((PMODE == MODE_HALO && p.h_kwbox)) {
                for (int j = 0; j < p.h_planes; j++)
                  tma_load_4d(&p.mapA[0], sa + j * p.h_plane_stride, &full[s], kb * p.h_cg, tw0 - p.h_pad + j,
                              th0 - p.h_pad, tn0);
              } else {
                for (int j = 0; j < p.h_planes; j++)
                  tma_load_4d(&p.mapA[0], sa + j * p.h_plane_stride, &full[s], kb * p.h_cg + 8 * j, tw0 - p.h_pad,
                              th0 - p.h_pad, tn0);
              }
            } else if (PMODE == MODE_FWD) {
              const uint32_t* tab = p.boxtab + kb * p.ga;
              for (int g = 0; g < p.ga; g++) {
                const uint32_t e = tab[g];
                tma_load_4d(&p.mapA[e & 3], sa + g * p.a_box_stride, &full[s], (int)((e >> 2) & 0xFFFF),
                            tw0 + (int)((e >> 18) & 127) - 64, th0 + (int)(e >> 25) - 64, tn0);
              }
              if (!p.b_res)
                for (int g = 0; g < p.gb; g++)
                  tma_load_2d(&p.mapB[0], sb + g * p.b_box_stride, &full[s], kb * BK + g * p.b_cel, n0);
            } else if (PMODE == MODE_WGRAD) {
              if ((PMODE == MODE_WGRAD ? p.w_pair : 0) == 2) {   // M atom 0 = dY rows one up (kh 2t+1), atom 1 = dY rows (kh 2t)
                for (int b = 0; b < 2; b++)
                  tma_load_4d(&p.mapA[0], sa + b * p.a_box_stride, &full[s], 0, pw, ph0 - 1 + b, pn);
              } else {
                for (int b = 0; b < ga_eff; b++)
                  tma_load_4d(&p.mapA[0], sa + b * p.a_box_stride, &full[s], m0 + b * p.a_cel, pw,
                              (PMODE == MODE_WGRAD ? p.w_pair : 0) == 3 ? ph0 - (p.w_kh - 1) : (PMODE == MODE_WGRAD ? p.w_pair : 0) ? ph0 - 1 : ph0, pn);
              }
              const uint32_t* tab = p.boxtab + nt * p.gb;
              for (int j = 0; j < p.gb; j++) {
                const uint32_t e = tab[j];
                tma_load_4d(&p.mapB[e & 3], sb + j * p.b_box_stride, &full[s], (int)((e >> 2) & 0xFFFF),
                            pw + (int)((e >> 18) & 127) - 64, ph0 + (int)(e >> 25) - 64, pn);
              }
            } else {  // DENSE
              for (int g = 0; g < p.ga; g++) {
                if (p.a_major == 0) tma_load_2d(&p.mapA[0], sa + g * p.a_box_stride, &full[s], kb * BK + g * p.a_cel, m0);
                else tma_load_2d(&p.mapA[0], sa + g * p.a_box_stride, &full[s], m0 + g * p.a_cel, kb * BK);
              }
              for (int g = 0; g < p.gb; g++) {
                if (p.b_major == 0) tma_load_2d(&p.mapB[0], sb + g * p.b_box_stride, &full[s], kb * BK + g * p.b_cel, n0);
                else tma_load_2d(&p.mapB[0], sb + g * p.b_box_stride, &full[s], n0 + g * p.b_cel, kb * BK);
              }
            }
          }
        }
        __syncwarp();
        if (PMODE == MODE_WGRAD) {
          pw += p.tw;
          if (pw >= p.ptiles_w * p.tw) {
            pw = 0;
            ph0 += p.th;
            if (ph0 >= p.ptiles_h * p.th) { ph0 = 0; pn += p.tn; }
          }
        }
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
    }
    if (PAIR) {
      // producer tail: every stage's last multicast release has landed in this CTA before it
      // may exit (the leader's commits write our barriers)
      for (int i = 0; i < p.stages; i++) {
        mbar_wait(&empty[s], ph ^ 1);
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
      for (int i = 0; i < p.stages_b; i++) {
        mbar_wait(&empty_b[sb_i], phb ^ 1);
        if (++sb_i == p.stages_b) { sb_i = 0; phb ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (PAIR && rank != 0) {
      // the peer CTA's MMA warp has no work: the leader issues for both SMs
    } else {
    const bool leader = elect_one();
    int s = 0;
    uint32_t ph = 0;
    int it = 0, lt = 0;
    int sbm = 0;         // HS weight-tap ring
    uint32_t phbm = 0;
    uint64_t adr[8], bdr[8];   // descriptor templates, read once (see issue_ksteps)
#pragma unroll
    for (int k = 0; k < 8; k++) { adr[k] = p.adesc[k]; bdr[k] = p.bdesc[k]; }
    const uint32_t idr = p.idesc;
    for (int u = cl; u < units; u += ncl, ++lt) {
      const int sp = (int)p.fd_mn.div((uint32_t)u);
      const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      const int acc = lt & (nacc - 1);
      if (lt == 0 && p.b_res) mbar_wait(bres_full, 0);
      mbar_wait(&tempty[acc], ((lt >> p.nacc_log2) & 1) ^ 1);
      if ((p.dbg & 32) && !(p.dbg & 64) && leader) TRACE(0, it);   // debug: slot 0 = accumulator wait passed
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * p.BN;
      if ((PMODE == MODE_HALO && p.hs)) {
        // per channel group: wait the halo, then per tap the weight box -> 4 MMAs (64 channels),
        // the tap's A start = kw box + kh KB (aligned SW128 starts, as in halo_kw_issue)
        uint32_t acc_flag = 0u;
        const uint32_t box16 = p.h_plane_stride >> 4;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a0 = adr[0] + ((smem0 + s * stage_bytes) >> 4);
          const int hkw = p.h_kw, ntap = p.h_kh * hkw;
          for (int t = 0, kh = 0, kw = 0; t < ntap; t++, kw = kw + 1 == hkw ? 0 : kw + 1, kh += kw == 0 ? 1 : 0) {
            mbar_wait(&full_b[sbm], phbm);
            tc_fence_after();
            const uint64_t b0 = bdr[0] + ((bres + sbm * p.b_tap_bytes) >> 4);
#pragma unroll
            for (int j = 0; j < 4; j++) {
              umma_t<PAIR>(tmem_d, a0 + (uint32_t)kw * box16 + (uint32_t)(kh * 64 + 2 * j), b0 + 2u * j, idr, acc_flag,
                           leader);
              acc_flag = 1u;
            }
            if (leader) commit_t<PAIR>(&empty_b[sbm]);
            __syncwarp();
            if (++sbm == p.stages_b) { sbm = 0; phbm ^= 1; }
          }
          if (leader) commit_t<PAIR>(&empty[s]);
          __syncwarp();
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
      } else if (p.kb_pair) {
        // gathered / dense K-blocks are only 4 MMAs each: the MMA warp's fixed cost per issue
        // batch (~450 cycles measured, independent of N) left the tensor pipe idle half the
        // time.  Two stages are waited for and issued as one batch of 8 MMAs.
        for (int kb = kb0; kb < kb1;) {
          const bool two = kb + 1 < kb1;
          const int s2 = s + 1 == p.stages ? 0 : s + 1;
          const uint32_t ph2 = s + 1 == p.stages ? ph ^ 1u : ph;
          mbar_wait(&full[s], ph);
          if (two) mbar_wait(&full[s2], ph2);
          tc_fence_after();
          if (leader) TRACE(1, it);
          const uint64_t sa = (smem0 + s * stage_bytes) >> 4;
          issue_ksteps<4, PAIR>(adr, bdr, idr, tmem_d, sa, sa + (a_stage >> 4), kb > kb0, leader);
          if (two) {
            const uint64_t sa2 = (smem0 + s2 * stage_bytes) >> 4;
            issue_ksteps<4, PAIR>(adr, bdr, idr, tmem_d, sa2, sa2 + (a_stage >> 4), true, leader);
          }
          if (leader) {
            commit_t<PAIR>(&empty[s]);
            if (two) commit_t<PAIR>(&empty[s2]);
            TRACE(2, it);
          }
          __syncwarp();
          const int n = two ? 2 : 1;
          kb += n;
          it += n;
          for (int i = 0; i < n; i++)
            if (++s == p.stages) { s = 0; ph ^= 1; }
        }
      } else
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        mbar_wait(&full[s], ph);
        if (!(p.dbg & 1024)) tc_fence_after();   // knob 1024: no per-K-block tcgen05 fence (experiment)
        if (leader) TRACE(1, it);
        if (p.dbg & 1) {
          if (leader) mbar_arrive(&empty[s]);
        } else {
          const uint64_t sa = (smem0 + s * stage_bytes) >> 4;
          if (PMODE == MODE_HALO) {
            {
            // every tap of this channel group reads the same halo planes at a row offset.
            // Offsets are plain uniform arithmetic (no table loads: with N = 64 an MMA is
            // only 48 smem-read cycles, so the issue loop must stay below that):
            //   A: tap (kh, kw) -> halo row kh*pitch + kw, 16-channel step j -> 2 planes
            //   B: 16-element K unit q = tap*cin/16 + kb*cg/16 + j -> slab q/4, step q%4
            const uint64_t a0 = p.adesc[0] + sa, b0 = p.bdesc[0] + (bres >> 4);
            const uint32_t nj = (uint32_t)p.h_cg >> 4, cin16 = (uint32_t)p.h_cin >> 4;
            const uint32_t plane2 = 2u * (p.h_plane_stride >> 4), slab16 = (uint32_t)(PAIR ? p.BN >> 1 : p.BN) * (BK * 2 / 16);
            uint32_t acc_flag = kb > kb0 ? 1u : 0u;
            const int geo = p.h_kh * 100 + p.h_kw * 10 + (int)nj;
            const uint32_t box16 = p.h_plane_stride >> 4;
            if ((PMODE == MODE_HALO && p.h_kwbox) && geo == 334) halo_kw_issue<3, 3, 4, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16, box16);
            else if ((PMODE == MODE_HALO && p.h_kwbox) && geo == 332) halo_kw_issue<3, 3, 2, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16, box16);
            else if (p.h_cg == 8) halo8_issue<3, 3, PAIR>(tmem_d, a0, p.adesc[1] + sa, b0, p.idesc, leader, slab16);
            else if (p.h_pitch == 16 && p.h_rowpad && geo == 332) halo_rows_issue_t<3, 3, 2, 8, 16, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_pitch == 16 && p.h_rowpad && geo == 442) halo_rows_issue_t<4, 4, 2, 8, 16, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_pitch == 16 && p.h_rows && geo == 334) halo_rows_issue_t<3, 3, 4, 8, 16, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rowpad && geo == 332) halo_rows_issue_t<3, 3, 2, 8, 8 + 3 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rowpad && geo == 442) halo_rows_issue_t<4, 4, 2, 8, 8 + 4 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rows && geo == 334) halo_rows_issue_t<3, 3, 4, 8, 8 + 3 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rows && geo == 114) halo_rows_issue_t<1, 1, 4, 8, 8 + 1 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rows && geo == 332) halo_rows_issue_t<3, 3, 2, 4, 8 + 3 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rows && geo == 112) halo_rows_issue_t<1, 1, 2, 4, 8 + 1 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (p.h_rows && geo == 442) halo_rows_issue_t<4, 4, 2, 4, 8 + 4 - 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 334) halo_issue<3, 3, 4, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 332) halo_issue<3, 3, 2, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 331) halo_issue<3, 3, 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 114) halo_issue<1, 1, 4, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 112) halo_issue<1, 1, 2, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else if (geo == 111) halo_issue<1, 1, 1, PAIR>(tmem_d, a0, b0, p.idesc, acc_flag, leader, kb, cin16, slab16);
            else {
            uint32_t qt = (uint32_t)kb * nj;
            for (int kh = 0; kh < p.h_kh; kh++) {
              const uint64_t arow = a0 + (uint32_t)(kh * p.h_pitch);
              for (int kw = 0; kw < p.h_kw; kw++, qt += cin16) {
#pragma unroll
                for (uint32_t j = 0; j < 4; j++) {
                  if (j < nj) {
                    const uint32_t q = qt + j;
                    umma_t<PAIR>(tmem_d, arow + (uint32_t)kw + j * plane2, b0 + (q >> 2) * slab16 + ((q & 3u) << 1),
                                 p.idesc, acc_flag, leader);
                    acc_flag = 1u;
                  }
                }
              }
            }
            }
            }
          } else {
            const uint64_t sb = p.b_res ? (uint64_t)((bres + kb * b_kb_bytes) >> 4) : sa + (a_stage >> 4);
            // compile-time step counts: the descriptors become uniform constant-bank operands
            // (a runtime-indexed p.adesc[k] is a per-thread indexed load in the issue loop)
            if (p.ksteps == 4 && (p.dbg & 512)) {   // profiling knob: every K-block's MMAs twice (results invalid)
              issue_ksteps<4, PAIR>(adr, bdr, idr, tmem_d, sa, sb, kb > kb0, leader);
              issue_ksteps<4, PAIR>(adr, bdr, idr, tmem_d, sa, sb, true, leader);
            } else if (p.ksteps == 4) issue_ksteps<4, PAIR>(adr, bdr, idr, tmem_d, sa, sb, kb > kb0, leader);
            else if (p.ksteps == 8) issue_ksteps<8, PAIR>(adr, bdr, idr, tmem_d, sa, sb, kb > kb0, leader);
            else
              for (int k = 0; k < p.ksteps; k++)
                umma_t<PAIR>(tmem_d, p.adesc[k] + sa, p.bdesc[k] + sb, p.idesc, (kb > kb0 || k > 0) ? 1u : 0u, leader);
          }
          if (leader) commit_t<PAIR>(&empty[s]);
        }
        if (leader) TRACE(2, it);
        __syncwarp();
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
      if (leader) commit_t<PAIR>(&tfull[acc]);
      if ((p.dbg & 64) && leader) TRACE(0, it - 1);   // debug: slot 0 = tile's accumulator commit issued
      __syncwarp();
    }
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int quarter = warp & 3;              // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;       // accumulator row (0..127)
    // row -> pixel offsets inside an NHWC M-tile (constant over tiles)
    const int wb = row % p.tw, r2 = row / p.tw, hb = r2 % p.th, nb = r2 / p.th;
    int lt = 0, stg_it = 0;
    // this warp's first row inside an NHWC M tile (constant over tiles)
    const int r0w = quarter * 32;
    const int w_off = r0w % p.tw, h_off = (r0w / p.tw) % p.th, n_off = r0w / (p.tw * p.th);
    // the accumulator buffers are released on the leader's barriers (pair) or our own
    const uint32_t tempty0 = PAIR ? mapa_rank0(smem_u32(&tempty[0])) : smem_u32(&tempty[0]);
    EpiK ek;
    ek.bias = pinp(p.bias); ek.st_ch = pin(p.st_ch); ek.swz = pin((int)p.st_swz); ek.f32 = pin(p.out_f32);
    ek.N = pin(p.N); ek.accum = pin(p.accum); ek.col_off = pin(p.col_off);
    const uint32_t stg_w = pinu(smem0 + p.stg_off + (uint32_t)(warp - 2) * p.stg_warp), stg_half = pinu(p.stg_warp >> 1);
    for (int u = cl; u < units; u += ncl, ++lt) {
      const int rest = (int)p.fd_m.div((uint32_t)u), mt = (u - rest * mtu) * (PAIR ? 2 : 1) + rank;
      const int sp = (int)p.fd_n.div((uint32_t)rest), nt = rest - sp * p.n_tiles;
      const int kb0 = sp * p.kb_per_split, kb1 = min(p.num_kb, kb0 + p.kb_per_split);
      if (p.epi_alt && (lt & 1) != ((warp - 2) >> 2)) continue;   // the other warp group's tile
      const int acc = lt & (nacc - 1);
      mbar_wait_lazy(&tfull[acc], (lt >> p.nacc_log2) & 1, (p.dbg & 128) != 0);
      if (warp == 2 && lane == 0) TRACE(3, lt);
      tc_fence_after();
      bool valid = true;
      int64_t dst_row = 0;
      if (p.st_tma) {
      } else if (p.out_mode == OUT_NHWC) {
        const int ow = (mt % p.ptiles_w) * p.tw + wb;
        const int q = mt / p.ptiles_w;
        const int oh = (q % p.ptiles_h) * p.th + hb;
        const int n = (q / p.ptiles_h) * p.tn + nb;
        valid = (row < p.tw * p.th * p.tn) && ow < p.OW && oh < p.OH && n < p.NIMG;
        dst_row = (((int64_t)n * p.OH + oh) * p.OW + ow);
      } else if (p.out_mode == OUT_ROWS) {
        const int m = mt * BM + row;
        valid = m < p.M;
        dst_row = m;
      } else if ((PMODE == MODE_WGRAD ? p.w_pair : 0)) {
        valid = 2 * nt + (quarter < 2 ? 1 : 0) < p.w_kh;
        dst_row = (int64_t)sp * p.part_rows + (row & 63);
      } else {
        const int m = mt * BM + row;
        valid = m < p.part_rows;
        dst_row = (int64_t)sp * p.part_rows + m;
      }
      const bool has_k = kb1 > kb0;
      const uint32_t tbase = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * p.BN;
      if (p.dbg & 8) {   // profiling knob: no epilogue work (results invalid)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) release_acc(tempty0, acc);
        if (warp == 2 && lane == 0) TRACE(4, lt);
        continue;
      }
      if (p.st_tma) {
        // box origin of this warp's 32 rows
        int c1 = 0, c2 = 0, c3 = 0;
        if (p.out_mode == OUT_NHWC) {
          const int q = (int)p.fd_pw.div((uint32_t)mt), q2 = (int)p.fd_ph.div((uint32_t)q);
          c1 = (mt - q * p.ptiles_w) * p.tw + w_off;
          c2 = (q - q2 * p.ptiles_h) * p.th + h_off;
          c3 = q2 * p.tn + n_off;
        } else {
          c1 = mt * BM + quarter * 32;
          c2 = p.out_mode == OUT_PARTIAL ? sp : 0;
        }
        // kh-paired wgrad: lane quarters 0-1 hold kh 2nt+1, quarters 2-3 kh 2nt, both for Cout 0..63;
        // kh-quad (Cout 32): lane quarter q holds kh = KH-1-q (q = KH.. unused), channel group nt
        const int pair_kh = (PMODE == MODE_WGRAD ? p.w_pair : 0) == 3 ? p.w_kh - 1 - quarter : 2 * nt + (quarter < 2 ? 1 : 0);
        const int colbase = (PMODE == MODE_WGRAD ? p.w_pair : 0) ? pair_kh * p.BN : nt * p.BN;
        if ((PMODE == MODE_WGRAD ? p.w_pair : 0)) c1 = (PMODE == MODE_WGRAD ? p.w_pair : 0) == 3 ? 0 : (quarter & 1) * 32;
        const uint32_t stg = stg_w;
        const int span = p.n_epi == 8 && !p.epi_alt ? p.BN >> 1 : p.BN;   // columns this warp stores
        const int cbeg = p.n_epi == 8 && !p.epi_alt && warp >= 6 ? span : 0;
        const bool rows_real = (PMODE == MODE_WGRAD ? p.w_pair : 0) ? (pair_kh >= 0 && pair_kh < p.w_kh) : quarter * 32 < p.st_rows;
        const int cend = rows_real ? cbeg + span : cbeg;   // short tile: nothing to store
        const bool one_chunk = span <= ek.st_ch;
        bool released = false;
        for (int c = cbeg; c < cend; c += ek.st_ch, ++stg_it) {
          if ((PMODE == MODE_WGRAD && p.w_halo) && (c & 63) >= p.w_cin) { --stg_it; continue; }   // zero-fill channels: nothing to store
          const uint32_t buf = stg + (stg_it & 1) * stg_half;
          // TMEM first: a single-chunk tile hands its accumulator back to the MMA warp before
          // waiting for the staging buffer
          uint32_t r[64];
          if (warp == 2 && lane == 0 && (p.dbg & 8192)) TRACE(6, lt);   // debug: before the TMEM load
          if (ek.st_ch == 64) { tmem_ld32(tbase + c, *reinterpret_cast<uint32_t(*)[32]>(r));
                               tmem_ld32(tbase + c + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32)); }
          else if (ek.st_ch == 32) tmem_ld32(tbase + c, *reinterpret_cast<uint32_t(*)[32]>(r));
          else tmem_ld16(tbase + c, r);
          tmem_wait();
          if (warp == 2 && lane == 0) TRACE(5, lt);
          if (one_chunk) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) release_acc(tempty0, acc);
            released = true;
          }
          if (lane == 0) bulk_wait_read1();        // the store that last used this buffer has read it
          __syncwarp();
          if (warp == 2 && lane == 0 && !(p.dbg & 8192)) TRACE(6, lt);
          if (ek.st_ch == 8) {   // 8 fp32 columns (32-byte rows): zero-padded 8-channel halo wgrad
            const uint32_t off0 = (uint32_t)lane * 32u, off1 = off0 + 16u;
            st_shared_v4(buf + (off0 ^ (((off0 >> 7) & ek.swz) << 4)), has_k ? r[0] : 0u, has_k ? r[1] : 0u,
                         has_k ? r[2] : 0u, has_k ? r[3] : 0u);
            st_shared_v4(buf + (off1 ^ (((off1 >> 7) & ek.swz) << 4)), has_k ? r[4] : 0u, has_k ? r[5] : 0u,
                         has_k ? r[6] : 0u, has_k ? r[7] : 0u);
          } else if (!(p.dbg & 4096)) {   // knob 4096: no staging (profiling, results invalid)
#pragma unroll
          for (int cc = 0; cc < 64; cc += 16)
            if (cc < ek.st_ch) stage16(ek, buf, lane, cc, nt * p.BN + c + cc, r + cc, has_k);
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            int c0 = ek.col_off + colbase + c;
            if ((PMODE == MODE_WGRAD && p.w_halo)) {   // halo wgrad tile: 64-column kw segments of the [kh][kw][cin] output row
              const int khh = (PMODE == MODE_WGRAD ? p.w_pair : 0) ? pair_kh : nt / p.w_groups;
              const int gg = (PMODE == MODE_WGRAD ? p.w_pair : 0) == 3 ? nt : (PMODE == MODE_WGRAD ? p.w_pair : 0) ? 0 : nt - (nt / p.w_groups) * p.w_groups;
              c0 = (khh * p.h_kw + (c >> 6)) * p.w_cin + gg * 64 + (c & 63);
            }
            if (p.dbg & 2048) {   // profiling knob: no output store (results invalid)
            } else if (ek.accum) tma_red_add_4d(&p.mapC, buf, c0, c1, c2, c3);
            else tma_store_4d(&p.mapC, buf, c0, c1, c2, c3);
            bulk_commit();
          }
          if (warp == 2 && lane == 0) TRACE(7, lt);
        }
        if (!released) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) release_acc(tempty0, acc);
        }
        if (warp == 2 && lane == 0) TRACE(4, lt);
        continue;
      }
      const int64_t rowoff = dst_row * p.ldc + p.col_off +
                             ((PMODE == MODE_WGRAD ? p.w_pair : 0) ? (2 * nt + (quarter < 2 ? 1 : 0)) * p.BN : nt * p.BN);
      int c = 0;
      for (; c + 32 <= p.BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tbase + c, r);
        tmem_wait();
        if (valid) {
          store16(p, rowoff + c, nt * p.BN + c, r, has_k);
          store16(p, rowoff + c + 16, nt * p.BN + c + 16, r + 16, has_k);
        }
      }
      if (c < p.BN) {
        uint32_t r[16];
        tmem_ld16(tbase + c, r);
        tmem_wait();
        if (valid) store16(p, rowoff + c, nt * p.BN + c, r, has_k);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) release_acc(tempty0, acc);
      if (warp == 2 && lane == 0) TRACE(4, lt);
    }
    if (p.st_tma && lane == 0) bulk_wait_all();
  }
  __syncwarp();
  tc_fence_before();
  if (PAIR) cluster_sync_all();   // the leader's MMAs into the peer's TMEM / smem are done
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tmem_cols));
  }
}
#undef PMODE

using GemmKernel = void (*)(const GemmParams);
GemmKernel kernel_for(int pair, int mode) {
  static const GemmKernel k[2][4] = {
      {umma_gemm_kernel<0, MODE_FWD>, umma_gemm_kernel<0, MODE_WGRAD>, umma_gemm_kernel<0, MODE_DENSE>,
       umma_gemm_kernel<0, MODE_HALO>},
      {umma_gemm_kernel<1, MODE_FWD>, umma_gemm_kernel<1, MODE_WGRAD>, umma_gemm_kernel<1, MODE_DENSE>,
       umma_gemm_kernel<1, MODE_HALO>}};
  return k[pair ? 1 : 0][mode & 3];
}

// ---------------------------------------------------------------------------------------
// Host side: tensor maps, descriptor templates, box tables, launch planning
// ---------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encoder() {
  if (g_encode) return CVB_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CVB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) { cvb_set_error("cuTensorMapEncodeTiled unavailable"); return CVB_ECUDA; }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return CVB_OK;
}

CUtensorMapSwizzle swz_of(int rowbytes) {
  return rowbytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : rowbytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
       : rowbytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
}

int encode(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
           const uint32_t* box, int rowbytes) {
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(rowbytes), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    cvb_set_error("cuTensorMapEncodeTiled failed (%d) rank=%d dims=%llu,%llu,%llu,%llu box=%u,%u,%u,%u", (int)r, rank,
                  (unsigned long long)dims[0], (unsigned long long)(rank > 1 ? dims[1] : 0),
                  (unsigned long long)(rank > 2 ? dims[2] : 0), (unsigned long long)(rank > 3 ? dims[3] : 0), box[0],
                  rank > 1 ? box[1] : 0, rank > 2 ? box[2] : 0, rank > 3 ? box[3] : 0);
    return CVB_EINVAL;
  }
  return CVB_OK;
}

// NHWC activation map (channel stride cstride, using channels [0, c)), box (cel, bw, bh, bn).
// parity (rh, rw) >= 0 builds the stride-2 view of rows rh::2 and cols rw::2.
int encode_nhwc(CUtensorMap* m, const void* base, int n, int h, int w, int c, int cstride, int cel, int bw, int bh,
                int bn, int rh = -1, int rw = -1) {
  const uint64_t es = 2;
  if (rh < 0) {
    uint64_t dims[4] = {(uint64_t)c, (uint64_t)w, (uint64_t)h, (uint64_t)n};
    uint64_t st[3] = {cstride * es, (uint64_t)w * cstride * es, (uint64_t)h * w * cstride * es};
    uint32_t box[4] = {(uint32_t)cel, (uint32_t)bw, (uint32_t)bh, (uint32_t)bn};
    return encode(m, base, 4, dims, st, box, cel * 2);
  }
  const char* b = reinterpret_cast<const char*>(base) + ((int64_t)rh * w + rw) * cstride * es;
  uint64_t w2 = (uint64_t)(w - rw + 1) / 2, h2 = (uint64_t)(h - rh + 1) / 2;
  if (w2 == 0) w2 = 1;
  if (h2 == 0) h2 = 1;
  uint64_t dims[4] = {(uint64_t)c, w2, h2, (uint64_t)n};
  uint64_t st[3] = {2 * cstride * es, 2 * (uint64_t)w * cstride * es, (uint64_t)h * w * cstride * es};
  uint32_t box[4] = {(uint32_t)cel, (uint32_t)bw, (uint32_t)bh, (uint32_t)bn};
  return encode(m, b, 4, dims, st, box, cel * 2);
}

// 2-D row-major [rows][cols] (ld elements per row), box (cel, brows)
int encode_2d(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld, int cel, int brows) {
  uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  uint64_t st[1] = {(uint64_t)ld * 2};
  uint32_t box[2] = {(uint32_t)cel, (uint32_t)brows};
  return encode(m, base, 2, dims, st, box, cel * 2);
}

int pick_cel(int c) {
  if (c % 64 == 0) return 64;
  if (c % 32 == 0) return 32;
  if (c % 16 == 0) return 16;
  if (c % 8 == 0) return 8;
  return 0;
}

uint32_t make_idesc(int a_major, int b_major, int bn, int m = BM) {
  uint32_t d = 0;
  d |= 1u << 4;                    // D = f32
  d |= 1u << 7;                    // A = bf16
  d |= 1u << 10;                   // B = bf16
  d |= (uint32_t)a_major << 15;
  d |= (uint32_t)b_major << 16;
  d |= (uint32_t)(bn >> 3) << 17;
  d |= (uint32_t)(m >> 4) << 24;
  return d;
}

// UMMA shared-memory descriptor (sm_100: version 1 at bits 46-47); start address relative.
uint64_t desc_tmpl(uint32_t rel_addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((rel_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
uint32_t layout_of(int rowbytes) { return rowbytes == 128 ? 2u : rowbytes == 64 ? 4u : rowbytes == 32 ? 6u : 0u; }

// Descriptor template of MMA k-step s (16 K elements) of one operand stage.
//   K-major : `rows` rows per box, boxes of cel K-elements at stride rows*R
//   MN-major: boxes of cel MN-elements x 64 K-rows at stride 64*R
uint64_t operand_desc(int major, int cel, int rows, int s, int krows = 64) {
  const int R = cel * 2;
  if (major == 0) {
    if (R == 16) return desc_tmpl(2 * s * rows * 16, rows * 16, 128, 0);
    const int kb = 32 * s;
    return desc_tmpl((kb / R) * rows * R + (kb % R), 16, 8 * R, layout_of(R));
  }
  if (R == 16) return desc_tmpl(s * 256, 128, krows * 16, 0);
  return desc_tmpl(s * 16 * R, krows * R, 8 * R, layout_of(R));
}

// TMA-store epilogue plan: output map + per-warp box (see GemmParams::st_tma).  Returns 0 and
// leaves st_tma = 0 when the tile geometry does not split into 32-row boxes (direct stores).
int plan_tma_store(GemmParams& p) {
  p.st_tma = 0;
  static int off = -1;
  if (off < 0) off = getenv("CVB_NO_TMA_STORE") ? 1 : 0;
  if (off) return CVB_OK;
  const int es = p.out_f32 ? 4 : 2;
  const int maxch = 128 / es;
  const int span = p.n_epi == 8 && !p.epi_alt ? p.BN / 2 : p.BN;   // columns per epilogue warp
  int ch = maxch;
  while (ch > 8 && span % ch) ch >>= 1;
  if (p.mode == MODE_WGRAD && p.w_halo && p.w_cin < ch) ch = p.w_cin;   // padded rows: store the real channels only
  if (span % ch || ch * es < 32) return CVB_OK;
  int bw = 32, bh = 1, bn = 1;
  uint64_t dims[4], st[3];
  const uint64_t ld = (uint64_t)p.ldc * es;
  if (((uintptr_t)p.out & 15) || (ld & 15)) return CVB_OK;
  if (p.out_mode == OUT_NHWC) {
    const int tile_rows = p.tw * p.th * p.tn;
    if (tile_rows > BM || tile_rows % 32) return CVB_OK;
    if (p.tw >= 32) {
      if (p.tw % 32) return CVB_OK;
      bw = 32;
    } else {
      if (32 % p.tw) return CVB_OK;
      bw = p.tw;
      const int hr = 32 / p.tw;
      if (p.th >= hr) {
        if (p.th % hr) return CVB_OK;
        bh = hr;
      } else {
        if (hr % p.th) return CVB_OK;
        bh = p.th;
        bn = hr / p.th;
      }
    }
    dims[0] = (uint64_t)(p.col_off + p.N); dims[1] = p.OW; dims[2] = p.OH; dims[3] = p.NIMG;
    st[0] = ld; st[1] = ld * p.OW; st[2] = ld * p.OW * p.OH;
    if (p.out_par == 1) {   // rows out_ph::2, cols out_pw::2 of the full image
      st[0] = 2 * ld; st[1] = 2 * ld * p.out_W; st[2] = ld * p.out_W * p.out_H;
    } else if (p.out_par == 2) {   // rows out_ph::2 of the full image
      st[0] = ld; st[1] = 2 * ld * p.out_W; st[2] = ld * p.out_W * p.out_H;
    }
  } else if (p.out_mode == OUT_ROWS) {
    dims[0] = (uint64_t)(p.col_off + p.N); dims[1] = (uint64_t)p.M; dims[2] = 1; dims[3] = 1;
    st[0] = ld; st[1] = ld * p.M; st[2] = ld * p.M;
  } else {
    dims[0] = (uint64_t)p.N; dims[1] = (uint64_t)p.part_rows; dims[2] = (uint64_t)p.splits; dims[3] = 1;
    st[0] = ld; st[1] = ld * p.part_rows; st[2] = ld * p.part_rows * p.splits;
  }
  uint32_t box[4] = {(uint32_t)ch, (uint32_t)bw, (uint32_t)bh, (uint32_t)bn};
  uint32_t ones[4] = {1, 1, 1, 1};
  const int rowbytes = ch * es;
  void* base = p.out;
  if (p.out_mode == OUT_NHWC && p.out_par)
    base = (char*)p.out + ((int64_t)p.out_ph * p.out_W + (p.out_par == 1 ? p.out_pw : 0)) * (int64_t)ld;
  CUresult r = g_encode(&p.mapC, p.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                        base, dims, st, box, ones, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(rowbytes),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return CVB_OK;   // geometry the encoder rejects: direct stores
  p.st_tma = 1;
  p.st_rows = p.out_mode == OUT_NHWC ? p.tw * p.th * p.tn : BM;
  p.st_ch = ch;
  p.st_swz = rowbytes == 128 ? 7u : rowbytes == 64 ? 3u : 1u;
  p.st_bw = bw; p.st_bh = bh; p.st_bn = bn;
  return CVB_OK;
}

int g_num_sms = 0;
unsigned long long g_attr_done = 0;   // one bit per device
long long* g_trace = nullptr;

int launch(GemmParams& p, cudaStream_t stream) {
  g_num_sms = cvb_num_sms();   // cached per device
  if (!p.kr) p.kr = BK;
  p.ksteps = p.kr / 16;
  if (!p.a_stage_bytes) p.a_stage_bytes = BM * p.kr * 2;
  // CTA pair for gathered convs / dgrads with streamed weights: the two SMs of a TPC share
  // one 256 x BN MMA, each loading its own 128-row A tile and HALF of the weight tile (the L2
  // traffic per tile drops from A + B to A + B/2 and the B smem reads halve)
  static int env_pair = -1;
  if (env_pair < 0) { const char* e = getenv("CVB_GEMM_PAIR"); env_pair = e ? atoi(e) : 1; }
  // HALO convs (resident weights, each CTA keeps half the weight rows): correct but measured
  // slower (conv 64->64 @32x32, batch 512: 49.9 -> 69.3 us; 32->32: 25.8 -> 38.7 us, it also
  // displaces the two-CTA-per-SM plan) -- opt-in only (CVB_GEMM_PAIR_HALO=1)
  static int env_pair_halo = -1;
  if (env_pair_halo < 0) { const char* e = getenv("CVB_GEMM_PAIR_HALO"); env_pair_halo = e ? atoi(e) : 0; }
  const bool pair_fwd = p.mode == MODE_FWD && !p.b_res && p.b_cel == 64 && p.gb == 1 && p.b_major == 0 && p.kr == BK;
  const bool pair_halo = (env_pair_halo && p.mode == MODE_HALO && p.b_res && p.b_cel == 64 && p.gb == 1) ||
                         (p.hs && p.BN % 32 == 0);
  // weight gradients with Cout a multiple of 256: the pair shares the input (B) boxes
  static int env_pair_wg = -1;
  if (env_pair_wg < 0) { const char* e = getenv("CVB_GEMM_PAIR_WGRAD"); env_pair_wg = e ? atoi(e) : 1; }
  const bool pair_wgrad = env_pair_wg && p.mode == MODE_WGRAD && !p.w_halo && !p.w_pair && p.M % 256 == 0 &&
                          p.gb % 2 == 0 && p.a_major == 1 && p.b_major == 1;
  if (env_pair && pair_wgrad && p.m_tiles % 2 == 0 && g_num_sms % 2 == 0 && p.BN % 32 == 0) {
    p.pair = 1;
    p.b_stage_bytes = (uint32_t)(p.BN / 2) * p.kr * 2;
    p.tx_bytes -= (uint32_t)(p.gb / 2) * p.kr * p.b_cel * 2;   // this CTA's half of the input boxes
  } else
  p.pair = (env_pair && (pair_fwd || pair_halo) && p.b_ptr && p.m_tiles % 2 == 0 && p.BN % 32 == 0 &&
            p.splits == 1 && g_num_sms % 2 == 0) ? 1 : 0;
  if (p.pair && p.mode != MODE_WGRAD) {
    int rc = encode_2d(&p.mapB[0], p.b_ptr, p.b_rows, p.b_cols, p.b_ld, p.b_cel, p.BN / 2);
    if (rc) return rc;
    if (p.hs) {
      p.b_tap_bytes /= 2;   // this CTA's half of every tap's weight box
    } else if (p.b_res) {
      p.b_res_bytes /= 2;   // this CTA's half of every weight slab
    } else {
      p.b_stage_bytes = (uint32_t)(p.BN / 2) * p.kr * 2;
      p.tx_bytes -= (uint32_t)(p.BN / 2) * p.b_cel * 2;   // this CTA's half of the weight box
    }
  }
  const uint32_t stage_bytes = p.a_stage_bytes + ((p.b_res || p.hs) ? 0u : (p.b_stage_bytes ? p.b_stage_bytes
                                                                                   : (uint32_t)p.BN * p.kr * 2));
  static int env_epi4 = -1;
  if (env_epi4 < 0) env_epi4 = getenv("CVB_EPI4") ? 1 : 0;
  // narrow tiles: two epilogue warps per TMEM lane quarter (each stores half the columns) so
  // the per-tile epilogue latency (TMEM load, staging, store issue) overlaps across warps
  static int env_alt = -1, env_nacc = -1;
  if (env_alt < 0) {
    const char* e = getenv("CVB_EPI_ALT");
    env_alt = e ? atoi(e) : 1;
    e = getenv("CVB_NACC");
    env_nacc = e ? atoi(e) : 4;
  }
  // two CTAs per SM for narrow HALO convs whose resident weights + 2 stages fit in half the
  // shared memory: two independent MMA issue streams share the SM's tensor core
  static int env_2cta = -1;
  if (env_2cta < 0) { const char* e = getenv("CVB_GEMM_2CTA"); env_2cta = e ? atoi(e) : 1; }   // measured +3% step
  const uint32_t half = 112u * 1024u;
  const bool two = env_2cta && !p.pair && p.mode == MODE_HALO && p.BN <= 32 &&
                   2 * stage_bytes + p.b_res_bytes + 16u * 1024u + 1280u <= half;
  // wide tiles with few K-blocks are epilogue-bound: two warps per TMEM lane quarter, each
  // draining half the columns (tiles of <= CVB_EPI8_MAXKB K-blocks, default 4: DenseNet +1.5%,
  // ResNet-18 neutral, same-box)
  static int env_epi8kb = -1;
  if (env_epi8kb < 0) { const char* e = getenv("CVB_EPI8_MAXKB"); env_epi8kb = e ? atoi(e) : 4; }
  const bool wide8 = env_epi8kb > 0 && p.mode != MODE_WGRAD && p.BN > 64 && p.BN % 64 == 0 &&
                     p.kb_per_split <= env_epi8kb;
  p.n_epi = (!env_epi4 && !two && ((p.BN <= 64 && p.BN % 32 == 0) || wide8)) ? 8 : 4;
  // narrow tiles: more TMEM accumulators (the epilogue of tile i no longer gates the MMAs of
  // tile i+2) and alternate-tile epilogue warp groups (two tiles drain concurrently)
  p.nacc_log2 = (env_nacc >= 4 && 4 * p.BN <= 512) ? 2 : 1;
  p.epi_alt = (p.n_epi == 8 && env_alt && p.nacc_log2 == 2 && !p.no_epi_alt) ? 1 : 0;
  plan_tma_store(p);
  if (!p.st_tma && p.n_epi == 8) { p.n_epi = 4; p.epi_alt = 0; plan_tma_store(p); }
  if (!p.st_tma) { p.n_epi = 4; p.epi_alt = 0; }
  p.stg_warp = p.st_tma ? 2u * 32u * (uint32_t)p.st_ch * (p.out_f32 ? 4u : 2u) : 0u;
  const uint32_t stg_bytes = p.st_tma ? (uint32_t)p.n_epi * p.stg_warp : 0u;
  if (p.st_tma && 2 * stage_bytes + p.b_res_bytes + stg_bytes > 224u * 1024u) {   // keep 2 stages: direct stores
    p.st_tma = 0;
    p.n_epi = 4;      // the direct-store epilogue is one warp per TMEM lane quarter, all columns
    p.epi_alt = 0;
    p.stg_warp = 0;
  }
  if (p.out_par && !p.st_tma) { cvb_set_error("parity output needs the TMA-store epilogue"); return CVB_EINVAL; }
  if ((p.w_groups > 1 || p.w_pair == 3 || (p.w_halo && p.w_cin < 64)) && !p.st_tma) { cvb_set_error("grouped halo wgrad needs the TMA-store epilogue"); return CVB_EINVAL; }
  const uint32_t stg = p.st_tma ? stg_bytes : 0u;
  if (p.hs) {   // two halo stages; the weight-tap ring takes the rest (<= 16 slots)
    p.stages_b = (int)((224u * 1024u - 2u * stage_bytes - stg) / p.b_tap_bytes);
    if (p.stages_b > 16) p.stages_b = 16;
    if (p.stages_b < 2) { cvb_set_error("halo stream: no room for the weight ring"); return CVB_EINVAL; }
    p.b_res_bytes = (uint32_t)p.stages_b * p.b_tap_bytes;
  }
  p.stages = (int)(((two ? half - 1280u : 224u * 1024u) - p.b_res_bytes - stg) / stage_bytes);
  if (p.stages > 8) p.stages = 8;
  if (p.hs) p.stages = 2;
  p.two_cta = two && p.stages >= 2 ? 1 : 0;
  if (two && !p.two_cta) p.stages = (int)((224u * 1024u - p.b_res_bytes - stg) / stage_bytes);
  static int env_stages = -1, env_dbg = -1;
  if (env_stages < 0) {
    const char* e = getenv("CVB_STAGES");
    env_stages = e ? atoi(e) : 0;
    const char* d = getenv("CVB_GEMM_DBG");
    env_dbg = d ? atoi(d) : 0;
  }
  if (env_stages > 0 && env_stages < p.stages) p.stages = env_stages;
  p.dbg = env_dbg;
  // Paired K-blocks halve the MMA warp's per-batch cost (conv 128->128 with the TMA loads
  // skipped: 57.6 -> 40.1 us), but with the loads on these convs sit at the L2 throughput cap
  // (~42 B/clk/SM: 576 KB of operands per 128x128 tile) and the pairing delays stage release:
  // measured +2.7% on the ResNet-18 GEMM class.  Opt-in (CVB_KB_PAIR=1) until operand reuse
  // lowers the L2 demand.
  // With the CTA pair (half the L2 demand) pairing is the default; CVB_KB_PAIR=0/1 forces it.
  static int pair_on = -1;
  if (pair_on < 0) { const char* e = getenv("CVB_KB_PAIR"); pair_on = e ? atoi(e) : 2; }
  const bool want_kb_pair = pair_on == 1 || (pair_on == 2 && p.pair);
  p.kb_pair = (want_kb_pair && p.mode != MODE_HALO && p.ksteps == 4 && !p.b_res && p.stages >= 4 && !(env_dbg & 1)) ? 1 : 0;
  p.trace = nullptr;
  if (env_dbg & 4) {
    static long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, 8 * 4096 * sizeof(long long));
    cudaMemsetAsync(tr, 0, 8 * 4096 * sizeof(long long), stream);
    p.trace = tr;
    g_trace = tr;
  }
  if (p.stages < 2) { cvb_set_error("BN too large"); return CVB_EINVAL; }
  p.stg_off = (uint32_t)p.stages * stage_bytes + p.b_res_bytes;   // 1024-aligned (stages, slabs are)
  size_t smem = (size_t)p.stages * stage_bytes + p.b_res_bytes + stg + 1024 + 512;   // barriers: 64 words
  if (cvb_first_on_device(&g_attr_done)) {
    for (int m = 0; m < 4; m++)
      for (int pr = 0; pr < 2; pr++)
        CVB_CUDA(cudaFuncSetAttribute(kernel_for(pr, m), cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  }
  p.idesc = make_idesc(p.a_major, p.b_major, p.BN, p.pair ? 2 * BM : BM);
  // smem box strides and descriptor templates
  p.a_box_stride = p.a_major == 0 ? BM * p.a_cel * 2 : p.kr * p.a_cel * 2;
  p.b_box_stride = p.b_major == 0 ? p.BN * p.b_cel * 2 : p.kr * p.b_cel * 2;
  for (int k = 0; k < p.ksteps; k++) {
    p.adesc[k] = operand_desc(p.a_major, p.a_cel, BM, k, p.kr);
    p.bdesc[k] = operand_desc(p.b_major, p.b_cel, p.BN, k, p.kr);
  }
  if (p.mode == MODE_HALO && !p.h_rows)   // no-swizzle K-major: LBO = next 8-channel plane, SBO = one halo row
    p.adesc[0] = desc_tmpl(0, p.h_plane_stride, (uint32_t)p.h_pitch * 16, 0);
  if (p.mode == MODE_WGRAD && p.w_halo) {
    // B = the (tw+KW-1)-wide halo box, MN-major, rows of R = cin*2 bytes (one pixel each).
    // k-step s = pixels [16s, 16s+16) of the tw x th box -> halo row (16s/tw)*(tw+KW-1) + 16s%tw;
    // the kw taps are the MN atoms of one MMA: LBO = one row (the next kw shift), SBO = 8 rows.
    const uint32_t R = (uint32_t)p.b_cel * 2, pitch = (uint32_t)(p.tw + p.h_kw - 1);
    for (int k = 0; k < p.ksteps; k++) {
      const uint32_t row = (uint32_t)(16 * k / p.tw) * pitch + (uint32_t)(16 * k % p.tw);
      p.bdesc[k] = desc_tmpl(row * R, R, 8 * R, layout_of((int)R));
      // kh pairs: A = one (bh+1)-row dY box; M atom 0 (kh 2t+1) starts at box row 0, atom 1
      // (kh 2t) one dY row later: LBO = one box row of pixels
      if (p.w_pair == 1) p.adesc[k] = desc_tmpl((uint32_t)(16 * k) * 128u, (uint32_t)p.tw * 128u, 8u * 128u, 2u);
      // kh-quad: 32-channel (64-byte, SW64) dY rows; M atom q = the box one pixel row further down
      if (p.w_pair == 3) p.adesc[k] = desc_tmpl((uint32_t)(16 * k) * 64u, (uint32_t)p.tw * 64u, 8u * 64u, 4u);
    }
  }
  if (p.mode == MODE_HALO && p.h_rows && p.h_kwbox)   // kw boxes: plain SW128 K-major, 8-row groups 1 KB apart
    p.adesc[0] = desc_tmpl(0, 16, 1024, 2u);
  else if (p.mode == MODE_HALO && p.h_rows)   // SW128/SW64 K-major rows: SBO = one halo row of 8-pixel groups
    p.adesc[0] = desc_tmpl(0, 16, (uint32_t)p.h_pitch * (p.h_rowpad ? 128 : p.h_cg * 2),
                           layout_of(p.h_rowpad ? 128 : p.h_cg * 2));
  if (p.mode == MODE_HALO && p.h_cg == 8) {   // tap pairs: second K half = next pixel / next row
    p.adesc[0] = desc_tmpl(0, 16, (uint32_t)p.h_pitch * 16, 0);
    p.adesc[1] = desc_tmpl(0, (uint32_t)(p.h_pitch - p.h_kw + 1) * 16, (uint32_t)p.h_pitch * 16, 0);
  }
  const int mtu = p.pair ? p.m_tiles / 2 : p.m_tiles;   // M scheduling units (tile pairs)
  const int units = mtu * p.n_tiles * p.splits;
  const int slots = p.pair ? g_num_sms / 2 : g_num_sms * (p.two_cta ? 2 : 1);
  const int grid = (units < slots ? units : slots) * (p.pair ? 2 : 1);
  p.fd_m = make_fastdiv((uint32_t)mtu);
  p.fd_n = make_fastdiv((uint32_t)p.n_tiles);
  p.fd_mn = make_fastdiv((uint32_t)(mtu * p.n_tiles));
  p.fd_pw = make_fastdiv((uint32_t)(p.ptiles_w > 0 ? p.ptiles_w : 1));
  p.fd_ph = make_fastdiv((uint32_t)(p.ptiles_h > 0 ? p.ptiles_h : 1));
  if (p.pair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3((2 + p.n_epi) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cvb_pdl_enabled() ? 2 : 1;
    cudaLaunchKernelEx(&cfg, kernel_for(1, p.mode), p);
  } else {
    cvb_launch(kernel_for(0, p.mode), grid, (2 + p.n_epi) * 32, smem, stream, p);
  }
  CVB_CHECK_LAUNCH();
  return CVB_OK;
}

int pick_bn(int n) {
  if (n <= 256) return (n + 15) / 16 * 16;
  int tiles = (n + 255) / 256;
  return ((n + tiles - 1) / tiles + 15) / 16 * 16;
}

// pixel box for an M tile of 128 output rows
void pick_mbox(int n, int oh, int ow, int& bw, int& bh, int& bn) {
  if (ow >= BM) { bw = BM; bh = 1; bn = 1; return; }
  bw = ow;
  int hmax = BM / ow;
  if (hmax >= oh) {
    bh = oh;
    bn = BM / (ow * oh);
    if (bn > n) bn = n;
    return;
  }
  int ht = (oh + hmax - 1) / hmax;
  bh = (oh + ht - 1) / ht;
  bn = 1;
}

int next_pow2(int x) { int q = 1; while (q < x) q <<= 1; return q; }

// pixel box for a 64-pixel K chunk (wgrad): exact 64 rows, OOB rows zero-filled by TMA
void pick_kbox(int oh, int ow, int rows, int& bw, int& bh, int& bn) {
  bw = next_pow2(ow) < rows ? next_pow2(ow) : rows;
  if (bw > 256) bw = 256;
  bh = rows / bw < next_pow2(oh) ? rows / bw : next_pow2(oh);
  bn = rows / (bw * bh);
}

// gathered-operand box: tap -> (parity map, dw, dh) for the conv geometry
uint32_t gather_entry(int k_elem, int cin, int ntaps, int KW, int pad, int stride) {
  const int tap = k_elem / cin, ci = k_elem - tap * cin;
  if (tap >= ntaps) return pack_box(0, cin, 0, 0);   // fully out of bounds -> zeros
  const int kh = tap / KW, kw = tap - kh * KW;
  const int dh = kh - pad, dw = kw - pad;
  if (stride == 1) return pack_box(0, ci, dw, dh);
  const int mi = ((dh & 1) << 1) | (dw & 1);
  return pack_box(mi, ci, dw >> 1, dh >> 1);
}

}  // namespace

// ---------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------

// Convolution forward as implicit GEMM (also serves dgrad):
//   y[n,oh,ow, yoff+co] = bias[co] + sum_{kh,kw,ci} x[n, oh*s-pad+kh, ow*s-pad+kw, ci] * w[co][kh][kw][ci]
// x: NHWC bf16 (channel stride xcs, channels [0,cin)), cin multiple of 8.
// w: bf16 [cout][kh*kw*cin] (K-major).  y: NHWC (bf16, or fp32 if y_f32) with channel stride ycs.
// Halo conv with streamed weights (see cvb_conv2d_fwd): stride 1, any KH x KW <= 3 x 3 with
// top/left padding pad (bottom/right overflow is TMA zero fill), 8 x 16 pixel tiles, the kw-box
// halo of one 64-channel group per K-block, one weight-tap box per ring slot.
static bool hs_fits(int n, int oh, int ow, int cin, int xcs, int cout) {
  return cin % 64 == 0 && cin >= 128 && cout % 32 == 0 && cout <= 256 && ow % 8 == 0 && oh % 16 == 0 && xcs % 8 == 0 &&
         n > 0;
}
static int plan_hs(GemmParams& p, const void* x, int n, int h, int w, int cin, int xcs, const void* wt, int cout, int kh, int kw,
            int pad, void* y, int oh, int ow, int ycs, int yoff, const float* bias, int y_f32, int accumulate) {
  memset(&p, 0, sizeof(p));
  const int Kh = kh * kw * cin, BNh = pick_bn(cout), hrows = 16 + kh - 1;
  p.mode = MODE_HALO;
  p.hs = 1;
  p.a_major = 0; p.b_major = 0;
  p.a_cel = 8; p.b_cel = 64;
  p.gb = 1;
  p.BN = BNh;
  p.M = n * oh * ow; p.N = cout;
  p.tw = 8; p.th = 16; p.tn = 1;
  p.ptiles_w = ow / 8; p.ptiles_h = oh / 16;
  p.m_tiles = p.ptiles_w * p.ptiles_h * n;
  p.n_tiles = 1; p.splits = 1;
  p.h_cin = cin; p.h_cg = 64; p.h_pad = pad; p.h_kh = kh; p.h_kw = kw;
  p.h_rows = 1; p.h_kwbox = 1; p.h_planes = kw; p.h_pitch = 8;
  p.h_box_bytes = 8u * (uint32_t)hrows * 128u;
  p.h_plane_stride = (p.h_box_bytes + 1023) / 1024 * 1024;
  p.a_stage_bytes = (uint32_t)kw * p.h_plane_stride;
  p.num_kb = cin / 64; p.kb_per_split = p.num_kb;
  p.OH = oh; p.OW = ow; p.NIMG = n;
  p.b_res = 0; p.b_res_bytes = 0;
  p.tx_bytes = (uint32_t)kw * p.h_box_bytes;
  p.b_tap_bytes = (uint32_t)BNh * 128u;   // launch(): halved for the CTA pair
  int rc;
  if ((rc = encode_nhwc(&p.mapA[0], x, n, h, w, cin, xcs, 64, 8, hrows, 1))) return rc;
  if ((rc = encode_2d(&p.mapB[0], wt, cout, Kh, Kh, 64, BNh))) return rc;
  p.b_ptr = wt; p.b_rows = cout; p.b_cols = Kh; p.b_ld = Kh;
  p.out_mode = OUT_NHWC; p.out_f32 = y_f32; p.out = y; p.ldc = ycs; p.col_off = yoff; p.bias = bias;
  p.accum = accumulate;
  return CVB_OK;
}

CVB_API int cvb_conv2d_fwd(const void* x, int n, int h, int w, int cin, int xcs, const void* wt, int cout, int kh,
                           int kw, int stride, int pad, void* y, int oh, int ow, int ycs, int yoff, const float* bias,
                           int y_f32, int accumulate, void* stream) {
  if (get_encoder()) return CVB_ECUDA;
  const int acel = pick_cel(cin);
  if (!acel || (stride != 1 && stride != 2) || cout % 8) { cvb_set_error("conv2d_fwd: unsupported shape"); return CVB_EINVAL; }
  static GemmParams p;   // large (boxes table): keep off the stack
  memset(&p, 0, sizeof(p));
  {
    // ---- 1x1 stride-1 convs: a plain GEMM over the pixel rows [n*h*w][cin] (stride xcs) --
    // 128-row tiles, no spatial boxes, TMA-stored rows at channel offset yoff.  The halo and
    // gathered plans tile the image in 8x16 / w x (128 / w) boxes: DenseNet's 56- and 28-wide
    // maps lost rows to partial boxes and stored 112-row tiles with per-thread stores
    // (measured 1x1 256->128 at 56x56, batch 128: halo 83.6, gathered 56.5 us).
    static int no_dense1 = -1;
    if (no_dense1 < 0) no_dense1 = getenv("CVB_NO_DENSE_1X1") ? 1 : 0;
    if (!no_dense1 && kh == 1 && kw == 1 && stride == 1 && pad == 0 && oh == h && ow == w && cin % 8 == 0 &&
        xcs % 8 == 0 && ycs % 8 == 0) {
      p.mode = MODE_DENSE;
      p.a_major = 0; p.b_major = 0;
      p.a_cel = pick_cel(cin) < 64 ? pick_cel(cin) : 64;
      p.b_cel = p.a_cel;
      p.BN = pick_bn(cout);
      p.ga = BK / p.a_cel;
      p.gb = BK / p.b_cel;
      const int M = n * h * w;
      p.M = M; p.N = cout;
      p.m_tiles = (M + BM - 1) / BM;
      p.n_tiles = (cout + p.BN - 1) / p.BN;
      p.num_kb = (cin + BK - 1) / BK;
      p.kb_per_split = p.num_kb;
      p.splits = 1;
      p.tw = 1; p.th = 1; p.tn = 1; p.ptiles_w = 1; p.ptiles_h = 1;
      int rc;
      if ((rc = encode_2d(&p.mapA[0], x, M, cin, xcs, p.a_cel, BM))) return rc;
      if ((rc = encode_2d(&p.mapB[0], wt, cout, cin, cin, p.b_cel, p.BN))) return rc;
      p.tx_bytes = p.ga * BM * p.a_cel * 2 + p.gb * p.BN * p.b_cel * 2;
      p.out_mode = OUT_ROWS; p.out_f32 = y_f32; p.out = y; p.ldc = ycs; p.col_off = yoff; p.bias = bias;
      p.accum = accumulate;
      return launch(p, (cudaStream_t)stream);
    }
  }
  {
    // ---- halo path: stride 1, 16-channel multiples, resident weights ----
    static int no_halo = -1;
    if (no_halo < 0) no_halo = getenv("CVB_NO_HALO") ? 1 : 0;
    const int K = kh * kw * cin;
    const int BN = pick_bn(cout);
    const uint32_t b_all = (uint32_t)((K + BK - 1) / BK) * BN * BK * 2;
    int cg = cin % 64 == 0 ? 64 : cin % 32 == 0 ? 32 : cin % 16 == 0 ? 16 : 0;
    if (cin == 8 && kh == 3 && kw == 3) cg = 8;   // stem: tap-pair MMAs (halo8_issue)
    if (!no_halo && stride == 1 && cg && cout <= 256 && b_all <= 96u * 1024u && kh <= 7 && kw <= 7) {
      p.mode = MODE_HALO;
      p.a_major = 0; p.b_major = 0;
      p.a_cel = 8; p.b_cel = 64;
      p.gb = 1;
      p.BN = BN;
      p.M = n * oh * ow; p.N = cout;
      p.tw = 8; p.th = 16; p.tn = 1;
      p.ptiles_w = (ow + 7) / 8;
      p.ptiles_h = (oh + 15) / 16;
      p.m_tiles = p.ptiles_w * p.ptiles_h * n;
      p.n_tiles = 1;
      p.splits = 1;
      p.h_cin = cin; p.h_cg = cg; p.h_planes = cg >= 8 ? cg / 8 : 1; p.h_pad = pad; p.h_kh = kh; p.h_kw = kw;
      p.h_pitch = 8 + kw - 1 + (cg == 8 ? 1 : 0);   // tap pairs read one pixel past the last tap
      static int dbg_rows = -1;   // profiling knob CVB_HALO_DBG_ROWS: load only this many halo rows (results invalid)
      if (dbg_rows < 0) { const char* e = getenv("CVB_HALO_DBG_ROWS"); dbg_rows = e ? atoi(e) : 0; }
      const int hrows = dbg_rows > 0 ? dbg_rows : 16 + kh - 1;
      static int no_rows = -1;
      if (no_rows < 0) no_rows = getenv("CVB_NO_HALO_ROWS") ? 1 : 0;
      static int rows32 = -1;
      if (rows32 < 0) rows32 = getenv("CVB_NO_HALO_ROWS32") ? 0 : 1;   // SW64 rows for 32-channel groups
      p.h_rows = (!no_rows && (cg == 64 || (cg == 32 && rows32)) &&
                  ((kh == 3 && kw == 3) || (kh == 1 && kw == 1) || (kh == 4 && kw == 4))) ? 1 : 0;
      static int rowpad = -1;
      if (rowpad < 0) rowpad = getenv("CVB_NO_ROWPAD") ? 0 : 1;
      p.h_rowpad = (p.h_rows && rowpad && cg == 32 && cin == 32 &&
                    ((kh == 3 && kw == 3) || (kh == 4 && kw == 4))) ? 1 : 0;
      if (p.h_rows) p.h_planes = 1;
      const int rowb = p.h_rowpad ? 128 : cg * 2;   // smem bytes per halo pixel row
      p.h_box_bytes = (uint32_t)p.h_pitch * hrows * (p.h_rows ? rowb : 16);
      p.h_plane_stride = (p.h_box_bytes + 127) / 128 * 128;
      p.a_stage_bytes = (p.h_planes * p.h_plane_stride + 1023) / 1024 * 1024;
      // UMMA reads a SW128 operand whose 8-row groups are 1280 B apart (the 10-pixel halo
      // pitch) at ~99 cycles per MMA, 1024/2048 B apart at the 40-64-cycle floor
      // (scripts/mma_rate.py): pad the halo pitch to 16 pixels (SBO = 2 KB).
      static int pitch16 = -1;
      if (pitch16 < 0) pitch16 = getenv("CVB_NO_PITCH16") ? 0 : 1;
      if (pitch16 && p.h_rows && rowb == 128 && kw > 1 && kw <= 9) {
        p.h_pitch = 16;
        p.h_box_bytes = 16u * (uint32_t)hrows * 128u;
        p.h_plane_stride = (p.h_box_bytes + 127) / 128 * 128;
        p.a_stage_bytes = (p.h_plane_stride + 1023) / 1024 * 1024;
      }
      static int kwbox = -1;
      if (kwbox < 0) kwbox = getenv("CVB_NO_KWBOX") ? 0 : 1;
      // (64-channel groups only: for the zero-padded 32-channel rows the 3x box writes cost more
      // than the aligned starts save -- measured conv 32->32 28.8 -> 29.3 us)
      if (kwbox && p.h_rows && !p.h_rowpad && rowb == 128 && kh == 3 && kw == 3) {
        const uint32_t box = 8u * (uint32_t)hrows * 128u, stride = (box + 1023) / 1024 * 1024;
        const uint32_t a_stage = (uint32_t)kw * stride;
        if (2 * a_stage + b_all + 32u * 1024u <= 224u * 1024u) {
          p.h_kwbox = 1;
          p.h_pitch = 8;
          p.h_planes = kw;
          p.h_box_bytes = box;
          p.h_plane_stride = stride;
          p.a_stage_bytes = a_stage;
          p.no_epi_alt = 2 * a_stage + b_all + 64u * 1024u > 224u * 1024u;
        }
      }
      p.num_kb = cin / cg;
      p.kb_per_split = p.num_kb;
      p.OH = oh; p.OW = ow; p.NIMG = n;
      p.b_res = 1;
      p.b_res_bytes = b_all;
      p.b_slabs = (K + BK - 1) / BK;
      p.h_mps = kh * kw * (cg / 16);   // MMAs per K-block (offsets computed in the issue loop)
      p.tx_bytes = p.h_planes * p.h_box_bytes;
      int rc;
      if ((rc = encode_nhwc(&p.mapA[0], x, n, h, w, cin, xcs, p.h_rows ? rowb / 2 : 8, p.h_pitch, hrows, 1))) return rc;
      if ((rc = encode_2d(&p.mapB[0], wt, cout, K, K, p.b_cel, p.BN))) return rc;
      p.b_ptr = wt; p.b_rows = cout; p.b_cols = K; p.b_ld = K;
      p.out_mode = OUT_NHWC; p.out_f32 = y_f32; p.out = y; p.ldc = ycs; p.col_off = yoff; p.bias = bias;
      p.accum = accumulate;
      return launch(p, (cudaStream_t)stream);
    }
  }
  {
    // ---- halo with streamed weights: wide stride-1 3x3 convs whose weights do not stay
    // resident (128+ channels).  The gathered plan reads the 128-pixel A box once per TAP from
    // L2 (9x per channel group) and is bounded by the L2 -> SM rate (~34 B/clk/SM measured,
    // ResNet-18 stage 2); here the kw-box halo is read once per channel group and only the
    // weights stream per tap (A + B per tap 24 -> ~14 KB with the CTA pair).
    static int no_hs = -1;
    if (no_hs < 0) no_hs = getenv("CVB_NO_HALO_STREAM") ? 1 : 0;
    const int Kh = kh * kw * cin, BNh = pick_bn(cout);
    const uint32_t b_all_h = (uint32_t)((Kh + BK - 1) / BK) * BNh * BK * 2;
    if (!no_hs && stride == 1 && kh == 3 && kw == 3 && pad == 1 && b_all_h > 96u * 1024u &&
        hs_fits(n, oh, ow, cin, xcs, cout)) {
      int rc = plan_hs(p, x, n, h, w, cin, xcs, wt, cout, kh, kw, pad, y, oh, ow, ycs, yoff, bias, y_f32, accumulate);
      if (rc) return rc;
      return launch(p, (cudaStream_t)stream);
    }
  }
  p.mode = MODE_FWD;
  p.a_major = 0; p.b_major = 0;
  p.a_cel = acel;
  const int K = kh * kw * cin;
  p.b_cel = 64;   // weights [cout][K]: 128-byte rows, K tail zero-filled by TMA
  p.ga = BK / p.a_cel;
  p.gb = BK / p.b_cel;
  p.BN = pick_bn(cout);
  p.M = n * oh * ow;
  p.N = cout;
  int bw, bh, bnn;
  pick_mbox(n, oh, ow, bw, bh, bnn);
  p.tw = bw; p.th = bh; p.tn = bnn;
  p.ptiles_w = (ow + bw - 1) / bw;
  p.ptiles_h = (oh + bh - 1) / bh;
  const int ptiles_n = (n + bnn - 1) / bnn;
  p.m_tiles = p.ptiles_w * p.ptiles_h * ptiles_n;
  p.n_tiles = (cout + p.BN - 1) / p.BN;
  p.splits = 1;
  p.num_kb = (K + BK - 1) / BK;
  p.kb_per_split = p.num_kb;
  p.OH = oh; p.OW = ow; p.NIMG = n;
  p.nbox = p.num_kb * p.ga;
  if (p.nbox > MAX_BOXES) { cvb_set_error("conv2d_fwd: K too large for the box table"); return CVB_EINVAL; }
  for (int i = 0; i < p.nbox; i++) p.boxtab[i] = gather_entry((i / p.ga) * BK + (i % p.ga) * acel, cin, kh * kw, kw, pad, stride);
  // small weight operands stay resident in smem for the CTA's whole tile loop
  const uint32_t b_all = (uint32_t)p.num_kb * p.BN * BK * 2;
  p.b_res = (p.n_tiles == 1 && b_all <= 96u * 1024u) ? 1 : 0;
  p.b_res_bytes = p.b_res ? b_all : 0;
  p.b_slabs = p.num_kb;
  p.tx_bytes = p.ga * bw * bh * bnn * p.a_cel * 2 + (p.b_res ? 0 : p.gb * p.BN * p.b_cel * 2);
  int rc;
  if (stride == 1) {
    if ((rc = encode_nhwc(&p.mapA[0], x, n, h, w, cin, xcs, acel, bw, bh, bnn))) return rc;
  } else {
    for (int rh = 0; rh < 2; rh++)
      for (int rw = 0; rw < 2; rw++)
        if ((rc = encode_nhwc(&p.mapA[rh * 2 + rw], x, n, h, w, cin, xcs, acel, bw, bh, bnn, rh, rw))) return rc;
  }
  if ((rc = encode_2d(&p.mapB[0], wt, cout, K, K, p.b_cel, p.BN))) return rc;
  p.b_ptr = wt; p.b_rows = cout; p.b_cols = K; p.b_ld = K;
  p.out_mode = OUT_NHWC; p.out_f32 = y_f32; p.out = y; p.ldc = ycs; p.col_off = yoff; p.bias = bias;
  p.accum = accumulate;
  return launch(p, (cudaStream_t)stream);
}

namespace {

// ---- stride-2 dgrad by output-parity classes ------------------------------------------
// dx[i] = sum_{o,k : 2o - pad + k = i} w[k] dy[o] (per spatial dim).  For output parity
// rho = i mod 2 only taps k == rho + pad (mod 2) contribute, with o = i/2 + (rho + pad - k)/2.
// So each of the 4 (rho_h, rho_w) classes is a stride-1 gather-conv of dY (no zero-upsampled
// copy, no multiplications by inserted zeros: 4x fewer MMAs than the upsampled form) with its
// own tap subset, written through a parity view of dx by the TMA-store epilogue.
struct ClassW {
  int ntaps[4];
  int64_t off[5];
  int kh[4][16], kw[4][16];
};

__global__ void dgrad_class_weights(const __nv_bfloat16* __restrict__ w, int cout, int KH, int KW, int cin, ClassW cw,
                                    __nv_bfloat16* __restrict__ out) {
  CVB_PDL_PROLOGUE();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cw.off[4]) return;
  int c = 0;
  while (i >= cw.off[c + 1]) c++;
  const int64_t local = i - cw.off[c];
  const int co = (int)(local % cout);
  const int64_t r = local / cout;
  const int nt = cw.ntaps[c];
  const int t = (int)(r % nt), ci = (int)(r / nt);
  out[i] = w[(((int64_t)co * KH + cw.kh[c][t]) * KW + cw.kw[c][t]) * cin + ci];
}

// One parity class: stride-1 gather conv of x (= dY) with explicit tap offsets (dh, dw),
// output through the parity view (ph, pw) of y [n][H][W][ycs].
int plan_gather_conv(GemmParams& p, const void* x, int n, int h, int w, int cin, int xcs, const void* wt, int cout,
                     int ntaps, const int* dh, const int* dw, void* y, int H, int W, int ycs, int ph, int pw,
                     int accumulate, int rows_only = 0) {
  const int acel = pick_cel(cin);
  if (!acel || cout % 8) { cvb_set_error("dgrad: unsupported channels"); return CVB_EINVAL; }
  memset(&p, 0, sizeof(p));
  const int oh = (H - ph + 1) / 2, ow = rows_only ? W : (W - pw + 1) / 2;
  p.mode = MODE_FWD;
  p.a_cel = acel;
  p.b_cel = 64;
  p.ga = BK / acel;
  p.gb = 1;
  p.BN = pick_bn(cout);
  p.M = n * oh * ow;
  p.N = cout;
  const int K = ntaps * cin;
  int bw, bh, bnn;
  pick_mbox(n, oh, ow, bw, bh, bnn);
  p.tw = bw; p.th = bh; p.tn = bnn;
  p.ptiles_w = (ow + bw - 1) / bw;
  p.ptiles_h = (oh + bh - 1) / bh;
  p.m_tiles = p.ptiles_w * p.ptiles_h * ((n + bnn - 1) / bnn);
  p.n_tiles = (cout + p.BN - 1) / p.BN;
  p.splits = 1;
  p.num_kb = (K + BK - 1) / BK;
  p.kb_per_split = p.num_kb;
  p.OH = oh; p.OW = ow; p.NIMG = n;
  p.nbox = p.num_kb * p.ga;
  if (p.nbox > MAX_BOXES) { cvb_set_error("dgrad: K too large for the box table"); return CVB_EINVAL; }
  for (int i = 0; i < p.nbox; i++) {
    const int k = (i / p.ga) * BK + (i % p.ga) * acel;
    const int tap = k / cin, ci = k - tap * cin;
    p.boxtab[i] = tap >= ntaps ? pack_box(0, cin, 0, 0) : pack_box(0, ci, dw[tap], dh[tap]);
  }
  const uint32_t b_all = (uint32_t)p.num_kb * p.BN * BK * 2;
  p.b_res = (p.n_tiles == 1 && b_all <= 96u * 1024u) ? 1 : 0;
  p.b_res_bytes = p.b_res ? b_all : 0;
  p.b_slabs = p.num_kb;
  p.tx_bytes = p.ga * bw * bh * bnn * acel * 2 + (p.b_res ? 0 : p.gb * p.BN * p.b_cel * 2);
  int rc;
  if ((rc = encode_nhwc(&p.mapA[0], x, n, h, w, cin, xcs, acel, bw, bh, bnn))) return rc;
  if ((rc = encode_2d(&p.mapB[0], wt, cout, K, K, p.b_cel, p.BN))) return rc;
  p.b_ptr = wt; p.b_rows = cout; p.b_cols = K; p.b_ld = K;
  p.out_mode = OUT_NHWC; p.out_f32 = 0; p.out = y; p.ldc = ycs; p.col_off = 0; p.bias = nullptr;
  p.accum = accumulate;
  p.out_par = rows_only ? 2 : 1; p.out_ph = ph; p.out_pw = pw; p.out_H = H; p.out_W = W;
  plan_tma_store(p);
  if (!p.st_tma) { cvb_set_error("dgrad: parity class geometry needs direct stores"); return CVB_EINVAL; }
  return CVB_OK;
}

}  // namespace

// dX of a stride-2 conv (w [cout][kh][kw][cin] bf16, pad) from dY [n][oh][ow][cout] (stride
// dycs): dx [n][h][w][cin] bf16 (stride dxcs), added into dx when accumulate.  wscratch holds
// cout*kh*kw*cin bf16 (the per-class weight matrices).  Returns CVB_EINVAL without launching
// anything when a class geometry is unsupported (the caller then uses the upsampled form).
// Classes without taps (e.g. odd positions of a 1x1 stride-2 conv) contribute nothing: the
// caller must accumulate (or have zeroed dx).
CVB_API int cvb_conv2d_dgrad_s2(const void* dy, int n, int oh, int ow, int cout, int dycs, const void* w, int cin,
                                int kh, int kw, int pad, void* dx, int h, int wd, int dxcs, int accumulate,
                                void* wscratch, void* stream) {
  if (get_encoder()) return CVB_ECUDA;
  static GemmParams plans[4];
  static int dh[4][16], dw[4][16];
  ClassW cw;
  memset(&cw, 0, sizeof(cw));
  int have = 0;
  for (int c = 0; c < 4; c++) {
    const int ph = c >> 1, pw = c & 1;
    int nt = 0;
    for (int y = 0; y < kh; y++)
      for (int x = 0; x < kw; x++)
        if (((y - ph - pad) & 1) == 0 && ((x - pw - pad) & 1) == 0) {
          if (nt >= 16) { cvb_set_error("dgrad_s2: kernel too large"); return CVB_EINVAL; }
          cw.kh[c][nt] = y; cw.kw[c][nt] = x;
          dh[c][nt] = (ph + pad - y) / 2; dw[c][nt] = (pw + pad - x) / 2;
          nt++;
        }
    cw.ntaps[c] = nt;
    cw.off[c + 1] = cw.off[c] + (int64_t)cin * nt * cout;
    if (!nt) continue;
    const void* wc = (const char*)wscratch + cw.off[c] * 2;
    int rc = plan_gather_conv(plans[c], dy, n, oh, ow, cout, dycs, wc, cin, nt, dh[c], dw[c], dx, h, wd, dxcs, ph, pw,
                              accumulate);
    if (rc) return rc;
    have |= 1 << c;
  }
  if (!accumulate && have != 15) { cvb_set_error("dgrad_s2: a parity class has no taps; accumulate into zeroed dx"); return CVB_EINVAL; }
  const int64_t total = cw.off[4];
  if (w) {   // w == NULL: wscratch already holds the class weights (cvb_transpose_batched jobs)
    cvb_launch(dgrad_class_weights, (unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream,
        (const __nv_bfloat16*)w, cout, kh, kw, cin, cw, (__nv_bfloat16*)wscratch);
    CVB_CHECK_LAUNCH();
  }
  for (int c = 0; c < 4; c++)
    if (have & (1 << c)) {
      int rc = launch(plans[c], (cudaStream_t)stream);
      if (rc) return rc;
    }
  return CVB_OK;
}

// dX of a 3x3 pad-1 stride-2 conv as TWO gather convs of dY, one per output ROW parity a, each
// producing both column parities at once: output "pixel" (i, j) of conv a holds the 2*cin
// channels (b, ci) = dx[2i + a][2j + b][ci] (adjacent in dx when dxcs == cin), so N = 2*cin
// and the four parity classes' 9 taps become 2 + 4 tap boxes of dY (dh-major, dw in {0, 1}):
//   conv 0: (dh, dw) = (0,0) (0,1);   conv 1: (0,0) (0,1) (1,0) (1,1)
// with weight rows (b, ci) of tap (dh, dw) = w[co][a + 1 - 2dh][b + 1 - 2dw][ci] (zero where that
// tap does not exist).  wrows = conv 0's [2cin][2][cout] then conv 1's [2cin][4][cout] bf16
// (written by cvb_transpose_batched jobs; the zero entries stay zero).  Against the four class
// convs (N = cin): half the dY box loads per output element and twice the MMA width.
CVB_API int cvb_conv2d_dgrad_s2_rows(const void* dy, int n, int oh, int ow, int cout, int dycs, int cin, void* dx,
                                     int h, int wd, int dxcs, int accumulate, const void* wrows, void* stream) {
  if (get_encoder()) return CVB_ECUDA;
  if (dxcs != cin || h != 2 * oh || wd != 2 * ow || cin % 8) {
    cvb_set_error("dgrad_s2_rows: needs dx [n][2oh][2ow][cin] contiguous");
    return CVB_EINVAL;
  }
  static GemmParams plans[2];
  static const int dh0[2] = {0, 0}, dw0[2] = {0, 1};
  static const int dh1[4] = {0, 0, 1, 1}, dw1[4] = {0, 1, 0, 1};
  const void* w1 = (const char*)wrows + (size_t)2 * cin * 2 * cout * 2;
  // dY maps of 16 x 16 and larger (ResNet-18 stage 2): the halo plan with streamed weights --
  // conv 0 is a 1 x 2 and conv 1 a 2 x 2 stride-1 conv of dY, no top/left padding (the
  // bottom/right overflow is TMA zero fill); the dY halo is read once per channel group
  static int no_hs = -1;
  if (no_hs < 0) no_hs = getenv("CVB_NO_DGRAD_ROWS_HS") ? 1 : 0;
  int rc;
  if (!no_hs && hs_fits(n, oh, ow, cout, dycs, 2 * cin)) {
    for (int a = 0; a < 2; a++) {
      if ((rc = plan_hs(plans[a], dy, n, oh, ow, cout, dycs, a ? w1 : wrows, 2 * cin, a ? 2 : 1, 2, 0, dx, oh, ow,
                        2 * dxcs, 0, nullptr, 0, accumulate)))
        return rc;
      plans[a].out_par = 2; plans[a].out_ph = a; plans[a].out_pw = 0; plans[a].out_H = h; plans[a].out_W = ow;
    }
  } else {
    rc = plan_gather_conv(plans[0], dy, n, oh, ow, cout, dycs, wrows, 2 * cin, 2, dh0, dw0, dx, h, ow, 2 * dxcs, 0, 0,
                          accumulate, 1);
    if (rc) return rc;
    rc = plan_gather_conv(plans[1], dy, n, oh, ow, cout, dycs, w1, 2 * cin, 4, dh1, dw1, dx, h, ow, 2 * dxcs, 1, 0,
                          accumulate, 1);
    if (rc) return rc;
  }
  for (int a = 0; a < 2; a++)
    if ((rc = launch(plans[a], (cudaStream_t)stream))) return rc;
  return CVB_OK;
}

// Weight gradient, fp32 partials: part[split][cout_rows][kh*kw*cin] (caller reduces with
// cvb_reduce_splits).  dy: NHWC bf16 [n][oh][ow][cout] (stride dycs); x: NHWC input.
// Returns the number of splits used through *splits_out (<= max_splits).
CVB_API int cvb_conv2d_wgrad(const void* dy, int n, int oh, int ow, int cout, int dycs, const void* x, int h, int w,
                             int cin, int xcs, int kh, int kw, int stride, int pad, float* part, int max_splits,
                             int* splits_out, void* stream) {
  if (get_encoder()) return CVB_ECUDA;
  const int acel = pick_cel(cout), bcel = pick_cel(cin);
  if (!acel || !bcel || (stride != 1 && stride != 2)) { cvb_set_error("conv2d_wgrad: unsupported shape"); return CVB_EINVAL; }
  static GemmParams p;
  memset(&p, 0, sizeof(p));
  p.mode = MODE_WGRAD;
  p.a_major = 1; p.b_major = 1;
  p.a_cel = acel; p.b_cel = bcel;
  const int Ncols = kh * kw * cin;
  int bn = pick_bn(Ncols);
  bn = (bn + bcel - 1) / bcel * bcel;      // an N tile is a whole number of B boxes
  if (bn > 256) bn = 256 / bcel * bcel;
  p.BN = bn;
  p.ga = BM / p.a_cel;
  p.gb = p.BN / p.b_cel;
  p.M = cout; p.N = Ncols;
  // 128 pixels per K-block halves the TMA issues per pixel (TMA issue, not the tensor core,
  // bounds these wgrads); measured better even when only 2 stages fit
  static int env_kr = -1;
  if (env_kr < 0) { const char* e = getenv("CVB_WGRAD_KR"); env_kr = e ? atoi(e) : 0; }
  p.kr = (BM + p.BN) * 128 * 2 * 2 + 32 * 1024 <= 224 * 1024 ? 128 : 64;
  if (env_kr == 64 || env_kr == 128) p.kr = env_kr;
  int bw, bh, bnn;
  pick_kbox(oh, ow, p.kr, bw, bh, bnn);
  p.tw = bw; p.th = bh; p.tn = bnn;
  p.ptiles_w = (ow + bw - 1) / bw;
  p.ptiles_h = (oh + bh - 1) / bh;
  const int ptiles_n = (n + bnn - 1) / bnn;
  p.num_kb = p.ptiles_w * p.ptiles_h * ptiles_n;
  p.m_tiles = (cout + BM - 1) / BM;
  p.n_tiles = (Ncols + p.BN - 1) / p.BN;
  g_num_sms = cvb_num_sms();   // cached per device
  int tiles = p.m_tiles * p.n_tiles;
  int splits = (g_num_sms + tiles - 1) / tiles;
  if (splits > max_splits) splits = max_splits;
  if (splits > p.num_kb) splits = p.num_kb;
  if (splits < 1) splits = 1;
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
  p.splits = splits;
  p.OH = oh; p.OW = ow; p.NIMG = n;
  p.nbox = p.n_tiles * p.gb;
  if (p.nbox > MAX_BOXES) { cvb_set_error("conv2d_wgrad: N too large for the box table"); return CVB_EINVAL; }
  for (int i = 0; i < p.nbox; i++) p.boxtab[i] = gather_entry(i * bcel, cin, kh * kw, kw, pad, stride);
  p.tx_bytes = p.ga * p.kr * acel * 2 + p.gb * p.kr * bcel * 2;
  p.a_box_bytes = p.kr * acel * 2;
  int rc;
  if ((rc = encode_nhwc(&p.mapA[0], dy, n, oh, ow, cout, dycs, acel, bw, bh, bnn))) return rc;
  static int no_whalo = -1;
  if (no_whalo < 0) no_whalo = getenv("CVB_NO_WGRAD_HALO") ? 1 : 0;
  // WGRAD halo: stride 1, one 64-channel group (one 128-byte SW128 row per pixel; the 32-channel
  // SW64 variant computes correctly but measured 2x slower), one image
  // row box whose width is a multiple of 16 pixels, whole kw rows per N tile (N = KW*cin <= 256).
  // cin = 64 * G (G > 1): N tile (kh, channel group g) = KW x 64 columns, one box of group g
  static int no_whalo_g = -1;
  if (no_whalo_g < 0) no_whalo_g = getenv("CVB_NO_WGRAD_HALO_GROUPS") ? 1 : 0;
  // (only for narrow Cout: with Cout = 128 the dY operand is re-read per (kh, g) tile and the
  // gathered plan measured faster -- stage-2 ResNet wgrad 57.5 vs 63.2 us)
  // cin = 32: loaded as 64-channel SW128 rows whose upper half is TMA zero fill (the SW64 form
  // read at half rate); the padded half's output columns are not stored (CVB_NO_WGRAD_ROWPAD)
  static int no_wpad = -1;
  if (no_wpad < 0) no_wpad = getenv("CVB_NO_WGRAD_ROWPAD") ? 1 : 0;
  // (cin = 16 and 8 too: 16 / 8-column store chunks of the real channels only)
  // (8 channels only with the kh-quad plan, Cout 32: kh-paired at Cout 64 it measured slower,
  // the ResNet-18 stem wgrad 37.6 -> 46.9 us)
  const bool wpad = (cin == 32 || cin == 16 || (cin == 8 && cout == 32)) && !no_wpad;
  const int wg = cin % 64 == 0 ? cin / 64 : wpad ? 1 : 0;
  if (!no_whalo && stride == 1 && wg >= 1 && (wg == 1 || (!no_whalo_g && cout <= 64)) && (bcel == 64 || wpad) &&
      bnn == 1 && bw % 16 == 0 &&
      kw * 64 <= 256 && oh == h && ow == w) {
    p.w_halo = 1;
    p.b_cel = 64;   // 64-channel SW128 rows (cin = 32: upper half zero fill)
    p.w_groups = wg;
    p.w_cin = cin;
    p.h_kw = kw;
    p.BN = kw * 64;
    p.gb = 1;
    p.n_tiles = kh * wg;
    const int hw_ = bw + kw - 1;
    p.b_stage_bytes = ((uint32_t)hw_ * bh * 64 * 2 + 1023) / 1024 * 1024;
    p.tx_bytes = p.ga * p.kr * acel * 2 + (uint32_t)hw_ * bh * 64 * 2;
    tiles = p.m_tiles * p.n_tiles;
    splits = (g_num_sms + tiles - 1) / tiles;
    if (splits > max_splits) splits = max_splits;
    if (splits > p.num_kb) splits = p.num_kb;
    if (splits < 1) splits = 1;
    p.kb_per_split = (p.num_kb + splits - 1) / splits;
    splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
    p.splits = splits;
    static int no_pair = -1;
    if (no_pair < 0) no_pair = getenv("CVB_NO_WGRAD_PAIR") ? 1 : 0;
    // Cout = 64 fills only half of the 128-row MMA: pair the kh rows instead.  With the input
    // box fixed at X rows (2t - pad + r), kh = 2t reads dY row r and kh = 2t+1 dY row r - 1, so
    // ONE dY box of bh+1 rows (starting a row early) carries both as the two M atoms.
    static int one_box = -1;   // default: one (bh+1)-row box (measured 47.0 vs 48.6 us, stage-1 ResNet wgrad)
    if (one_box < 0) one_box = getenv("CVB_WGRAD_PAIR_TWOBOX") ? 0 : 1;
    // Cout = 32: a quarter of the MMA rows -- pack up to four kh rows as the M atoms of ONE
    // (bh + KH - 1)-row dY box (atom q = kh KH-1-q, one box row = one pixel row further down);
    // an N tile is then one 64-channel input group with every kh and kw (CVB_NO_WGRAD_QUAD=1: off)
    static int no_quad = -1;
    if (no_quad < 0) no_quad = getenv("CVB_NO_WGRAD_QUAD") ? 1 : 0;
    if (!no_quad && cout == 32 && acel == 32 && kh >= 2 && kh <= 4 && (bw * 64) % 1024 == 0 && p.w_groups >= 1) {
      p.w_pair = 3;
      p.w_kh = kh;
      p.n_tiles = wg;
      p.ptiles_h = (oh + kh - 1 + bh - 1) / bh;   // the pixel range runs KH-1 rows past the image
      p.num_kb = p.ptiles_w * p.ptiles_h * ((n + bnn - 1) / bnn);
      p.a_stage_bytes = ((uint32_t)bw * (bh + kh - 1) * 64u + 1023u) / 1024u * 1024u;
      p.tx_bytes = (uint32_t)bw * (bh + kh - 1) * 64u + (uint32_t)hw_ * bh * 64 * 2;
      if ((rc = encode_nhwc(&p.mapA[0], dy, n, oh, ow, cout, dycs, acel, bw, bh + kh - 1, bnn))) return rc;
      tiles = p.m_tiles * p.n_tiles;
      splits = (g_num_sms + tiles - 1) / tiles;
      if (splits > max_splits) splits = max_splits;
      if (splits > p.num_kb) splits = p.num_kb;
      if (splits < 1) splits = 1;
      p.kb_per_split = (p.num_kb + splits - 1) / splits;
      splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
      p.splits = splits;
    } else if (!no_pair && cout == 64 && kh >= 2 && wg == 1) {
      p.w_pair = one_box ? 1 : 2;
      p.w_kh = kh;
      p.n_tiles = (kh + 1) / 2;
      // kh = 2t+1 pairs dY row r-1 with the input rows of kh = 2t at row r: its last dY row
      // (oh-1) is reached only from K row oh -> the pixel range runs one row past the image
      // (that row is TMA zero fill for kh = 2t)
      p.ptiles_h = (oh + 1 + bh - 1) / bh;
      p.num_kb = p.ptiles_w * p.ptiles_h * ((n + bnn - 1) / bnn);
      if (p.w_pair == 1) {   // one (bh+1)-row box, M atoms one box row apart (LBO = a row of pixels)
        p.a_stage_bytes = ((uint32_t)bw * (bh + 1) * 128u + 1023u) / 1024u * 1024u;
        p.tx_bytes = (uint32_t)bw * (bh + 1) * 128u + (uint32_t)hw_ * bh * 64 * 2;
        if ((rc = encode_nhwc(&p.mapA[0], dy, n, oh, ow, cout, dycs, acel, bw, bh + 1, bnn))) return rc;
      } else {               // two boxes of the same dY channels, one row apart (standard MN atoms)
        p.tx_bytes = 2u * (uint32_t)bw * bh * 128u + (uint32_t)hw_ * bh * 64 * 2;
      }
      tiles = p.m_tiles * p.n_tiles;
      splits = (g_num_sms + tiles - 1) / tiles;
      if (splits > max_splits) splits = max_splits;
      if (splits > p.num_kb) splits = p.num_kb;
      if (splits < 1) splits = 1;
      p.kb_per_split = (p.num_kb + splits - 1) / splits;
      splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
      p.splits = splits;
    }
    p.nbox = p.n_tiles;
    if (p.nbox > MAX_BOXES) { cvb_set_error("conv2d_wgrad: too many halo tiles"); return CVB_EINVAL; }
    for (int t = 0; t < p.n_tiles; t++)   // row kh = t (paired: kh = 2t and 2t+1; groups: t / G), all kw
      p.boxtab[t] = p.w_pair == 3 ? pack_box(0, t * 64, -pad, -pad)
                  : p.w_pair ? pack_box(0, 0, -pad, 2 * t - pad) : pack_box(0, (t % wg) * 64, -pad, t / wg - pad);
    if ((rc = encode_nhwc(&p.mapB[0], x, n, h, w, cin, xcs, 64, hw_, bh, bnn))) return rc;
    p.out_mode = OUT_PARTIAL; p.out_f32 = 1; p.out = part; p.ldc = Ncols; p.col_off = 0; p.part_rows = cout;
    *splits_out = splits;
    return launch(p, (cudaStream_t)stream);
  }
  if (stride == 1) {
    if ((rc = encode_nhwc(&p.mapB[0], x, n, h, w, cin, xcs, bcel, bw, bh, bnn))) return rc;
  } else {
    for (int rh = 0; rh < 2; rh++)
      for (int rw = 0; rw < 2; rw++)
        if ((rc = encode_nhwc(&p.mapB[rh * 2 + rw], x, n, h, w, cin, xcs, bcel, bw, bh, bnn, rh, rw))) return rc;
  }
  p.out_mode = OUT_PARTIAL; p.out_f32 = 1; p.out = part; p.ldc = Ncols; p.col_off = 0; p.part_rows = cout;
  *splits_out = splits;
  return launch(p, (cudaStream_t)stream);
}

// Dense GEMM: C[m][n] (+bias[n]) = sum_k A(m,k) B(n,k)
//   A: a_major 0 -> row-major [M][K] (lda), 1 -> row-major [K][M] (lda)
//   B: b_major 0 -> row-major [N][K] (ldb), 1 -> row-major [K][N] (ldb)
// C row-major [M][ldc] bf16 or fp32; split-K > 1 writes fp32 partials [split][M][ldc].
CVB_API int cvb_gemm_ex(const void* a, int a_major, int64_t lda, const void* b, int b_major, int64_t ldb, int M, int N,
                        int K, void* c, int64_t ldc, int c_f32, const float* bias, int splits, int accumulate,
                        int max_bn, void* stream);
CVB_API int cvb_gemm(const void* a, int a_major, int64_t lda, const void* b, int b_major, int64_t ldb, int M, int N,
                     int K, void* c, int64_t ldc, int c_f32, const float* bias, int splits, int accumulate,
                     void* stream) {
  return cvb_gemm_ex(a, a_major, lda, b, b_major, ldb, M, N, K, c, ldc, c_f32, bias, splits, accumulate, 256, stream);
}

// max_bn (16..256, multiple of 16): narrower N tiles -> more (m, n) tiles and fewer split-K
// partial bytes for small-M FC layers.
CVB_API int cvb_gemm_ex(const void* a, int a_major, int64_t lda, const void* b, int b_major, int64_t ldb, int M, int N,
                        int K, void* c, int64_t ldc, int c_f32, const float* bias, int splits, int accumulate,
                        int max_bn, void* stream) {
  if (get_encoder()) return CVB_ECUDA;
  static GemmParams p;
  memset(&p, 0, sizeof(p));
  p.mode = MODE_DENSE;
  p.a_major = a_major; p.b_major = b_major;
  p.a_cel = 64; p.b_cel = 64;
  if (K % 8 || (a_major && M % 8) || (b_major && N % 8)) { cvb_set_error("gemm: unsupported shape"); return CVB_EINVAL; }
  if (a_major == 0) p.a_cel = pick_cel(K) ? (pick_cel(K) < 64 ? pick_cel(K) : 64) : 8;
  if (b_major == 0) p.b_cel = pick_cel(K) ? (pick_cel(K) < 64 ? pick_cel(K) : 64) : 8;
  p.BN = pick_bn(N);
  if (max_bn >= 16 && max_bn < p.BN) p.BN = max_bn / 16 * 16;
  if (b_major == 1) { p.BN = (p.BN + 63) / 64 * 64; if (p.BN > 256) p.BN = 256; }
  p.ga = a_major == 0 ? BK / p.a_cel : BM / p.a_cel;
  p.gb = b_major == 0 ? BK / p.b_cel : p.BN / p.b_cel;
  p.M = M; p.N = N;
  p.m_tiles = (M + BM - 1) / BM;
  p.n_tiles = (N + p.BN - 1) / p.BN;
  p.num_kb = (K + BK - 1) / BK;
  if (splits < 1) splits = 1;
  if (splits > p.num_kb) splits = p.num_kb;
  p.kb_per_split = (p.num_kb + splits - 1) / splits;
  p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
  p.tw = 1; p.th = 1; p.tn = 1; p.ptiles_w = 1; p.ptiles_h = 1;
  int rc;
  if (a_major == 0) { if ((rc = encode_2d(&p.mapA[0], a, M, K, lda, p.a_cel, BM))) return rc; }
  else { if ((rc = encode_2d(&p.mapA[0], a, K, M, lda, p.a_cel, BK))) return rc; }
  if (b_major == 0) { if ((rc = encode_2d(&p.mapB[0], b, N, K, ldb, p.b_cel, p.BN))) return rc; }
  else { if ((rc = encode_2d(&p.mapB[0], b, K, N, ldb, p.b_cel, BK))) return rc; }
  p.tx_bytes = (a_major == 0 ? p.ga * BM * p.a_cel * 2 : p.ga * BK * p.a_cel * 2) +
               (b_major == 0 ? p.gb * p.BN * p.b_cel * 2 : p.gb * BK * p.b_cel * 2);
  if (p.splits > 1) { p.out_mode = OUT_PARTIAL; p.out_f32 = 1; p.part_rows = M; }
  else { p.out_mode = OUT_ROWS; p.out_f32 = c_f32; }
  p.out = c; p.ldc = ldc; p.bias = p.splits > 1 ? nullptr : bias;
  p.accum = p.splits > 1 ? 0 : accumulate;
  return launch(p, (cudaStream_t)stream);
}

// ---- microbenchmark of the raw tcgen05.mma issue rate (debug aid, not on the hot path) ---
// issuers = 1 or 2 warps (warps 0 and 2), each with its own accumulator and mbarrier; the
// MMAs are committed once at the end.  Returns cycles for n_mma MMAs per issuer.
__global__ void __launch_bounds__(96, 1) mma_rate_kernel(int n_mma, int bn, int issuers, int a_halo, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_init(&bar[2], 1); mbar_init(&bar[3], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arrive(&bar[2]);   // phase 0 complete: a wait on it passes at once
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int me = warp == 0 ? 0 : warp == 2 ? 1 : -1;
  if (me >= 0 && me < (issuers == 3 ? 1 : issuers)) {
    const uint32_t tmem = slot + (uint32_t)me * 256u;
    const bool leader = elect_one();
    const uint64_t sa = smem_u32(smem) >> 4, sb = sa + (16384 >> 4);
    const uint64_t d0 = (uint64_t)1 | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
    // halo-like A: no swizzle, LBO = 2944 B (next 8-channel plane), SBO = 160 B (next halo row)
    const uint64_t dh = ((uint64_t)(2944 >> 4) << 16) | ((uint64_t)(160 >> 4) << 32) | ((uint64_t)1 << 46);
    const uint64_t da = a_halo ? dh : d0;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(bn >> 3) << 17) | (8u << 24);
    if (a_halo >= 11) {   // 11: A/B filled with random bf16 values, 12: with zeros (data dependence)
      uint32_t x = 0x9e3779b9u * (blockIdx.x + 1) + threadIdx.x;
      for (int i = threadIdx.x & 31; i < 16384; i += 32) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem)[i] = a_halo == 11 ? ((x & 0x3fff3fffu) | 0x3c003c00u) : 0u;
      }
      __syncwarp();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    long long t0 = clock64();
    if (leader) {
      if (a_halo == 10) {
        // halo rows with a 16-pixel pitch (SBO = 2048 B) and the 3x3 row-shifted starts
        const uint64_t dp = ((uint64_t)1 << 16) | ((uint64_t)(2048 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        for (int i = 0; i < n_mma; i++) {
          const int t = (i >> 1) % 9, j = i & 1;
          const uint32_t aoff = (uint32_t)((t / 3) * 16 + t % 3) * 8u + (uint32_t)j * 2u;
          umma_bf16(tmem + ((i / 18) & 1) * 32u, dp + sa + aoff, d0 + sb + j * 2, idesc, (i % 18) ? 1u : 0u);
        }
      } else if (a_halo == 8 || a_halo == 9) {
        // distinct A tiles: 8 = aligned starts walking 9 x 2 KB-apart tiles (SW128, SBO 1 KB),
        // 9 = the same walk shifted by one row (misaligned)
        const uint64_t dk = ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        for (int i = 0; i < n_mma; i++) {
          const int t = (i >> 1) % 9, j = i & 1;
          const uint32_t aoff = (uint32_t)t * 128u + (a_halo == 9 ? 8u : 0u) + (uint32_t)j * 2u;
          umma_bf16(tmem + ((i / 18) & 1) * 32u, dk + sa + aoff, d0 + sb + j * 2, idesc, (i % 18) ? 1u : 0u);
        }
      } else if (a_halo >= 5) {
        // one issuer alternating between two accumulators (two independent chains);
        // 5 = SW128 aligned A, 6 = row-shifted SW128 halo A, 7 = four accumulators aligned
        const uint64_t dr = ((uint64_t)1 << 16) | ((uint64_t)(1280 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        const int nch = a_halo == 7 ? 4 : 2;
        for (int i = 0; i < n_mma; i++) {
          const int t = (i >> 1) % 9, j = i & 1;
          const uint32_t aoff = (a_halo == 6 ? (uint32_t)((t / 3) * 10 + t % 3) * 8u : 0u) + (uint32_t)j * 2u;
          umma_bf16(tmem + (uint32_t)(i % nch) * (uint32_t)bn, (a_halo == 6 ? dr : d0) + sa + aoff, d0 + sb + j * 2,
                    idesc, i >= nch ? 1u : 0u);
        }
      } else if (a_halo == 3 || a_halo == 4) {
        // SW128 halo rows (pitch 10 pixels of 128 B, SBO = 1280 B): 3 = the rowpad conv's
        // row-shifted 3x3 start sequence, 4 = the same descriptors without the row shift
        const uint64_t dr = ((uint64_t)1 << 16) | ((uint64_t)(1280 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
        for (int i = 0; i < n_mma; i++) {
          const int t = (i >> 1) % 9, j = i & 1;
          const uint32_t aoff = (a_halo == 3 ? (uint32_t)((t / 3) * 10 + t % 3) * 8u : 0u) + (uint32_t)j * 2u;
          umma_bf16(tmem + ((i / 18) & 1) * 32u, dr + sa + aoff, d0 + sb + j * 2, idesc, (i % 18) ? 1u : 0u);
        }
      } else if (a_halo == 2) {   // the halo conv's exact 3x3 x 2-plane offset sequence, 2 accumulators
        for (int i = 0; i < n_mma; i++) {
          const int t = (i >> 1) % 9, j = i & 1;
          const uint32_t aoff = (uint32_t)((t / 3) * 10 + t % 3) + (uint32_t)j * 368u;
          umma_bf16(tmem + ((i / 18) & 1) * 32u, dh + sa + aoff, d0 + sb + j * 2, idesc, (i % 18) ? 1u : 0u);
          if (issuers == 3 && i % 18 == 17) umma_commit(&bar[1]);   // per-tile commit, never waited on
        }
      } else if (a_halo >= 13 && a_halo <= 16) {
        // the GEMM kernel's per-K-block synchronisation after every 4 MMAs: 13 = full-barrier
        // wait + tcgen05 fence + commit, 14 = commit only, 15 = fence only, 16 = wait only
        for (int i = 0; i < n_mma; i++) {
          umma_bf16(tmem, d0 + sa + (i & 3) * 2, d0 + sb + (i & 3) * 2, idesc, 1u);
          if ((i & 3) == 3) {
            if (a_halo == 13 || a_halo == 16) mbar_wait(&bar[2], 0);
            if (a_halo == 13 || a_halo == 15) tc_fence_after();
            if (a_halo == 13 || a_halo == 14) umma_commit(&bar[3]);
          }
        }
      } else {
        for (int i = 0; i < n_mma; i++) umma_bf16(tmem, da + sa + (i & 3) * (a_halo ? 1 : 2), d0 + sb + (i & 3) * 2, idesc, 1u);
      }
      umma_commit(&bar[me]);
    }
    __syncwarp();
    mbar_wait(&bar[me], 0);
    long long t1 = clock64();
    if (leader && blockIdx.x == 0) out[me] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}

CVB_API long long cvb_debug_mma_cycles(int n_mma, int bn, int issuers, int a_halo) {
  long long* d = nullptr;
  long long h[2] = {-1, -1};
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  // a_halo >= 100: the same probe on every SM at once (a_halo - 100), CTA 0 reports
  const int grid = a_halo >= 100 ? cvb_num_sms() : 1;
  if (a_halo >= 100) a_halo -= 100;
  mma_rate_kernel<<<grid, 96, 64 * 1024>>>(n_mma, bn, issuers, a_halo, d);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h[0] > h[1] ? h[0] : h[1];
}

// ---- microbenchmark of the TMA issue rate (debug aid) -----------------------------------
struct TmaProbe { CUtensorMap map; };
__global__ void __launch_bounds__(32, 1) tma_rate_kernel(const __grid_constant__ TmaProbe tp, int n_tma, int dims,
                                                        int box_bytes, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncwarp();
  const bool leader = elect_one();
  long long t0 = clock64();
  if (leader) {
    prefetch_map(&tp.map);
    mbar_expect_tx(&bar, (uint32_t)n_tma * box_bytes);
    for (int i = 0; i < n_tma; i++) {
      const uint32_t dst = smem_u32(smem) + (i & 7) * box_bytes;
      if (dims == 4) tma_load_4d(&tp.map, dst, &bar, 0, (i & 3), (i >> 2) & 3, 0);
      else tma_load_2d(&tp.map, dst, &bar, 0, (i & 15) * 8);
    }
  }
  __syncwarp();
  long long t1 = clock64();
  mbar_wait(&bar, 0);
  long long t2 = clock64();
  if (leader) { out[0] = t1 - t0; out[1] = t2 - t0; }
}

// returns issue cycles for n_tma loads (low 32 bits: issue, high: until all landed)
CVB_API long long cvb_debug_tma_cycles(int n_tma, int dims, int cel) {
  if (get_encoder()) return -1;
  TmaProbe tp;
  void* buf = nullptr;
  cudaMalloc(&buf, 64 << 20);
  int rc;
  if (dims == 4) rc = encode_nhwc(&tp.map, buf, 4, 64, 64, 64, 64, cel, 32, 4, 1);
  else rc = encode_2d(&tp.map, buf, 4096, 4096, 4096, cel, 128);
  if (rc) { cudaFree(buf); return -2; }
  const int box_bytes = dims == 4 ? 128 * cel * 2 : 128 * cel * 2;
  long long* d = nullptr;
  long long h[2] = {-1, -1};
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(tma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  tma_rate_kernel<<<1, 32, 8 * box_bytes + 1024>>>(tp, n_tma, dims, box_bytes, d);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(buf);
  return (h[1] << 32) | (h[0] & 0xffffffff);
}

CVB_API int cvb_debug_trace(long long* host_out) {
  if (!g_trace) return -1;
  cudaDeviceSynchronize();
  cudaMemcpy(host_out, g_trace, 8 * 4096 * sizeof(long long), cudaMemcpyDeviceToHost);
  return 0;
}

CVB_API int cvb_gemm_splits_used(int K, int splits) {
  int num_kb = (K + BK - 1) / BK;
  if (splits < 1) splits = 1;
  if (splits > num_kb) splits = num_kb;
  int per = (num_kb + splits - 1) / splits;
  return (num_kb + per - 1) / per;
}
