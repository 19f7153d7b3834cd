// paper_1412_6862_b200/csrc/hamming.cu -- sm_100a kernels + C ABI (include/hamming.h).
//
// Hot path: per-codeword Hamming decode of a bit-packed
// packet of concatenated perfect (2^m-1, 2^m-1-m) codewords -- the paper's
// checksum kernel (Algorithm 1) and error kernel (ED, EC, RR)
// fused into one HBM pass.  B200 design:
//
//   * Work unit = a warp tile of 1024 codewords.  Because n and k are odd or
//     small, 32 codewords of one lane occupy exactly n input words and k output
//     words (gcd(n, 32) = 1 for odd n), so a warp tile is 128*n input bytes and
//     128*k output bytes: always 16-byte aligned, always a whole number of words.
//   * a1 load/unpack: one elected lane moves the tile HBM -> shared memory with a
//     1-D TMA bulk copy (cp.async.bulk + mbarrier complete_tx), STAGES deep per
//     warp; each lane then reads its own n words (lane stride n words is odd, so
//     the reads are bank-conflict free) and extracts codeword c with compile-time
//     funnel shifts (bit offset c*n - 1 is a constant after unrolling).
//   * a2 syndrome: one POPC per syndrome bit on the codeword AND the index-set
//     mask M_j (P:L98 index sets; "modulo 2 (XOR)").  For m = 6 the two
//     32-bit halves are folded first (positions p and p+32 share their low five
//     bits), so every mask is 32-bit.
//   * a3 ED/EC: v ^= 1 << s with the dummy bit 0 standing in for "no error" --
//     branch free, no divergence (the paper's Fermi divergence problem).
//   * a4 RR: m-1 shift-and-mask steps (the pext of the data mask).
//   * a5 merge/pack: each lane ORs its k-bit results into k registers at
//     compile-time offsets, stores them to shared memory (odd stride again),
//     and the elected lane writes the whole tile back with one bulk S2G copy.
//   * a6 syndromes: 32 bytes per lane, two 16-byte streaming stores (the warp
//     writes 1 KiB contiguous).
//   * a7 count: per-lane register count -> warp __reduce_add_sync -> block
//     shared-memory sum -> one 64-bit atomic per CTA.
//   * Persistent grid: one CTA per SM (or more for small m), each warp runs an
//     independent grid-stride loop over tiles; no __syncthreads in the loop.
//
// The ragged tail (< 1024 codewords) runs the same lane function in a one-warp
// kernel with bounded, zero-filled loads; it also writes *corrected first so the
// main kernel can accumulate into it (stream order), i.e. the count is
// overwritten without a memset.
//
// Nothing here is shared with oracle/ (the CPU checker).

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <type_traits>

#include "hamming.h"

namespace {

// ------------------------------------------------------------------ geometry
template <int M>
struct Geo {
  static constexpr int n = (1 << M) - 1;
  static constexpr int k = n - M;
};

constexpr int kTileCw = 1024;  // codewords per warp tile (32 lanes x 32)

// Parity mask of index set I_j on a register v whose bit p holds position p
// (bit 0 = dummy), positions 1..min(n, 31).  (I_j = {p : bit j of p}.)
__host__ __device__ constexpr uint32_t pmask(int n, int j) {
  uint32_t mk = 0;
  for (int p = 1; p <= n && p < 32; ++p)
    if ((p >> j) & 1) mk |= (1u << p);
  return mk;
}

// Redundancy removal, group g (positions 2^g+1 .. 2^(g+1)-1): after shifting v
// right by g+2 the group lands on data bits [2^g-g-1, 2^(g+1)-g-2].
__host__ __device__ constexpr uint32_t dmask(int g) {
  return ((1u << ((1 << g) - 1)) - 1u) << ((1 << g) - g - 1);
}

// --------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
#ifndef HAM_WAIT_MODE
#define HAM_WAIT_MODE 0
#endif
#ifndef HAM_WAIT_NS
#define HAM_WAIT_NS 100000
#endif
// Wait for an mbarrier phase.  Mode 0: the try_wait loop (the hardware may
// suspend the thread inside try_wait for a system-dependent time); mode 1:
// try_wait with an explicit suspend-time hint (HAM_WAIT_NS); mode 2: a failed
// try_wait backs off with __nanosleep(HAM_WAIT_NS) -- modes 1, 2 are power
// experiments (tools/power_probe.py).
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#if HAM_WAIT_MODE == 1
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "HAM_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra HAM_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase), "r"(HAM_WAIT_NS)
      : "memory");
#elif HAM_WAIT_MODE == 2
  while (!mbar_try(bar, phase)) __nanosleep(HAM_WAIT_NS);
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "HAM_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra HAM_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
#endif
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 1-D TMA: global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// 2-D TMA (tensor map, e.g. 128-byte swizzled): global -> shared.
__device__ __forceinline__ void tensor_g2s_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tensor_g2s_3d(void* dst, const void* tmap, int x, int y, int z, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_addr(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// TMA tensor stores (shared -> global through a tensor map), bulk-group completion.
__device__ __forceinline__ void tensor_s2g_2d(const void* tmap, int x, int y, const void* src, uint64_t pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(
                   tmap),
               "r"(x), "r"(y), "r"(smem_addr(src)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void tensor_s2g_3d(const void* tmap, int x, int y, int z, const void* src, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(tmap),
      "r"(x), "r"(y), "r"(z), "r"(smem_addr(src)), "l"(pol)
      : "memory");
}
// 1-D TMA: shared -> global, bulk-group completion.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// A CTA-wide table copied from global memory by ONE TMA bulk copy (thread 0
// issues it; the caller's other set-up runs meanwhile): cta_table_copy_begin,
// then a __syncthreads, then cta_table_copy_wait on every thread.  `bar` is a
// __shared__ mbarrier used once per launch.
__device__ __forceinline__ void cta_table_copy_begin(void* dst, const void* src, uint32_t bytes, int tid, uint64_t* bar) {
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, bytes);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
  }
}
__device__ __forceinline__ void cta_table_copy_wait(uint64_t* bar) { mbar_wait(bar, 0); }
__device__ __forceinline__ void st_global_cs_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// ------------------------------------------------- compile-time bit plumbing
// Read `width` (<= 32) bits starting at lane-stream bit b from the register
// array w[0..NW); bits past the array read as 0.  b is a constant after unrolling.
template <int NW>
__device__ __forceinline__ uint32_t take_bits(const uint32_t (&w)[NW], int b) {
  const int q = b >> 5, r = b & 31;
  const uint32_t a = (q < NW) ? w[q] : 0u;
  if (r == 0) return a;
  const uint32_t c = (q + 1 < NW) ? w[q + 1] : 0u;
  return __funnelshift_r(a, c, r);
}
// OR a clean `width`-bit value into the register array o at lane-stream bit b.
template <int NO>
__device__ __forceinline__ void put_bits(uint32_t (&o)[NO], int b, uint32_t val, int width) {
  const int q = b >> 5, r = b & 31;
  o[q] |= val << r;
  if (r != 0 && r + width > 32) o[q + 1] |= val >> (32 - r);
}

// OR bits [pos, pos+len) of src into the output stream at bit b: one shift and
// one LOP3 per output word touched (all shifts are constants after unrolling).
// Used to move each redundancy-removal group straight to its final position.
template <int NO>
__device__ __forceinline__ void put_field(uint32_t (&o)[NO], int b, uint32_t src, int pos, int len) {
  const int q = b >> 5, r = b & 31;
  const uint32_t m = (len >= 32) ? 0xFFFFFFFFu : ((1u << len) - 1u);
  const uint32_t x = (r >= pos) ? (src << (r - pos)) : (src >> (pos - r));
  o[q] |= x & (m << r);
  if (r + len > 32) o[q + 1] |= (src >> (pos + 32 - r)) & (m >> (32 - r));
}

// Count of nonzero syndrome bytes in the lane's 8 side words (s <= 63, so
// adding 0x7F to a byte never carries into the next one).
__device__ __forceinline__ uint32_t count_nonzero_bytes(const uint32_t (&w)[8]) {
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += ((w[i] + 0x7F7F7F7Fu) & 0x80808080u) >> 7;
  return (acc * 0x01010101u) >> 24;  // four byte lanes of at most 8 each
}

// The same count with one POPC per word: for the table decoders, whose XU
// pipe is otherwise idle and whose ALU pipe is the tighter one.
__device__ __forceinline__ uint32_t count_nonzero_bytes_xu(const uint32_t (&w)[8]) {
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t t;
    asm("mad.lo.u32 %0, %1, 1, 2139062143;" : "=r"(t) : "r"(w[i]));  // + 0x7F7F7F7F on the FMA pipe
    c += __popc(t & 0x80808080u);
  }
  return c;
}

// --------------------------------------------------------- per-codeword math
// Decode one codeword given as v = (lo, hi): bit p of v holds position p
// (hi bit i = position 32 + i; hi unused for m <= 5).  Returns the syndrome s
// and the corrected data bits (dlo: data bits 0.., dhi for m = 6:
// data bits 26..56).
template <int M>
__device__ __forceinline__ uint32_t decode_cw(uint32_t lo, uint32_t hi, uint32_t& dlo, uint32_t& dhi) {
  constexpr int n = Geo<M>::n;
  uint32_t s;
  if constexpr (M <= 5) {
    s = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) s |= static_cast<uint32_t>(__popc(lo & pmask(n, j)) & 1) << j;  // a2
    lo ^= 1u << s;                                                                               // a3
    uint32_t d = 0;
#pragma unroll
    for (int g = 1; g < M; ++g) d |= (lo >> (g + 2)) & dmask(g);  // a4
    dlo = d;
    dhi = 0;
  } else {
    const uint32_t x = lo ^ hi;  // fold: positions p and p+32 agree in bits 0..4
    s = static_cast<uint32_t>(__popc(hi) & 1) << 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) s |= static_cast<uint32_t>(__popc(x & pmask(31, j)) & 1) << j;
    const uint64_t f = 1ull << s;
    lo ^= static_cast<uint32_t>(f);
    hi ^= static_cast<uint32_t>(f >> 32);
    uint32_t d = 0;
#pragma unroll
    for (int g = 1; g < 5; ++g) d |= (lo >> (g + 2)) & dmask(g);
    dlo = d;        // data bits 0..25 (positions 3..31)
    dhi = hi >> 1;  // data bits 26..56 (positions 33..63)
  }
  return s;
}

// The syndrome alone (a2): s = sum_j 2^j parity(v & M_j), folded for m = 6.
template <int M>
__device__ __forceinline__ uint32_t syndrome_cw(uint32_t lo, uint32_t hi) {
  constexpr int n = Geo<M>::n;
  uint32_t s = 0;
  if constexpr (M <= 5) {
#pragma unroll
    for (int j = 0; j < M; ++j) s |= static_cast<uint32_t>(__popc(lo & pmask(n, j)) & 1) << j;
  } else {
    const uint32_t x = lo ^ hi;
    s = static_cast<uint32_t>(__popc(hi) & 1) << 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) s |= static_cast<uint32_t>(__popc(x & pmask(31, j)) & 1) << j;
  }
  return s;
}

// Encode one message (dlo, dhi as produced by decode_cw) into v = (lo, hi):
// data at non-power-of-two positions, parity 2^j = XOR over I_j \ {2^j}.
template <int M>
__device__ __forceinline__ void encode_cw(uint32_t dlo, uint32_t dhi, uint32_t& lo, uint32_t& hi) {
  constexpr int n = Geo<M>::n;
  constexpr int G = (M <= 5) ? M : 5;
  uint32_t v = 0;
#pragma unroll
  for (int g = 1; g < G; ++g) v |= (dlo & dmask(g)) << (g + 2);
  uint32_t h = (M == 6) ? (dhi << 1) : 0u;
  uint32_t s = 0;
  if constexpr (M <= 5) {
#pragma unroll
    for (int j = 0; j < M; ++j) s |= static_cast<uint32_t>(__popc(v & pmask(n, j)) & 1) << j;
  } else {
    const uint32_t x = v ^ h;
    s = static_cast<uint32_t>(__popc(h) & 1) << 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) s |= static_cast<uint32_t>(__popc(x & pmask(31, j)) & 1) << j;
  }
#pragma unroll
  for (int j = 0; j < G; ++j) v |= ((s >> j) & 1u) << (1 << j);
  if constexpr (M == 6) h |= (s >> 5) & 1u;
  lo = v;
  hi = h;
}

// Emit codeword v (bit p = position p) as stream bits [b, b+n).
template <int M, int NO>
__device__ __forceinline__ void put_codeword(uint32_t (&o)[NO], int b, uint32_t lo, uint32_t hi) {
  constexpr int n = Geo<M>::n;
  if constexpr (M <= 4) {
    put_bits(o, b, (lo >> 1) & ((1u << n) - 1u), n);
  } else if constexpr (M == 5) {
    put_bits(o, b, lo >> 1, 31);
  } else {
    put_bits(o, b, (lo >> 1) | (hi << 31), 32);
    put_bits(o, b + 32, hi >> 1, 31);
  }
}

// ------------------------------------------------------------ tile operators
// Each operator processes the 32 codewords of one lane: `in` = the lane's
// IN_W input words, `out` = its OUT_W output words (both in shared memory),
// `side` = 8 words of per-codeword bytes (syndromes).
// `valid` = number of the lane's 32 codewords that exist (32 except in the tail).

// EXT = false: the perfect (2^m-1, 2^m-1-m) code, codeword c = lane-stream
// bits [c n, c n + n).  EXT = true: extended Hamming / SECDED (SURVEY.md 8(f)
// f4, reading R17), codeword c = bits [c 2^m, (c+1) 2^m) with bit 0 the
// overall parity -- register bit p is position p in both cases (bit 0 is the
// dummy resp. the parity bit), so a2..a5 are shared.
// Shared-memory 16-byte unit of tile unit g (stream order) for tiles loaded
// by the swizzled tensor map, lanes owning IN_W words each.  The map views
// the tile as 128-byte rows; with RPL = IN_W / 32 >= 2 rows per lane it is
// 3-D and lands row h of lane l at smem row r = h * 32 + l (so the 8 lanes of
// a 128-bit access phase sit in 8 different rows), otherwise r = the stream
// row.  CU_TENSOR_MAP_SWIZZLE_128B then puts unit c of row r at c ^ (r & 7).
template <int IN_W>
__host__ __device__ __forceinline__ constexpr uint32_t swz_unit(uint32_t g) {
  constexpr uint32_t RPL = IN_W / 32;
  const uint32_t row = g >> 3;
  const uint32_t r = (RPL >= 2) ? (row % RPL) * 32 + row / RPL : row;
  return r * 8 + ((g ^ r) & 7u);
}

// flags byte of a SECDED codeword from its syndrome and overall parity
__device__ __forceinline__ uint32_t secded_flags(uint32_t s, uint32_t par) {
  return s | (par << 6) | ((static_cast<uint32_t>(s != 0) & (par ^ 1u)) << 7);
}
// the same for four codewords at once: S4 holds s_k in byte k (s_k < 64), P4 holds P_k at bit
// 8k + 6; byte k of the result is secded_flags(s_k, P_k) (s_k + 0x7F carries into bit 7 iff
// s_k != 0, never out of the byte)
__device__ __forceinline__ uint32_t secded_flags4(uint32_t S4, uint32_t P4) {
  const uint32_t nz = (S4 + 0x7F7F7F7Fu) & 0x80808080u;
  return S4 | P4 | (nz & ~(P4 << 1));
}

template <int M, bool EXT = false>
struct DecodeOp {
  static constexpr int CW_BITS = EXT ? (1 << M) : Geo<M>::n;
  static constexpr int IN_W = CW_BITS;  // 32 codewords of a lane
  static constexpr int OUT_W = Geo<M>::k;
  static constexpr int IN_BITS = CW_BITS;  // per codeword
  static constexpr bool HAS_SIDE = true;
  static constexpr int NCOUNT = EXT ? 2 : 1;
  static constexpr int SHARED = 0;  // CTA-shared bytes (lookup tables)
  // SECDED lanes own 2^m words: a power-of-two stride would put all lanes'
  // reads of their own codewords in the same banks, so SECDED tiles are
  // loaded by a TMA tensor map with the 128-byte swizzle and read back
  // through swz_unit (below).
  static constexpr bool SWZ = EXT;
  struct NoArgs {};
  struct TmapArgs {
    CUtensorMap tmap;  // the input as rows of 128 bytes, box = one tile
  };
  using Args = typename std::conditional<EXT, TmapArgs, NoArgs>::type;
  __device__ __forceinline__ static void cta_init(uint8_t*, int, int) {}
  // counts from the side bytes: perfect code -- nonzero syndromes; SECDED --
  // [corrected (bit 6), double errors detected (bit 7)]
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) {
    if constexpr (EXT) {
      uint32_t c = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) c += __popc(sw[i] & 0x40404040u);
      return c;
    } else {
      return count_nonzero_bytes(sw);
    }
  }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&sw)[8]) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) c += __popc(sw[i] & 0x80808080u);
    return c;
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                  uint32_t (&side)[8], uint64_t /*cw0*/, int /*valid*/,
                                                  const Args&, const uint8_t* /*sh*/) {
    constexpr int n = Geo<M>::n, k = Geo<M>::k;
    uint32_t w[IN_W];
    if constexpr (SWZ) {  // `in` is the tile base; this lane's 16-byte units through the swizzle
      constexpr int CPL = IN_W / 4;
      const uint32_t l = threadIdx.x & 31u;
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const uint4 v = reinterpret_cast<const uint4*>(in)[swz_unit<IN_W>(l * CPL + u)];
        w[4 * u] = v.x;
        w[4 * u + 1] = v.y;
        w[4 * u + 2] = v.z;
        w[4 * u + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < IN_W; ++i) w[i] = in[i];
    }
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    uint32_t o[k];
#pragma unroll
    for (int i = 0; i < k; ++i) o[i] = 0;
    uint32_t S4 = 0, P4 = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      uint32_t lo, hi = 0;
      if constexpr (EXT) {  // word-aligned 2^m-bit codewords
        if constexpr (M == 6) {
          lo = w[2 * c];
          hi = w[2 * c + 1];
        } else {
          lo = take_bits(w, c * CW_BITS);
        }
      } else if (c == 0) {  // v = w << 1 (no previous codeword: dummy bit 0 = 0)
        lo = w[0] << 1;
        if constexpr (M == 6) hi = __funnelshift_l(w[0], w[1], 1);
      } else {  // v = lane-stream bits [c*n - 1, c*n - 1 + 32*(1 or 2))
        lo = take_bits(w, c * n - 1);
        if constexpr (M == 6) hi = take_bits(w, c * n + 31);
      }
      const uint32_t s = syndrome_cw<M>(lo, hi);  // a2
      uint32_t par = 0;
      if constexpr (EXT) {  // overall parity P decides: P = 1 correct, P = 0 and s != 0 detect
        if constexpr (M == 6) par = __popc(lo ^ hi) & 1u;
        else if constexpr (M == 5) par = __popc(lo) & 1u;
        else par = __popc(lo & ((1u << CW_BITS) - 1u)) & 1u;
        if constexpr (M <= 5) {  // a3: flip position s only when P = 1 (s = 0: the parity bit)
          lo ^= par << s;
        } else {
          const uint64_t f = static_cast<uint64_t>(par) << s;
          lo ^= static_cast<uint32_t>(f);
          hi ^= static_cast<uint32_t>(f >> 32);
        }
      } else if constexpr (M <= 5) {  // a3 (s = 0 flips the dummy bit 0)
        lo ^= 1u << s;
      } else {
        const uint64_t f = 1ull << s;
        lo ^= static_cast<uint32_t>(f);
        hi ^= static_cast<uint32_t>(f >> 32);
      }
      // a4 + a5: each redundancy-removal group (positions 2^g+1 .. 2^(g+1)-1,
      // data bits from 2^g-g-1) goes straight to its place in the output stream
#pragma unroll
      for (int g = 1; g < (M <= 5 ? M : 5); ++g)
        put_field(o, c * k + (1 << g) - g - 1, lo, (1 << g) + 1, (1 << g) - 1);
      if constexpr (M == 6) put_field(o, c * k + 26, hi, 1, 31);
      if constexpr (EXT) {  // flags bytes {s, P << 6, (s != 0 and P = 0) << 7}, four at a time
        S4 |= s << (8 * (c & 3));
        P4 |= par << (8 * (c & 3) + 6);
        if ((c & 3) == 3) {
          side[c >> 2] |= secded_flags4(S4, P4);
          S4 = P4 = 0;
        }
      } else {
        side[c >> 2] |= s << (8 * (c & 3));
      }
    }
#pragma unroll
    for (int i = 0; i < k; ++i) out[i] = o[i];
  }
};

// ----------------------------------------------------- lookup-table decoders
// For m = 3 and 4 the POPC-per-index-set syndrome is bound by the XU pipe
// (16 lanes/clk/SM) long before HBM is; a shared-memory
// table turns the whole per-codeword decode (a2..a4) into one LDS on the
// otherwise idle LSU pipe.  The table entries are produced by decode_cw<M>
// itself, so the table IS the POPC decoder, evaluated once per index.

// Lane-stream bits starting at b, placed at bit `at` of the result (bits below
// `at` hold the preceding stream bits).  b and at are constants after unrolling.
template <int NW>
__device__ __forceinline__ uint32_t field_at(const uint32_t (&w)[NW], int b, int at) {
  return (b >= at) ? take_bits(w, b - at) : (w[0] << (at - b));
}

// PRMT selectors that move byte 1 of the second operand into byte i of the first.
__device__ __forceinline__ uint32_t insert_byte1(uint32_t word, uint32_t e, int i) {
  const uint32_t sel = (i == 0) ? 0x3215u : (i == 1) ? 0x3250u : (i == 2) ? 0x3510u : 0x5210u;
  return __byte_perm(word, e, sel);
}

// (7,4): per-lane replicated 128-entry table of 8-byte entries {data nibble
// replicated into all eight nibbles, s | (s != 0) << 16}; lane l reads entry
// [x][l], always its own bank pair (32 KB, conflict-free).  The replicated
// nibble goes to its place in the output word with one LOP3 against a constant
// mask (no shift); the syndrome bytes of four codewords become one side word by
// three PRMTs, and the count is the high half of the plain sum of the .y words
// (the low halves add up to at most 32 x 7, no carry into bit 16).
struct DecodeLut3Op {
  static constexpr int NCOUNT = 1;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return count_nonzero_bytes_xu(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }
  static constexpr int IN_W = 7, OUT_W = 4, IN_BITS = 7;
  static constexpr bool HAS_SIDE = true;
  static constexpr bool LANE_COUNT = true;
  static constexpr int SHARED = 128 * 32 * 8;
  struct Args {};

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    uint2* L = reinterpret_cast<uint2*>(sh);
    for (int e = tid; e < 128 * 32; e += nth) {
      uint32_t dlo, dhi;
      const uint32_t s = decode_cw<3>(static_cast<uint32_t>(e >> 5) << 1, 0u, dlo, dhi);
      L[e] = make_uint2(dlo * 0x11111111u, s | (static_cast<uint32_t>(s != 0) << 16));
    }
  }

  __device__ __forceinline__ static uint32_t lane_count(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                        uint32_t (&side)[8], uint64_t, int, const Args&,
                                                        const uint8_t* sh) {
    uint32_t w[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) w[i] = in[i];
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    const uint32_t lane8 = (threadIdx.x & 31u) << 3;
    uint32_t o[4] = {0, 0, 0, 0};
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // codewords 4j .. 4j+3
      uint32_t y[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = 4 * j + i;
        const uint32_t off = (field_at(w, 7 * c, 8) & 0x7F00u) | lane8;  // (x * 32 + lane) * 8
        const uint2 e = *reinterpret_cast<const uint2*>(sh + off);
        o[c >> 3] |= e.x & (0xFu << ((4 * c) & 31));
        y[i] = e.y;
      }
      acc += y[0] + y[1] + y[2] + y[3];
      side[j] = __byte_perm(__byte_perm(y[0], y[1], 0x0040u), __byte_perm(y[2], y[3], 0x0040u), 0x5410u);
    }
    *reinterpret_cast<uint4*>(out) = make_uint4(o[0], o[1], o[2], o[3]);
    return acc >> 16;
  }
};

// (7,4), two codewords per lookup: a 16384-entry table (64 KB, built per CTA)
// indexed by the 14 stream bits of a codeword PAIR, entry = {the two corrected
// data nibbles (byte 0), the two syndromes (bytes 1, 2), the number of nonzero
// syndromes (byte 3)} -- every field is decode_cw<3> of one half.  Per pair:
// one funnel shift + one LOP3 form the byte address, one LDS; the data bytes of
// four pairs become one output word by three PRMTs, the syndrome bytes of two
// pairs one side word by one PRMT, and the count is one add of byte 3.  The
// per-codeword table decoder (DecodeLut3Op) spent ~5 ALU instructions per
// codeword and bound the pipe (ncu: ALU 75 %, issue 74 %); this one ~2.
struct DecodeLut3PairOp {
  static constexpr int NCOUNT = 1;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return count_nonzero_bytes_xu(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }
  static constexpr int IN_W = 7, OUT_W = 4, IN_BITS = 7;
  static constexpr bool HAS_SIDE = true;
  static constexpr bool LANE_COUNT = true;  // lane_count() returns the lane's nonzero-syndrome count
  static constexpr int SHARED = 16384 * 4 + 128 * 4;
  struct Args {};

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    uint32_t* P = reinterpret_cast<uint32_t*>(sh);
    uint32_t* E1 = P + 16384;  // single codewords: data | s << 8
    for (int e = tid; e < 128; e += nth) {
      uint32_t dlo, dhi;
      const uint32_t s = decode_cw<3>(static_cast<uint32_t>(e) << 1, 0u, dlo, dhi);
      E1[e] = dlo | (s << 8);
    }
    __syncthreads();  // cta_init is called by every thread of the CTA
    for (int x = tid; x < 16384; x += nth) {
      const uint32_t a = E1[x & 127], b = E1[x >> 7];
      const uint32_t sa = a >> 8, sb = b >> 8;
      P[x] = (a & 0xFu) | ((b & 0xFu) << 4) | (sa << 8) | (sb << 16) |
             ((static_cast<uint32_t>(sa != 0) + static_cast<uint32_t>(sb != 0)) << 24);
    }
  }

  __device__ __forceinline__ static uint32_t lane_count(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                        uint32_t (&side)[8], uint64_t, int, const Args&,
                                                        const uint8_t* sh) {
    uint32_t w[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) w[i] = in[i];
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    uint32_t e[16];
#pragma unroll
    for (int c2 = 0; c2 < 16; ++c2) {  // pair c2 = codewords 2 c2, 2 c2 + 1 = lane-stream bits 14 c2 ..
      const uint32_t off = field_at(w, 14 * c2, 2) & 0xFFFCu;  // 4 x (14-bit index)
      e[c2] = *reinterpret_cast<const uint32_t*>(sh + off);
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int c2 = 0; c2 < 16; ++c2) cnt += e[c2] >> 24;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t t01 = __byte_perm(e[4 * i], e[4 * i + 1], 0x0040u);
      const uint32_t t23 = __byte_perm(e[4 * i + 2], e[4 * i + 3], 0x0040u);
      out[i] = __byte_perm(t01, t23, 0x5410u);  // data bytes of pairs 4i .. 4i+3
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) side[j] = __byte_perm(e[2 * j], e[2 * j + 1], 0x6521u);  // s of codewords 4j..4j+3
    return cnt;
  }
};

// (15,11): one 32768-entry table of 16-bit entries (64 KB, shared by the CTA),
// entry = corrected data (bits 0..10) | syndrome << 12.  Built once per device
// in global memory, copied into shared memory at CTA start.
__device__ __align__(16) uint16_t g_lut15[32768];

// (31,26) half-word table: for a 15-bit chunk x (bit p-1 = position p) the
// UNcorrected redundancy removal (bits 0..10), the syndrome contribution
// XOR{p} (bits 11..14) and the parity of x (bit 15).
__device__ __align__(16) uint16_t g_lut15raw[32768];

__global__ void init_lut15_kernel() {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < 32768) {
    uint32_t dlo, dhi;
    const uint32_t v = static_cast<uint32_t>(x) << 1;
    const uint32_t s = decode_cw<4>(v, 0u, dlo, dhi);
    g_lut15[x] = static_cast<uint16_t>(dlo | (s << 12));
    uint32_t raw = 0;
#pragma unroll
    for (int g = 1; g < 4; ++g) raw |= (v >> (g + 2)) & dmask(g);
    g_lut15raw[x] = static_cast<uint16_t>(raw | (s << 11) | ((static_cast<uint32_t>(__popc(x)) & 1u) << 15));
  }
}

// (31,26): a codeword is two 15-bit table lookups -- positions 1..15 and
// positions 17..31 -- plus position 16:  s = S(lo) ^ S(hi) ^ 16 (parity(hi) ^
// bit16), data = RR(lo) | hi << 11, corrected by a per-lane flip-mask table
// F[s] (4 KB, conflict-free).  No POPC: the XU pipe, which bounds the
// POPC decoder at m = 5, is left idle.
struct DecodeLut5Op {
  static constexpr int NCOUNT = 1;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return count_nonzero_bytes_xu(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }
  static constexpr int IN_W = 31, OUT_W = 26, IN_BITS = 31;
  static constexpr bool HAS_SIDE = true;
  static constexpr int SHARED = 32768 * 2 + 32 * 32 * 4;
  struct Args {};

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    __shared__ __align__(8) uint64_t tbar;
    cta_table_copy_begin(sh, g_lut15raw, 32768 * 2, tid, &tbar);  // one TMA copy of the 64 KB table
    uint32_t* F = reinterpret_cast<uint32_t*>(sh + 32768 * 2);
    for (int e = tid; e < 32 * 32; e += nth) {  // F[s][lane] = the data bit of position s (0 if parity)
      const uint32_t v = (e >> 5) ? (1u << (e >> 5)) : 0u;  // a word with only position s set
      uint32_t raw = 0;
#pragma unroll
      for (int g = 1; g < 5; ++g) raw |= (v >> (g + 2)) & dmask(g);
      F[e] = raw;
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    cta_table_copy_wait(&tbar);
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&,
                                              const uint8_t* sh) {
    uint32_t w[31];
#pragma unroll
    for (int i = 0; i < 31; ++i) w[i] = in[i];
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    const uint32_t lane4 = (threadIdx.x & 31u) << 2;
    uint32_t o[26];
#pragma unroll
    for (int i = 0; i < 26; ++i) o[i] = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t alo = field_at(w, 31 * c, 1) & 0xFFFEu;       // positions 1..15, x 2
      const uint32_t h = take_bits(w, 31 * c + 15);                 // bit 0 = position 16, 1.. = 17..31
      const uint32_t elo = *reinterpret_cast<const uint16_t*>(sh + alo);
      const uint32_t ehi = *reinterpret_cast<const uint16_t*>(sh + (h & 0xFFFEu));
      const uint32_t t = elo ^ ehi;
      const uint32_t s = ((t >> 11) & 0xFu) | ((((ehi >> 15) ^ h) & 1u) << 4);
      const uint32_t f = *reinterpret_cast<const uint32_t*>(sh + 65536 + (s << 7) + lane4);
      const uint32_t d = ((elo & 0x7FFu) | ((h << 10) & 0x3FFF800u)) ^ f;
      put_bits(o, 26 * c, d, 26);
      side[c >> 2] |= s << (8 * (c & 3));
    }
#pragma unroll
    for (int i = 0; i < 26; ++i) out[i] = o[i];
  }
};

struct DecodeLut4Op {
  static constexpr int NCOUNT = 1;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return count_nonzero_bytes_xu(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }
  static constexpr int IN_W = 15, OUT_W = 11, IN_BITS = 15;
  static constexpr bool HAS_SIDE = true;
  static constexpr int SHARED = 32768 * 2;
  struct Args {};

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int) {
    __shared__ __align__(8) uint64_t tbar;
    cta_table_copy_begin(sh, g_lut15, SHARED, tid, &tbar);  // one TMA copy of the 64 KB table
    __syncthreads();  // the barrier is initialised before anyone waits on it
    cta_table_copy_wait(&tbar);
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&,
                                              const uint8_t* sh) {
    uint32_t w[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) w[i] = in[i];
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    uint32_t o[11];
#pragma unroll
    for (int i = 0; i < 11; ++i) o[i] = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t off = field_at(w, 15 * c, 1) & 0xFFFEu;  // x * 2
      const uint32_t e = *reinterpret_cast<const uint16_t*>(sh + off);
      const int b = 11 * c, q = b >> 5, r = b & 31;
      o[q] |= (e << r) & (0x7FFu << r);
      if (r > 21) o[q + 1] |= (e >> (32 - r)) & (0x7FFu >> (32 - r));
      side[c >> 2] = insert_byte1(side[c >> 2], e, c & 3);  // byte 1 = d8..d10, 0, s
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) side[i] = (side[i] >> 4) & 0x0F0F0F0Fu;
#pragma unroll
    for (int i = 0; i < 11; ++i) out[i] = o[i];
  }
};


// ------------------------------------------------ SECDED table decoders
// Extended Hamming (2^m bits, bit 0 = overall parity P): the same decisions
// as DecodeOp<m, true> -- P = 1: correct position s (s = 0: the parity bit);
// P = 0, s != 0: double error detected, data left as received -- with the
// syndrome from tables instead of POPCs.  The lane reads its 2^m words
// through the swizzled tensor-map layout (swz_unit), like DecodeOp<m, true>.
template <int IN_W>
__device__ __forceinline__ void load_swizzled(const uint32_t* __restrict__ tile, uint32_t (&w)[IN_W]) {
  constexpr int CPL = IN_W / 4;
  const uint32_t l = threadIdx.x & 31u;
#pragma unroll
  for (int u = 0; u < CPL; ++u) {
    const uint4 v = reinterpret_cast<const uint4*>(tile)[swz_unit<IN_W>(l * CPL + u)];
    w[4 * u] = v.x;
    w[4 * u + 1] = v.y;
    w[4 * u + 2] = v.z;
    w[4 * u + 3] = v.w;
  }
}


// (8,4): a codeword is one byte; per-lane replicated 256-entry table of 8-byte
// entries {final data nibble replicated into all eight nibbles, flags} (64 KB),
// placed as in DecodeLut3Op.
struct DecodeSecded3Op {
  static constexpr int NCOUNT = 2;
  static constexpr int IN_W = 8, OUT_W = 4, IN_BITS = 8;
  static constexpr bool HAS_SIDE = true;
  static constexpr bool SWZ = true;
  static constexpr int SHARED = 256 * 32 * 8;
  struct Args {
    CUtensorMap tmap;
  };
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) c += __popc(sw[i] & 0x40404040u);
    return c;
  }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&sw)[8]) {
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) c += __popc(sw[i] & 0x80808080u);
    return c;
  }

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    uint2* L = reinterpret_cast<uint2*>(sh);
    for (int e = tid; e < 256 * 32; e += nth) {
      uint32_t v = static_cast<uint32_t>(e >> 5);  // bit p = position p, bit 0 = P
      const uint32_t s = syndrome_cw<3>(v, 0u);
      const uint32_t par = static_cast<uint32_t>(__popc(v)) & 1u;
      v ^= par << s;
      const uint32_t d = ((v >> 3) & 1u) | ((v >> 4) & 0xEu);  // positions 3, 5, 6, 7
      L[e] = make_uint2(d * 0x11111111u, secded_flags(s, par));
    }
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&,
                                              const uint8_t* sh) {
    uint32_t w[8];
    load_swizzled<8>(in, w);
    __syncwarp();  // every lane has its input words: the tile may be overwritten in place
    const uint32_t lane8 = (threadIdx.x & 31u) << 3;
    uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      // (x * 32 + lane) * 8 with x = byte c of the lane's words
      const int bo = 8 * (c & 3);
      const uint32_t off = ((bo <= 8 ? (w[c >> 2] << (8 - bo)) : (w[c >> 2] >> (bo - 8))) & 0xFF00u) | lane8;
      const uint2 e = *reinterpret_cast<const uint2*>(sh + off);
      o[c >> 3] |= e.x & (0xFu << ((4 * c) & 31));
      side[c >> 2] |= e.y << bo;
    }
    *reinterpret_cast<uint4*>(out) = make_uint4(o[0], o[1], o[2], o[3]);
  }
};

// (16,11): positions 1..15 through the (15,11) table g_lut15 (corrected data |
// s << 12), P = parity of the 16 bits (one POPC); a detected double error
// takes the uncorrected data back by XOR-ing the data bit of position s
// (per-lane table F[s], 2 KB, conflict-free).
struct DecodeSecded4Op {
  static constexpr int NCOUNT = 2;
  static constexpr int IN_W = 16, OUT_W = 11, IN_BITS = 16;
  static constexpr bool HAS_SIDE = true;
  static constexpr bool SWZ = true;
  static constexpr int SHARED = 32768 * 2 + 16 * 32 * 4;
  struct Args {
    CUtensorMap tmap;
  };
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return DecodeSecded3Op::count0(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&sw)[8]) { return DecodeSecded3Op::count1(sw); }

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    __shared__ __align__(8) uint64_t tbar;
    cta_table_copy_begin(sh, g_lut15, 32768 * 2, tid, &tbar);  // one TMA copy of the 64 KB table
    uint32_t* F = reinterpret_cast<uint32_t*>(sh + 32768 * 2);
    for (int e = tid; e < 16 * 32; e += nth) {  // F[s][lane] = the data bit of position s (0 if parity)
      const uint32_t v = (e >> 5) ? (1u << (e >> 5)) : 0u;
      uint32_t raw = 0;
#pragma unroll
      for (int g = 1; g < 4; ++g) raw |= (v >> (g + 2)) & dmask(g);
      F[e] = raw;
    }
    __syncthreads();  // the barrier is initialised before anyone waits on it
    cta_table_copy_wait(&tbar);
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&,
                                              const uint8_t* sh) {
    uint32_t w[16];
    load_swizzled<16>(in, w);
    __syncwarp();
    const uint32_t lane4 = (threadIdx.x & 31u) << 2;
    uint32_t o[11];
#pragma unroll
    for (int i = 0; i < 11; ++i) o[i] = 0;
    uint32_t S4 = 0, P4 = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t cw = (w[c >> 1] >> (16 * (c & 1))) & 0xFFFFu;
      const uint32_t e = *reinterpret_cast<const uint16_t*>(sh + (cw & 0xFFFEu));  // positions 1..15, x 2
      const uint32_t s = e >> 12, par = static_cast<uint32_t>(__popc(cw)) & 1u;
      const uint32_t f = *reinterpret_cast<const uint32_t*>(sh + 65536 + (s << 7) + lane4);
      const uint32_t d = (e ^ (par ? 0u : f)) & 0x7FFu;
      const int b = 11 * c, q = b >> 5, r = b & 31;
      o[q] |= d << r;
      if (r > 21) o[q + 1] |= d >> (32 - r);
      S4 |= s << (8 * (c & 3));
      P4 |= par << (8 * (c & 3) + 6);
      if ((c & 3) == 3) {
        side[c >> 2] |= secded_flags4(S4, P4);
        S4 = P4 = 0;
      }
    }
#pragma unroll
    for (int i = 0; i < 11; ++i) out[i] = o[i];
  }
};

// (32,26): a codeword is one word; positions 1..15 and 17..31 through the
// half-word table g_lut15raw (uncorrected RR | syndrome part << 11 | parity
// << 15) as in DecodeLut5Op; P = both parities ^ bit 16 ^ bit 0 -- no POPC.
struct DecodeSecded5Op {
  static constexpr int NCOUNT = 2;
  static constexpr int IN_W = 32, OUT_W = 26, IN_BITS = 32;
  static constexpr bool HAS_SIDE = true;
  static constexpr bool SWZ = true;
  static constexpr int SHARED = 32768 * 2 + 32 * 32 * 4;
  struct Args {
    CUtensorMap tmap;
  };
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&sw)[8]) { return DecodeSecded3Op::count0(sw); }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&sw)[8]) { return DecodeSecded3Op::count1(sw); }

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) { DecodeLut5Op::cta_init(sh, tid, nth); }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&,
                                              const uint8_t* sh) {
    uint32_t w[32];
    load_swizzled<32>(in, w);
    __syncwarp();
    const uint32_t lane4 = (threadIdx.x & 31u) << 2;
    uint32_t o[26];
#pragma unroll
    for (int i = 0; i < 26; ++i) o[i] = 0;
    uint32_t S4 = 0, P4 = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t x = w[c];
      const uint32_t elo = *reinterpret_cast<const uint16_t*>(sh + (x & 0xFFFEu));          // positions 1..15
      const uint32_t h = x >> 16;                                                            // 16, 17..31
      const uint32_t ehi = *reinterpret_cast<const uint16_t*>(sh + (h & 0xFFFEu));
      const uint32_t t = elo ^ ehi;
      const uint32_t s = ((t >> 11) & 0xFu) | ((((ehi >> 15) ^ h) & 1u) << 4);
      const uint32_t par = ((t >> 15) ^ h ^ x) & 1u;  // parities of both halves, bit 16, bit 0
      const uint32_t f = *reinterpret_cast<const uint32_t*>(sh + 65536 + (s << 7) + lane4);
      const uint32_t d = ((elo & 0x7FFu) | ((h << 10) & 0x3FFF800u)) ^ (par ? f : 0u);
      put_bits(o, 26 * c, d, 26);
      S4 |= s << (8 * (c & 3));
      P4 |= par << (8 * (c & 3) + 6);
      if ((c & 3) == 3) {
        side[c >> 2] |= secded_flags4(S4, P4);
        S4 = P4 = 0;
      }
    }
#pragma unroll
    for (int i = 0; i < 26; ++i) out[i] = o[i];
  }
};

// SECDED: set bit 0 (position 0) to the parity of positions 1..n and emit the
// whole 2^m-bit codeword at lane-stream bit b.
template <int M, int NO>
__device__ __forceinline__ void put_ext_codeword(uint32_t (&o)[NO], int b, uint32_t lo, uint32_t hi) {
  if constexpr (M == 6) {
    lo = (lo & ~1u) | (static_cast<uint32_t>(__popc((lo & ~1u) ^ hi)) & 1u);
    o[b >> 5] = lo;
    o[(b >> 5) + 1] = hi;
  } else {
    constexpr int W = 1 << M;
    constexpr uint32_t mask = (W == 32) ? 0xFFFFFFFFu : ((1u << W) - 1u);
    lo &= mask & ~1u;
    lo |= static_cast<uint32_t>(__popc(lo)) & 1u;
    put_bits(o, b, lo, W);
  }
}

template <int M, bool EXT = false>
struct EncodeOp {
  static constexpr int CW_BITS = EXT ? (1 << M) : Geo<M>::n;
  static constexpr int IN_W = Geo<M>::k;
  static constexpr int OUT_W = CW_BITS;
  static constexpr int IN_BITS = Geo<M>::k;
  static constexpr bool HAS_SIDE = false;
  static constexpr int NCOUNT = 1;
  static constexpr int SHARED = 0;
  // SECDED (32,26) / (64,57) output: a lane's 2^m-word stride would put every
  // lane's stores in the same banks, so the tile is written through the
  // swizzle (swz_unit) and stored by a tensor map.
  static constexpr bool SWZ_OUT = EXT && M >= 5;
  struct NoArgs {};
  struct OutArgs {
    CUtensorMap tmap_out;
  };
  using Args = typename std::conditional<SWZ_OUT, OutArgs, NoArgs>::type;
  __device__ __forceinline__ static void cta_init(uint8_t*, int, int) {}

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                  uint32_t (&)[8], uint64_t, int, const Args&, const uint8_t*) {
    constexpr int n = Geo<M>::n, k = Geo<M>::k;
    uint32_t w[k];
#pragma unroll
    for (int i = 0; i < k; ++i) w[i] = in[i];
    uint32_t o[OUT_W];
#pragma unroll
    for (int i = 0; i < OUT_W; ++i) o[i] = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      uint32_t dlo, dhi = 0;
      if constexpr (M <= 5) {
        dlo = take_bits(w, c * k);
        if constexpr (k < 32) dlo &= (1u << k) - 1u;
      } else {
        dlo = take_bits(w, c * k) & ((1u << 26) - 1u);
        dhi = take_bits(w, c * k + 26) & 0x7FFFFFFFu;
      }
      uint32_t lo, hi;
      encode_cw<M>(dlo, dhi, lo, hi);
      if constexpr (EXT) put_ext_codeword<M>(o, c * CW_BITS, lo, hi);
      else put_codeword<M>(o, c * n, lo, hi);
    }
    if constexpr (SWZ_OUT) {  // `out` is the output tile base
      const uint32_t l = threadIdx.x & 31u;
#pragma unroll
      for (int u = 0; u < OUT_W / 4; ++u)
        reinterpret_cast<uint4*>(out - l * OUT_W)[swz_unit<OUT_W>(l * (OUT_W / 4) + u)] =
            make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < OUT_W; ++i) out[i] = o[i];
    }
    (void)n;
  }
};

// Table encoders (m = 3, 4; perfect and SECDED): the codeword is linear in
// the data, so it is the XOR of one table entry per data chunk, each entry
// the whole codeword (in stream form) of that chunk alone.  m = 3: a data
// byte is two codewords, one 256-entry lookup per pair; m = 4: two lookups
// (data bits 0..5, 6..10) per codeword.  Per-lane replicated tables (entry e
// for lane l at word e * 32 + l: conflict free), built at CTA start from
// encode_cw itself.  No POPC: the POPC encoder is XU-bound at m = 3, 4.
template <int M, bool EXT = false>
struct EncodeLutOp {
  static_assert(M == 3 || M == 4, "table encoders: m = 3, 4");
  static constexpr int CW_BITS = EXT ? (1 << M) : Geo<M>::n;
  static constexpr int k = Geo<M>::k;
  static constexpr int IN_W = k, OUT_W = CW_BITS, IN_BITS = k;
  static constexpr bool HAS_SIDE = false;
  static constexpr int NCOUNT = 1;
  static constexpr int ENTRIES = (M == 3) ? 256 : 64 + 32;
  static constexpr int SHARED = ENTRIES * 32 * 4;
  // (16,11) SECDED tiles (a lane's 16 output words: bank conflicts on a linear layout) go out
  // through the 128-byte swizzle and a tensor-map store, as EncodeOp<5/6, true>: 0.81 -> 0.88 of
  // the copy peak; (8,4) measured better linear (0.88 vs 0.85)
  static constexpr bool SWZ_OUT = EXT && M == 4;
  struct NoArgs {};
  struct OutArgs {
    CUtensorMap tmap_out;
  };
  using Args = typename std::conditional<SWZ_OUT, OutArgs, NoArgs>::type;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&)[8]) { return 0; }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }

  // one codeword of data d, in stream form (perfect: positions 1..n; SECDED: bit 0 = P)
  __device__ __forceinline__ static uint32_t codeword(uint32_t d) {
    uint32_t lo, hi;
    encode_cw<M>(d, 0u, lo, hi);
    if constexpr (EXT) return (lo & ~1u) | (static_cast<uint32_t>(__popc(lo & ~1u)) & 1u);
    else return lo >> 1;
  }

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    uint32_t* T = reinterpret_cast<uint32_t*>(sh);
    for (int e = tid; e < ENTRIES * 32; e += nth) {
      const uint32_t x = static_cast<uint32_t>(e >> 5);
      if constexpr (M == 3) T[e] = codeword(x & 0xFu) | (codeword(x >> 4) << CW_BITS);  // a pair
      else T[e] = x < 64 ? codeword(x) : codeword((x - 64) << 6);
    }
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&)[8], uint64_t, int, const Args&, const uint8_t* sh) {
    uint32_t w[k];
#pragma unroll
    for (int i = 0; i < k; ++i) w[i] = in[i];
    const uint32_t lane4 = (threadIdx.x & 31u) << 2;
    uint32_t o[OUT_W];
#pragma unroll
    for (int i = 0; i < OUT_W; ++i) o[i] = 0;
    if constexpr (M == 3) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {  // codewords 2q, 2q+1 = data byte q
        const uint32_t off = (((w[q >> 2] >> (8 * (q & 3))) & 0xFFu) << 7) | lane4;
        put_bits(o, 2 * q * CW_BITS, *reinterpret_cast<const uint32_t*>(sh + off), 2 * CW_BITS);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const uint32_t d = take_bits(w, c * k) & 0x7FFu;
        const uint32_t v = *reinterpret_cast<const uint32_t*>(sh + (((d & 63u) << 7) | lane4)) ^
                           *reinterpret_cast<const uint32_t*>(sh + ((((d >> 6) + 64u) << 7) | lane4));
        put_bits(o, c * CW_BITS, v, CW_BITS);
      }
    }
    if constexpr (SWZ_OUT) {  // `out` is the output tile base
      const uint32_t l = threadIdx.x & 31u;
#pragma unroll
      for (int u = 0; u < OUT_W / 4; ++u)
        reinterpret_cast<uint4*>(out - l * OUT_W)[swz_unit<OUT_W>(l * (OUT_W / 4) + u)] =
            make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < OUT_W; ++i) out[i] = o[i];
    }
  }
};

// m = 5 table encoder (perfect and SECDED): the codeword is linear in the 26
// data bits, so it is the XOR of four table entries, one per data chunk (bits
// 0..6, 7..13, 14..19, 20..25), each entry the whole codeword (stream form;
// SECDED: with its overall-parity contribution in bit 0) of that chunk alone.
// Per-lane replicated (entry e for lane l at word e * 32 + l: conflict free),
// 384 entries = 48 KB, built at CTA start from encode_cw itself.  The POPC
// encoder needs 5 (SECDED 6) POPCs per codeword and is XU-bound there.
template <bool EXT>
struct EncodeLut5Op {
  static constexpr int CW_BITS = EXT ? 32 : 31;
  static constexpr int k = 26;
  static constexpr int IN_W = k, OUT_W = CW_BITS, IN_BITS = k;
  static constexpr bool HAS_SIDE = false;
  static constexpr int NCOUNT = 1;
  static constexpr int ENTRIES = 128 + 128 + 64 + 64;
  static constexpr int SHARED = ENTRIES * 32 * 4;
  static constexpr bool SWZ_OUT = EXT;  // (32,26) tiles: the swizzled tensor-map store of EncodeOp<5, true>
  struct NoArgs {};
  struct OutArgs {
    CUtensorMap tmap_out;
  };
  using Args = typename std::conditional<SWZ_OUT, OutArgs, NoArgs>::type;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&)[8]) { return 0; }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }

  __device__ __forceinline__ static uint32_t codeword(uint32_t d) {
    uint32_t lo, hi;
    encode_cw<5>(d, 0u, lo, hi);
    if constexpr (EXT) return (lo & ~1u) | (static_cast<uint32_t>(__popc(lo & ~1u)) & 1u);
    else return lo >> 1;
  }

  __device__ __forceinline__ static void cta_init(uint8_t* sh, int tid, int nth) {
    uint32_t* T = reinterpret_cast<uint32_t*>(sh);
    for (int e = tid; e < ENTRIES * 32; e += nth) {
      const uint32_t x = static_cast<uint32_t>(e >> 5);
      const uint32_t d = x < 128 ? x : x < 256 ? (x - 128) << 7 : x < 320 ? (x - 256) << 14 : (x - 320) << 20;
      T[e] = codeword(d);
    }
  }

  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&)[8], uint64_t, int, const Args&, const uint8_t* sh) {
    uint32_t w[k];
#pragma unroll
    for (int i = 0; i < k; ++i) w[i] = in[i];
    const uint32_t lane4 = (threadIdx.x & 31u) << 2;
    const uint8_t* t0 = sh + lane4;
    const uint8_t* t1 = sh + (128u << 7) + lane4;
    const uint8_t* t2 = sh + (256u << 7) + lane4;
    const uint8_t* t3 = sh + (320u << 7) + lane4;
    uint32_t o[OUT_W];
#pragma unroll
    for (int i = 0; i < OUT_W; ++i) o[i] = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t d = take_bits(w, c * k);
      const uint32_t v = *reinterpret_cast<const uint32_t*>(t0 + ((d & 0x7Fu) << 7)) ^
                         *reinterpret_cast<const uint32_t*>(t1 + (((d >> 7) & 0x7Fu) << 7)) ^
                         *reinterpret_cast<const uint32_t*>(t2 + (((d >> 14) & 0x3Fu) << 7)) ^
                         *reinterpret_cast<const uint32_t*>(t3 + (((d >> 20) & 0x3Fu) << 7));
      if constexpr (EXT) o[c] = v;
      else put_bits(o, c * CW_BITS, v, CW_BITS);
    }
    if constexpr (SWZ_OUT) {  // `out` is the output tile base
      const uint32_t l = threadIdx.x & 31u;
#pragma unroll
      for (int u = 0; u < OUT_W / 4; ++u)
        reinterpret_cast<uint4*>(out - l * OUT_W)[swz_unit<OUT_W>(l * (OUT_W / 4) + u)] =
            make_uint4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < OUT_W; ++i) out[i] = o[i];
    }
  }
};

// splitmix64 output function (Steele, Lea & Flood 2014) -- written here
// independently of oracle/oracle.c; the two are compared byte for byte.
__device__ __forceinline__ uint64_t sm64_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int M, bool EXT = false>
struct GenerateOp {
  static constexpr int CW_BITS = EXT ? (1 << M) : Geo<M>::n;
  static constexpr int IN_W = 0;
  static constexpr int OUT_W = CW_BITS;
  static constexpr int IN_BITS = 0;
  static constexpr bool HAS_SIDE = false;
  static constexpr int NCOUNT = 1;
  static constexpr int SHARED = 0;
  struct Args {
    uint64_t seed, c_first, thresh, q2thresh;
    int all;
  };
  __device__ __forceinline__ static void cta_init(uint8_t*, int, int) {}

  __device__ __forceinline__ static void lane(const uint32_t*, uint32_t* __restrict__ out, uint32_t (&)[8],
                                                  uint64_t cw0, int valid, const Args& a, const uint8_t*) {
    constexpr int n = Geo<M>::n, k = Geo<M>::k;
    constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
    uint32_t o[OUT_W];
#pragma unroll
    for (int i = 0; i < OUT_W; ++i) o[i] = 0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint64_t g = a.c_first + cw0 + c;
      const uint64_t base = a.seed + 4 * g * kGamma;
      const uint64_t u0 = sm64_mix(base + 1 * kGamma);
      const uint64_t u1 = sm64_mix(base + 2 * kGamma);
      const uint64_t u2 = sm64_mix(base + 3 * kGamma);
      const uint64_t u3 = sm64_mix(base + 4 * kGamma);
      uint32_t dlo, dhi = 0;
      if constexpr (M <= 5) {
        dlo = static_cast<uint32_t>(u0) & ((1u << k) - 1u);
      } else {
        dlo = static_cast<uint32_t>(u0) & ((1u << 26) - 1u);
        dhi = static_cast<uint32_t>(u0 >> 26) & 0x7FFFFFFFu;
      }
      uint32_t lo, hi;
      encode_cw<M>(dlo, dhi, lo, hi);
      const bool ev = a.all || (u1 < a.thresh);
      const bool two = (u2 >> 32) < a.q2thresh;
      uint64_t f;
      if constexpr (EXT) {  // bit indices over the whole 2^m-bit codeword (0 = the parity bit)
        lo = (lo & ~1u) | (static_cast<uint32_t>(__popc((lo & ~1u) ^ hi)) & 1u);
        const uint32_t b1 = __umulhi(static_cast<uint32_t>(u3), static_cast<uint32_t>(CW_BITS));
        uint32_t b2 = b1 + 1u + __umulhi(static_cast<uint32_t>(u3 >> 32), static_cast<uint32_t>(CW_BITS - 1));
        b2 = (b2 >= static_cast<uint32_t>(CW_BITS)) ? b2 - CW_BITS : b2;
        f = ev ? (1ull << b1) : 0ull;
        f ^= (ev && two) ? (1ull << b2) : 0ull;
      } else {
        const uint32_t p1 = 1u + __umulhi(static_cast<uint32_t>(u3), static_cast<uint32_t>(n));
        uint32_t p2 = p1 + __umulhi(static_cast<uint32_t>(u3 >> 32), static_cast<uint32_t>(n - 1));  // (p1-1)+1+x
        p2 = (p2 >= static_cast<uint32_t>(n) ? p2 - n : p2) + 1u;
        f = ev ? (1ull << p1) : 0ull;
        f ^= (ev && two) ? (1ull << p2) : 0ull;
      }
      lo ^= static_cast<uint32_t>(f);
      hi ^= static_cast<uint32_t>(f >> 32);
      if (c >= valid) {  // past the end of the packet (tail only): emit zeros
        lo = 0;
        hi = 0;
      }
      if constexpr (EXT) {
        if constexpr (M == 6) {
          o[2 * c] = lo;
          o[2 * c + 1] = hi;
        } else {
          put_bits(o, c * CW_BITS, lo & ((CW_BITS == 32) ? 0xFFFFFFFFu : ((1u << CW_BITS) - 1u)), CW_BITS);
        }
      } else {
        put_codeword<M>(o, c * n, lo, hi);
      }
    }
#pragma unroll
    for (int i = 0; i < OUT_W; ++i) out[i] = o[i];
  }
};
// ------------------------------------------------------------------ kernels
template <class Op, class = void>
struct Swizzled {
  static constexpr bool value = false;
};
template <class Op>
struct Swizzled<Op, decltype(void(Op::SWZ))> {
  static constexpr bool value = Op::SWZ;
};

template <class Op, class = void>
struct SwizzledOut {
  static constexpr bool value = false;
};
template <class Op>
struct SwizzledOut<Op, decltype(void(Op::SWZ_OUT))> {
  static constexpr bool value = Op::SWZ_OUT;
};

// Ops that count inside the lane function (LANE_COUNT) return the count from
// lane_count(); the others are counted from their side words by count0().
template <class Op, class = void>
struct LaneCount {
  static constexpr bool value = false;
};
template <class Op>
struct LaneCount<Op, decltype(void(Op::LANE_COUNT))> {
  static constexpr bool value = Op::LANE_COUNT;
};

template <class Op>
__device__ __forceinline__ uint32_t run_lane(const uint32_t* in, uint32_t* out, uint32_t (&side)[8], uint64_t g,
                                             int valid, const typename Op::Args& args, const uint8_t* sh) {
  if constexpr (LaneCount<Op>::value) {
    return Op::lane_count(in, out, side, g, valid, args, sh);
  } else {
    Op::lane(in, out, side, g, valid, args, sh);
    if constexpr (Op::HAS_SIDE) return Op::count0(side);
    return 0;
  }
}

template <class Op>
struct TileBytes {
  static constexpr int IN = Op::IN_W * 128;   // 32 lanes x IN_W words x 4 B
  static constexpr int OUT = Op::OUT_W * 128;
  static constexpr bool SWZ = Swizzled<Op>::value;
  // output tiles written through the same swizzle and stored by a tensor map
  static constexpr bool SWZ_OUT = SwizzledOut<Op>::value;
  __host__ __device__ static constexpr uint32_t staged_out(uint32_t i) {
    if constexpr (SWZ_OUT) {
      return (swz_unit<Op::OUT_W>(i >> 4) << 4) | (i & 15u);
    } else {
      return i;
    }
  }
  // shared-memory byte offset of tile byte i (128-byte swizzle for SWZ tiles)
  __host__ __device__ static constexpr uint32_t staged(uint32_t i) {
    if constexpr (SWZ) {
      return (swz_unit<Op::IN_W>(i >> 4) << 4) | (i & 15u);
    } else {
      return i;
    }
  }
};

// Issue the TMA load of one input tile into a stage.
template <class Op>
__device__ __forceinline__ void load_tile(uint8_t* stage, const uint8_t* in, uint64_t t, uint64_t* bar,
                                          const typename Op::Args& args, uint64_t pol) {
  constexpr int IN = TileBytes<Op>::IN;
  mbar_arrive_expect_tx(bar, IN);
  if constexpr (TileBytes<Op>::SWZ) {
    if constexpr (Op::IN_W / 32 >= 2) tensor_g2s_3d(stage, &args.tmap, 0, static_cast<int>(t * 32), 0, bar, pol);
    else tensor_g2s_2d(stage, &args.tmap, 0, static_cast<int>(t * (IN / 128)), bar, pol);
  } else {
    bulk_g2s(stage, in + t * IN, IN, bar, pol);
  }
}

// The ragged last tile (rem < 1024 codewords) of a launch: bounded 16-byte
// loads with zero fill, input pad bits past rem codewords cleared, the same
// lane function, bounded stores.  Runs in the warp that owns the tile.
template <class Op>
__device__ __noinline__ uint32_t run_tail_tile(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                               uint8_t* __restrict__ side, uint64_t tile, uint32_t rem,
                                               uint64_t in_total, uint64_t out_total, uint8_t* ibuf,
                                               uint32_t* obuf, int lane, const typename Op::Args& args,
                                               const uint8_t* sh, uint32_t& cnt2) {
  constexpr int IN = TileBytes<Op>::IN, OUT = TileBytes<Op>::OUT;
  if constexpr (IN > 0) {
    const uint64_t ib0 = tile * IN;
    const uint64_t nb = in_total - ib0;  // bytes of this tile that exist (< IN)
    using TB = TileBytes<Op>;
    for (int i = lane * 16; i < IN; i += 512) {  // 16-byte units, placed as the TMA would place them
      uint8_t* dst = ibuf + TB::staged(i);
      if (static_cast<uint64_t>(i) + 16 <= nb) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(in + ib0 + i);
      } else {
        for (int b = 0; b < 16; ++b) dst[b] = (static_cast<uint64_t>(i + b) < nb) ? in[ib0 + i + b] : 0;
      }
    }
    __syncwarp();
    const uint64_t vbits = static_cast<uint64_t>(rem) * Op::IN_BITS;  // clear the input pad bits
    uint32_t* iw = reinterpret_cast<uint32_t*>(ibuf);
    for (int i = lane; i < IN / 4; i += 32) {
      const uint64_t b = static_cast<uint64_t>(i) * 32;
      uint32_t& x = iw[TB::staged(4u * i) / 4];
      if (b >= vbits) x = 0;
      else if (b + 32 > vbits) x &= (1u << (vbits - b)) - 1u;
    }
    __syncwarp();
  }
  const int valid = max(0, min(32, static_cast<int>(rem) - lane * 32));
  uint32_t sidew[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const uint32_t lc = run_lane<Op>(reinterpret_cast<const uint32_t*>(ibuf) + (TileBytes<Op>::SWZ ? 0 : lane * Op::IN_W),
                                   obuf + lane * Op::OUT_W, sidew, tile * kTileCw + lane * 32, valid, args, sh);
  __syncwarp();
  const uint64_t ob0 = tile * OUT;
  const uint64_t nbo = out_total - ob0;
  const uint8_t* ob = reinterpret_cast<const uint8_t*>(obuf);
  for (int i = lane * 16; static_cast<uint64_t>(i) < nbo; i += 512) {  // 16-byte units, un-swizzled
    const uint8_t* srcu = ob + TileBytes<Op>::staged_out(static_cast<uint32_t>(i));
    if (static_cast<uint64_t>(i) + 16 <= nbo) {
      *reinterpret_cast<uint4*>(out + ob0 + i) = *reinterpret_cast<const uint4*>(srcu);
    } else {
      for (int b = 0; static_cast<uint64_t>(i + b) < nbo; ++b) out[ob0 + i + b] = srcu[b];
    }
  }
  uint32_t cnt = 0;
  if constexpr (Op::HAS_SIDE) {
    if (side != nullptr) {
      uint8_t* sp = side + tile * kTileCw + lane * 32;
      for (int c = 0; c < valid; ++c) sp[c] = static_cast<uint8_t>(sidew[c >> 2] >> (8 * (c & 3)));
    }
    cnt = lc;  // codewords past `valid` decode zeros: s = 0, no flags
    if constexpr (Op::NCOUNT > 1) cnt2 += Op::count1(sidew);
  }
  return cnt;
}

// Persistent warp-tile pipeline, one launch per call: each warp owns STAGES
// tile buffers filled by TMA bulk loads (mbarrier-tracked) and walks full tiles
// gw, gw + nw, ...; the warp next in line after the last full tile also takes
// the ragged tail.  Decoders write their (smaller) output tile IN PLACE over
// the consumed input tile and bulk-store it from there; the stage is refilled
// at the next iteration, once that store has read it.  Ops whose output is
// larger than the input (encode, generate) use two separate output buffers.
// The corrected count (zeroed on the stream by the launcher) is reduced
// warp -> CTA -> one atomic.
template <class Op, bool WANT_IN_PLACE = true>
struct TileLayout {
  static constexpr int IN = TileBytes<Op>::IN, OUT = TileBytes<Op>::OUT;
  static constexpr bool IN_PLACE = WANT_IN_PLACE && IN > 0 && OUT <= IN;
  static constexpr int OUT_BUFS = IN_PLACE ? 0 : 2;
  static constexpr bool ALIGN1K = TileBytes<Op>::SWZ || TileBytes<Op>::SWZ_OUT;
  // byte offset of the output buffers (after the input stages)
  __host__ __device__ static constexpr int out_off(int stages) {
    return ALIGN1K ? (stages * IN + 1023) / 1024 * 1024 : stages * IN;
  }
  // swizzled buffers stay 1024-byte aligned from warp to warp
  __host__ __device__ static constexpr int warp_bytes(int stages) {
    return ALIGN1K ? (out_off(stages) + OUT_BUFS * OUT + 1023) / 1024 * 1024 : stages * IN + OUT_BUFS * OUT;
  }
};

#ifdef HAM_TIMING  // debug builds only: per-CTA %globaltimer stamps (tools/timing_probe.py)
__device__ unsigned long long g_timing[1024 * 4];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define HAM_STAMP(i) \
  if (threadIdx.x == 0 && blockIdx.x < 1024) g_timing[blockIdx.x * 4 + (i)] = gtimer()
#else
#define HAM_STAMP(i)
#endif

// Per-launch scratch for the count and the dynamic tail, one per (device,
// stream) (host map below; never shared by two launches that can run at the
// same time): every CTA adds its partial count to `sum`, and the LAST CTA to
// arrive at `done` writes the total into the caller's count (overwrite, or add
// in accumulate mode) and resets the slot to zero for the stream's next
// launch -- so a call needs no cudaMemsetAsync of the count before its kernel.
// `claim` hands out the dynamically scheduled tail tiles.
struct LaunchSlot {
  unsigned long long sum[2];
  unsigned int claim;
  unsigned int done;
};
constexpr int kSlots = 256;
__device__ LaunchSlot g_slots[kSlots];  // zero-initialised at module load

constexpr uint32_t kNoTile = 0xFFFFFFFFu;

template <class Op, int WARPS, int STAGES, bool INPLACE>
__global__ void __launch_bounds__(WARPS * 32, 1)
    tiles_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, uint8_t* __restrict__ side,
                 uint64_t n_full, uint32_t rem, uint64_t in_total, uint64_t out_total,
                 unsigned long long* __restrict__ counter, int store_count, LaunchSlot* __restrict__ slot,
                 uint64_t static_end, int accumulate, const __grid_constant__ typename Op::Args args) {
  using TL = TileLayout<Op, INPLACE>;
  constexpr int IN = TL::IN, OUT = TL::OUT;
  constexpr int WARP_SMEM = TL::warp_bytes(STAGES);
  static_assert(STAGES <= 32, "stage tile ids live one per lane");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned long long block_cnt[2];

  HAM_STAMP(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* const sh = smem;  // Op::SHARED bytes of CTA-wide tables first
  // 128-byte-swizzled TMA destinations must be 1024-byte aligned
  uint8_t* const tiles = smem + Op::SHARED +
                         ((TileBytes<Op>::SWZ || TileBytes<Op>::SWZ_OUT)
                              ? ((1024u - (smem_addr(smem + Op::SHARED) & 1023u)) & 1023u)
                              : 0u);
  uint8_t* wbase = tiles + warp * WARP_SMEM;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tiles + WARPS * WARP_SMEM) + warp * STAGES;
  // global warp index, CTA-minor: the last, partial round of tiles (n_full % nw
  // of them) lands on one warp of as many different SMs as possible rather
  // than on every warp of the first few CTAs
  const uint64_t gw = static_cast<uint64_t>(warp) * gridDim.x + blockIdx.x;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * WARPS;
  const uint64_t pol = policy_evict_first();
  // Schedule: tiles [0, static_end) round-robin (warp gw takes gw, gw + nw, ...:
  // rs = static_end / nw of them each, no communication); tiles [static_end,
  // n_full] -- n_full itself being the ragged tail when rem > 0 -- claimed one at
  // a time from slot->claim, so the last rounds balance across warps and SMs.
  // Without a dynamic part (static_end == n_full) the warp next in line takes
  // the tail, as before.
  const bool dyn = static_end < n_full;
  const uint64_t rs = dyn ? static_end / nw : ~0ull;
  bool exhausted = false, do_tail = false;
  // tile of this warp's j-th sequence slot; claims are made by lane 0 in sequence
  // order (every lane calls this, uniformly)
  auto seq_tile = [&](uint64_t j) -> uint32_t {
    if (!dyn) {
      const uint64_t t = gw + j * nw;
      return t < n_full ? static_cast<uint32_t>(t) : kNoTile;
    }
    if (j < rs) return static_cast<uint32_t>(gw + j * nw);
    if (exhausted) return kNoTile;
    uint32_t d = 0;
    if (lane == 0) d = atomicAdd(&slot->claim, 1u);
    d = __shfl_sync(0xffffffffu, d, 0);
    const uint64_t t = static_end + d;
    if (t >= n_full) {  // the ragged tail (t == n_full, rem > 0) or nothing: no more tiles
      exhausted = true;
      if (t == n_full && rem > 0) do_tail = true;
      return kNoTile;
    }
    return static_cast<uint32_t>(t);
  };

  if (threadIdx.x < 2) block_cnt[threadIdx.x] = 0;
  uint32_t stage_tile = kNoTile;  // lane s: the tile in stage s
  if constexpr (IN > 0) {
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
      fence_mbar_init();
    }
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      const uint32_t t = seq_tile(s);
      if (lane == s) stage_tile = t;
      if (lane == 0 && t != kNoTile) load_tile<Op>(wbase + s * IN, in, t, &bars[s], args, pol);
    }
    __syncwarp();
  }

  // the CTA's tables are built while the first tiles are in flight (the
  // prologue's TMA loads land in the warp stages, disjoint from the tables)
  if constexpr (Op::SHARED > 0) {
    Op::cta_init(sh, threadIdx.x, blockDim.x);
    __syncthreads();
  }

  uint32_t cnt = 0, cnt2 = 0;
  for (uint32_t it = 0;; ++it) {
    const int st = static_cast<int>(it % STAGES);
    uint64_t t;
    if constexpr (IN > 0) {
      t = (it < rs) ? gw + static_cast<uint64_t>(it) * nw : __shfl_sync(0xffffffffu, stage_tile, st);
      if (t >= n_full) break;  // kNoTile, or past the full tiles (static schedule)
    } else {
      t = gw + static_cast<uint64_t>(it) * nw;  // no input: a plain grid-stride walk
      if (t >= n_full) break;
    }
    uint32_t* obuf;
    if constexpr (TL::IN_PLACE) {
      mbar_wait(&bars[st], (it / STAGES) & 1u);
#ifdef HAM_TIMING
      if (it == 0) HAM_STAMP(1);
#endif
      obuf = reinterpret_cast<uint32_t*>(wbase + st * IN);
    } else {
      if constexpr (IN > 0) mbar_wait(&bars[st], (it / STAGES) & 1u);
      obuf = reinterpret_cast<uint32_t*>(wbase + TL::out_off(STAGES) + (it & 1u) * OUT);
      if (lane == 0) bulk_wait_read<1>();  // the store issued two tiles ago has read obuf
      __syncwarp();
    }
    uint32_t sidew[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint32_t* ibuf = reinterpret_cast<const uint32_t*>(wbase + st * IN);
    const uint32_t lc = run_lane<Op>(ibuf + (TileBytes<Op>::SWZ ? 0 : lane * Op::IN_W), obuf + lane * Op::OUT_W,
                                     sidew, t * kTileCw + lane * 32, 32, args, sh);
    fence_proxy_async_smem();  // make this lane's st.shared visible to the bulk copy
    __syncwarp();
    if (lane == 0) {
      if constexpr (TileBytes<Op>::SWZ_OUT) {
        if constexpr (Op::OUT_W / 32 >= 2) tensor_s2g_3d(&args.tmap_out, 0, static_cast<int>(t * 32), 0, obuf, pol);
        else tensor_s2g_2d(&args.tmap_out, 0, static_cast<int>(t * (OUT / 128)), obuf, pol);
      } else {
        bulk_s2g(out + t * OUT, obuf, OUT, pol);
      }
      bulk_commit();
    }
    // the tile to prefetch: IN_PLACE refills the stage of the PREVIOUS tile (its in-place
    // store was issued a whole tile ago, so waiting for it to have read shared memory is
    // free); otherwise this tile's stage, whose input the lane function has consumed
    if constexpr (IN > 0) {
      if (!TL::IN_PLACE || it > 0) {
        const int ps = TL::IN_PLACE ? static_cast<int>((it - 1) % STAGES) : st;
        const uint32_t nt = seq_tile(static_cast<uint64_t>(it) + STAGES - (TL::IN_PLACE ? 1 : 0));
        if (lane == ps) stage_tile = nt;
        if (lane == 0 && nt != kNoTile) {
          if constexpr (TL::IN_PLACE) bulk_wait_read<1>();
          load_tile<Op>(wbase + ps * IN, in, nt, &bars[ps], args, pol);
        }
      }
    }
    if constexpr (Op::HAS_SIDE) {
      if (side != nullptr) {
        uint8_t* sp = side + t * kTileCw + lane * 32;
        st_global_cs_v4(sp, sidew[0], sidew[1], sidew[2], sidew[3]);
        st_global_cs_v4(sp + 16, sidew[4], sidew[5], sidew[6], sidew[7]);
      }
      cnt += lc;
      if constexpr (Op::NCOUNT > 1) cnt2 += Op::count1(sidew);
    }
  }
  if (rem > 0 && (dyn ? do_tail : gw == n_full % nw)) {  // the ragged tail tile
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    uint8_t* tail_out = TL::IN_PLACE ? wbase : wbase + TL::out_off(STAGES);
    cnt += run_tail_tile<Op>(in, out, side, n_full, rem, in_total, out_total, wbase,
                             reinterpret_cast<uint32_t*>(tail_out), lane, args, sh, cnt2);
  }
  HAM_STAMP(2);
  if (lane == 0) bulk_wait<0>();
  HAM_STAMP(3);

  if (counter != nullptr || slot != nullptr) {
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if constexpr (Op::NCOUNT > 1) cnt2 = __reduce_add_sync(0xffffffffu, cnt2);
    __syncthreads();
    if (lane == 0 && cnt) atomicAdd(&block_cnt[0], static_cast<unsigned long long>(cnt));
    if constexpr (Op::NCOUNT > 1)
      if (lane == 0 && cnt2) atomicAdd(&block_cnt[1], static_cast<unsigned long long>(cnt2));
    __syncthreads();
    if (slot != nullptr) {
      if (threadIdx.x == 0) {
        // the last CTA to arrive publishes the total and resets the slot (threadFence reduction)
        for (int i = 0; i < Op::NCOUNT; ++i)
          if (block_cnt[i]) atomicAdd(&slot->sum[i], block_cnt[i]);
        __threadfence();
        if (atomicAdd(&slot->done, 1u) == gridDim.x - 1) {
          __threadfence();
          for (int i = 0; i < Op::NCOUNT; ++i) {
            const unsigned long long tot = atomicExch(&slot->sum[i], 0ull);
            if (counter != nullptr) {
              if (accumulate) atomicAdd(&counter[i], tot);
              else counter[i] = tot;
            }
          }
          slot->claim = 0;
          slot->done = 0;
        }
      }
    } else if (threadIdx.x < Op::NCOUNT) {
      const unsigned long long v = block_cnt[threadIdx.x];
      if (store_count) counter[threadIdx.x] = v;  // a single-CTA launch owns the count: no memset needed
      else if (v) atomicAdd(&counter[threadIdx.x], v);
    }
  }
}

// ---------------------------------------------------------- host-side state
thread_local char g_err[512] = "";
thread_local int g_launches = 0;
thread_local int g_grid = 0;

hamming_status set_err(hamming_status s, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return s;
}
hamming_status cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
  return HAMMING_E_CUDA;
}

constexpr int kMaxDev = 64;
std::atomic<int> g_sm_count[kMaxDev];

int sm_count(int dev) {
  int v = (dev >= 0 && dev < kMaxDev) ? g_sm_count[dev].load(std::memory_order_relaxed) : 0;
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    if (dev >= 0 && dev < kMaxDev) g_sm_count[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// One-time kernel attribute setup per (kernel, device) -- the dynamic shared
// memory limit raised to the 227 KB maximum, optionally the full carveout --
// and memoised occupancy per (kernel, device, block size, shared memory), so
// a warm call makes no attribute or occupancy query (latency-bound small
// packet calls of the packet / long-code launchers).
struct OccKey {
  const void* fn;
  int dev, threads;
  size_t smem;
  bool operator<(const OccKey& o) const {
    return std::tie(fn, dev, threads, smem) < std::tie(o.fn, o.dev, o.threads, o.smem);
  }
};
std::mutex g_occ_mu;
std::map<OccKey, int> g_occ;
std::set<std::pair<const void*, int>> g_attr_done;

hamming_status kernel_blocks_per_sm(const void* fn, int dev, int threads, size_t smem, bool carveout, int& occ) {
  std::lock_guard<std::mutex> lock(g_occ_mu);
  const OccKey key{fn, dev, threads, smem};
  const auto it = g_occ.find(key);
  if (it != g_occ.end()) {
    occ = it->second;
    return HAMMING_OK;
  }
  if (g_attr_done.count({fn, dev}) == 0) {
    // the opt-in maximum per block less the kernel's static shared memory
    int optin = 0;
    cudaFuncAttributes fa{};
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess) return cuda_fail(e, "kernel attributes");
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - static_cast<int>(fa.sharedSizeBytes));
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(max dynamic shared memory)");
    if (carveout) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(carveout)");
    }
    g_attr_done.insert({fn, dev});
  }
  int v = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, threads, smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
  occ = std::max(1, v);
  g_occ[key] = occ;
  return HAMMING_OK;
}

// The launch slot of (device, stream): a stream's launches run one after
// another, so they can share one slot; launches on different streams get
// different slots.  nullptr (use the memset + atomics path) when the stream is
// being captured into a CUDA graph -- a replay may run on another stream,
// concurrently with eager launches on this one -- or when every slot is taken.
std::mutex g_slot_mu;
std::map<std::pair<int, cudaStream_t>, int> g_slot_of;
int g_slots_used[kMaxDev];

LaunchSlot* launch_slot(int dev, cudaStream_t st) {
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  // the per-thread default stream has one handle value for every host thread's
  // own stream: launches from two threads could run at once on one slot
  if (st == cudaStreamPerThread) return nullptr;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  static LaunchSlot* base[kMaxDev] = {};
  std::lock_guard<std::mutex> lock(g_slot_mu);
  if (base[dev] == nullptr) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_slots) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    base[dev] = static_cast<LaunchSlot*>(p);
  }
  const auto key = std::make_pair(dev, st);
  auto it = g_slot_of.find(key);
  if (it == g_slot_of.end()) {
    if (g_slots_used[dev] >= kSlots) return nullptr;
    it = g_slot_of.emplace(key, g_slots_used[dev]++).first;
  }
  return base[dev] + it->second;
}

template <class Op, int WARPS, int STAGES, bool INPLACE = true>
struct Launcher {
  static constexpr int IN = TileBytes<Op>::IN, OUT = TileBytes<Op>::OUT;
  static constexpr size_t SMEM = Op::SHARED + ((TileBytes<Op>::SWZ || TileBytes<Op>::SWZ_OUT) ? 1024 : 0) +
                                 static_cast<size_t>(WARPS) * TileLayout<Op, INPLACE>::warp_bytes(STAGES) +
                                 WARPS * STAGES * 8;
  static_assert(SMEM <= 227 * 1024, "shared memory budget");

  // dyn_rounds > 0: the last ~dyn_rounds rounds of tiles are claimed dynamically
  // (decoders with few tiles per warp, where one round is several % of the call)
  static hamming_status run(const uint8_t* in, uint8_t* out, uint8_t* side, uint64_t n_cw, uint64_t in_total,
                            uint64_t out_total, unsigned long long* counter, const typename Op::Args& args,
                            cudaStream_t stream, bool accumulate = false, int dyn_rounds = 0) {
    static std::atomic<int> configured[kMaxDev];
    static std::atomic<int> blocks_per_sm[kMaxDev];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    auto kfn = tiles_kernel<Op, WARPS, STAGES, INPLACE>;
    if (dev < 0 || dev >= kMaxDev || !configured[dev].load(std::memory_order_acquire)) {
      e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(SMEM));
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
#ifdef HAM_CARVEOUT
      e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, HAM_CARVEOUT);
      if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(carveout)");
#endif
      int occ = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, WARPS * 32, SMEM);
      if (e != cudaSuccess) return cuda_fail(e, "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      if (dev >= 0 && dev < kMaxDev) {
        blocks_per_sm[dev].store(std::max(1, occ), std::memory_order_relaxed);
        configured[dev].store(1, std::memory_order_release);
      }
    }
    const int bps = (dev >= 0 && dev < kMaxDev) ? blocks_per_sm[dev].load(std::memory_order_relaxed) : 1;
    const uint64_t n_full = n_cw / kTileCw;
    const uint32_t rem = static_cast<uint32_t>(n_cw - n_full * kTileCw);
    int launches = 0;
    int grid = 0;
    const uint64_t n_tiles = n_full + (rem > 0 ? 1 : 0);
    if (n_tiles > 0) {
      const uint64_t want = (n_tiles + WARPS - 1) / WARPS;
      int sms = sm_count(dev);
#ifdef HAM_GRID_TUNE  // tuning builds only: the number of SMs the tile grid covers, from the environment
      if (const char* ev = getenv("HAM_GRID_SMS")) sms = std::max(1, std::min(sms, atoi(ev)));
#endif
      grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sms) * bps));
    }
    const int store_count = (counter != nullptr && !accumulate && grid == 1) ? 1 : 0;
    // the slot: the count without a memset (multi-CTA launches) and the dynamic tail
    LaunchSlot* slot = nullptr;
    if (grid > 1 && (counter != nullptr || dyn_rounds > 0)) slot = launch_slot(dev, stream);
    uint64_t static_end = n_full;
    if (slot != nullptr && dyn_rounds > 0 && n_full < (1ull << 31)) {
      const uint64_t nw = static_cast<uint64_t>(grid) * WARPS;
      const uint64_t rounds = n_full / nw;
      static_end = (rounds > static_cast<uint64_t>(dyn_rounds) ? rounds - dyn_rounds : 0) * nw;
    }
    if (counter != nullptr && !accumulate && !store_count && slot == nullptr) {  // overwritten, stream-ordered
      e = cudaMemsetAsync(counter, 0, Op::NCOUNT * sizeof(unsigned long long), stream);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(corrected)");
    }
    if (grid > 0) {
      kfn<<<grid, WARPS * 32, SMEM, stream>>>(in, out, side, n_full, rem, in_total, out_total, counter,
                                              store_count, slot, static_end, accumulate ? 1 : 0, args);
      ++launches;
      e = cudaGetLastError();
      if (e != cudaSuccess) return cuda_fail(e, "tiles kernel launch");
    }
    g_launches = launches;
    g_grid = grid;
    return HAMMING_OK;
  }
};

// Per-m launch shapes: warps per CTA x TMA stages per warp.
template <int M> struct Shape;
template <> struct Shape<2> { static constexpr int W = 16, S = 4; };
template <> struct Shape<3> { static constexpr int W = 16, S = 4; };
template <> struct Shape<4> { static constexpr int W = 16, S = 4; };
template <> struct Shape<5> { static constexpr int W = 12, S = 3; };
template <> struct Shape<6> { static constexpr int W = 7, S = 2; };

// The 2-D, 128-byte-swizzled tensor map over the full tiles of a SECDED input
// (rows of 128 bytes, one box = one tile of `tile_bytes`).  The driver entry
// point is resolved once through the runtime (no -lcuda).
hamming_status make_tile_tmap(CUtensorMap* map, const void* base, uint64_t n_full, int tile_bytes) {
  memset(map, 0, sizeof(*map));
  if (n_full == 0) return HAMMING_OK;  // no TMA loads: the tail loader handles everything
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (encode == nullptr) return set_err(HAMMING_E_CUDA, "cuTensorMapEncodeTiled entry point not found");
  const uint64_t rows = n_full * static_cast<uint64_t>(tile_bytes / 128);
  if (rows > (1ull << 31)) return set_err(HAMMING_E_RANGE, "input too large for one tensor map");
  const cuuint32_t rpl = static_cast<cuuint32_t>(tile_bytes / (32 * 128));  // 128-byte rows per lane
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r;
  if (rpl >= 2) {  // {byte, lane, row of the lane}: smem box order [row of lane][lane][128 B]
    const cuuint64_t dims[3] = {128, rows / rpl, rpl};
    const cuuint64_t strides[2] = {128ull * rpl, 128};
    const cuuint32_t box[3] = {128, 32, rpl};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[2] = {128, rows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {128, static_cast<cuuint32_t>(tile_bytes / 128)};
    r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return set_err(HAMMING_E_CUDA, "cuTensorMapEncodeTiled failed");
  return HAMMING_OK;
}

template <class Op, int WARPS, int STAGES>
hamming_status run_swizzled(const uint8_t* in, uint8_t* out, uint8_t* side, uint64_t N, uint64_t ib, uint64_t ob,
                            unsigned long long* counter, cudaStream_t st) {
  typename Op::Args a;
  const hamming_status s = make_tile_tmap(&a.tmap, in, N / kTileCw, TileBytes<Op>::IN);
  if (s != HAMMING_OK) return s;
  return Launcher<Op, WARPS, STAGES, true>::run(in, out, side, N, ib, ob, counter, a, st);
}

template <class Op, int WARPS, int STAGES>
hamming_status run_swizzled_out(const uint8_t* in, uint8_t* out, uint64_t N, uint64_t ib, uint64_t ob,
                                cudaStream_t st) {
  typename Op::Args a;
  const hamming_status s = make_tile_tmap(&a.tmap_out, out, N / kTileCw, TileBytes<Op>::OUT);
  if (s != HAMMING_OK) return s;
  return Launcher<Op, WARPS, STAGES, false>::run(in, out, nullptr, N, ib, ob, nullptr, a, st);
}

bool ranges_overlap(const void* a, uint64_t na, const void* b, uint64_t nb) {
  if (!a || !b || !na || !nb) return false;
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + nb && y < x + na;
}
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool bits_overflow(int m, uint64_t N) {
  const uint64_t n = (1ull << m) - 1;
  return N > (~0ull) / n;
}

// Decode launch shapes: warps per CTA, TMA stages per warp, output in place
// (DESIGN.md section 5).  Overridable at build time for tuning sweeps only.
#ifndef HAM_W2
#define HAM_W2 16
#endif
#ifndef HAM_S2
#define HAM_S2 8
#endif
#ifndef HAM_IP2
#define HAM_IP2 true
#endif
#ifndef HAM_W3
#define HAM_W3 16
#endif
#ifndef HAM_S3
#define HAM_S3 12
#endif
#ifndef HAM_M3_OP
#define HAM_M3_OP DecodeLut3Op
#endif
#ifndef HAM_IP3
#define HAM_IP3 true
#endif
#ifndef HAM_W4
#define HAM_W4 8
#endif
#ifndef HAM_S4
#define HAM_S4 8
#endif
#ifndef HAM_IP4
#define HAM_IP4 true
#endif
#ifndef HAM_W5
#define HAM_W5 12
#endif
#ifndef HAM_S5
#define HAM_S5 3
#endif
#ifndef HAM_IP5
#define HAM_IP5 true
#endif
#ifndef HAM_W6
#define HAM_W6 8
#endif
#ifndef HAM_S6
#define HAM_S6 3
#endif
#ifndef HAM_IP6
#define HAM_IP6 true
#endif

// Rounds of tiles claimed dynamically at the end of a decode launch (0 = all
// static); measured, tools/tune_shapes.py.  The claims go through one L2
// atomic, so codes with many (short) tiles per warp keep the static schedule.
#ifndef HAM_DYN3
#define HAM_DYN3 0
#endif
#ifndef HAM_DYN4
#define HAM_DYN4 0
#endif
#ifndef HAM_DYN5
#define HAM_DYN5 2
#endif
#ifndef HAM_DYN6
#define HAM_DYN6 2
#endif

// Below this many codewords a call uses the light small-packet launch.
constexpr uint64_t kSmallPacketCw = 1u << 16;

// Small calls (at most kSmallCallBits coded bits, e.g. the BJ configs[0] 4 KB packet and the C2
// sizes up to 2 MiB): the tile pipeline gives every lane 32 consecutive codewords, so a 4 KB (7,4)
// packet kept ~150 lanes busy for 32 dependent decodes each and a call cost ~10 us of device time
// (ncu: 3065 warp instructions in 12.7 us on one SM).  Instead CTAs of 1024 threads each take
// small_call_cw<m>() consecutive codewords (a multiple of 32, so every CTA's input and output start on a
// word), stage their stream in shared memory with coalesced 16-byte loads, decode one codeword per
// thread at a time (a2..a4 as decode_cw), gather the data bits with shared atomics and write whole
// words, the syndromes and the count.  One CTA writes the count itself; several publish it through
// the stream's launch slot (the last CTA to finish writes it and resets the slot, as tiles_kernel)
// or, without a slot (graph capture), add into a count zeroed by a memset first.
constexpr uint64_t kSmallCallBits = 1u << 24;  // 2 MiB of coded stream
constexpr int kSmallCallThreads = 1024;
#ifndef HAM_SMALL_PDL
#define HAM_SMALL_PDL 1
#endif
constexpr int kSmallCallPdl = HAM_SMALL_PDL;  // programmatic dependent launch of small calls (0: plain launch)
// codewords per CTA: the most (a multiple of 1024, at most 16384) whose stream and data images fit
// the default 48 KB of shared memory -- 16384 for m = 2, 3 (BJ configs[0] is one CTA), 14336 for
// m = 4, 6144 for m = 5, 3072 for m = 6
template <int M>
__host__ __device__ constexpr uint32_t small_call_cw() {
  constexpr uint32_t bits = Geo<M>::n + Geo<M>::k;
  uint32_t c = 16384;
  while (c > 1024 && c * bits / 8 + 256 > 48 * 1024) c -= 1024;
  return c;
}

template <int M>
__global__ void __launch_bounds__(kSmallCallThreads)
    small_decode_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, uint8_t* __restrict__ syn,
                        uint32_t N, uint32_t in_total, uint32_t out_total, unsigned long long* __restrict__ counter,
                        int accumulate, LaunchSlot* __restrict__ slot, uint32_t CPB) {
  constexpr uint32_t n = Geo<M>::n, k = Geo<M>::k;
  extern __shared__ __align__(16) uint32_t small_sm[];
  __shared__ uint32_t cnt_s;  // 32-bit: a CTA holds at most 16384 codewords
  // programmatic dependent launch: this grid may be resident before the previous kernel on the stream
  // has finished (launch_small_decode sets the attribute); every global access waits for it here, and
  // the next small call may start launching at once
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t c0 = blockIdx.x * CPB, nc = min(CPB, N - c0);
  // this CTA's stream: bits [c0 n, (c0 + nc) n), byte ib0 = c0 n / 8 (a multiple of 4)
  const uint32_t ib0 = c0 / 8 * n, in_bytes = min(in_total - ib0, (nc * n + 7) / 8 + 8);
  const uint32_t ob0 = c0 / 8 * k, out_bytes = min(out_total - ob0, (nc * k + 7) / 8);
  const uint32_t in_words = (in_bytes + 15) / 16 * 4 + 4;  // + a zero 16-byte unit: reads past the end
  const uint32_t out_words = (nc * k + 31) / 32;
  uint32_t* sin = small_sm;
  uint32_t* sout = small_sm + in_words;
  const uint32_t tid = threadIdx.x;
  const uint8_t* src = in + ib0;
  for (uint32_t u = tid; u < in_words / 4; u += blockDim.x) {  // 16-byte units, zero past in_bytes
    uint4 v = make_uint4(0, 0, 0, 0);
    if (16 * u + 16 <= in_bytes && ((ib0 & 15u) == 0)) {
      v = __ldg(reinterpret_cast<const uint4*>(src) + u);
    } else if (16 * u < in_bytes) {
      uint32_t wv[4] = {0, 0, 0, 0};
      for (uint32_t b = 16 * u; b < in_bytes && b < 16 * u + 16; ++b)
        wv[(b >> 2) & 3] |= static_cast<uint32_t>(src[b]) << (8 * (b & 3));
      v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    reinterpret_cast<uint4*>(sin)[u] = v;
  }
  for (uint32_t i = tid; i < out_words; i += blockDim.x) sout[i] = 0;
  if (tid == 0) cnt_s = 0;
  __syncthreads();
  uint32_t cnt = 0;
  for (uint32_t c = tid; c < nc; c += blockDim.x) {
    const uint32_t b = c * n, q = b >> 5, r = b & 31u;
    const uint32_t lo = __funnelshift_r(sin[q], sin[q + 1], r);  // stream bits b .. b + 31
    // v: bit p = position p (bit 0 a zero dummy); bits past n belong to the next codeword and are
    // ignored by decode_cw's masks (m <= 5) or shifted out (m = 6)
    const uint32_t vlo = lo << 1;
    uint32_t vhi = 0;
    if constexpr (M == 6) vhi = (__funnelshift_r(sin[q + 1], sin[q + 2], r) << 1) | (lo >> 31);
    uint32_t dlo, dhi;
    const uint32_t s = decode_cw<M>(vlo, vhi, dlo, dhi);
    const uint32_t P = c * k, pw = P >> 5, pr = P & 31u;
    if constexpr (M <= 5) {
      atomicOr(&sout[pw], dlo << pr);
      if (pr + k > 32) atomicOr(&sout[pw + 1], dlo >> (32 - pr));
    } else {
      const uint64_t d = static_cast<uint64_t>(dlo) | (static_cast<uint64_t>(dhi) << 26);  // 57 bits
      const uint64_t x = d << pr;
      atomicOr(&sout[pw], static_cast<uint32_t>(x));
      atomicOr(&sout[pw + 1], static_cast<uint32_t>(x >> 32));
      if (pr + k > 64) atomicOr(&sout[pw + 2], static_cast<uint32_t>(d >> (64 - pr)));
    }
    if (syn != nullptr) syn[c0 + c] = static_cast<uint8_t>(s);
    cnt += (s != 0);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((tid & 31u) == 0 && cnt != 0) atomicAdd(&cnt_s, cnt);
  __syncthreads();
  uint8_t* dst = out + ob0;
  for (uint32_t i = tid; i < out_words; i += blockDim.x) {  // only data bits were OR-ed in: pad bits are 0
    const uint32_t v = sout[i];
    if (4 * i + 4 <= out_bytes) {
      reinterpret_cast<uint32_t*>(dst)[i] = v;
    } else {
      for (uint32_t b = 4 * i; b < out_bytes; ++b) dst[b] = static_cast<uint8_t>(v >> (8 * (b & 3)));
    }
  }
  if (tid == 0) {
    const unsigned long long cs = cnt_s;
    if (gridDim.x == 1) {
      if (accumulate) atomicAdd(counter, cs);
      else *counter = cs;
    } else if (slot != nullptr) {  // the last CTA to arrive publishes the total and resets the slot
      if (cs) atomicAdd(&slot->sum[0], cs);
      __threadfence();
      if (atomicAdd(&slot->done, 1u) == gridDim.x - 1) {
        __threadfence();
        const unsigned long long tot = atomicExch(&slot->sum[0], 0ull);
        if (accumulate) atomicAdd(counter, tot);
        else *counter = tot;
        slot->claim = 0;
        slot->done = 0;
      }
    } else if (cs) {  // count zeroed by the launcher (or accumulating)
      atomicAdd(counter, cs);
    }
  }
}

template <int M>
hamming_status launch_small_decode(const uint8_t* in, uint64_t N, uint8_t* out, uint8_t* syn,
                                   unsigned long long* counter, cudaStream_t st, bool accumulate) {
  const uint32_t ib = static_cast<uint32_t>((Geo<M>::n * N + 7) / 8), ob = static_cast<uint32_t>((Geo<M>::k * N + 7) / 8);
  // one CTA when the call fits one (no count to publish across CTAs); otherwise 2048 codewords per
  // CTA, so that mid-size calls spread over many SMs (measured: 64 KiB of (15,11) in a CUDA graph
  // 12.3 us with 3 CTAs of 14336 codewords, 8.2 us with 18 of 2048)
  const uint32_t CPB = N <= small_call_cw<M>() ? static_cast<uint32_t>(N) : 2048u;
  const uint32_t grid = static_cast<uint32_t>((N + CPB - 1) / CPB);
  const uint32_t cpb = static_cast<uint32_t>(std::min<uint64_t>(N, CPB));
  const size_t smem = 4 * (((Geo<M>::n * cpb + 7) / 8 + 8 + 15) / 16 * 4 + 4 + (Geo<M>::k * cpb + 31) / 32);
  LaunchSlot* slot = nullptr;
  if (grid > 1) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    slot = launch_slot(dev, st);
    if (slot == nullptr && !accumulate) {  // no slot (graph capture): count zeroed first, then added
      e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(corrected)");
    }
  }
  // programmatic stream serialisation: back-to-back small calls (C1, graph-batched packets) overlap the
  // next call's launch with this one's execution; the kernel's griddepcontrol.wait keeps stream order
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kSmallCallThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = kSmallCallPdl;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, small_decode_kernel<M>, in, out, syn, static_cast<uint32_t>(N), ib, ob,
                                     counter, accumulate ? 1 : 0, slot, CPB);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "small decode launch");
  g_launches = 1;
  g_grid = static_cast<int>(grid);
  return HAMMING_OK;
}

// Per-device build of the (15,11) table in global memory, once it succeeds: a
// failed build (e.g. a first call made while the caller's stream is being
// captured into a CUDA graph, where the build's own stream sync is not
// allowed) is reported and retried by the next call, never latched.
std::mutex g_lut15_mu;
std::atomic<bool> g_lut15_ok[kMaxDev];

hamming_status ensure_lut15(int dev, cudaStream_t caller) {
  if (dev < 0 || dev >= kMaxDev) return set_err(HAMMING_E_CUDA, "device index out of range");
  if (g_lut15_ok[dev].load(std::memory_order_acquire)) return HAMMING_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(caller, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return set_err(HAMMING_E_CUDA,
                   "the (15,11)/(31,26) lookup table is built by the first eager call on a device; "
                   "make one call outside CUDA-graph capture first");
  std::lock_guard<std::mutex> lock(g_lut15_mu);
  if (g_lut15_ok[dev].load(std::memory_order_acquire)) return HAMMING_OK;
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    init_lut15_kernel<<<32768 / 256, 256, 0, s>>>();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "building the (15,11) table");
  g_lut15_ok[dev].store(true, std::memory_order_release);
  return HAMMING_OK;
}

hamming_status launch_long_decode(int m, const uint8_t* in, uint64_t N, uint8_t* out, uint8_t* syn,
                                  unsigned long long* counter, cudaStream_t st, bool accumulate);

hamming_status decode_dispatch(int m, const uint8_t* in, uint64_t N, uint8_t* out, uint8_t* syn,
                               unsigned long long* counter, cudaStream_t st, bool accumulate) {
  if (m == 7 || m == 8) return launch_long_decode(m, in, N, out, syn, counter, st, accumulate);
  const uint64_t n = (1ull << m) - 1, k = n - m;
  const uint64_t ib = (n * N + 7) / 8, ob = (k * N + 7) / 8;
  if (N > 0 && n * N <= kSmallCallBits) {  // a single small call: one CTA, no tile pipeline
    switch (m) {
      case 2: return launch_small_decode<2>(in, N, out, syn, counter, st, accumulate);
      case 3: return launch_small_decode<3>(in, N, out, syn, counter, st, accumulate);
      case 4: return launch_small_decode<4>(in, N, out, syn, counter, st, accumulate);
      case 5: return launch_small_decode<5>(in, N, out, syn, counter, st, accumulate);
      case 6: return launch_small_decode<6>(in, N, out, syn, counter, st, accumulate);
    }
  }
  if (N < kSmallPacketCw) {
    // Small packets are latency-bound: a light CTA (4 warps, 2 stages, no
    // table to build or copy) launches and finishes fastest; from 4 full tiles
    // on, 8 warps, so that the ragged tail gets a warp of its own instead of
    // queueing behind a full tile (C1, a 4 KB (7,4) packet: 6.2 -> 4.0 us per
    // packet in a CUDA graph).
    switch (m) {
#define HAMMING_SMALL_CASE(MM)                                                                               \
  case MM:                                                                                                   \
    return N >= 4 * kTileCw                                                                                  \
               ? Launcher<DecodeOp<MM>, 8, 2, true>::run(in, out, syn, N, ib, ob, counter, {}, st, accumulate) \
               : Launcher<DecodeOp<MM>, 4, 2, true>::run(in, out, syn, N, ib, ob, counter, {}, st, accumulate);
      HAMMING_SMALL_CASE(2)
      HAMMING_SMALL_CASE(3)
      HAMMING_SMALL_CASE(4)
      HAMMING_SMALL_CASE(5)
      HAMMING_SMALL_CASE(6)
#undef HAMMING_SMALL_CASE
    }
  }
  switch (m) {
    case 2:
      return Launcher<DecodeOp<2>, HAM_W2, HAM_S2, HAM_IP2>::run(in, out, syn, N, ib, ob, counter, {}, st,
                                                                 accumulate);
    case 3:
      return Launcher<HAM_M3_OP, HAM_W3, HAM_S3, HAM_IP3>::run(in, out, syn, N, ib, ob, counter, {}, st,
                                                                  accumulate, HAM_DYN3);
    case 4: {
      int dev = 0;
      const cudaError_t e = cudaGetDevice(&dev);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
      const hamming_status rc = ensure_lut15(dev, st);
      if (rc != HAMMING_OK) return rc;
      return Launcher<DecodeLut4Op, HAM_W4, HAM_S4, HAM_IP4>::run(in, out, syn, N, ib, ob, counter, {}, st,
                                                                  accumulate, HAM_DYN4);
    }
    case 5: {
      int dev = 0;
      const cudaError_t e = cudaGetDevice(&dev);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
      const hamming_status rc = ensure_lut15(dev, st);
      if (rc != HAMMING_OK) return rc;
      return Launcher<DecodeLut5Op, HAM_W5, HAM_S5, HAM_IP5>::run(in, out, syn, N, ib, ob, counter, {}, st,
                                                                  accumulate, HAM_DYN5);
    }
    case 6:
      return Launcher<DecodeOp<6>, HAM_W6, HAM_S6, HAM_IP6>::run(in, out, syn, N, ib, ob, counter, {}, st,
                                                                 accumulate, HAM_DYN6);
  }
  return set_err(HAMMING_E_INVALID_M, "decode: m must be in [2, 6]");
}

constexpr uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

struct HostSlotLayout {
  uint64_t rx, data, syn, slot;
};

HostSlotLayout host_slot_layout(int m, uint64_t chunk, int with_syn) {
  const uint64_t n = (1ull << m) - 1, k = n - m;
  HostSlotLayout L;
  L.rx = align256((n * chunk + 7) / 8);
  L.data = align256((k * chunk + 7) / 8);
  L.syn = with_syn ? align256(chunk) : 0;
  L.slot = L.rx + L.data + L.syn;
  return L;
}

#include "packets.cuh"

}  // namespace

// =================================================================== C ABI
#ifdef HAM_PROBE
// ------------------------------------------------ power/bandwidth probes
// Tools-only build (-DHAM_PROBE, tools/power_probe.py): the (63,57) tile
// pipeline with the decode taken out, to split the decode's power between
// the TMA round trip through shared memory and the arithmetic.
//   kind 0 (ProbeTmaOp): the lane does nothing -- TMA in, the first 57 x 128
//     bytes of the tile TMA out, zero syndrome bytes stored: the same HBM
//     bytes as the decode, no shared-memory loads or stores by the SM.
//   kind 1 (ProbeLdsOp): the lane also loads its 63 words from shared memory
//     and stores 57 of them back (the decode's LDS/STS traffic, no math).
struct ProbeTmaOp {
  static constexpr int NCOUNT = 1;
  __device__ __forceinline__ static uint32_t count0(const uint32_t (&)[8]) { return 0; }
  __device__ __forceinline__ static uint32_t count1(const uint32_t (&)[8]) { return 0; }
  static constexpr int IN_W = 63, OUT_W = 57, IN_BITS = 63;
  static constexpr bool HAS_SIDE = true;
  static constexpr int SHARED = 0;
  struct Args {};
  __device__ __forceinline__ static void cta_init(uint8_t*, int, int) {}
  __device__ __forceinline__ static void lane(const uint32_t* __restrict__, uint32_t* __restrict__, uint32_t (&)[8],
                                              uint64_t, int, const Args&, const uint8_t*) {}
};
struct ProbeLdsOp : ProbeTmaOp {
  __device__ __forceinline__ static void lane(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                              uint32_t (&side)[8], uint64_t, int, const Args&, const uint8_t*) {
    uint32_t w[63];
#pragma unroll
    for (int i = 0; i < 63; ++i) w[i] = in[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 57; ++i) out[i] = w[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) side[i] = w[57 + i % 6] & 0x01010101u;
  }
};
// kind 3 (ProbeCopyTileOp): whole (63,57)-sized tiles TMA in and the same
//   tile TMA out, no side stores: a TMA copy through shared memory.
// kind 4: a plain grid-stride LDG.128 / STG.128 copy kernel (no shared memory).
struct ProbeCopyTileOp : ProbeTmaOp {
  static constexpr int OUT_W = 63;
  static constexpr bool HAS_SIDE = false;
};
__global__ void probe_copy_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, uint64_t n16) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i];
}
#endif

extern "C" {

int hamming_abi_version(void) { return HAMMING_ABI_VERSION; }

#ifdef HAM_PROBE
hamming_status hamming_probe_tiles(int kind, const void* rx_dev, uint64_t N, void* data_dev, uint8_t* syn_dev,
                                   unsigned long long* counter, void* stream) {
  const uint64_t ib = (63 * N + 7) / 8, ob = (57 * N + 7) / 8;
  const auto* in = static_cast<const uint8_t*>(rx_dev);
  auto* out = static_cast<uint8_t*>(data_dev);
  auto st = static_cast<cudaStream_t>(stream);
  if (kind == 0) return Launcher<ProbeTmaOp, HAM_W6, HAM_S6, HAM_IP6>::run(in, out, syn_dev, N, ib, ob, counter, {}, st);
  if (kind == 1) return Launcher<ProbeLdsOp, HAM_W6, HAM_S6, HAM_IP6>::run(in, out, syn_dev, N, ib, ob, counter, {}, st);
  if (kind == 2) return Launcher<ProbeTmaOp, HAM_W6, HAM_S6, HAM_IP6>::run(in, out, nullptr, N, ib, ob, counter, {}, st);
  // kinds 3, 4 move ib + ob + N bytes too: ib read and (ob + N) ~ ib written (the same HBM volume)
  if (kind == 3) return Launcher<ProbeCopyTileOp, HAM_W6, HAM_S6, HAM_IP6>::run(in, out, nullptr, N, ib, ib, nullptr, {}, st);
  const uint64_t n16 = ib / 16;
  probe_copy_kernel<<<148 * 8, 512, 0, st>>>(reinterpret_cast<const uint4*>(in), reinterpret_cast<uint4*>(out), n16);
  return cudaGetLastError() == cudaSuccess ? HAMMING_OK : HAMMING_E_CUDA;
}
#endif
#ifdef HAM_TIMING
int hamming_debug_timing(unsigned long long* host_out, int n) {
  return cudaMemcpyFromSymbol(host_out, g_timing, sizeof(unsigned long long) * n) == cudaSuccess ? 0 : 1;
}
#endif

uint64_t hamming_coded_bytes(int m, uint64_t N) {
  if (m < 2 || m > 8 || bits_overflow(m, N)) return 0;
  const uint64_t n = (1ull << m) - 1;
  return (n * N + 7) / 8;
}

uint64_t hamming_data_bytes(int m, uint64_t N) {
  if (m < 2 || m > 8 || bits_overflow(m, N)) return 0;
  const uint64_t k = (1ull << m) - 1 - m;
  return (k * N + 7) / 8;
}

const char* hamming_status_string(hamming_status s) {
  switch (s) {
    case HAMMING_OK: return "ok";
    case HAMMING_E_INVALID_M: return "invalid m (decode: 2..8; encode/generate: 2..6; SECDED: 3..6)";
    case HAMMING_E_NULL: return "required pointer is NULL";
    case HAMMING_E_MISALIGNED: return "device buffer not 16-byte aligned";
    case HAMMING_E_OVERLAP: return "input and output buffers overlap";
    case HAMMING_E_RANGE: return "size or probability out of range";
    case HAMMING_E_CUDA: return "CUDA error";
    case HAMMING_E_ARG: return "invalid argument";
  }
  return "unknown status";
}

const char* hamming_last_error(void) { return g_err; }
int hamming_last_launch_count(void) { return g_launches; }
int hamming_last_grid_blocks(void) { return g_grid; }

hamming_status hamming_decode(int m, const void* rx_dev, uint64_t N, void* data_dev, uint8_t* syn_dev,
                              unsigned long long* corrected_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 2 || m > 8) return set_err(HAMMING_E_INVALID_M, "hamming_decode: m must be in [2, 8]");
  if (bits_overflow(m, N)) return set_err(HAMMING_E_RANGE, "hamming_decode: n * n_codewords overflows");
  if (corrected_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_decode: corrected is NULL");
  if (N > 0 && (rx_dev == nullptr || data_dev == nullptr))
    return set_err(HAMMING_E_NULL, "hamming_decode: rx or data is NULL");
  if (!aligned16(rx_dev) || !aligned16(data_dev) || !aligned16(syn_dev))
    return set_err(HAMMING_E_MISALIGNED, "hamming_decode: rx, data and syndromes must be 16-byte aligned");
  const uint64_t ib = hamming_coded_bytes(m, N), ob = hamming_data_bytes(m, N);
  const uint64_t sb = syn_dev ? N : 0;
  if (ranges_overlap(rx_dev, ib, data_dev, ob) || ranges_overlap(rx_dev, ib, syn_dev, sb) ||
      ranges_overlap(data_dev, ob, syn_dev, sb) || ranges_overlap(rx_dev, ib, corrected_dev, 8) ||
      ranges_overlap(data_dev, ob, corrected_dev, 8) || ranges_overlap(syn_dev, sb, corrected_dev, 8))
    return set_err(HAMMING_E_OVERLAP, "hamming_decode: buffers overlap");
  return decode_dispatch(m, static_cast<const uint8_t*>(rx_dev), N, static_cast<uint8_t*>(data_dev), syn_dev,
                         corrected_dev, static_cast<cudaStream_t>(stream), false);
}

// encoder launch shapes (warps x stages), tunable with -D (tools/tune_shapes.py encode)
#ifndef HAM_ENC_W3
#define HAM_ENC_W3 16
#define HAM_ENC_S3 8
#endif
#ifndef HAM_ENC_W4
#define HAM_ENC_W4 16
#define HAM_ENC_S4 4
#endif
#ifndef HAM_ENC_W5
#define HAM_ENC_W5 10
#define HAM_ENC_S5 2
#endif
#ifndef HAM_SENC_W3
#define HAM_SENC_W3 16
#define HAM_SENC_S3 8
#endif
#ifndef HAM_SENC_W4
#define HAM_SENC_W4 16
#define HAM_SENC_S4 3
#endif
#ifndef HAM_SENC_W5
#define HAM_SENC_W5 4
#define HAM_SENC_S5 8
#endif
#ifndef HAM_SENC_W6
#define HAM_SENC_W6 6
#define HAM_SENC_S6 2
#endif
hamming_status hamming_encode(int m, const void* data_dev, uint64_t N, void* rx_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 2 || m > 6) return set_err(HAMMING_E_INVALID_M, "hamming_encode: m must be in [2, 6]");
  if (bits_overflow(m, N)) return set_err(HAMMING_E_RANGE, "hamming_encode: n * n_codewords overflows");
  if (N == 0) return HAMMING_OK;
  if (data_dev == nullptr || rx_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_encode: NULL buffer");
  if (!aligned16(data_dev) || !aligned16(rx_dev))
    return set_err(HAMMING_E_MISALIGNED, "hamming_encode: buffers must be 16-byte aligned");
  const uint64_t ib = hamming_data_bytes(m, N), ob = hamming_coded_bytes(m, N);
  if (ranges_overlap(data_dev, ib, rx_dev, ob)) return set_err(HAMMING_E_OVERLAP, "hamming_encode: overlap");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint8_t* in = static_cast<const uint8_t*>(data_dev);
  uint8_t* out = static_cast<uint8_t*>(rx_dev);
  switch (m) {
    case 2: return Launcher<EncodeOp<2>, Shape<2>::W, Shape<2>::S>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
    case 3: return Launcher<EncodeLutOp<3>, HAM_ENC_W3, HAM_ENC_S3>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
    case 4: return Launcher<EncodeLutOp<4>, HAM_ENC_W4, HAM_ENC_S4>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
    case 5: return Launcher<EncodeLut5Op<false>, HAM_ENC_W5, HAM_ENC_S5>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
    case 6: return Launcher<EncodeOp<6>, Shape<6>::W, Shape<6>::S>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
  }
  return set_err(HAMMING_E_INVALID_M, "hamming_encode: m must be in [2, 6]");
}

hamming_status hamming_channel_generate(int m, uint64_t seed, uint64_t c_first, uint64_t N, uint64_t thresh,
                                        int all, uint64_t q2thresh, void* rx_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 2 || m > 6) return set_err(HAMMING_E_INVALID_M, "hamming_channel_generate: m must be in [2, 6]");
  if (bits_overflow(m, N)) return set_err(HAMMING_E_RANGE, "hamming_channel_generate: size overflows");
  if (q2thresh > (1ull << 32)) return set_err(HAMMING_E_RANGE, "hamming_channel_generate: q2thresh > 2^32");
  if (N == 0) return HAMMING_OK;
  if (rx_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_channel_generate: rx is NULL");
  if (!aligned16(rx_dev)) return set_err(HAMMING_E_MISALIGNED, "hamming_channel_generate: rx misaligned");
  const uint64_t ob = hamming_coded_bytes(m, N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* out = static_cast<uint8_t*>(rx_dev);
  switch (m) {
#define HAMMING_GEN_CASE(MM)                                                                                 \
  case MM: {                                                                                                 \
    typename GenerateOp<MM>::Args a{seed, c_first, thresh, q2thresh, all};                                  \
    return Launcher<GenerateOp<MM>, 4, 1>::run(nullptr, out, nullptr, N, 0, ob, nullptr, a, st);            \
  }
    HAMMING_GEN_CASE(2)
    HAMMING_GEN_CASE(3)
    HAMMING_GEN_CASE(4)
    HAMMING_GEN_CASE(5)
    HAMMING_GEN_CASE(6)
#undef HAMMING_GEN_CASE
  }
  return set_err(HAMMING_E_INVALID_M, "hamming_channel_generate: m must be in [2, 6]");
}

size_t hamming_host_workspace_bytes(int m, uint64_t chunk_codewords, int n_streams, int with_syndromes) {
  if (m < 2 || m > 8 || n_streams < 1 || n_streams > 4 || chunk_codewords == 0 ||
      bits_overflow(m, chunk_codewords))
    return 0;
  return static_cast<size_t>(256 + n_streams * host_slot_layout(m, chunk_codewords, with_syndromes).slot);
}

hamming_status hamming_decode_host(int m, const void* rx_host, uint64_t N, void* data_host, uint8_t* syn_host,
                                   unsigned long long* corrected_host, void* workspace_dev,
                                   uint64_t chunk, int n_streams) {
  g_launches = 0;
  g_grid = 0;
  if (m < 2 || m > 8) return set_err(HAMMING_E_INVALID_M, "hamming_decode_host: m must be in [2, 8]");
  if (bits_overflow(m, N)) return set_err(HAMMING_E_RANGE, "hamming_decode_host: size overflows");
  if (corrected_host == nullptr || workspace_dev == nullptr)
    return set_err(HAMMING_E_NULL, "hamming_decode_host: corrected or workspace is NULL");
  if (N > 0 && (rx_host == nullptr || data_host == nullptr))
    return set_err(HAMMING_E_NULL, "hamming_decode_host: rx or data is NULL");
  if (n_streams < 1 || n_streams > 4 || chunk == 0 || chunk % kTileCw != 0)
    return set_err(HAMMING_E_ARG, "hamming_decode_host: need 1 <= n_streams <= 4, chunk a multiple of 1024");
  if (!aligned16(workspace_dev)) return set_err(HAMMING_E_MISALIGNED, "hamming_decode_host: workspace misaligned");
  const uint64_t n = (1ull << m) - 1, k = n - m;
  const HostSlotLayout L = host_slot_layout(m, chunk, syn_host != nullptr);
  uint8_t* ws = static_cast<uint8_t*>(workspace_dev);
  unsigned long long* total = reinterpret_cast<unsigned long long*>(ws);
  // the pipeline's streams and event: created once per (thread, device) and reused, so a
  // call makes no stream / event create or destroy (never destroyed: they live as long as
  // the thread, and tearing them down at thread exit could race the runtime's own exit)
  struct HostPipe {
    cudaStream_t s[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ready = nullptr;
  };
  static thread_local HostPipe pipes[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return set_err(HAMMING_E_CUDA, "device index out of range");
  HostPipe& P = pipes[dev];
  for (int i = 0; i < 4 && e == cudaSuccess; ++i)
    if (P.s[i] == nullptr) e = cudaStreamCreateWithFlags(&P.s[i], cudaStreamNonBlocking);
  if (e == cudaSuccess && P.ready == nullptr) e = cudaEventCreateWithFlags(&P.ready, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(e, "hamming_decode_host: stream setup");
  cudaStream_t* streams = P.s;
  cudaEvent_t ready = P.ready;
  hamming_status rc = HAMMING_OK;
  int launches = 0;
  e = cudaMemsetAsync(total, 0, sizeof(unsigned long long), streams[0]);
  if (e == cudaSuccess) e = cudaEventRecord(ready, streams[0]);
  for (int i = 1; i < n_streams && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(streams[i], ready, 0);
  if (e != cudaSuccess) rc = cuda_fail(e, "hamming_decode_host setup");
  const uint8_t* hin = static_cast<const uint8_t*>(rx_host);
  uint8_t* hout = static_cast<uint8_t*>(data_host);
  for (uint64_t c0 = 0, i = 0; rc == HAMMING_OK && c0 < N; c0 += chunk, ++i) {
    const uint64_t cn = std::min<uint64_t>(chunk, N - c0);
    const int sl = static_cast<int>(i % n_streams);
    cudaStream_t s = streams[sl];
    uint8_t* d_rx = ws + 256 + sl * L.slot;
    uint8_t* d_data = d_rx + L.rx;
    uint8_t* d_syn = syn_host ? d_data + L.data : nullptr;
    const uint64_t ib = (n * cn + 7) / 8, ob = (k * cn + 7) / 8;
    e = cudaMemcpyAsync(d_rx, hin + c0 * n / 8, ib, cudaMemcpyHostToDevice, s);  // PS
    if (e != cudaSuccess) { rc = cuda_fail(e, "hamming_decode_host H2D"); break; }
    rc = decode_dispatch(m, d_rx, cn, d_data, d_syn, total, s, true);                   // DKE
    if (rc != HAMMING_OK) break;
    launches += g_launches;
    e = cudaMemcpyAsync(hout + c0 * k / 8, d_data, ob, cudaMemcpyDeviceToHost, s);      // PR
    if (e == cudaSuccess && syn_host) e = cudaMemcpyAsync(syn_host + c0, d_syn, cn, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) { rc = cuda_fail(e, "hamming_decode_host D2H"); break; }
  }
  for (int i = 0; i < n_streams; ++i) {
    if (streams[i]) {
      const cudaError_t e2 = cudaStreamSynchronize(streams[i]);
      if (e2 != cudaSuccess && rc == HAMMING_OK) rc = cuda_fail(e2, "hamming_decode_host sync");
    }
  }
  if (rc == HAMMING_OK) {
    e = cudaMemcpy(corrected_host, total, sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "hamming_decode_host count D2H");
  }
  g_launches = launches;
  return rc;
}

// ---------------------------------------------------- SECDED (extended Hamming)
uint64_t hamming_secded_coded_bytes(int m, uint64_t N) {
  if (m < 3 || m > 6 || N > (~0ull >> m)) return 0;
  return (N << m) / 8;
}

// SECDED launch shapes (warps x stages), tunable with -D (tools/tune_shapes.py secded)
#ifndef HAM_SEC_W3
#define HAM_SEC_W3 16
#define HAM_SEC_S3 4
#endif
#ifndef HAM_SEC_W4
#define HAM_SEC_W4 16
#define HAM_SEC_S4 3
#endif
#ifndef HAM_SEC_W5
#define HAM_SEC_W5 12
#define HAM_SEC_S5 3
#endif
#ifndef HAM_SEC_W6
#define HAM_SEC_W6 8
#define HAM_SEC_S6 3
#endif
hamming_status hamming_decode_secded(int m, const void* rx_dev, uint64_t N, void* data_dev, uint8_t* flags_dev,
                                     unsigned long long* counts_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 3 || m > 6) return set_err(HAMMING_E_INVALID_M, "hamming_decode_secded: m must be in [3, 6]");
  if (N > (~0ull >> m)) return set_err(HAMMING_E_RANGE, "hamming_decode_secded: size overflows");
  if (counts_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_decode_secded: counts is NULL");
  if (N > 0 && (rx_dev == nullptr || data_dev == nullptr))
    return set_err(HAMMING_E_NULL, "hamming_decode_secded: rx or data is NULL");
  if (!aligned16(rx_dev) || !aligned16(data_dev) || !aligned16(flags_dev))
    return set_err(HAMMING_E_MISALIGNED, "hamming_decode_secded: buffers must be 16-byte aligned");
  const uint64_t ib = hamming_secded_coded_bytes(m, N), ob = hamming_data_bytes(m, N), sb = flags_dev ? N : 0;
  if (ranges_overlap(rx_dev, ib, data_dev, ob) || ranges_overlap(rx_dev, ib, flags_dev, sb) ||
      ranges_overlap(data_dev, ob, flags_dev, sb) || ranges_overlap(rx_dev, ib, counts_dev, 16) ||
      ranges_overlap(data_dev, ob, counts_dev, 16) || ranges_overlap(flags_dev, sb, counts_dev, 16))
    return set_err(HAMMING_E_OVERLAP, "hamming_decode_secded: buffers overlap");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint8_t* in = static_cast<const uint8_t*>(rx_dev);
  uint8_t* out = static_cast<uint8_t*>(data_dev);
  if (m == 4 || m == 5) {  // the (15,11) / half-word tables
    int dev = 0;
    const cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    const hamming_status rc = ensure_lut15(dev, st);
    if (rc != HAMMING_OK) return rc;
  }
  if (N < kSmallPacketCw) {
    switch (m) {
      case 3: return run_swizzled<DecodeSecded3Op, 4, 2>(in, out, flags_dev, N, ib, ob, counts_dev, st);
      case 4: return run_swizzled<DecodeSecded4Op, 4, 2>(in, out, flags_dev, N, ib, ob, counts_dev, st);
      case 5: return run_swizzled<DecodeSecded5Op, 4, 2>(in, out, flags_dev, N, ib, ob, counts_dev, st);
      case 6: return run_swizzled<DecodeOp<6, true>, 4, 2>(in, out, flags_dev, N, ib, ob, counts_dev, st);
    }
  }
  switch (m) {
    case 3: return run_swizzled<DecodeSecded3Op, HAM_SEC_W3, HAM_SEC_S3>(in, out, flags_dev, N, ib, ob, counts_dev, st);
    case 4: return run_swizzled<DecodeSecded4Op, HAM_SEC_W4, HAM_SEC_S4>(in, out, flags_dev, N, ib, ob, counts_dev, st);
    case 5: return run_swizzled<DecodeSecded5Op, HAM_SEC_W5, HAM_SEC_S5>(in, out, flags_dev, N, ib, ob, counts_dev, st);
    case 6: return run_swizzled<DecodeOp<6, true>, HAM_SEC_W6, HAM_SEC_S6>(in, out, flags_dev, N, ib, ob, counts_dev, st);
  }
  return set_err(HAMMING_E_INVALID_M, "hamming_decode_secded: m must be in [3, 6]");
}

hamming_status hamming_encode_secded(int m, const void* data_dev, uint64_t N, void* rx_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 3 || m > 6) return set_err(HAMMING_E_INVALID_M, "hamming_encode_secded: m must be in [3, 6]");
  if (N > (~0ull >> m)) return set_err(HAMMING_E_RANGE, "hamming_encode_secded: size overflows");
  if (N == 0) return HAMMING_OK;
  if (data_dev == nullptr || rx_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_encode_secded: NULL buffer");
  if (!aligned16(data_dev) || !aligned16(rx_dev))
    return set_err(HAMMING_E_MISALIGNED, "hamming_encode_secded: buffers must be 16-byte aligned");
  const uint64_t ib = hamming_data_bytes(m, N), ob = hamming_secded_coded_bytes(m, N);
  if (ranges_overlap(data_dev, ib, rx_dev, ob)) return set_err(HAMMING_E_OVERLAP, "hamming_encode_secded: overlap");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint8_t* in = static_cast<const uint8_t*>(data_dev);
  uint8_t* out = static_cast<uint8_t*>(rx_dev);
  switch (m) {
    case 3: return Launcher<EncodeLutOp<3, true>, HAM_SENC_W3, HAM_SENC_S3, false>::run(in, out, nullptr, N, ib, ob, nullptr, {}, st);
    case 4: return run_swizzled_out<EncodeLutOp<4, true>, HAM_SENC_W4, HAM_SENC_S4>(in, out, N, ib, ob, st);
    case 5: return run_swizzled_out<EncodeLut5Op<true>, HAM_SENC_W5, HAM_SENC_S5>(in, out, N, ib, ob, st);
    case 6: return run_swizzled_out<EncodeOp<6, true>, HAM_SENC_W6, HAM_SENC_S6>(in, out, N, ib, ob, st);
  }
  return set_err(HAMMING_E_INVALID_M, "hamming_encode_secded: m must be in [3, 6]");
}

hamming_status hamming_channel_generate_secded(int m, uint64_t seed, uint64_t c_first, uint64_t N, uint64_t thresh,
                                               int all, uint64_t q2thresh, void* rx_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  if (m < 3 || m > 6) return set_err(HAMMING_E_INVALID_M, "hamming_channel_generate_secded: m must be in [3, 6]");
  if (N > (~0ull >> m)) return set_err(HAMMING_E_RANGE, "hamming_channel_generate_secded: size overflows");
  if (q2thresh > (1ull << 32)) return set_err(HAMMING_E_RANGE, "hamming_channel_generate_secded: q2thresh > 2^32");
  if (N == 0) return HAMMING_OK;
  if (rx_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_channel_generate_secded: rx is NULL");
  if (!aligned16(rx_dev)) return set_err(HAMMING_E_MISALIGNED, "hamming_channel_generate_secded: rx misaligned");
  const uint64_t ob = hamming_secded_coded_bytes(m, N);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* out = static_cast<uint8_t*>(rx_dev);
  switch (m) {
#define HAMMING_SECDED_GEN(MM)                                                                      \
  case MM: {                                                                                        \
    typename GenerateOp<MM, true>::Args a{seed, c_first, thresh, q2thresh, all};                    \
    return Launcher<GenerateOp<MM, true>, 4, 1, false>::run(nullptr, out, nullptr, N, 0, ob, nullptr, a, st); \
  }
    HAMMING_SECDED_GEN(3)
    HAMMING_SECDED_GEN(4)
    HAMMING_SECDED_GEN(5)
    HAMMING_SECDED_GEN(6)
#undef HAMMING_SECDED_GEN
  }
  return set_err(HAMMING_E_INVALID_M, "hamming_channel_generate_secded: m must be in [3, 6]");
}

// ------------------------------------------------- packets (the paper's workload)
uint64_t hamming_packet_coded_bytes(uint32_t msg_bytes, int t) {
  PacketGeom g;
  if (packet_geom(msg_bytes, t, g) != HAMMING_OK) return 0;
  return (g.coded_bits + 7) / 8;
}

hamming_status hamming_packet_layout(uint32_t msg_bytes, int t, uint32_t* seg_k, uint32_t* seg_n) {
  PacketGeom g;
  const hamming_status rc = packet_geom(msg_bytes, t, g);
  if (rc != HAMMING_OK) return rc;
  if (seg_k == nullptr || seg_n == nullptr) return set_err(HAMMING_E_NULL, "hamming_packet_layout: NULL output");
  for (int i = 0; i < t; ++i) {
    seg_k[i] = g.k[i];
    seg_n[i] = g.n[i];
  }
  return HAMMING_OK;
}

hamming_status hamming_packet_launch_shape(uint32_t msg_bytes, int t, uint64_t rx_stride, uint64_t n_packets,
                                           int sms, int* warps, int* G, int* L, int* ctas, int* smem) {
  PacketGeom g;
  hamming_status rc = packet_geom(msg_bytes, t, g);
  if (rc != HAMMING_OK) return rc;
  if (rx_stride % 16 != 0 || rx_stride < (g.coded_bits + 7) / 8)
    return set_err(HAMMING_E_ARG, "hamming_packet_launch_shape: rx_stride must be a multiple of 16 >= the coded bytes");
  PacketTables T;
  rc = build_packet_tables(g, T);
  if (rc != HAMMING_OK) return rc;
  BatchGeom bg;
  rc = batch_geom(g, T, rx_stride, std::min<uint64_t>(n_packets, 1ull << 31), sms, bg);
  if (rc != HAMMING_OK) return rc;
  const uint64_t bytes = bg.tab_bytes + static_cast<uint64_t>(bg.warps) * bg.warp_bytes;
  if (warps) *warps = static_cast<int>(bg.warps);
  if (G) *G = static_cast<int>(bg.G);
  if (L) *L = static_cast<int>(bg.L);
  if (ctas) *ctas = static_cast<int>(std::min<uint64_t>(228ull * 1024 / (bytes + 1536), 32 / bg.warps));
  if (smem) *smem = static_cast<int>(bytes);
  return HAMMING_OK;
}

static hamming_status packet_common(uint32_t msg_bytes, int t, uint64_t pk_stride, const void* pk, PacketGeom& g,
                                    const char* who) {
  const hamming_status rc = packet_geom(msg_bytes, t, g);
  if (rc != HAMMING_OK) return rc;
  if (pk_stride < g.in_bytes || (pk_stride & 15u) != 0) {
    snprintf(g_err, sizeof(g_err), "%s: packet stride must be a multiple of 16 and >= %u", who, g.in_bytes);
    return HAMMING_E_ARG;
  }
  if (!aligned16(pk)) return set_err(HAMMING_E_MISALIGNED, "packets: packet buffer must be 16-byte aligned");
  return HAMMING_OK;
}

hamming_status hamming_decode_packets(uint32_t msg_bytes, int t, const void* rx_dev, uint64_t rx_stride,
                                      uint64_t n_packets, void* msg_dev, uint64_t msg_stride,
                                      uint16_t* syndromes_dev, uint8_t* status_dev,
                                      unsigned long long* counts_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  PacketGeom g;
  hamming_status rc = packet_common(msg_bytes, t, rx_stride, rx_dev, g, "hamming_decode_packets");
  if (rc != HAMMING_OK) return rc;
  if (n_packets > 0 && (rx_dev == nullptr || msg_dev == nullptr))
    return set_err(HAMMING_E_NULL, "hamming_decode_packets: NULL buffer");
  if (msg_stride < msg_bytes) return set_err(HAMMING_E_ARG, "hamming_decode_packets: msg_stride < msg_bytes");
  if (n_packets > (~0ull) / rx_stride || n_packets > (~0ull) / msg_stride ||
      n_packets > (~0ull) / (2ull * static_cast<uint64_t>(t)))
    return set_err(HAMMING_E_RANGE, "hamming_decode_packets: n_packets * stride overflows");
  if ((reinterpret_cast<uintptr_t>(syndromes_dev) & 1u) != 0 || (reinterpret_cast<uintptr_t>(counts_dev) & 7u) != 0)
    return set_err(HAMMING_E_MISALIGNED,
                   "hamming_decode_packets: syndromes must be 2-byte and counts 8-byte aligned");
  {
    const void* buf[5] = {rx_dev, msg_dev, syndromes_dev, status_dev, counts_dev};
    const uint64_t len[5] = {rx_stride * n_packets, msg_stride * n_packets, 2ull * t * n_packets, n_packets,
                             counts_dev ? 16u : 0u};
    for (int i = 0; i < 5; ++i)
      for (int j = i + 1; j < 5; ++j)
        if (ranges_overlap(buf[i], len[i], buf[j], len[j]))
          return set_err(HAMMING_E_OVERLAP, "hamming_decode_packets: buffers overlap");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PacketArgs a{};  // counts: overwritten by the kernel itself (launch_packets_decode), no memset
  a.in = static_cast<const uint8_t*>(rx_dev);
  a.in_stride = rx_stride;
  a.out = static_cast<uint8_t*>(msg_dev);
  a.out_stride = msg_stride;
  a.syn = syndromes_dev;
  a.status = status_dev;
  a.counts = counts_dev;
  a.n_packets = n_packets;
  return launch_packets_decode(g, a, st);
}

hamming_status hamming_encode_packets(uint32_t msg_bytes, int t, const void* msg_dev, uint64_t msg_stride,
                                      uint64_t n_packets, void* rx_dev, uint64_t rx_stride, void* stream) {
  g_launches = 0;
  g_grid = 0;
  PacketGeom g;
  hamming_status rc = packet_common(msg_bytes, t, rx_stride, rx_dev, g, "hamming_encode_packets");
  if (rc != HAMMING_OK) return rc;
  if (n_packets > 0 && (rx_dev == nullptr || msg_dev == nullptr))
    return set_err(HAMMING_E_NULL, "hamming_encode_packets: NULL buffer");
  if (msg_stride < msg_bytes) return set_err(HAMMING_E_ARG, "hamming_encode_packets: msg_stride < msg_bytes");
  if (n_packets > (~0ull) / rx_stride || n_packets > (~0ull) / msg_stride)
    return set_err(HAMMING_E_RANGE, "hamming_encode_packets: n_packets * stride overflows");
  if (n_packets > 0 && ranges_overlap(msg_dev, msg_stride * n_packets, rx_dev, rx_stride * n_packets))
    return set_err(HAMMING_E_OVERLAP, "hamming_encode_packets: buffers overlap");
  PacketArgs a{};
  a.in = static_cast<const uint8_t*>(msg_dev);
  a.in_stride = msg_stride;
  a.out = static_cast<uint8_t*>(rx_dev);
  a.out_stride = rx_stride;
  a.n_packets = n_packets;
  return launch_packets<kPktEncode>(g, a, static_cast<cudaStream_t>(stream));
}

hamming_status hamming_packet_channel_generate(uint32_t msg_bytes, int t, uint64_t seed, uint64_t g_first,
                                               uint64_t n_packets, uint64_t thresh, int all, void* rx_dev,
                                               uint64_t rx_stride, void* msg_dev, void* stream) {
  g_launches = 0;
  g_grid = 0;
  PacketGeom g;
  hamming_status rc = packet_common(msg_bytes, t, rx_stride, rx_dev, g, "hamming_packet_channel_generate");
  if (rc != HAMMING_OK) return rc;
  if (n_packets > 0 && rx_dev == nullptr) return set_err(HAMMING_E_NULL, "hamming_packet_channel_generate: NULL rx");
  if (n_packets > (~0ull) / rx_stride || n_packets > (~0ull) / msg_bytes)
    return set_err(HAMMING_E_RANGE, "hamming_packet_channel_generate: n_packets * stride overflows");
  PacketArgs a{};
  a.out = static_cast<uint8_t*>(rx_dev);
  a.out_stride = rx_stride;
  a.n_packets = n_packets;
  a.seed = seed;
  a.g_first = g_first;
  a.thresh = thresh;
  a.all = all;
  a.gen_msg = static_cast<uint8_t*>(msg_dev);
  return launch_packets<kPktGenerate>(g, a, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
