// paper_1412_6862_b200/csrc/packets.cuh -- the paper's own workload (SURVEY.md
// 8(f) row f2), included into hamming.cu's anonymous namespace.
//
// A packet of msg_bytes message bytes is split into t segments ("splits
// the message into t segments H_1 ... H_t, where t is the error tolerance";
// near-equal, larger first: DESIGN.md reading R14) and every segment is one
// SHORTENED Hamming codeword: k_i message bits, the minimal r_i with
// 2^r >= k + r + 1 ("|H_i| = 7+4 = 11 bits and |R| = 4"), n_i = k_i + r_i,
// n up to 8013 bits on the paper's grid (M = 400..2000 B, t = 2..6).
// The encoded packet is H = H_1 + ... + H_t, LSB-first (reading R4).
//
// GPU design.  Encoder / synthetic channel (not the hot path): one warp per
// packet, the packet staged in shared memory.  Decoder: packets_decode_kernel
// (below) -- a warp decodes a batch of packets from shared memory in passes
// driven by host-built per-word slice tables; its syndrome is the checksum
// vector of P:L160 over 64-position chunks, s > n is the uncorrectable path
// (reading R15; SPEC detect_and_correct).  m = 7, 8 perfect-code streams:
// perfect_long_kernel (end of file).

constexpr int kPktMaxSeg = 16;
constexpr int kPktMaxMsgBytes = 4096;
#ifndef HAM_PKT_WARPS
#define HAM_PKT_WARPS 16
#endif
constexpr int kPktWarps = HAM_PKT_WARPS;

struct PacketGeom {
  uint32_t msg_bytes, t, coded_bits, in_bytes;  // in_bytes = coded bytes rounded up to 16
  uint32_t in_cap, msg_cap;                     // per-warp shared buffer sizes (bytes, 16-aligned)
  uint32_t off[kPktMaxSeg];                     // segment bit offset in the packet stream
  uint32_t n[kPktMaxSeg], k[kPktMaxSeg], r[kPktMaxSeg];
  uint32_t moff[kPktMaxSeg];                    // segment bit offset in the message
};

// host: the layout (same rule as the oracle's, written independently)
hamming_status packet_geom(uint32_t msg_bytes, int t, PacketGeom& g) {
  if (t < 1 || t > kPktMaxSeg) return set_err(HAMMING_E_ARG, "packets: t must be in [1, 16]");
  if (msg_bytes < 1 || msg_bytes > kPktMaxMsgBytes)
    return set_err(HAMMING_E_ARG, "packets: msg_bytes must be in [1, 4096]");
  const uint32_t bits = msg_bytes * 8u;
  if (bits < static_cast<uint32_t>(t)) return set_err(HAMMING_E_ARG, "packets: fewer message bits than segments");
  memset(&g, 0, sizeof(g));
  g.msg_bytes = msg_bytes;
  g.t = static_cast<uint32_t>(t);
  uint32_t off = 0, moff = 0;
  for (int i = 0; i < t; ++i) {
    const uint32_t k = bits / t + (static_cast<uint32_t>(i) < bits % t ? 1u : 0u);
    uint32_t r = 0;
    while ((1u << r) < k + r + 1) ++r;
    g.k[i] = k;
    g.r[i] = r;
    g.n[i] = k + r;
    g.off[i] = off;
    g.moff[i] = moff;
    off += k + r;
    moff += k;
  }
  g.coded_bits = off;
  g.in_bytes = ((off + 7) / 8 + 15) / 16 * 16;
  g.in_cap = g.in_bytes + 32;  // 16-byte front pad (decode) + slack for funnel reads past the end
  g.msg_cap = (msg_bytes + 15) / 16 * 16 + 16;
  return HAMMING_OK;
}

// 32 stream bits starting at bit o of a shared-memory word array.
__device__ __forceinline__ uint32_t sm_bits32(const uint32_t* w, uint32_t o) {
  const uint32_t q = o >> 5;
  return __funnelshift_r(w[q], w[q + 1], o & 31u);  // shift 0 returns w[q]
}

__device__ __forceinline__ uint32_t low_mask(uint32_t c) { return c >= 32 ? 0xFFFFFFFFu : ((1u << c) - 1u); }

// XOR of the indices of the set bits of a 32-bit word (5 POPCs).
__device__ __forceinline__ uint32_t xor_of_indices(uint32_t x) {
  return (static_cast<uint32_t>(__popc(x & 0xAAAAAAAAu) & 1) << 0) |
         (static_cast<uint32_t>(__popc(x & 0xCCCCCCCCu) & 1) << 1) |
         (static_cast<uint32_t>(__popc(x & 0xF0F0F0F0u) & 1) << 2) |
         (static_cast<uint32_t>(__popc(x & 0xFF00FF00u) & 1) << 3) |
         (static_cast<uint32_t>(__popc(x & 0xFFFF0000u) & 1) << 4);
}

// The decode buffer holds the packet from bit kPadBits on (one zero-padded
// 16-byte slot in front), so position 0 of the first segment -- stream bit -1
// -- is still inside the buffer and every chunk is one funnel shift.
constexpr uint32_t kPadBits = 128;


// Encoder side: codeword word cw (positions 32 cw .. 32 cw + 31) of segment
// (k, moff) built from the message words `msg` -- data positions only (parity
// positions and position 0 left 0).
__device__ __forceinline__ uint32_t segment_code_word(const uint32_t* msg, uint32_t n, uint32_t moff, uint32_t cw) {
  uint32_t out = 0;
  uint32_t p = max(32u * cw, 3u), p1 = min(32u * cw + 32u, n + 1);
  while (p < p1) {
    const uint32_t j = 31u - __clz(p);  // 2^j <= p < 2^(j+1)
    if (p == (1u << j)) {               // parity position
      ++p;
      continue;
    }
    const uint32_t run_end = min(p1, 2u << j);
    const uint32_t take = run_end - p;
    const uint32_t d = p - j - 2;
    out |= (sm_bits32(msg, moff + d) & low_mask(take)) << (p - 32u * cw);
    p = run_end;
  }
  return out;
}

// Encode the message in shared memory `msg` into the packet stream `w`
// (zeroed here, in_cap bytes) -- the "exact reverse process": data at
// the non-power-of-two positions, then parity bit 2^q = bit q of the syndrome
// of the data-only word (even parity over every I_q).  Warp-collective.
__device__ __forceinline__ void encode_packet_warp(const PacketGeom& g, const uint32_t* msg, uint32_t* w, int lane) {
  for (uint32_t i = lane; i < g.in_cap / 4; i += 32) w[i] = 0;
  __syncwarp();
  for (uint32_t i = 0; i < g.t; ++i) {
    const uint32_t off = g.off[i], n = g.n[i], moff = g.moff[i], r = g.r[i];
    const uint32_t words = (n + 32) / 32;  // position words 0 .. n/32
    uint32_t X = 0, P = 0;
    for (uint32_t cw = lane; cw < words; cw += 32) {
      uint32_t x = segment_code_word(msg, n, moff, cw);  // bit b = position 32cw + b
      X ^= x;
      P ^= (static_cast<uint32_t>(__popc(x)) & 1u) * (32u * cw);
      // position p sits at stream bit off + p - 1
      uint32_t base;
      if (cw == 0) {
        x >>= 1;  // drop position 0
        base = off;
      } else {
        base = off + 32 * cw - 1;
      }
      const uint32_t q = base >> 5, rr = base & 31u;
      if (x) {
        atomicOr(&w[q], x << rr);
        if (rr) atomicOr(&w[q + 1], x >> (32 - rr));
      }
    }
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) {
      X ^= __shfl_xor_sync(0xffffffffu, X, sh);
      P ^= __shfl_xor_sync(0xffffffffu, P, sh);
    }
    const uint32_t s = P ^ xor_of_indices(X);  // syndrome of the data-only word
    if (static_cast<uint32_t>(lane) < r && ((s >> lane) & 1u)) {
      const uint32_t b = off + (1u << lane) - 1;
      atomicOr(&w[b >> 5], 1u << (b & 31));
    }
    __syncwarp();
  }
}

__device__ __forceinline__ uint64_t pkt_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

enum PacketMode { kPktEncode = 1, kPktGenerate = 2 };

struct PacketArgs {
  const uint8_t* in;   // decode: received packets; encode: messages
  uint64_t in_stride;
  uint8_t* out;        // decode: messages; encode/generate: packets
  uint64_t out_stride;
  uint16_t* syn;       // decode: n_packets * t syndromes (nullable)
  uint8_t* status;     // decode: n_packets statuses (nullable)
  unsigned long long* counts;  // decode: [corrected segments, uncorrectable segments] (nullable)
  uint64_t n_packets;
  // generate
  uint64_t seed, g_first, thresh;
  int all;
  uint8_t* gen_msg;    // generate: sent messages (nullable), msg_bytes apart
  // decode counts without a memset: one CTA writes them (store_count), several publish through the
  // stream's launch slot (the last CTA writes the total and resets the slot), else per-CTA atomics
  // onto counts zeroed by the host; accumulate: add instead of overwrite (launches after the first)
  LaunchSlot* slot;
  int store_count, accumulate;
};

// Encoder / synthetic channel: one warp per packet (not on the hot path).
template <int MODE>
__global__ void __launch_bounds__(kPktWarps * 32)
    packets_kernel(const __grid_constant__ PacketGeom g, const __grid_constant__ PacketArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* wb = smem + warp * (g.in_cap + g.msg_cap);
  uint32_t* w = reinterpret_cast<uint32_t*>(wb);                  // packet stream
  uint32_t* mbuf = reinterpret_cast<uint32_t*>(wb + g.in_cap);    // message
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kPktWarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kPktWarps;
  for (uint64_t pk = gw; pk < a.n_packets; pk += nw) {
    uint8_t* mb = reinterpret_cast<uint8_t*>(mbuf);
    if constexpr (MODE == kPktEncode) {
      const uint8_t* src = a.in + pk * a.in_stride;
      for (uint32_t i = lane; i < g.msg_bytes; i += 32) mb[i] = src[i];
    } else {
      const uint64_t key = pkt_mix(a.seed + (a.g_first + pk + 1) * 0x9E3779B97F4A7C15ull);
      for (uint32_t q = lane; q < (g.msg_bytes + 7) / 8; q += 32) {
        const uint64_t u = pkt_mix(key + (static_cast<uint64_t>(q) + 1) * 0x9E3779B97F4A7C15ull);
        for (uint32_t b = 0; b < 8 && 8 * q + b < g.msg_bytes; ++b) mb[8 * q + b] = static_cast<uint8_t>(u >> (8 * b));
      }
    }
    for (uint32_t i = g.msg_bytes + lane; i < g.msg_cap; i += 32) mb[i] = 0;
    __syncwarp();
    encode_packet_warp(g, mbuf, w, lane);
    if constexpr (MODE == kPktGenerate) {
      const uint64_t key = pkt_mix(a.seed + (a.g_first + pk + 1) * 0x9E3779B97F4A7C15ull);
      const uint32_t W = (g.msg_bytes + 7) / 8;
      if (lane < static_cast<int>(g.t)) {
        const uint64_t ue = pkt_mix(key + (static_cast<uint64_t>(W) + 2 * lane + 1) * 0x9E3779B97F4A7C15ull);
        const uint64_t up = pkt_mix(key + (static_cast<uint64_t>(W) + 2 * lane + 2) * 0x9E3779B97F4A7C15ull);
        if (a.all || ue < a.thresh) {
          const uint32_t p = 1u + __umulhi(static_cast<uint32_t>(up), g.n[lane]);
          const uint32_t b = g.off[lane] + p - 1;
          atomicXor(&w[b >> 5], 1u << (b & 31));
        }
      }
      __syncwarp();
      if (a.gen_msg != nullptr) {
        uint8_t* gm = a.gen_msg + pk * g.msg_bytes;
        for (uint32_t i = lane; i < g.msg_bytes; i += 32) gm[i] = mb[i];
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(a.out + pk * a.out_stride);
    for (uint32_t i = lane; i < g.in_bytes / 16; i += 32) dst[i] = reinterpret_cast<const uint4*>(w)[i];
    __syncwarp();
  }
}

template <int MODE>
hamming_status launch_packets(const PacketGeom& g, const PacketArgs& a, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const size_t smem = static_cast<size_t>(kPktWarps) * (g.in_cap + g.msg_cap);
  auto kfn = packets_kernel<MODE>;
  int occ = 0;
  const hamming_status rc = kernel_blocks_per_sm(reinterpret_cast<const void*>(kfn), dev, kPktWarps * 32, smem,
                                                 false, occ);
  if (rc != HAMMING_OK) return rc;
  const uint64_t want = (a.n_packets + kPktWarps - 1) / kPktWarps;
  const int grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sm_count(dev)) * std::max(1, occ)));
  if (grid > 0) {
    kfn<<<grid, kPktWarps * 32, smem, st>>>(g, a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "packets kernel launch");
  }
  g_launches = grid > 0 ? 1 : 0;
  g_grid = grid;
  return HAMMING_OK;
}

// ---------------------------------------------------------------------------
// Packet decode.  A warp stages a BATCH of G consecutive packets in shared
// memory (TMA bulk, double-buffered) and decodes it in passes:
//   S  (syndrome, the checksum vector) -- per (packet, segment) item,
//      by a group of L lanes: s = XOR_j [32 j * parity(x_j)] ^ S5(XOR_j x_j);
//      the item's lead lane then writes the syndrome, the packet status and
//      the counts, applies a correctable s as a flip of the STREAM bit at
//      position s, and -- with HX (every k >= 96) -- compacts the segment's
//      head in place (the 57 data bits of positions 0..63 moved to 7..63) and
//      assembles the message word straddling the segment's start;
//   R  (redundancy removal + merger) -- one lane per 32-bit
//      message word.  The geometry is the same for every packet, so the host
//      precomputes, per message word, where its bits sit in the packet stream
//      as slices that stay inside one run (positions 2^j+1 .. 2^(j+1)-1) of
//      one segment.  From data index 57 on (after HX: everywhere) a run is
//      >= 57 bits long, so a word is one or two slices: two funnel shifts and
//      one merge.  "Head words" -- across a segment boundary, or without HX
//      near a segment head (runs of 1, 3, 7, 15, 31 bits) -- are skipped and
//   H  (only without HX) built by one lane each from their piece list.
// Every message word is written exactly once (X, R or H), so nothing is zeroed.
// ---------------------------------------------------------------------------
constexpr uint32_t kPktMaxWords = kPktMaxMsgBytes / 4;
#ifndef HAM_PKT_STAGES
#define HAM_PKT_STAGES 2
#endif
#ifndef HAM_PKT_MSGBUF
#define HAM_PKT_MSGBUF 1
#endif
constexpr uint32_t kPktStages = HAM_PKT_STAGES;   // input batches per warp (1 decoding + prefetch)
constexpr int kPktMsgBufs = HAM_PKT_MSGBUF;       // message buffers per warp
constexpr uint32_t kPktMaxSpecial = 80;   // <= 57 t / 32 + 2 t + 1 head words
constexpr uint32_t kPktMaxPieces = 640;

struct PacketTables {
  uint32_t Wp;                    // message words per packet, ceil(msg_bytes / 4)
  uint32_t n_special, n_pieces;
  uint32_t mag_t, mag_ns;  // floor(2^32 / d), d = t, n_special (divmod_small)
  uint32_t headx;                 // 1: segment heads are compacted in place first (pass X, kPktHeadxMinK)
  uint32_t Wfull, rem, mag_rem;   // pass R: Wp = Wfull + rem, Wfull a multiple of 32; floor(2^32 / rem)
  // src0 (bits 0..15) | nb0 (bits 16..21): a word is slice 0 (nb0 bits) and, if nb0 < 32, slice 1 =
  // the stream one bit after slice 0 ends (a skipped parity position); head words: 32 << 16
  uint32_t word0[kPktMaxWords];
  uint32_t special[kPktMaxSpecial + 1];  // word index | first piece << 16; [n_special]: end
  uint32_t piece[kPktMaxPieces];         // src (bits 0..15) | len (16..21) | pos (24..28)
  uint16_t piece_word[kPktMaxPieces];    // the head word a piece belongs to
  // with headx, the word straddling the start of segment i (i >= 1) is assembled by pass X:
  // bw[i] = its word index (0xFFFFFFFF: segment i starts word-aligned), bsrc[i] = src | nb0 << 16
  // of the last blen[i] data bits of segment i-1 (two slices, as in pass R), which fill its low bits
  uint32_t bw[kPktMaxSeg], bsrc[kPktMaxSeg], blen[kPktMaxSeg];
};
// src = bit of the packet stream (from its first bit) holding the slice's first data bit.

// host: data index -> run j: the data bits of run j (positions 2^j+1 .. 2^(j+1)-1)
// are d in [2^j - j - 1, 2^(j+1) - j - 3]; position = d + j + 2
uint32_t host_run_of(uint32_t d) {
  uint32_t j = 1;
  while (d >= (2u << j) - j - 2) ++j;
  return j;
}

// Pass X (heads compacted in place) needs every segment's 57-bit head window
// (positions 7..63) at least 32 bits clear of the next segment's, so that no
// two lanes rewrite the same stream word: k >= 96 gives n >= 103.
constexpr uint32_t kPktHeadxMinK = 96;

hamming_status build_packet_tables(const PacketGeom& g, PacketTables& T, bool allow_headx = true) {
  const uint32_t bits = g.msg_bytes * 8u;
  T.Wp = (g.msg_bytes + 3) / 4;
  uint32_t kmin = ~0u;
  for (uint32_t i = 0; i < g.t; ++i) kmin = std::min(kmin, g.k[i]);
  T.headx = (allow_headx && kmin >= kPktHeadxMinK) ? 1u : 0u;
  T.n_special = 0;
  T.n_pieces = 0;
  uint32_t seg = 0;
  for (uint32_t W = 0; W < T.Wp; ++W) {
    uint32_t src[32], len[32], pos[32], np = 0;
    uint32_t d = 32u * W;
    const uint32_t dend = std::min(32u * W + 32u, bits);
    while (d < dend) {
      while (d >= g.moff[seg] + g.k[seg]) ++seg;
      const uint32_t dl = d - g.moff[seg];
      if (T.headx && dl < 57) {  // after pass X: data bits 0..56 at positions 7..63, contiguous
        const uint32_t take = std::min(57u - dl, dend - d);
        src[np] = g.off[seg] + dl + 6;
        len[np] = take;
        pos[np] = d - 32u * W;
        ++np;
        d += take;
        continue;
      }
      const uint32_t j = host_run_of(dl);
      const uint32_t run_end = std::min((2u << j) - j - 2, g.k[seg]);
      const uint32_t take = std::min(run_end - dl, dend - d);
      src[np] = g.off[seg] + dl + j + 1;  // position dl + j + 2 is packet bit off + position - 1
      len[np] = take;
      pos[np] = d - 32u * W;
      ++np;
      d += take;
    }
    if (np == 1 || (np == 2 && src[1] == src[0] + len[0] + 1)) {  // slice 1 = the stream one bit later
      T.word0[W] = src[0] | (len[0] << 16);
    } else {
      if (T.n_special >= kPktMaxSpecial || T.n_pieces + np > kPktMaxPieces)
        return set_err(HAMMING_E_ARG, "packets: piece table overflow");
      T.word0[W] = 33u << 16;  // head word: not written by pass R
      T.special[T.n_special++] = W | (T.n_pieces << 16);
      for (uint32_t i = 0; i < np; ++i) {
        T.piece_word[T.n_pieces] = static_cast<uint16_t>(W);
        T.piece[T.n_pieces++] = src[i] | (len[i] << 16) | (pos[i] << 24);
      }
    }
  }
  T.special[T.n_special] = T.n_pieces << 16;
  for (uint32_t i = 0; i < kPktMaxSeg; ++i) T.bw[i] = 0xFFFFFFFFu, T.bsrc[i] = 0, T.blen[i] = 0;
  if (T.headx) {  // every head word must be one segment boundary: <= 2 tail slices, then the head
    for (uint32_t e = 0; e < T.n_special; ++e) {
      const uint32_t W = T.special[e] & 0xFFFFu, p0 = T.special[e] >> 16, p1 = T.special[e + 1] >> 16;
      uint32_t lt = 0, nt = 0, src0 = 0, len0 = 0;
      bool ok = p1 > p0;
      for (uint32_t q = p0; ok && q < p1; ++q) {
        const uint32_t src = T.piece[q] & 0xFFFFu, len = (T.piece[q] >> 16) & 63u, pos = T.piece[q] >> 24;
        if (q + 1 < p1) {  // a tail slice of segment i - 1
          if (nt == 0) src0 = src, len0 = len;
          else ok = ok && nt == 1 && src == src0 + len0 + 1;
          ok = ok && pos == lt;
          lt += len;
          ++nt;
        } else {  // the head of segment i: data index 0 at position 7
          uint32_t i = 1;
          while (i < g.t && g.moff[i] != 32u * W + lt) ++i;
          ok = ok && nt >= 1 && i < g.t && pos == lt && len == 32u - lt && src == g.off[i] + 6;
          if (ok) {
            T.bw[i] = W;
            T.bsrc[i] = src0 | ((nt == 1 ? 32u : len0) << 16);
            T.blen[i] = lt;
          }
        }
      }
      if (!ok) return build_packet_tables(g, T, false);  // not expected; decode without pass X
    }
  }
  auto mag = [](uint32_t d) { return d <= 1 ? 0xFFFFFFFFu : static_cast<uint32_t>((1ull << 32) / d); };
  T.mag_t = mag(g.t);
  T.mag_ns = mag(T.n_special);
  T.Wfull = T.Wp / 32 * 32;
  T.rem = T.Wp - T.Wfull;
  T.mag_rem = mag(T.rem);
  return HAMMING_OK;
}

// pass R: words (np = 1) or packets (np > 1) per unrolled step
constexpr uint32_t kPktRU = 4;

struct BatchGeom {
  uint32_t warps;      // warps per CTA (<= kPktWarps)
  uint32_t G;          // packets per batch
  uint32_t L;          // lanes per item in pass S (power of two)
  uint32_t in_cap;     // bytes per input buffer: 16 pad + G*stride + 16 slack
  uint32_t msg_cap;    // bytes of the message buffer: G packets of Wp words (+ slack)
  uint32_t warp_bytes; // 2*in_cap + msg_cap + status words
  uint32_t tab_bytes;  // CTA tables in front of the warp areas
  uint32_t slot_words; // shared-memory words from one staged packet to the next (>= rx_stride / 4)
  uint32_t copy_bytes; // 0: a batch is one TMA copy of G strides; else one copy of this many bytes per
                       // packet into its slot (restaged at slot_words to spread pass S over the banks)
};

hamming_status batch_geom(const PacketGeom& g, const PacketTables& T, uint64_t stride, uint64_t n_packets, int sms,
                          BatchGeom& b) {
  // a warp stages kPktStages whole strides: larger strides cannot be staged
  if (stride > (200u << 10) / kPktStages)
    return set_err(HAMMING_E_ARG, "packets: rx_stride too large to stage in shared memory (max 100 KiB)");
  uint32_t maxn = 0;
  for (uint32_t i = 0; i < g.t; ++i) maxn = max(maxn, g.n[i]);
  constexpr uint64_t kSmemSM = 227ull * 1024;
  b.tab_bytes = (16 * T.Wp + 8 * T.n_pieces + 8 * T.n_special + 4 * 7 * kPktMaxSeg + 15) / 16 * 16;
  // with head compaction (T.headx) the messages are written in place over the input stage: no
  // message buffer
  auto in_cap = [&](uint64_t G) { return 16 + G * stride + 16; };
  auto msg_cap = [&](uint64_t G) { return T.headx ? 0ull : (G * T.Wp * 4 + 15) / 16 * 16 + 16; };
  // kPktStages input buffers (TMA prefetch depth), kPktMsgBufs message buffers (bulk stores in flight),
  // statuses and the boundary words of pass X
  auto warp_bytes = [&](uint64_t G) {
    return kPktStages * in_cap(G) + kPktMsgBufs * msg_cap(G) + 16 * ((G * 4 * (1 + g.t) + 15) / 16);
  };
  // Launch shape by an issue model, over every warps-per-CTA w and packets-per-batch G
  // that fit: per packet, pass S costs ceil(G t / (32 / L)) rounds of a fixed set-up + epilogue
  // (~60 warp instructions with L >= 8, ~75 below) plus ceil(C64 / 4L) unrolled blocks of ~42 each,
  // pass R ~14 (one packet per batch) or ~9.5 warp instructions per 32 message words, and every batch
  // ~170 more; the issue rate falls off below 16 warps per SM as (W / 16)^0.7 (measured: 8 warps per
  // SM lose ~25 % against 12, 24 gain ~20 % in issue but pay more per-batch work, profiles/
  // r02_packets_tune.txt), and the last wave of batches counts as a whole wave.
  const uint32_t c64 = (maxn + 1) / 64 + 1;
  auto best_L = [&](uint64_t G, uint32_t& L) {
    const uint32_t items = static_cast<uint32_t>(G) * g.t;
    double best = 1e300;
    for (uint32_t l = 1; l <= 32; l *= 2) {
      const uint64_t rounds = (items + 32 / l - 1) / (32 / l);
      const double cost = static_cast<double>(rounds) * ((l >= 8 ? 60.0 : 75.0) + 42.0 * ((c64 + 4 * l - 1) / (4 * l)));
      if (cost < best) best = cost, L = l;
    }
    return best;
  };
  double score = 1e300;
  b.warps = 0;
  for (uint32_t w = 4; w <= static_cast<uint32_t>(kPktWarps); w += 2) {
    for (uint64_t G = 1; G <= 64; ++G) {
      const uint64_t smem = b.tab_bytes + w * warp_bytes(G);
      if (smem > kSmemSM) break;
      // 228 KB per SM, 1 KB reserved per CTA (+ the kernel's static tables); 64 registers per
      // thread cap an SM at 32 warps
      const uint64_t ctas = std::min<uint64_t>(228ull * 1024 / (smem + 1536), 32 / w);
      if (ctas == 0) continue;
      const double W = static_cast<double>(ctas * w);
      uint32_t L = 1;
      const double r_pp = (T.Wp / 32.0) * (G == 1 ? 14.0 : 9.5);
      const double per_packet = (best_L(G, L) + 170.0) / static_cast<double>(G) + r_pp;
      const double issue = std::pow(std::min(1.0, W / 16.0), 0.7);
      const uint64_t batches = (n_packets + G - 1) / G, slots = static_cast<uint64_t>(std::max(1, sms)) * ctas * w;
      const uint64_t waves = std::max<uint64_t>(1, (batches + slots - 1) / slots);
      const double eff = static_cast<double>(batches) / static_cast<double>(waves * slots);
      const double sc = per_packet / issue / std::max(eff, 1e-9);
      if (sc < score * 0.999) score = sc, b.warps = w, b.G = static_cast<uint32_t>(G), b.L = L;
    }
  }
#ifdef HAM_PKT_BUDGET  // tuning builds: the pre-round-2 budget rule
  {
    const uint64_t per = kPktStages * stride + (T.headx ? 0ull : kPktMsgBufs * 4ull * T.Wp) + 4 + 4ull * g.t;
    b.G = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((HAM_PKT_BUDGET - 96) / per, 64)));
    b.warps = kPktWarps;
    uint32_t L = 1;
    best_L(b.G, L);
    b.L = L;
  }
#endif
#ifdef HAM_PKT_L
  b.L = HAM_PKT_L;
#endif
#ifdef HAM_PKT_TUNE  // tuning builds only: warps per CTA and packets per batch from the environment
  if (const char* e = getenv("HAM_PKT_W")) b.warps = static_cast<uint32_t>(atoi(e));
  if (const char* e = getenv("HAM_PKT_G")) {
    b.G = static_cast<uint32_t>(atoi(e));
    uint32_t L = 1;
    best_L(b.G, L);
    b.L = L;
  }
#endif
#ifdef HAM_PKT_TUNE  // tuning builds only: lanes per item from the environment
  if (const char* e = getenv("HAM_PKT_L")) b.L = static_cast<uint32_t>(atoi(e));
#endif
  if (b.warps == 0) return set_err(HAMMING_E_ARG, "packets: one packet (rx_stride) does not fit shared memory");
  // Pass S reads 32 / L items at once at unrelated offsets; with the packets at their global stride
  // the same segment of packets p and p + 4 (any stride = 8 mod 32 words, e.g. M = 400) shares a
  // bank.  Restage the batch at slot_words = 4 (stride / 16 + j), j < 8 (TMA needs 16-byte slots),
  // choosing the j whose first round puts the fewest lanes on one bank (ties: the smallest j; j = 0
  // keeps the single TMA copy per batch).
  b.slot_words = static_cast<uint32_t>(stride / 4);
  b.copy_bytes = 0;
  {
    auto worst = [&](uint32_t sw) {
      uint32_t cnt[32] = {0}, mx = 0;
      const uint32_t items = std::min<uint32_t>(b.G * g.t, 32 / b.L);
      for (uint32_t it = 0; it < items; ++it) {
        const uint32_t pk = it / g.t, seg = it % g.t;
        const uint32_t base = (pk * sw * 32 + g.off[seg] + kPadBits - 1) >> 5;
        for (uint32_t q = 0; q < b.L; ++q) mx = std::max(mx, ++cnt[(base + 2 * q) & 31u]);
      }
      return mx;
    };
    uint32_t best_sw = b.slot_words, best = worst(b.slot_words);
    const uint32_t copy = (g.coded_bits + 7) / 8 + 15 - ((g.coded_bits + 7) / 8 + 15) % 16;  // coded bytes, to 16
    for (uint32_t j = 1; j < 8 && b.G > 1; ++j) {
      const uint32_t sw = static_cast<uint32_t>(stride / 4) + 4 * j;
      const uint32_t wv = worst(sw);
      if (wv < best) best = wv, best_sw = sw;
    }
    // only if the larger slots keep the CTAs per SM the shape was chosen with
    auto ctas_at = [&](uint32_t sw) {
      const uint64_t ic = 16 + static_cast<uint64_t>(b.G) * sw * 4 + 16;
      const uint64_t wbytes = kPktStages * ic + kPktMsgBufs * msg_cap(b.G) + 16 * ((b.G * 4ull * (1 + g.t) + 15) / 16);
      return 228ull * 1024 / (b.tab_bytes + b.warps * wbytes + 1536);
    };
    if (best_sw != b.slot_words && ctas_at(best_sw) >= ctas_at(b.slot_words)) {
      b.slot_words = best_sw;
      b.copy_bytes = copy;
    }
  }
  b.in_cap = static_cast<uint32_t>(16 + static_cast<uint64_t>(b.G) * b.slot_words * 4 + 16);
  b.msg_cap = static_cast<uint32_t>(msg_cap(b.G));
  b.warp_bytes = static_cast<uint32_t>(kPktStages * b.in_cap + kPktMsgBufs * b.msg_cap +
                                       16 * ((static_cast<uint64_t>(b.G) * 4 * (1 + g.t) + 15) / 16));
  while (b.warps > 1 && b.tab_bytes + static_cast<uint64_t>(b.warps) * b.warp_bytes > kSmemSM) --b.warps;
  if (b.tab_bytes + static_cast<uint64_t>(b.warp_bytes) > kSmemSM)
    return set_err(HAMMING_E_ARG, "packets: one packet (rx_stride) does not fit shared memory");
  return HAMMING_OK;
}

// The same syndrome over 64-position chunks (three shared loads per 64
// positions): chunk J = positions 64 J .. 64 J + 63 = (lo, hi) with
// Y_J = lo ^ hi, so X = XOR_J Y_J and
//   XOR_j [32 j par(x_j)] = 64 XOR_J [J par(Y_J)] ^ 32 par(XOR_J hi_J).
// Lane q takes J = q + L m, m = 4 blk + it (it < 4 unrolled), over the full
// chunks (64 J + 63 <= n; position 0's garbage bit counts for nothing, as
// above); with J = q | (L m): XOR over odd-parity J of J =
// q par(X) ^ L (4 BB ^ par(A0) ^ 2 par(A1)).  The group's rank-0 lane adds
// the tail (positions 64 Jf .. n, at most two masked 32-bit chunks).
template <uint32_t L>
__device__ __forceinline__ uint32_t group_syndrome64(const uint32_t* w, uint32_t off, uint32_t n, bool active,
                                                     uint32_t q, uint32_t mq, uint32_t gid) {
  const uint32_t o = off + kPadBits - 1;
  const uint32_t rb = o & 31u;
  const uint32_t np1 = active ? n + 1 : 0;  // positions 0 .. n
  const uint32_t full = np1 / 64;           // full 64-position chunks
  const uint32_t rest = np1 - 64 * full;    // positions of the partial chunk J = full (0 .. 63)
  const uint32_t nch = full + (rest != 0 ? 1u : 0u);
  // the partial chunk is a chunk like the others with the positions past n masked off: its
  // 64 full par(Y) and 32 par(hi) terms are exactly the generic ones
  const uint32_t mlo = __funnelshift_lc(0xFFFFFFFFu, 0u, rest);
  const uint32_t mhi = __funnelshift_lc(0xFFFFFFFFu, 0u, rest > 32 ? rest - 32 : 0u);
  const uint32_t* wq = w + (o >> 5) + 2 * q;
  uint32_t X = 0, H = 0, A0 = 0, A1 = 0, BB = 0;
  // one block = 4 chunks per lane; blocks below full / 4L are complete for every lane of the
  // group, so only the last block tests which of its chunks exist (and masks the partial one)
  auto block = [&](uint32_t blk, auto checked) {
    const uint32_t* wb = wq + 8 * L * blk;
    const int cnt = static_cast<int>(nch - 4 * L * blk) - static_cast<int>(q);
    uint32_t Xb = 0;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (!decltype(checked)::value || static_cast<int>(L) * it < cnt) {
        const uint32_t w0 = wb[2 * L * it], w1 = wb[2 * L * it + 1], w2 = wb[2 * L * it + 2];
        uint32_t hi = __funnelshift_r(w1, w2, rb), lo = __funnelshift_r(w0, w1, rb);
        if constexpr (decltype(checked)::value) {
          if (rest != 0 && static_cast<int>(L) * it == cnt - 1) {  // chunk J = full
            lo &= mlo;
            hi &= mhi;
          }
        }
        const uint32_t y = lo ^ hi;
        Xb ^= y;
        H ^= hi;
        if (it & 1) A0 ^= y;
        if (it & 2) A1 ^= y;
      }
    }
    X ^= Xb;
    BB ^= (__popc(Xb) & 1u) ? blk : 0u;
  };
  const uint32_t nb = full / (4 * L);
  for (uint32_t blk = 0; blk < nb; ++blk) block(blk, std::false_type{});
  if (4 * L * nb < nch) block(nb, std::true_type{});
  uint32_t P = (64u * ((q * (__popc(X) & 1u)) ^ L * ((4u * BB) ^ (__popc(A0) & 1u) ^ ((__popc(A1) & 1u) << 1)))) ^
               (32u * (__popc(H) & 1u));
  if constexpr (L == 32) {
    X = __reduce_xor_sync(0xffffffffu, X);
    P = __reduce_xor_sync(0xffffffffu, P);
  } else {
#pragma unroll
    for (uint32_t sh = L >> 1; sh > 0; sh >>= 1) {
      X ^= __shfl_xor_sync(0xffffffffu, X, sh);
      P ^= __shfl_xor_sync(0xffffffffu, P, sh);
    }
  }
  if constexpr (L >= 8) {  // S5(X) by five lanes of the group at once: lane q < 5 holds bit q
    const uint32_t bal = __ballot_sync(0xffffffffu, __popc(X & mq) & 1u);
    return P ^ ((bal >> (gid * L)) & 31u);
  } else {
    return P ^ xor_of_indices(X);
  }
}

// mask of the bit indices with bit q set (0xAAAAAAAA, 0xCCCCCCCC, ... 0xFFFF0000), 0 for q >= 5
__device__ __forceinline__ uint32_t index_bit_mask(uint32_t q) {
  if (q >= 5) return 0u;
  const uint32_t h = 1u << q;
  return (0xFFFFFFFFu / ((1u << h) + 1u)) << h;
}

// q = u / d, r = u % d from mag = floor(2^32 / d) (2^32 - 1 for d = 1): the
// estimate is q or q - 1, one correction step.
__device__ __forceinline__ uint32_t divmod_small(uint32_t u, uint32_t d, uint32_t mag, uint32_t& r) {
  uint32_t q = __umulhi(u, mag);
  r = u - q * d;
  if (r >= d) {
    ++q;
    r -= d;
  }
  return q;
}

// Pass R for U packets of one message word (descriptor d): all 2U loads first, then the U stores
// (the message words land in the input stage, below every stream word still to be read).
template <uint32_t U>
__device__ __forceinline__ void rr_step(const uint32_t* wp, uint32_t* mp, const uint4& d, uint32_t wstride,
                                        uint32_t mstride) {
  uint32_t x0[U], x1[U];
#pragma unroll
  for (uint32_t u = 0; u < U; ++u) x0[u] = wp[u * wstride], x1[u] = wp[u * wstride + 1];
#pragma unroll
  for (uint32_t u = 0; u < U; ++u)
    mp[u * mstride] = (__funnelshift_r(x0[u], x1[u], d.y) & d.z) | (__funnelshift_rc(x0[u], x1[u], d.w) & ~d.z);
}

template <uint32_t L, bool HX>
__global__ void __launch_bounds__(kPktWarps * 32)
    packets_decode_kernel(const __grid_constant__ PacketGeom g, const __grid_constant__ BatchGeom bg,
                          const __grid_constant__ PacketArgs a, const __grid_constant__ PacketTables T) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned long long cta_counts[2];
  __shared__ __align__(8) uint64_t bars_all[kPktWarps * kPktStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Wp = T.Wp, nsp = HX ? 0u : T.n_special;  // with HX pass X writes the head words
  // CTA tables: word descriptors {word, shift, mask of slice 0, keep}, head-word
  // pieces {src | len | pos, word}, per-segment geometry
  uint4* wdesc = reinterpret_cast<uint4*>(smem);
  uint2* pieces = reinterpret_cast<uint2*>(smem + 16 * Wp);
  uint2* spec = pieces + T.n_pieces;  // head words {word, first piece | end piece << 16}
  uint32_t* sg = reinterpret_cast<uint32_t*>(spec + T.n_special);  // [off | n | k | moff] x kPktMaxSeg
  for (uint32_t i = threadIdx.x; i < Wp; i += blockDim.x) {
    const uint32_t s0 = T.word0[i] & 0xFFFFu, nb = T.word0[i] >> 16;
    const bool head = nb > 32;  // head words: pass R skips them (pass H, or with HX pass X, writes them)
    // .w: the shift of slice 1 (1..32, the skipped parity bit), 0 for a head word (pass R skips it)
    wdesc[i] = make_uint4(s0 >> 5, s0 & 31u, nb >= 32 ? 0xFFFFFFFFu : (1u << nb) - 1u, head ? 0u : (s0 & 31u) + 1u);
  }
  for (uint32_t i = threadIdx.x; i < T.n_pieces; i += blockDim.x) pieces[i] = make_uint2(T.piece[i], T.piece_word[i]);
  for (uint32_t i = threadIdx.x; i < T.n_special; i += blockDim.x)
    spec[i] = make_uint2(T.special[i] & 0xFFFFu, (T.special[i] >> 16) | (T.special[i + 1] & 0xFFFF0000u));
  if (threadIdx.x < g.t) {
    sg[threadIdx.x] = g.off[threadIdx.x];
    sg[kPktMaxSeg + threadIdx.x] = g.n[threadIdx.x];
    sg[2 * kPktMaxSeg + threadIdx.x] = g.k[threadIdx.x];
    sg[3 * kPktMaxSeg + threadIdx.x] = g.moff[threadIdx.x];
    sg[4 * kPktMaxSeg + threadIdx.x] = T.bw[threadIdx.x];
    sg[5 * kPktMaxSeg + threadIdx.x] = T.bsrc[threadIdx.x];
    sg[6 * kPktMaxSeg + threadIdx.x] = T.blen[threadIdx.x];
  }
  uint8_t* wb = smem + bg.tab_bytes + warp * bg.warp_bytes;
  uint32_t* pst = reinterpret_cast<uint32_t*>(wb + kPktStages * bg.in_cap + kPktMsgBufs * bg.msg_cap);  // statuses
  uint32_t* bside = pst + bg.G;  // HX: the boundary message words of the batch's items, [packet][segment]
  uint64_t* bars = bars_all + warp * kPktStages;
  if (threadIdx.x < 2) cta_counts[threadIdx.x] = 0;
  __syncthreads();
  // one launch covers fewer than 2^31 packets (the host splits larger calls), so the batch
  // arithmetic is 32-bit; only the global addresses are 64-bit
  const uint32_t nP = static_cast<uint32_t>(a.n_packets);
  const uint32_t n_batches = (nP + bg.G - 1) / bg.G;
  const uint32_t gw = static_cast<uint32_t>(warp) * gridDim.x + blockIdx.x;  // CTA-minor (see tiles_kernel)
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  const uint64_t pol = policy_evict_first();
  const uint32_t q = static_cast<uint32_t>(lane) & (L - 1), gid = static_cast<uint32_t>(lane) / L;
  const uint32_t groups = 32 / L;
  const uint32_t mq = index_bit_mask(q);  // pass S, L >= 8: this lane's bit of S5
  const uint32_t in_stride = static_cast<uint32_t>(a.in_stride);
  const uint32_t wstride = bg.slot_words;  // shared-memory words from one packet's slot to the next
  const uint32_t stride_bits = wstride * 32;
  uint32_t n_corr = 0, n_fail = 0;
  // stage batch b into stage s (warp-uniform call): one TMA copy of the batch's strides, or with
  // restaging one copy per packet into its slot, issued by lane p (lane 0 arms the barrier first)
  auto load_batch = [&](uint32_t s, uint32_t b) {
    const uint32_t npb = min(nP - b * bg.G, bg.G);
    const uint8_t* src = a.in + static_cast<uint64_t>(b) * bg.G * in_stride;
    uint8_t* dst = wb + s * bg.in_cap + 16;
    if (bg.copy_bytes == 0) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&bars[s], npb * in_stride);
        bulk_g2s(dst, src, npb * in_stride, &bars[s], pol);
      }
    } else {
      if (lane == 0) mbar_arrive_expect_tx(&bars[s], npb * bg.copy_bytes);
      __syncwarp();
      for (uint32_t p = lane; p < npb; p += 32)
        bulk_g2s(dst + p * wstride * 4, src + p * in_stride, bg.copy_bytes, &bars[s], pol);
    }
  };
  if (lane == 0) {
    for (uint32_t s = 0; s < kPktStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  for (uint32_t s = 0; s < kPktStages; ++s)
    if (gw + s * nw < n_batches) load_batch(s, gw + s * nw);
  __syncwarp();
  // contiguous 16-byte-aligned messages leave by one TMA bulk store per batch (decided once:
  // with msg_bytes a multiple of 16 every batch's start stays aligned)
  const bool bulk_out = a.out_stride == g.msg_bytes && (g.msg_bytes & 15u) == 0 &&
                        (reinterpret_cast<uintptr_t>(a.out) & 15u) == 0;
  uint32_t it = 0;
  for (uint32_t b = gw; b < n_batches; b += nw, ++it) {
    const uint32_t buf = it % kPktStages;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(wb + buf * bg.in_cap);
    const uint32_t p0 = b * bg.G;
    const uint32_t np = min(nP - p0, bg.G);
    // messages: with HX in place -- packet p's message words over the start of its own slot of
    // the input stage (word W of a message never lands above the stream words it is built from,
    // see pass R), so no message buffer; otherwise a separate buffer, packet pk at word pk * Wp
    uint32_t* mbuf = HX ? const_cast<uint32_t*>(w) + 4
                        : reinterpret_cast<uint32_t*>(wb + kPktStages * bg.in_cap + (it % kPktMsgBufs) * bg.msg_cap);
    const uint32_t mstride = HX ? wstride : Wp;  // words from one packet's message to the next
    uint16_t* syn_b = a.syn != nullptr ? a.syn + static_cast<uint64_t>(p0) * g.t : nullptr;
    if constexpr (!HX) {
      if (lane == 0) bulk_wait_read<kPktMsgBufs - 1>();  // the bulk store that last used this mbuf has read it
    }
    // G <= 64: two predicated stores (a lane-strided loop here compiles to ~40 instructions of unroll set-up)
    if (static_cast<uint32_t>(lane) < np) pst[lane] = 0;
    if (static_cast<uint32_t>(lane) + 32 < np) pst[lane + 32] = 0;
    mbar_wait(&bars[buf], (it / kPktStages) & 1u);
    __syncwarp();
    {  // pass S: per (packet, segment) item, by groups of L lanes: the checksum vector of the
       // stream as received, then the item's epilogue -- syndrome out, packet status (max), counts, the
       // correction as a flip of the stream bit at position s (ED/EC) -- and, with HX, pass X:
       // the item's head compacted in place (the m = 6 RR of positions 0..63) for passes R and H
      uint32_t* wm = const_cast<uint32_t*>(w);
      const uint32_t items = np * g.t;
#pragma unroll 1
      for (uint32_t base = 0; base < items; base += groups) {
        const bool active = base + gid < items;
        uint32_t seg;
        const uint32_t pk = divmod_small(active ? base + gid : 0, g.t, T.mag_t, seg);
        const uint32_t n = active ? sg[kPktMaxSeg + seg] : 0;
        const uint32_t off = pk * stride_bits + sg[seg];
        const uint32_t s = group_syndrome64<L>(w, off, n, active, q, mq, gid);
        // every lane's loads of this round are done (the group reduction above is warp-synchronous):
        // flipping a bit of this item cannot race with another item's reads, whose chunks never
        // count a bit outside their own positions 0..n
        const bool lead = active && q == 0;
        if (lead) {
          const bool corr = s != 0 && s <= n;
          const bool fail = s > n;
          if (syn_b != nullptr) syn_b[pk * g.t + seg] = static_cast<uint16_t>(s);
          if (corr || fail) atomicMax(&pst[pk], fail ? 2u : 1u);
          n_corr += corr;
          n_fail += fail;
          if (corr) {  // position s is buffer bit kPadBits + off + s - 1
            const uint32_t fb = kPadBits + off + s - 1;
            atomicXor(&wm[fb >> 5], 1u << (fb & 31u));
          }
        }
        if constexpr (HX) {
          __syncwarp();  // every flip of this round has landed before a head word is rewritten
          if (lead) {
            const uint32_t o = off + kPadBits - 1;  // buffer bit of position 0
            uint32_t* wq = wm + (o >> 5);
            const uint32_t r = o & 31u;
            const uint32_t w0 = wq[0], w1 = wq[1], w2 = wq[2];
            // bit p of (x0, x1) = position p (p < 32 in x0)
            const uint32_t x0 = __funnelshift_r(w0, w1, r), x1 = __funnelshift_r(w1, w2, r);
            // data positions 3, 5..7, 9..15, 17..31, 33..63 -> bits 0..56 (the m = 6 compaction,
            // App. A) in 32-bit halves: d0 = bits 0..31 (positions 3..38), d1 = bits 32..56 (39..63)
            const uint32_t d0 = ((x0 >> 3) & 0x1u) | ((x0 >> 4) & 0xeu) | ((x0 >> 5) & 0x7f0u) |
                                ((x0 >> 6) & 0x3fff800u) | ((x1 << 25) & 0xfc000000u);
            const uint32_t d1 = x1 >> 7;
            // positions 0..6 kept, data at 7..63
            const uint32_t lo = (x0 & 0x7fu) | (d0 << 7), hi = (d0 >> 25) | (d1 << 7);
            const uint32_t lm = (1u << r) - 1u;
            // plain read-modify-write: with k >= 96 no other item's head window or flip shares these
            // words in this round, and the bits outside positions 7..63 are written back unchanged
            wq[0] = (w0 & lm) | (lo << r);
            wq[1] = __funnelshift_l(lo, hi, r);
            wq[2] = (w2 & ~lm) | __funnelshift_l(hi, 0u, r);
            const uint32_t W = sg[4 * kPktMaxSeg + seg];
            if (W != 0xFFFFFFFFu) {  // the message word straddling this segment's start (pass R skips it):
              // the last lt data bits of segment seg - 1 (corrected: its round came first), then the head
              const uint32_t bs = sg[5 * kPktMaxSeg + seg], lt = sg[6 * kPktMaxSeg + seg];
              const uint32_t s0 = kPadBits + pk * stride_bits + (bs & 0xFFFFu), nb0 = bs >> 16;
              const uint32_t a0 = wm[s0 >> 5], a1 = wm[(s0 >> 5) + 1];
              const uint32_t m0 = __funnelshift_lc(0xFFFFFFFFu, 0u, nb0);
              const uint32_t tail = ((__funnelshift_r(a0, a1, s0) & m0) | (__funnelshift_rc(a0, a1, (s0 & 31u) + 1) & ~m0)) &
                                    __funnelshift_lc(0xFFFFFFFFu, 0u, lt);
              bside[pk * g.t + seg] = tail | (d0 << lt);  // written into place after pass R
            }
          }
        }
      }
    }
    __syncwarp();
    if constexpr (HX) {  // refill the previous stage once its in-place bulk stores have read it
      if (it > 0) {
        bulk_wait_read<0>();  // every lane: the stores it issued for the previous batch
        __syncwarp();
        const uint32_t nx = b + (kPktStages - 1) * nw;
        const uint32_t ps = (it + kPktStages - 1) % kPktStages;
        if (nx < n_batches) load_batch(ps, nx);
      }
    }
    {  // pass R: every word as one or two slices (lane: word W of every packet of the batch).
       // Loads are issued kRU words (or packets) at a time before any store, so a
       // warp has kRU independent shared-memory round trips in flight instead of one
       // (the stores go to the message buffer, which no load of this pass reads).
      constexpr uint32_t kRU = kPktRU;
      // slice 1 is the stream one bit further on (the parity position skipped)
      auto rr = [](uint32_t a0, uint32_t a1, const uint4& d) {
        return (__funnelshift_r(a0, a1, d.y) & d.z) | (__funnelshift_rc(a0, a1, d.w) & ~d.z);
      };
      if (np == 1) {  // one packet per batch (long packets): kRU words per lane per step, then single words
        const uint32_t Wstep = Wp / (32 * kRU) * (32 * kRU);
        for (uint32_t W0 = lane; W0 < Wstep; W0 += 32 * kRU) {
          uint4 d[kRU];
          uint32_t x0[kRU], x1[kRU];
#pragma unroll
          for (uint32_t u = 0; u < kRU; ++u) d[u] = wdesc[W0 + 32 * u];
#pragma unroll
          for (uint32_t u = 0; u < kRU; ++u) x0[u] = w[4 + d[u].x], x1[u] = w[5 + d[u].x];
#pragma unroll
          for (uint32_t u = 0; u < kRU; ++u)
            if (d[u].w) mbuf[W0 + 32 * u] = rr(x0[u], x1[u], d[u]);  // d.w = 0: a head word
        }
#pragma unroll 1
        for (uint32_t W = Wstep + lane; W < Wp; W += 32) {
          const uint4 d = wdesc[W];
          const uint32_t a0 = w[4 + d.x], a1 = w[5 + d.x];
          if (d.w) mbuf[W] = rr(a0, a1, d);
        }
      } else {
        for (uint32_t W = lane; W < T.Wfull; W += 32) {
          const uint4 d = wdesc[W];  // {word, shift, mask of slice 0, shift + 1 (0: head word)}
          if (d.w == 0) continue;    // a head word: pass X (or H) writes it
          const uint32_t* wp = w + 4 + d.x;  // (after the 16-byte pad)
          uint32_t* mp = mbuf + W;  // packet p's word W at mbuf + p * mstride
          // kRU packets per step, then one exact step of the rest (no predicated-off slots: the
          // compiler would otherwise issue every slot of a wide unrolled step for np = 2 .. 3)
          uint32_t p = 0;
#pragma unroll 1
          for (; p + kRU <= np; p += kRU, wp += kRU * wstride, mp += kRU * mstride) rr_step<kRU>(wp, mp, d, wstride, mstride);
          switch (np - p) {
            case 3: rr_step<3>(wp, mp, d, wstride, mstride); break;
            case 2: rr_step<2>(wp, mp, d, wstride, mstride); break;
            case 1: rr_step<1>(wp, mp, d, wstride, mstride); break;
            default: break;
          }
        }
        // the last Wp mod 32 words of every packet, flattened over (packet, word)
        #pragma unroll 1
        for (uint32_t e = lane; e < np * T.rem; e += 32) {
          uint32_t c;
          const uint32_t p = divmod_small(e, T.rem, T.mag_rem, c);
          const uint32_t W = T.Wfull + c;
          const uint4 d = wdesc[W];
          const uint32_t* wp = w + 4 + d.x + p * wstride;
          const uint32_t a0 = wp[0], a1 = wp[1];
          if (d.w) mbuf[p * mstride + W] = rr(a0, a1, d);
        }
      }
    }
    __syncwarp();
    if (nsp > 0) {  // pass H: head words (segment boundaries; without pass X also segment heads), one lane per word
#pragma unroll 1
      for (uint32_t e = lane; e < np * nsp; e += 32) {
        uint32_t c;
        const uint32_t p = divmod_small(e, nsp, T.mag_ns, c);
        const uint2 sp = spec[c];
        const uint32_t pb = kPadBits + p * stride_bits;
        uint32_t v = 0;
#pragma unroll 1
        for (uint32_t i = sp.y & 0xFFFFu; i < (sp.y >> 16); ++i) {
          const uint32_t pc = pieces[i].x;
          const uint32_t s0 = pb + (pc & 0xFFFFu), len = (pc >> 16) & 63u;
          const uint32_t x = __funnelshift_r(w[s0 >> 5], w[(s0 >> 5) + 1], s0) & __funnelshift_lc(0xFFFFFFFFu, 0u, len);
          v |= x << ((pc >> 24) & 31u);
        }
        mbuf[p * Wp + sp.x] = v;
      }
    }
    __syncwarp();
    if constexpr (HX) {  // the boundary words pass X assembled, now that pass R has read the stream
      __syncwarp();
#pragma unroll 1
      for (uint32_t e = lane; e < np * g.t; e += 32) {
        uint32_t seg;
        const uint32_t p = divmod_small(e, g.t, T.mag_t, seg);
        const uint32_t W = sg[4 * kPktMaxSeg + seg];
        if (W != 0xFFFFFFFFu) mbuf[p * mstride + W] = bside[e];
      }
    } else {
      const uint32_t nx = b + kPktStages * nw;  // buffer consumed: prefetch the batch two steps ahead
      if (nx < n_batches) load_batch(buf, nx);
    }
    // write the batch's messages (packet pk at word pk * mstride of mbuf) and statuses
    const uint8_t* mb = reinterpret_cast<const uint8_t*>(mbuf);
    const uintptr_t ob = reinterpret_cast<uintptr_t>(a.out + static_cast<uint64_t>(p0) * a.out_stride);
    if (bulk_out) {
      fence_proxy_async_smem();  // this lane's st.shared / atomics visible to the bulk copy
      __syncwarp();
      if constexpr (HX) {  // one bulk store per packet, from its slot, issued by lane p
        for (uint32_t pk = lane; pk < np; pk += 32)
          bulk_s2g(reinterpret_cast<void*>(ob + pk * g.msg_bytes), mbuf + pk * mstride, g.msg_bytes, pol);
        bulk_commit();
      } else if (lane == 0) {
        bulk_s2g(reinterpret_cast<void*>(ob), mbuf, np * g.msg_bytes, pol);
        bulk_commit();
      }
    } else if ((g.msg_bytes & 3u) == 0 && (a.out_stride & 3u) == 0 && (ob & 3u) == 0) {
      __syncwarp();
      for (uint32_t pk = 0; pk < np; ++pk) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(ob + pk * a.out_stride);
        for (uint32_t i = lane; i < Wp; i += 32) dst[i] = mbuf[pk * mstride + i];
      }
    } else {
      __syncwarp();
      for (uint32_t pk = 0; pk < np; ++pk) {
        uint8_t* dst = reinterpret_cast<uint8_t*>(ob + pk * a.out_stride);
        for (uint32_t i = lane; i < g.msg_bytes; i += 32) dst[i] = mb[pk * mstride * 4 + i];
      }
    }
    if (a.status != nullptr) {
      if (static_cast<uint32_t>(lane) < np) a.status[p0 + lane] = static_cast<uint8_t>(pst[lane]);
      if (static_cast<uint32_t>(lane) + 32 < np) a.status[p0 + lane + 32] = static_cast<uint8_t>(pst[lane + 32]);
    }
    __syncwarp();
  }
  bulk_wait<0>();  // every lane: its last bulk stores have completed before shared memory goes away
  if (a.counts != nullptr) {
    n_corr = __reduce_add_sync(0xffffffffu, n_corr);
    n_fail = __reduce_add_sync(0xffffffffu, n_fail);
    if (lane == 0) {
      if (n_corr) atomicAdd(&cta_counts[0], static_cast<unsigned long long>(n_corr));
      if (n_fail) atomicAdd(&cta_counts[1], static_cast<unsigned long long>(n_fail));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (a.store_count) {  // a single-CTA launch owns the counts
        for (int i = 0; i < 2; ++i) a.counts[i] = (a.accumulate ? a.counts[i] : 0ull) + cta_counts[i];
      } else if (a.slot != nullptr) {  // the last CTA to arrive publishes the totals and resets the slot
        for (int i = 0; i < 2; ++i)
          if (cta_counts[i]) atomicAdd(&a.slot->sum[i], cta_counts[i]);
        __threadfence();
        if (atomicAdd(&a.slot->done, 1u) == gridDim.x - 1) {
          __threadfence();
          for (int i = 0; i < 2; ++i) {
            const unsigned long long tot = atomicExch(&a.slot->sum[i], 0ull);
            a.counts[i] = (a.accumulate ? a.counts[i] : 0ull) + tot;
          }
          a.slot->claim = 0;
          a.slot->done = 0;
        }
      } else {
        if (cta_counts[0]) atomicAdd(&a.counts[0], cta_counts[0]);
        if (cta_counts[1]) atomicAdd(&a.counts[1], cta_counts[1]);
      }
    }
  }
}

hamming_status launch_packets_decode(const PacketGeom& g, const PacketArgs& a, cudaStream_t st) {
  static thread_local PacketTables T;  // rebuilt only when the geometry changes
  static thread_local uint32_t T_msg = 0, T_t = 0;
  if (T_msg != g.msg_bytes || T_t != g.t) {
    T_msg = 0;
    const hamming_status rc = build_packet_tables(g, T);
    if (rc != HAMMING_OK) return rc;
    T_msg = g.msg_bytes;
    T_t = g.t;
  }
  BatchGeom bg;
  int dev0 = 0;
  if (cudaGetDevice(&dev0) != cudaSuccess) dev0 = 0;
  hamming_status rc = batch_geom(g, T, a.in_stride, std::min<uint64_t>(a.n_packets, 1ull << 31), sm_count(dev0), bg);
  if (rc != HAMMING_OK) return rc;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const size_t smem = bg.tab_bytes + static_cast<size_t>(bg.warps) * bg.warp_bytes;
  if (smem > 227 * 1024) return set_err(HAMMING_E_ARG, "packets: shared memory budget exceeded");
  void (*kfn)(PacketGeom, BatchGeom, PacketArgs, PacketTables) = nullptr;
#define HAM_PKT_KFN(HX)                                   \
  switch (bg.L) {                                         \
    case 1: kfn = packets_decode_kernel<1, HX>; break;    \
    case 2: kfn = packets_decode_kernel<2, HX>; break;    \
    case 4: kfn = packets_decode_kernel<4, HX>; break;    \
    case 8: kfn = packets_decode_kernel<8, HX>; break;    \
    case 16: kfn = packets_decode_kernel<16, HX>; break;  \
    default: kfn = packets_decode_kernel<32, HX>; break;  \
  }
  if (T.headx) {
    HAM_PKT_KFN(true)
  } else {
    HAM_PKT_KFN(false)
  }
#undef HAM_PKT_KFN
  // the full shared-memory carveout so several CTAs fit per SM
  int occ = 0;
  rc = kernel_blocks_per_sm(reinterpret_cast<const void*>(kfn), dev, bg.warps * 32, smem, true, occ);
  if (rc != HAMMING_OK) return rc;
  // the kernel's batch arithmetic is 32-bit: one launch per 2^31 packets (counts accumulate)
  constexpr uint64_t kMaxPackets = 1ull << 31;
  int launches = 0, grid = 0;
  LaunchSlot* slot = (a.counts != nullptr) ? launch_slot(dev, st) : nullptr;
  if (a.counts != nullptr && a.n_packets == 0) {  // nothing to decode: the counts are still overwritten
    e = cudaMemsetAsync(a.counts, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counts)");
  }
  for (uint64_t first = 0; first < a.n_packets; first += kMaxPackets) {
    PacketArgs c = a;
    c.n_packets = std::min(kMaxPackets, a.n_packets - first);
    c.in = a.in + first * a.in_stride;
    c.out = a.out + first * a.out_stride;
    if (a.syn != nullptr) c.syn = a.syn + first * g.t;
    if (a.status != nullptr) c.status = a.status + first;
    const uint64_t batches = (c.n_packets + bg.G - 1) / bg.G;
    const uint64_t want = (batches + bg.warps - 1) / bg.warps;
    grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sm_count(dev)) * std::max(1, occ)));
    c.accumulate = first > 0 ? 1 : 0;
    c.store_count = grid == 1 ? 1 : 0;
    c.slot = grid > 1 ? slot : nullptr;
    if (a.counts != nullptr && grid > 1 && slot == nullptr && first == 0) {  // no slot (graph capture): memset + atomics
      e = cudaMemsetAsync(a.counts, 0, 2 * sizeof(unsigned long long), st);
      if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counts)");
    }
    kfn<<<grid, bg.warps * 32, smem, st>>>(g, bg, c, T);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "packets decode launch");
    ++launches;
  }
  g_launches = launches;
  g_grid = grid;
  return HAMMING_OK;
}

struct LongArgs {
  const uint8_t* in;
  uint8_t* out;
  uint8_t* syn;
  unsigned long long* counter;
  uint64_t N, in_total, out_total;
  uint32_t n, k, store_count;
};

// ---------------------------------------------------------------------------
// Longer perfect codes, m = 7, 8 ((127,120), (255,247)):
// one lane per codeword, 2^m codewords per batch.  With n = 2^m - 1 a batch
// of 2^m codewords is exactly n UNITS of 2^m bits (UW = 2^m / 32 words, 16-
// or 32-byte aligned), and codeword c's window -- positions 0..2^m-1, i.e.
// stream bits [c n - 1, c n - 1 + 2^m) -- starts in unit c-1 at bit
// 2^m - 1 - c.  With c = lane + 32 i that is word UW-1-i (the same for the
// whole warp: i is unrolled) at bit 31 - lane, so a lane loads its own unit
// c with vector loads and takes the tail words of unit c-1 from lane-1 by
// shuffle (lane 0: from lane 31's previous unit): no bank conflicts, one
// funnel shift per window word.  Syndrome: position p = 32 j + b, so
// s = S5(XOR_j v_j) ^ 32 XOR_j [j par(v_j)] (m + 2 POPCs); flip; redundancy
// removal = the (31,26) compaction of v_0 then v_1 >> 1, v_2 >> 1, v_3
// (m = 8: v_4 >> 1, v_5..v_7); the k data bits are funnel-shifted to their
// bit offset k*lane in the 32-codeword output block (k words, aligned), the
// word shared with the next lane passed up by one shuffle, and staged in
// shared memory for one TMA bulk store per batch.
// ---------------------------------------------------------------------------
template <int M>
struct LongGeo {
  static constexpr int UW = (1 << M) / 32;          // words per unit (= per codeword window)
  static constexpr int n = (1 << M) - 1, k = n - M;
  static constexpr int KW = (k + 31) / 32;           // data words per codeword
  static constexpr int B = 1 << M;                   // codewords per batch
  static constexpr int IN_BYTES = n * UW * 4;        // = B n / 8
  static constexpr int OUT_BYTES = B * k / 8;
};

template <int M>
__device__ __forceinline__ uint32_t long_batch(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                               uint8_t* __restrict__ sbuf, uint32_t nvalid, uint32_t lane) {
  using G = LongGeo<M>;
  constexpr int UW = G::UW, k = G::k, KW = G::KW;
  uint32_t cnt = 0;
  uint32_t Uprev[UW];
#pragma unroll
  for (int j = 0; j < UW; ++j) Uprev[j] = 0;  // unit -1: only position 0 of codeword 0 (ignored)
#pragma unroll
  for (int i = 0; i < G::B / 32; ++i) {
    const uint32_t c = lane + 32u * i;
    uint32_t P[2 * UW];  // units c-1 and c
    const uint4* up = reinterpret_cast<const uint4*>(in + c * UW);
#pragma unroll
    for (int q = 0; q < UW / 4; ++q) {
      const uint4 x = up[q];
      P[UW + 4 * q] = x.x;
      P[UW + 4 * q + 1] = x.y;
      P[UW + 4 * q + 2] = x.z;
      P[UW + 4 * q + 3] = x.w;
    }
    const int w0 = UW - 1 - i;  // first window word (a constant: i is unrolled)
#pragma unroll
    for (int j = 0; j < UW; ++j) {
      if (j >= w0) {
        const uint32_t send = (lane == 31) ? Uprev[j] : P[UW + j];
        P[j] = __shfl_sync(0xffffffffu, send, (lane + 31) & 31);
      } else {
        P[j] = 0;
      }
    }
#pragma unroll
    for (int j = 0; j < UW; ++j) Uprev[j] = P[UW + j];
    const uint32_t r = 31u - lane;
    uint32_t v[UW];
#pragma unroll
    for (int j = 0; j < UW; ++j) v[j] = __funnelshift_r(P[w0 + j], P[w0 + j + 1], r);
    // syndrome (a2): low five bits from the XOR of the window words, high bits from their parities
    uint32_t X = 0;
#pragma unroll
    for (int j = 0; j < UW; ++j) X ^= v[j];
    uint32_t s = xor_of_indices(X);
#pragma unroll
    for (int b = 0; (1 << b) < UW; ++b) {
      uint32_t y = 0;
#pragma unroll
      for (int j = 0; j < UW; ++j)
        if ((j >> b) & 1) y ^= v[j];
      s |= (static_cast<uint32_t>(__popc(y)) & 1u) << (5 + b);
    }
    // a3: flip position s (s = 0: the dummy position 0)
    const uint32_t fbit = 1u << (s & 31u);
#pragma unroll
    for (int j = 0; j < UW; ++j) v[j] ^= ((s >> 5) == static_cast<uint32_t>(j)) ? fbit : 0u;
    // a4: redundancy removal into D (k bits)
    uint32_t D[KW];
#pragma unroll
    for (int j = 0; j < KW; ++j) D[j] = 0;
    uint32_t d0 = 0;
#pragma unroll
    for (int g = 1; g < 5; ++g) d0 |= (v[0] >> (g + 2)) & dmask(g);
    put_bits(D, 0, d0, 26);
    put_bits(D, 26, v[1] >> 1, 31);
    put_bits(D, 57, v[2] >> 1, 31);
    put_bits(D, 88, v[3], 32);
    if constexpr (M == 8) {
      put_bits(D, 120, v[4] >> 1, 31);
      put_bits(D, 151, v[5], 32);
      put_bits(D, 183, v[6], 32);
      put_bits(D, 215, v[7], 32);
    }
    // a5: place the k bits at bit k*lane of this iteration's k-word output block
    const uint32_t b0 = static_cast<uint32_t>(k) * lane, sh = b0 & 31u, q0 = b0 >> 5;
    const uint32_t nw = ((b0 + k - 1) >> 5) - q0 + 1;
    const bool end_partial = ((b0 + k) & 31u) != 0;
    uint32_t O[KW + 1];
    O[0] = D[0] << sh;
#pragma unroll
    for (int j = 1; j < KW; ++j) O[j] = __funnelshift_l(D[j - 1], D[j], sh);
    O[KW] = __funnelshift_l(D[KW - 1], 0u, sh);
    const uint32_t tail = (nw - 1 == static_cast<uint32_t>(KW)) ? O[KW] : O[KW - 1];
    const uint32_t prev = __shfl_up_sync(0xffffffffu, tail, 1);
    if (sh != 0) O[0] |= prev;  // the word shared with lane - 1 (never lane 0: blocks are word-aligned)
    uint32_t* ob = out + i * k + q0;
#pragma unroll
    for (int j = 0; j <= KW; ++j)
      if (static_cast<uint32_t>(j) < nw && !(static_cast<uint32_t>(j) + 1 == nw && end_partial)) ob[j] = O[j];
    sbuf[c] = static_cast<uint8_t>(s);  // staged: the batch's B syndrome bytes leave by one bulk store
    cnt += (c < nvalid) & (s != 0);
  }
  return cnt;
}

template <int M, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    perfect_long_kernel(const __grid_constant__ LongArgs a) {
  using G = LongGeo<M>;
  constexpr uint32_t IN_B = G::IN_BYTES, OUT_B = G::OUT_BYTES, SYN_B = G::B;
  // two input buffers (TMA prefetch), one output buffer {data, syndromes}: measured, a second
  // output buffer (no wait for the previous batch's store) costs more in warps per SM than the
  // wait does ((127,120) 0.94 -> 0.86, round 2)
  constexpr uint32_t WARP_BYTES = 2 * IN_B + OUT_B + SYN_B;  // every part a multiple of 16 bytes
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned long long cta_count;
  __shared__ __align__(8) uint64_t bars_all[WARPS * 2];
  const int warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31u;
  uint8_t* wb = smem + warp * WARP_BYTES;
  uint64_t* bars = bars_all + warp * 2;
  if (threadIdx.x == 0) cta_count = 0;
  __syncthreads();
  const uint64_t n_full = a.N / G::B;
  const uint64_t n_batches = (a.N + G::B - 1) / G::B;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * WARPS + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * WARPS;
  const uint64_t pol = policy_evict_first();
  uint32_t cnt = 0;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    for (uint32_t s = 0; s < 2; ++s) {
      const uint64_t b = gw + s * nw;
      if (b < n_full) {
        mbar_arrive_expect_tx(&bars[s], IN_B);
        bulk_g2s(wb + s * IN_B, a.in + b * IN_B, IN_B, &bars[s], pol);
      }
    }
  }
  __syncwarp();
  uint32_t it = 0;
  for (uint64_t b = gw; b < n_batches; b += nw, ++it) {
    const uint32_t buf = it & 1u;
    uint8_t* ib = wb + buf * IN_B;
    const bool full = b < n_full;
    const uint32_t nvalid = full ? G::B : static_cast<uint32_t>(a.N - b * G::B);
    uint32_t* obuf = reinterpret_cast<uint32_t*>(wb + 2 * IN_B);
    uint8_t* sbuf = wb + 2 * IN_B + OUT_B;
    if (lane == 0) bulk_wait_read<0>();  // the previous batch's bulk stores have read obuf and sbuf
    if (full) {
      mbar_wait(&bars[buf], (it >> 1) & 1u);
    } else {  // the ragged last batch: bounded, zero-padded loads (TMA moves whole 16-byte units)
      const uint64_t ib0 = b * IN_B, nbytes = a.in_total - ib0;
      for (uint32_t i = lane; i < IN_B; i += 32) ib[i] = i < nbytes ? a.in[ib0 + i] : 0;
    }
    __syncwarp();
    cnt += long_batch<M>(reinterpret_cast<const uint32_t*>(ib), obuf, sbuf, nvalid, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0 && full) {
      bulk_s2g(a.out + b * OUT_B, obuf, OUT_B, pol);
      if (a.syn != nullptr) bulk_s2g(a.syn + b * SYN_B, sbuf, SYN_B, pol);
      bulk_commit();
      const uint64_t nx = b + 2 * nw;  // the input buffer is consumed: prefetch two batches ahead
      if (nx < n_full) {
        mbar_arrive_expect_tx(&bars[buf], IN_B);
        bulk_g2s(ib, a.in + nx * IN_B, IN_B, &bars[buf], pol);
      }
    }
    if (!full) {  // bounded byte stores of the ragged batch
      const uint64_t ob0 = b * OUT_B, nbytes = a.out_total - ob0;
      const uint8_t* mb = reinterpret_cast<const uint8_t*>(obuf);
      const uint32_t last_bits = static_cast<uint32_t>((a.N * G::k) & 7u);  // valid bits of the last byte
      for (uint32_t i = lane; i < nbytes && i < OUT_B; i += 32) {
        uint8_t x = mb[i];
        if (i + 1 == nbytes && last_bits != 0) x &= static_cast<uint8_t>((1u << last_bits) - 1u);  // pad bits 0
        a.out[ob0 + i] = x;
      }
      if (a.syn != nullptr)
        for (uint32_t i = lane; i < nvalid; i += 32) a.syn[b * SYN_B + i] = sbuf[i];
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait<0>();
  if (a.counter != nullptr) {
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0 && cnt) atomicAdd(&cta_count, static_cast<unsigned long long>(cnt));
    __syncthreads();
    if (threadIdx.x == 0) {
      if (a.store_count) *a.counter = cta_count;
      else if (cta_count) atomicAdd(a.counter, cta_count);
    }
  }
}

template <int M, int WARPS>
hamming_status launch_perfect_long(const LongArgs& a0, cudaStream_t st, bool accumulate) {
  using G = LongGeo<M>;
  LongArgs a = a0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  auto kfn = perfect_long_kernel<M, WARPS>;
  const size_t smem = static_cast<size_t>(WARPS) * (2 * G::IN_BYTES + G::OUT_BYTES + G::B);
  int occ = 0;
  const hamming_status rc = kernel_blocks_per_sm(reinterpret_cast<const void*>(kfn), dev, WARPS * 32, smem, true, occ);
  if (rc != HAMMING_OK) return rc;
  const uint64_t batches = (a.N + G::B - 1) / G::B;
  const uint64_t want = (batches + WARPS - 1) / WARPS;
  const int grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sm_count(dev)) * std::max(1, occ)));
  a.store_count = (a.counter != nullptr && !accumulate && grid == 1) ? 1u : 0u;
  if (a.counter != nullptr && !accumulate && !a.store_count) {
    e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(corrected)");
  }
  if (grid > 0) {
    kfn<<<grid, WARPS * 32, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "long decode launch");
  }
  g_launches = grid > 0 ? 1 : 0;
  g_grid = grid;
  return HAMMING_OK;
}

hamming_status launch_long_decode(int m, const uint8_t* in, uint64_t N, uint8_t* out, uint8_t* syn,
                                  unsigned long long* counter, cudaStream_t st, bool accumulate) {
  LongArgs a{};
  a.n = (1u << m) - 1;
  a.k = a.n - static_cast<uint32_t>(m);
  a.in = in;
  a.out = out;
  a.syn = syn;
  a.counter = counter;
  a.N = N;
  a.in_total = (static_cast<uint64_t>(a.n) * N + 7) / 8;
  a.out_total = (static_cast<uint64_t>(a.k) * N + 7) / 8;
#ifndef HAM_LONG_W7
#define HAM_LONG_W7 16
#endif
#ifndef HAM_LONG_W8
#define HAM_LONG_W8 8
#endif
  if (N == 0 && counter != nullptr && !accumulate) {
    const cudaError_t e0 = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(corrected)");
    g_launches = 0;
    g_grid = 0;
    return HAMMING_OK;
  }
  if (m == 7) return launch_perfect_long<7, HAM_LONG_W7>(a, st, accumulate);
  return launch_perfect_long<8, HAM_LONG_W8>(a, st, accumulate);
}
