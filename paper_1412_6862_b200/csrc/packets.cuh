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
// GPU design: one warp per packet (grid-stride over packets), the packet
// staged in shared memory with coalesced 128-bit loads.
// Per segment:
//   syndrome (the checksum vector): position p = 32 j + b, so
//     s = XOR_j [32 j * parity(x_j)]  ^  S5( XOR_j x_j ),
//   where x_j is the 32-position chunk j and S5(x) = XOR of the bit indices
//   of x (five POPCs).  S5 is linear, so each lane XORs its chunks and pays
//   one POPC per chunk for the parity; one warp XOR-reduction; S5 once.
//   ED/EC: s = 0 clean; 1 <= s <= n flip bit s (one lane, in shared memory);
//   s > n names a non-existent position: uncorrectable, bits left as received
//   (reading R15; SPEC detect_and_correct).
//   RR + merger: data index d of position p in run j (2^j < p < 2^(j+1)) is
//   p - j - 2, so every 32-bit word of the message is 1..3 funnel-shifted
//   slices of the packet stream; lanes build consecutive message words.

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

// Data index -> run: the data bits of run j (positions 2^j+1 .. 2^(j+1)-1) are
// d in [2^j - j - 1, 2^(j+1) - j - 3]; position = d + j + 2.  Closed form
// j = floor(log2(d + floor(log2(d + 2)) + 2)) (checked exhaustively for
// d < 200000, far past the largest segment).
__device__ __forceinline__ uint32_t run_of(uint32_t d) {
  const uint32_t j0 = 31u - __clz(d + 2);
  return 31u - __clz(d + j0 + 2);
}

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
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(packets)");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kPktWarps * 32, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy(packets)");
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
// memory (TMA bulk, double-buffered) and decodes it in three passes:
//   R  (redundancy removal + merger) -- one lane per 32-bit
//      message word.  The geometry is the same for every packet, so the host
//      precomputes, per message word, where its bits sit in the packet stream
//      as "pieces": maximal slices that stay inside one run (positions
//      2^j+1 .. 2^(j+1)-1) of one segment.  From data index 57 on a run is
//      >= 63 bits long, so almost every word is one or two slices: two funnel
//      shifts and one merge.  The few words near a segment head (data index
//      < 57: runs of 1, 3, 7, 15, 31 bits) or across a segment boundary are
//   H  ("head" words) built by one lane each from their piece list;
//   S  (syndrome, the checksum vector) -- per (packet, segment) item,
//      by a group of L lanes: s = XOR_j [32 j * parity(x_j)] ^ S5(XOR_j x_j);
//      a correctable s flips the corrected data bit of the message in place.
// Every message word is written exactly once (R or H), so nothing is zeroed.
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
  uint32_t mag_t, mag_ns, mag_wp, mag_np;  // floor(2^32 / d), d = t, n_special, Wp, n_pieces (divmod_small)
  // src0 (bits 0..15) | nb0 (bits 16..21): a word is slice 0 (nb0 bits) and, if nb0 < 32, slice 1 =
  // the stream one bit after slice 0 ends (a skipped parity position); head words: 32 << 16
  uint32_t word0[kPktMaxWords];
  uint32_t special[kPktMaxSpecial + 1];  // word index | first piece << 16; [n_special]: end
  uint32_t piece[kPktMaxPieces];         // src (bits 0..15) | len (16..21) | pos (24..28)
  uint16_t piece_word[kPktMaxPieces];    // the head word a piece belongs to
};
// src = bit of the packet stream (from its first bit) holding the slice's first data bit.

// host: data index -> run j (data indices of run j: 2^j-j-1 .. 2^(j+1)-j-3)
uint32_t host_run_of(uint32_t d) {
  uint32_t j = 1;
  while (d >= (2u << j) - j - 2) ++j;
  return j;
}

hamming_status build_packet_tables(const PacketGeom& g, PacketTables& T) {
  const uint32_t bits = g.msg_bytes * 8u;
  T.Wp = (g.msg_bytes + 3) / 4;
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
      T.word0[W] = 33u << 16;  // head word: pass R writes 0, pass H ORs its pieces in
      T.special[T.n_special++] = W | (T.n_pieces << 16);
      for (uint32_t i = 0; i < np; ++i) {
        T.piece_word[T.n_pieces] = static_cast<uint16_t>(W);
        T.piece[T.n_pieces++] = src[i] | (len[i] << 16) | (pos[i] << 24);
      }
    }
  }
  T.special[T.n_special] = T.n_pieces << 16;
  auto mag = [](uint32_t d) { return d <= 1 ? 0xFFFFFFFFu : static_cast<uint32_t>((1ull << 32) / d); };
  T.mag_t = mag(g.t);
  T.mag_ns = mag(T.n_special);
  T.mag_wp = mag(T.Wp);
  T.mag_np = mag(T.n_pieces);
  return HAMMING_OK;
}

struct BatchGeom {
  uint32_t G;          // packets per batch
  uint32_t L;          // lanes per item in pass S (power of two)
  uint32_t in_cap;     // bytes per input buffer: 16 pad + G*stride + 16 slack
  uint32_t msg_cap;    // bytes of the message buffer: G packets of Wp words (+ slack)
  uint32_t warp_bytes; // 2*in_cap + msg_cap + status words
  uint32_t tab_bytes;  // CTA tables in front of the warp areas
};

hamming_status batch_geom(const PacketGeom& g, const PacketTables& T, uint64_t stride, BatchGeom& b) {
  uint32_t maxn = 0;
  for (uint32_t i = 0; i < g.t; ++i) maxn = max(maxn, g.n[i]);
  const uint32_t chunks = (maxn + 32) / 32;
  uint32_t L = 1;
  while (L < 32 && L * 8 < chunks) L *= 2;
#ifndef HAM_PKT_BUDGET
#define HAM_PKT_BUDGET (6 * 1024)
#endif
  const uint64_t budget = HAM_PKT_BUDGET;  // shared bytes per warp (tuned: tools/tune_shapes.py packets)
  const uint64_t per = kPktStages * stride + kPktMsgBufs * 4ull * T.Wp + 4 + 4ull * g.t;
  uint64_t G = budget > 96 ? (budget - 96) / per : 1;
  G = std::max<uint64_t>(1, std::min<uint64_t>(G, 64));
  b.G = static_cast<uint32_t>(G);
  b.L = L;
  b.in_cap = static_cast<uint32_t>(16 + G * stride + 16);
  b.msg_cap = static_cast<uint32_t>((G * T.Wp * 4 + 15) / 16 * 16 + 16);
  // kPktStages input buffers (TMA prefetch depth), kPktMsgBufs message buffers (bulk stores in flight)
  b.warp_bytes = kPktStages * b.in_cap + kPktMsgBufs * b.msg_cap +
                 static_cast<uint32_t>(16 * ((G * 4 * (1 + g.t) + 15) / 16));  // + statuses, item syndromes
  b.tab_bytes = (16 * T.Wp + 8 * T.n_pieces + 4 * 4 * kPktMaxSeg + 15) / 16 * 16;
  if (b.tab_bytes + b.warp_bytes * 2ull > 227ull * 1024)
    return set_err(HAMMING_E_ARG, "packets: batch does not fit shared memory");
  return HAMMING_OK;
}

// Syndrome of item (off, n) by a group of L lanes (rank q); all 32 lanes call
// it together (inactive groups pass active = false).  Interior chunks need no
// mask; the group's rank-0 lane adds the first chunk (position 0 masked off)
// and the last one (positions past n masked off).
__device__ __forceinline__ uint32_t group_syndrome(const uint32_t* w, uint32_t off, uint32_t n, bool active,
                                                   uint32_t q, uint32_t L) {
  const uint32_t chunks = active ? (n + 32) / 32 : 0;
  const uint32_t o = off + kPadBits - 1;
  const uint32_t qb = o >> 5, rb = o & 31u;
  uint32_t X = 0, P = 0;
  for (uint32_t j = 1 + q; j + 1 < chunks; j += L) {
    const uint32_t x = __funnelshift_r(w[qb + j], w[qb + j + 1], rb);
    X ^= x;
    P ^= (static_cast<uint32_t>(__popc(x)) & 1u) * (32u * j);
  }
  if (active && q == 0) {
    uint32_t x0 = __funnelshift_r(w[qb], w[qb + 1], rb) & 0xFFFFFFFEu;
    if (chunks == 1) x0 &= low_mask(n + 1);
    X ^= x0;
    if (chunks > 1) {
      const uint32_t j = chunks - 1;
      const uint32_t x = __funnelshift_r(w[qb + j], w[qb + j + 1], rb) & low_mask(n - 32 * j + 1);
      X ^= x;
      P ^= (static_cast<uint32_t>(__popc(x)) & 1u) * (32u * j);
    }
  }
  if (L == 32) {  // one REDUX each for a whole-warp item
    X = __reduce_xor_sync(0xffffffffu, X);
    P = __reduce_xor_sync(0xffffffffu, P);
  } else {
    for (uint32_t sh = L >> 1; sh > 0; sh >>= 1) {
      X ^= __shfl_xor_sync(0xffffffffu, X, sh);
      P ^= __shfl_xor_sync(0xffffffffu, P, sh);
    }
  }
  return P ^ xor_of_indices(X);
}

// The same syndrome with L a compile-time group size and no per-chunk POPC.
// Lane q takes chunks j = q + L m, m = 8 blk + it (it < 8, unrolled), over
// j = 0 .. C-2 unmasked (position 0 sits in chunk 0, which contributes 0 to
// both halves of s whatever its bits), and the group's rank-0 lane adds the
// last chunk masked to positions <= n.  The high part XOR_j [32 j par(x_j)]
// is rebuilt at the end from parities of a few accumulators: with q < L a
// power of two, j = q | (L m), so XOR over odd-parity chunks of j is
// q*par(X) ^ L*(8*BB ^ par(A0) ^ 2 par(A1) ^ 4 par(A2)), where A_b is the XOR
// of the chunks whose `it` has bit b and BB the XOR of the block indices with
// an odd block parity.
template <uint32_t L>
__device__ __forceinline__ uint32_t group_syndrome_l(const uint32_t* w, uint32_t off, uint32_t n, bool active,
                                                     uint32_t q) {
  const uint32_t C = active ? (n + 32) / 32 : 0;
  const uint32_t o = off + kPadBits - 1;
  const uint32_t* wq = w + (o >> 5) + q;
  const uint32_t rb = o & 31u;
  uint32_t X = 0, A0 = 0, A1 = 0, A2 = 0, BB = 0;
  const uint32_t interior = C > 0 ? C - 1 : 0;  // chunks 0 .. C-2
  for (uint32_t blk = 0; 8 * L * blk < interior; ++blk) {
    const uint32_t* wb = wq + 8 * L * blk;
    // chunks of this lane in the block: j = q + 8 L blk + L it < interior
    const int cnt = static_cast<int>(interior - 8 * L * blk) - static_cast<int>(q);
    uint32_t Xb = 0;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      if (static_cast<int>(L) * it < cnt) {
        const uint32_t x = __funnelshift_r(wb[L * it], wb[L * it + 1], rb);
        Xb ^= x;
        if (it & 1) A0 ^= x;
        if (it & 2) A1 ^= x;
        if (it & 4) A2 ^= x;
      }
    }
    X ^= Xb;
    BB ^= (__popc(Xb) & 1u) ? blk : 0u;
  }
  uint32_t P = 32u * ((q * (__popc(X) & 1u)) ^
                      L * ((8u * BB) ^ (__popc(A0) & 1u) ^ ((__popc(A1) & 1u) << 1) ^ ((__popc(A2) & 1u) << 2)));
  if (active && q == 0) {  // the last chunk, positions past n masked off
    const uint32_t j = C - 1;
    const uint32_t x = __funnelshift_r(w[(o >> 5) + j], w[(o >> 5) + j + 1], rb) & low_mask(n - 32 * j + 1);
    X ^= x;
    P ^= (__popc(x) & 1u) ? 32u * j : 0u;
  }
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
  return P ^ xor_of_indices(X);
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
                                                     uint32_t q) {
  const uint32_t o = off + kPadBits - 1;
  const uint32_t rb = o & 31u;
  const uint32_t full = active ? (n + 1) / 64 : 0;  // full 64-position chunks
  const uint32_t* wq = w + (o >> 5) + 2 * q;
  uint32_t X = 0, H = 0, A0 = 0, A1 = 0, BB = 0;
  for (uint32_t blk = 0; 4 * L * blk < full; ++blk) {
    const uint32_t* wb = wq + 8 * L * blk;
    const int cnt = static_cast<int>(full - 4 * L * blk) - static_cast<int>(q);
    uint32_t Xb = 0;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      if (static_cast<int>(L) * it < cnt) {
        const uint32_t w0 = wb[2 * L * it], w1 = wb[2 * L * it + 1], w2 = wb[2 * L * it + 2];
        const uint32_t hi = __funnelshift_r(w1, w2, rb);
        const uint32_t y = __funnelshift_r(w0, w1, rb) ^ hi;
        Xb ^= y;
        H ^= hi;
        if (it & 1) A0 ^= y;
        if (it & 2) A1 ^= y;
      }
    }
    X ^= Xb;
    BB ^= (__popc(Xb) & 1u) ? blk : 0u;
  }
  uint32_t P = (64u * ((q * (__popc(X) & 1u)) ^ L * ((4u * BB) ^ (__popc(A0) & 1u) ^ ((__popc(A1) & 1u) << 1)))) ^
               (32u * (__popc(H) & 1u));
  if (active && q == 0) {  // the tail: positions 64 full .. n (fewer than 64)
    const uint32_t j = 2 * full, b0 = (o >> 5) + j;
    const uint32_t rest = n + 1 - 64 * full;  // positions left, 0 .. 63
    const uint32_t lo = __funnelshift_r(w[b0], w[b0 + 1], rb) & __funnelshift_lc(0xFFFFFFFFu, 0u, rest);
    const uint32_t hi = __funnelshift_r(w[b0 + 1], w[b0 + 2], rb) &
                        __funnelshift_lc(0xFFFFFFFFu, 0u, rest > 32 ? rest - 32 : 0u);
    X ^= lo ^ hi;
    P ^= ((__popc(lo) & 1u) ? 32u * j : 0u) ^ ((__popc(hi) & 1u) ? 32u * (j + 1) : 0u);
  }
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
  return P ^ xor_of_indices(X);
}

// The first 57 data bits of an item (positions 3..63 -- runs 1..5, where
// the run boundaries are dense) by the fixed compaction of the (63,57) code:
// v = positions 0..63, groups g = 1..4 from the low word, positions 33..63
// from the high word.  Bits past k are garbage and are masked by the caller.
__device__ __forceinline__ uint64_t rr_head57(const uint32_t* w, uint32_t off) {
  const uint32_t o = off + kPadBits - 1;  // buffer bit of position 0
  const uint32_t q = o >> 5, r = o & 31u;
  const uint32_t lo = __funnelshift_r(w[q], w[q + 1], r);
  const uint32_t hi = __funnelshift_r(w[q + 1], w[q + 2], r);
  uint32_t d = 0;
#pragma unroll
  for (int g = 1; g < 5; ++g) d |= (lo >> (g + 2)) & dmask(g);
  return static_cast<uint64_t>(d) | (static_cast<uint64_t>(hi >> 1) << 26);
}

// One message word of an item, general form (edge words, words holding
// d < 57): bits of the word outside [moff, moff + k) are 0.
__device__ __forceinline__ uint32_t item_word_general(const uint32_t* w, uint64_t head, uint32_t off, uint32_t k,
                                                      uint32_t moff, uint32_t mw) {
  const uint32_t d0 = max(32u * mw, moff) - moff;
  const uint32_t d1 = min(32u * mw + 32u, moff + k) - moff;
  const uint32_t sh = moff + d0 - 32u * mw;  // bit of the word that receives d0
  uint32_t v = 0;
  if (d0 < 57u) {
    const uint32_t e = min(d1, 57u);
    v = (static_cast<uint32_t>(head >> d0) & low_mask(e - d0)) << sh;
  }
  if (d1 > 57u) {
    const uint32_t dd = max(d0, 57u);
    const uint32_t j = run_of(dd);
    const uint32_t nb = min(32u, (2u << j) - j - 2 - dd);  // bits before the next run starts
    const uint32_t src = off + kPadBits + dd + j + 1;
    const uint32_t x0 = sm_bits32(w, src), x1 = sm_bits32(w, src + 1);
    const uint32_t part = ((x0 & low_mask(nb)) | (x1 & ~low_mask(nb))) & low_mask(d1 - dd);
    v |= part << (sh + dd - d0);
  }
  return v;
}

// Redundancy removal + merger for one item by its group: lane q builds message
// words mw0 + q, mw0 + q + L, ...  Data index d sits in run j at buffer bit
// off + kPadBits + d + j + 1.  d < 57 comes from rr_head57; from d = 57 on
// every run is >= 63 bits long, so a 32-bit window holds at most one run
// boundary: an interior word is two funnel-shifted slices one bit apart,
// merged at the boundary (branch free, the run tracked incrementally per
// lane).  Interior words are stored; the item's edge words (shared with
// neighbours) and the words holding d < 57 take the general path and are
// OR-ed atomically.  fb = message bit to flip (the corrected data bit) or ~0.
__device__ __forceinline__ void group_rr(const uint32_t* w, uint32_t* mbuf, uint32_t off, uint32_t k,
                                         uint32_t moff, uint32_t fb, uint32_t q, uint32_t L) {
  const uint32_t mw0 = moff / 32, mw1 = (moff + k + 31) / 32;
  // interior words: wholly inside the item and wholly at d >= 57
  const uint32_t ia = max((moff + 57 + 31) / 32, (moff + 31) / 32), ib = (moff + k) / 32;
  uint64_t head = 0;
  if (q < 3) head = rr_head57(w, off);  // the words holding d < 57 are the first (at most) three
  // general words: the head [mw0, min(ia, mw1)) and the tail [max(ib, ia), mw1) -- a few each
  const bool has_interior = ia < ib;
  const uint32_t he = has_interior ? ia : mw1, ts = has_interior ? ib : mw1;
  for (uint32_t i = q; i < (he - mw0) + (mw1 - ts); i += L) {
    const uint32_t mw = (i < he - mw0) ? mw0 + i : ts + (i - (he - mw0));
    uint32_t v = item_word_general(w, head, off, k, moff, mw);
    if ((fb >> 5) == mw) v ^= 1u << (fb & 31u);
    atomicOr(&mbuf[mw], v);
  }
  // interior words, lane q: ia + q', ia + q' + L, ... with q' the lane's slot in that sequence
  uint32_t mw = ia + ((q + L - (ia - mw0) % L) % L);
  if (has_interior && mw < ib) {
    uint32_t dd = 32u * mw - moff;
    uint32_t j = run_of(dd);
    uint32_t nxt = (2u << j) - j - 2;   // first data index of run j + 1
    const uint32_t base = off + kPadBits + 1;
    for (; mw < ib; mw += L, dd += 32u * L) {
      while (dd >= nxt) {
        ++j;
        nxt = (2u << j) - j - 2;
      }
      const uint32_t src = base + dd + j;
      const uint32_t qw = src >> 5, r = src & 31u;
      const uint32_t a0 = w[qw], a1 = w[qw + 1];
      const uint32_t x0 = __funnelshift_r(a0, a1, r);                          // run j
      const uint32_t x1 = (r == 31u) ? a1 : __funnelshift_r(a0, a1, r + 1);   // run j + 1: one bit later
      const uint32_t lm = low_mask(min(32u, nxt - dd));
      uint32_t v = (x0 & lm) | (x1 & ~lm);
      if ((fb >> 5) == mw) v ^= 1u << (fb & 31u);
      mbuf[mw] = v;
    }
  }
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

template <uint32_t L>
__global__ void __launch_bounds__(kPktWarps * 32)
    packets_decode_kernel(const __grid_constant__ PacketGeom g, const __grid_constant__ BatchGeom bg,
                          const __grid_constant__ PacketArgs a, const __grid_constant__ PacketTables T) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned long long cta_counts[2];
  __shared__ __align__(8) uint64_t bars_all[kPktWarps * kPktStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Wp = T.Wp, npc = T.n_pieces;
  // CTA tables: word descriptors {word, shift, mask of slice 0, keep}, head-word
  // pieces {src | len | pos, word}, per-segment geometry
  uint4* wdesc = reinterpret_cast<uint4*>(smem);
  uint2* pieces = reinterpret_cast<uint2*>(smem + 16 * Wp);
  uint32_t* sg = reinterpret_cast<uint32_t*>(pieces + T.n_pieces);  // [off | n | k | moff] x kPktMaxSeg
  for (uint32_t i = threadIdx.x; i < Wp; i += blockDim.x) {
    const uint32_t s0 = T.word0[i] & 0xFFFFu, nb = T.word0[i] >> 16;
    const bool head = nb > 32;  // head words are 0 after pass R and OR-ed together by pass H
    wdesc[i] = make_uint4(s0 >> 5, s0 & 31u, nb >= 32 ? 0xFFFFFFFFu : (1u << nb) - 1u, head ? 0u : 0xFFFFFFFFu);
  }
  for (uint32_t i = threadIdx.x; i < T.n_pieces; i += blockDim.x) pieces[i] = make_uint2(T.piece[i], T.piece_word[i]);
  if (threadIdx.x < g.t) {
    sg[threadIdx.x] = g.off[threadIdx.x];
    sg[kPktMaxSeg + threadIdx.x] = g.n[threadIdx.x];
    sg[2 * kPktMaxSeg + threadIdx.x] = g.k[threadIdx.x];
    sg[3 * kPktMaxSeg + threadIdx.x] = g.moff[threadIdx.x];
  }
  uint8_t* wb = smem + bg.tab_bytes + warp * bg.warp_bytes;
  uint32_t* pst = reinterpret_cast<uint32_t*>(wb + kPktStages * bg.in_cap + kPktMsgBufs * bg.msg_cap);  // statuses
  uint32_t* sbuf = pst + bg.G;  // per-item syndromes of the batch
  uint64_t* bars = bars_all + warp * kPktStages;
  if (threadIdx.x < 2) cta_counts[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t n_batches = (a.n_packets + bg.G - 1) / bg.G;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kPktWarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kPktWarps;
  const uint64_t pol = policy_evict_first();
  const uint32_t q = static_cast<uint32_t>(lane) & (L - 1), gid = static_cast<uint32_t>(lane) / L;
  const uint32_t groups = 32 / L;
  const uint32_t stride_bits = static_cast<uint32_t>(a.in_stride * 8);
  uint32_t n_corr = 0, n_fail = 0;
  auto batch_bytes = [&](uint64_t b) -> uint32_t {
    const uint64_t p0 = b * bg.G;
    const uint64_t left = a.n_packets - p0;
    return static_cast<uint32_t>((left < bg.G ? left : bg.G) * a.in_stride);
  };
  if (lane == 0) {
    for (uint32_t s = 0; s < kPktStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    for (uint32_t s = 0; s < kPktStages; ++s) {
      const uint64_t b = gw + s * nw;
      if (b < n_batches) {
        mbar_arrive_expect_tx(&bars[s], batch_bytes(b));
        bulk_g2s(wb + s * bg.in_cap + 16, a.in + b * bg.G * a.in_stride, batch_bytes(b), &bars[s], pol);
      }
    }
  }
  __syncwarp();
  uint32_t it = 0;
  for (uint64_t b = gw; b < n_batches; b += nw, ++it) {
    const uint32_t buf = it % kPktStages;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(wb + buf * bg.in_cap);
    const uint64_t p0 = b * bg.G;
    const uint64_t left = a.n_packets - p0;
    const uint32_t np = static_cast<uint32_t>(left < bg.G ? left : bg.G);
    uint32_t* mbuf = reinterpret_cast<uint32_t*>(wb + kPktStages * bg.in_cap + (it % kPktMsgBufs) * bg.msg_cap);
    if (lane == 0) bulk_wait_read<kPktMsgBufs - 1>();  // the bulk store that last used this mbuf has read it
    for (uint32_t i = lane; i < np; i += 32) pst[i] = 0;
    mbar_wait(&bars[buf], (it / kPktStages) & 1u);
    __syncwarp();
    {  // pass R: every word as one or two slices (lane: word W of every packet of the batch)
      const uint32_t wstride = static_cast<uint32_t>(a.in_stride / 4);
      if (np == 1) {  // one packet per batch (long packets): no inner loop
        for (uint32_t W = lane; W < Wp; W += 32) {
          const uint4 d = wdesc[W];
          const uint32_t a0 = w[4 + d.x], a1 = w[5 + d.x];
          mbuf[W] = ((__funnelshift_r(a0, a1, d.y) & d.z) | (__funnelshift_rc(a0, a1, d.y + 1) & ~d.z)) & d.w;
        }
      } else
      for (uint32_t W = lane; W < Wp; W += 32) {
        const uint4 d = wdesc[W];  // {word, shift, mask of slice 0, 0 for a head word}
        const uint32_t* wp = w + 4 + d.x;  // (after the 16-byte pad)
        uint32_t* mp = mbuf + W;
        for (uint32_t p = 0; p < np; ++p, wp += wstride, mp += Wp) {
          const uint32_t a0 = wp[0], a1 = wp[1];
          // slice 1 is the stream one bit further on (the parity position skipped)
          *mp = ((__funnelshift_r(a0, a1, d.y) & d.z) | (__funnelshift_rc(a0, a1, d.y + 1) & ~d.z)) & d.w;
        }
      }
    }
    __syncwarp();
    if (npc > 0) {  // pass H: head words, one piece per lane, OR-ed in
      for (uint32_t e = lane; e < np * npc; e += 32) {
        uint32_t c;
        const uint32_t p = divmod_small(e, npc, T.mag_np, c);
        const uint2 pc = pieces[c];
        const uint32_t s0 = kPadBits + p * stride_bits + (pc.x & 0xFFFFu), len = (pc.x >> 16) & 63u;
        const uint32_t x = __funnelshift_r(w[s0 >> 5], w[(s0 >> 5) + 1], s0) & __funnelshift_lc(0xFFFFFFFFu, 0u, len);
        atomicOr(&mbuf[p * Wp + pc.y], x << ((pc.x >> 24) & 31u));
      }
    }
    __syncwarp();
    {  // pass S: syndromes per (packet, segment) item, by groups of L lanes
      const uint32_t items = np * g.t;
      for (uint32_t base = 0; base < items; base += groups) {
        const bool active = base + gid < items;
        uint32_t seg;
        const uint32_t pk = divmod_small(active ? base + gid : 0, g.t, T.mag_t, seg);
        const uint32_t n = active ? sg[kPktMaxSeg + seg] : 0;
        const uint32_t off = pk * stride_bits + sg[seg];
        const uint32_t s = group_syndrome64<L>(w, off, n, active, q);
        if (active && q == 0) sbuf[base + gid] = s;
      }
    }
    __syncwarp();
    // per item: syndrome out, packet status, counts; a correctable error flips its data bit
    for (uint32_t i = lane; i < np * g.t; i += 32) {
      uint32_t seg;
      const uint32_t pk = divmod_small(i, g.t, T.mag_t, seg);
      const uint32_t s = sbuf[i], n = sg[kPktMaxSeg + seg];
      const bool corr = s != 0 && s <= n;
      const bool fail = s > n;
      if (a.syn != nullptr) a.syn[p0 * g.t + i] = static_cast<uint16_t>(s);
      if (corr || fail) atomicMax(&pst[pk], fail ? 2u : 1u);
      n_corr += corr;
      n_fail += fail;
      if (corr && (s & (s - 1)) != 0) {  // a data position: message bit moff + s - floor(log2 s) - 2
        const uint32_t fb = sg[3 * kPktMaxSeg + seg] + s - (31u - __clz(s)) - 2;
        atomicXor(&mbuf[pk * Wp + (fb >> 5)], 1u << (fb & 31u));
      }
    }
    __syncwarp();
    if (lane == 0) {  // buffer consumed: prefetch the batch two steps ahead
      const uint64_t nx = b + kPktStages * nw;
      if (nx < n_batches) {
        mbar_arrive_expect_tx(&bars[buf], batch_bytes(nx));
        bulk_g2s(wb + buf * bg.in_cap + 16, a.in + nx * bg.G * a.in_stride, batch_bytes(nx), &bars[buf], pol);
      }
    }
    // write the batch's messages (packet pk at word pk * Wp of mbuf) and statuses
    const uint8_t* mb = reinterpret_cast<const uint8_t*>(mbuf);
    const uintptr_t ob = reinterpret_cast<uintptr_t>(a.out + p0 * a.out_stride);
    if (a.out_stride == g.msg_bytes && (g.msg_bytes & 15u) == 0 && (ob & 15u) == 0) {
      fence_proxy_async_smem();  // this lane's st.shared / atomics visible to the bulk copy
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(reinterpret_cast<void*>(ob), mbuf, np * g.msg_bytes, pol);
        bulk_commit();
      }
    } else if ((g.msg_bytes & 3u) == 0 && (a.out_stride & 3u) == 0 && (ob & 3u) == 0) {
      for (uint32_t pk = 0; pk < np; ++pk) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(ob + pk * a.out_stride);
        for (uint32_t i = lane; i < Wp; i += 32) dst[i] = mbuf[pk * Wp + i];
      }
    } else {
      for (uint32_t pk = 0; pk < np; ++pk) {
        uint8_t* dst = reinterpret_cast<uint8_t*>(ob + pk * a.out_stride);
        for (uint32_t i = lane; i < g.msg_bytes; i += 32) dst[i] = mb[pk * Wp * 4 + i];
      }
    }
    if (a.status != nullptr)
      for (uint32_t i = lane; i < np; i += 32) a.status[p0 + i] = static_cast<uint8_t>(pst[i]);
    __syncwarp();
  }
  if (lane == 0) bulk_wait<0>();  // the last bulk stores have completed before shared memory goes away
  if (a.counts != nullptr) {
    n_corr = __reduce_add_sync(0xffffffffu, n_corr);
    n_fail = __reduce_add_sync(0xffffffffu, n_fail);
    if (lane == 0) {
      if (n_corr) atomicAdd(&cta_counts[0], static_cast<unsigned long long>(n_corr));
      if (n_fail) atomicAdd(&cta_counts[1], static_cast<unsigned long long>(n_fail));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (cta_counts[0]) atomicAdd(&a.counts[0], cta_counts[0]);
      if (cta_counts[1]) atomicAdd(&a.counts[1], cta_counts[1]);
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
  hamming_status rc = batch_geom(g, T, a.in_stride, bg);
  if (rc != HAMMING_OK) return rc;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const size_t smem = bg.tab_bytes + static_cast<size_t>(kPktWarps) * bg.warp_bytes;
  if (smem > 227 * 1024) return set_err(HAMMING_E_ARG, "packets: shared memory budget exceeded");
  void (*kfn)(PacketGeom, BatchGeom, PacketArgs, PacketTables) = nullptr;
  switch (bg.L) {
    case 1: kfn = packets_decode_kernel<1>; break;
    case 2: kfn = packets_decode_kernel<2>; break;
    case 4: kfn = packets_decode_kernel<4>; break;
    case 8: kfn = packets_decode_kernel<8>; break;
    case 16: kfn = packets_decode_kernel<16>; break;
    default: kfn = packets_decode_kernel<32>; break;
  }
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(packets decode)");
  // ask for the full shared-memory carveout so several CTAs fit per SM
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(carveout)");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kPktWarps * 32, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy(packets decode)");
  const uint64_t batches = (a.n_packets + bg.G - 1) / bg.G;
  const uint64_t want = (batches + kPktWarps - 1) / kPktWarps;
  const int grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sm_count(dev)) * std::max(1, occ)));
  if (grid > 0) {
    kfn<<<grid, kPktWarps * 32, smem, st>>>(g, bg, a, T);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "packets decode launch");
  }
  g_launches = grid > 0 ? 1 : 0;
  g_grid = grid;
  return HAMMING_OK;
}

// ---------------------------------------------------------------------------
// Longer perfect codes, m = 7, 8 ((127,120), (255,247)):
// the same item engine over a stream of codewords -- a batch is 128
// codewords (16n input bytes, 16k output bytes, both 16-byte aligned), items
// are codewords (off = c n, moff = c k), one lane per codeword.
// ---------------------------------------------------------------------------
struct LongArgs {
  const uint8_t* in;
  uint8_t* out;
  uint8_t* syn;
  unsigned long long* counter;
  uint64_t N, in_total, out_total;
  uint32_t n, k, store_count;
};

constexpr uint32_t kLongBatch = 128;

__global__ void __launch_bounds__(kPktWarps * 32)
    long_decode_kernel(const __grid_constant__ LongArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ unsigned long long cta_count;
  __shared__ __align__(8) uint64_t bars_all[kPktWarps * 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t in_b = 16 * a.n, out_b = 16 * a.k;
  const uint32_t in_cap = 16 + in_b + 16, msg_cap = out_b + 16;
  uint8_t* wb = smem + warp * (2 * in_cap + msg_cap);
  uint32_t* mbuf = reinterpret_cast<uint32_t*>(wb + 2 * in_cap);
  uint64_t* bars = bars_all + warp * 2;
  if (threadIdx.x == 0) cta_count = 0;
  __syncthreads();
  const uint64_t n_full = a.N / kLongBatch;
  const uint64_t n_batches = (a.N + kLongBatch - 1) / kLongBatch;
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kPktWarps + warp;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kPktWarps;
  const uint64_t pol = policy_evict_first();
  uint32_t cnt = 0;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    for (uint32_t s = 0; s < 2; ++s) {
      const uint64_t b = gw + s * nw;
      if (b < n_full) {
        mbar_arrive_expect_tx(&bars[s], in_b);
        bulk_g2s(wb + s * in_cap + 16, a.in + b * in_b, in_b, &bars[s], pol);
      }
    }
  }
  __syncwarp();
  uint32_t it = 0;
  for (uint64_t b = gw; b < n_batches; b += nw, ++it) {
    const uint32_t buf = it & 1u;
    uint8_t* wbytes = wb + buf * in_cap;
    const uint32_t* w = reinterpret_cast<const uint32_t*>(wbytes);
    const bool full = b < n_full;
    const uint32_t nb = full ? kLongBatch : static_cast<uint32_t>(a.N - b * kLongBatch);
    for (uint32_t i = lane; i < (out_b + 3) / 4; i += 32) mbuf[i] = 0;
    if (full) {
      mbar_wait(&bars[buf], (it >> 1) & 1u);
    } else {  // the ragged last batch: bounded loads (TMA needs whole 16-byte units)
      const uint64_t ib0 = b * in_b, nbytes = a.in_total - ib0;
      for (uint32_t i = lane; i < in_b; i += 32) wbytes[16 + i] = i < nbytes ? a.in[ib0 + i] : 0;
    }
    __syncwarp();
    for (uint32_t c = lane; c < kLongBatch; c += 32) {  // all lanes take part in every round
      const bool active = c < nb;
      const uint32_t off = c * a.n, moff = c * a.k;
      const uint32_t s = group_syndrome(w, off, a.n, active, 0, 1);
      if (!active) continue;
      uint32_t fb = 0xFFFFFFFFu;
      if (s != 0 && (s & (s - 1)) != 0) fb = moff + s - (31u - __clz(s)) - 2;
      group_rr(w, mbuf, off, a.k, moff, fb, 0, 1);
      if (a.syn != nullptr) a.syn[b * kLongBatch + c] = static_cast<uint8_t>(s);
      cnt += (s != 0);
    }
    __syncwarp();
    if (lane == 0 && full) {  // buffer consumed: prefetch the batch two steps ahead
      const uint64_t nx = b + 2 * nw;
      if (nx < n_full) {
        mbar_arrive_expect_tx(&bars[buf], in_b);
        bulk_g2s(wbytes + 16, a.in + nx * in_b, in_b, &bars[buf], pol);
      }
    }
    uint8_t* dst = a.out + b * out_b;
    if (full) {
      for (uint32_t i = lane; i < out_b / 16; i += 32)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(mbuf)[i];
    } else {
      const uint64_t nbytes = a.out_total - b * out_b;
      const uint8_t* mb = reinterpret_cast<const uint8_t*>(mbuf);
      for (uint32_t i = lane; i < nbytes; i += 32) dst[i] = mb[i];
    }
    __syncwarp();
  }
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
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const size_t smem = static_cast<size_t>(kPktWarps) * (2 * (16 + 16 * a.n + 16) + 16 * a.k + 16);
  e = cudaFuncSetAttribute(long_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(long decode)");
  e = cudaFuncSetAttribute(long_decode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(carveout)");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, long_decode_kernel, kPktWarps * 32, smem);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy(long decode)");
  const uint64_t batches = (N + kLongBatch - 1) / kLongBatch;
  const uint64_t want = (batches + kPktWarps - 1) / kPktWarps;
  const int grid = static_cast<int>(std::min<uint64_t>(want, static_cast<uint64_t>(sm_count(dev)) * std::max(1, occ)));
  a.store_count = (counter != nullptr && !accumulate && grid == 1) ? 1u : 0u;
  if (counter != nullptr && !accumulate && !a.store_count) {
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(corrected)");
  }
  if (grid > 0) {
    long_decode_kernel<<<grid, kPktWarps * 32, smem, st>>>(a);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "long decode launch");
  } else if (counter != nullptr && !accumulate) {
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(corrected)");
  }
  g_launches = grid > 0 ? 1 : 0;
  g_grid = grid;
  return HAMMING_OK;
}
