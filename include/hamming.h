/*
 * include/hamming.h -- C ABI of the B200-native batched Hamming decoder.
 *
 * Method: Islam, Kim & Kim, "Computationally Efficient Implementation of a
 * Hamming Code Decoder using Graphics Processing Unit" (arXiv 1412.6862;
 * /root/reference/PAPER.md cited as P:L<line>).  The decoder is "splitter,
 * decoder, and merger" with "error detection (ED), error correction (EC),
 * and redundancy remover (RR)" (Fig. 1), the syndrome ("checksum
 * vector") being the modulo-2 sum over each index set I_j (P:L98, P:L160
 * Algorithm 1 Step 4).  This library decodes packets of concatenated perfect
 * (n, k) = (2^m - 1, 2^m - 1 - m) codewords, m in [2, 8] (m = 7, 8 -- the
 * (127,120) and (255,247) codes of SURVEY.md 8(f) f4 -- through the long-
 * codeword engine; encode and the synthetic channel cover m in [2, 6]),
 * extended-Hamming (SECDED) codewords, and the paper's own packets of
 * shortened codes.
 *
 * Stream layout (readings R3, R4):
 *   - stream bit b is bit (b & 7) of byte b >> 3 (LSB-first), i.e. bit
 *     (b & 31) of little-endian 32-bit word b >> 5;
 *   - codeword c occupies stream bits [c*n, c*n + n); its 1-based position p
 *     is stream bit c*n + p - 1; parity bits sit at positions 1, 2, 4, ...;
 *   - the data stream holds codeword c's k message bits at [c*k, c*k + k),
 *     message bit 1 first (= the non-power-of-two positions, ascending).
 *
 * Conventions shared by every entry point:
 *   - Pointers named *_dev are DEVICE memory, pointers named *_host are HOST
 *     memory; all are owned by the caller.  The library allocates nothing
 *     except where an entry point says so, and keeps no state beyond a
 *     thread-local error string and a per-device attribute cache.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device entry points are asynchronous on it; argument errors
 *     are returned synchronously before anything is launched; faults during
 *     kernel execution surface at the caller's next synchronisation.
 *   - Outputs are bit-exact and independent of the launch configuration.
 *   - Reentrant: concurrent calls on distinct buffers / streams are safe.
 *   - No host fallback: every step runs in this library's sm_100a kernels.
 */
#ifndef HAMMING_H_
#define HAMMING_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HAMMING_ABI_VERSION 1

typedef enum {
    HAMMING_OK = 0,
    HAMMING_E_INVALID_M = 1,   /* m out of range for the entry point */
    HAMMING_E_NULL = 2,        /* a required pointer is NULL while n_codewords > 0 */
    HAMMING_E_MISALIGNED = 3,  /* a device buffer is not 16-byte aligned */
    HAMMING_E_OVERLAP = 4,     /* input and output ranges overlap (no in-place) */
    HAMMING_E_RANGE = 5,       /* n * n_codewords bits overflows uint64, or bad p/q2 */
    HAMMING_E_CUDA = 6,        /* CUDA launch/config error; see hamming_last_error() */
    HAMMING_E_ARG = 7          /* any other invalid argument */
} hamming_status;

/* ---------------------------------------------------------------- decode */

/* hamming_decode -- the hot path.
 * For every codeword c < n_codewords of the received packet `rx_dev`:
 *   s_c = sum_j 2^j * XOR{ bit at position p : p in I_j }
 *   if s_c != 0 the bit at position s_c is flipped              (P:L59 ED/EC)
 *   the k bits at non-power-of-two positions are kept, in order (P:L59 RR)
 *   and written to data bits [c*k, c*k + k)                     (P:L68 merger)
 * Arguments:
 *   m            code order, n = 2^m - 1, k = n - m, 2 <= m <= 8.
 *   rx_dev       hamming_coded_bytes(m, N) bytes, 16-byte aligned; pad bits
 *                past n*N in the last byte are ignored.  Never written.
 *   n_codewords  N (64-bit; 0 is a valid no-op that sets *corrected = 0).
 *   data_dev     hamming_data_bytes(m, N) bytes, 16-byte aligned; fully
 *                overwritten, pad bits past k*N written as 0.
 *   syndromes_dev  N bytes, 16-byte aligned, or NULL to skip: s_c in [0, n];
 *                the per-codeword corrected flag is (s_c != 0).
 *   corrected_dev  one device uint64, OVERWRITTEN (stream-ordered) with
 *                #{c : s_c != 0} -- corrections performed, miscorrections of
 *                multi-bit errors included (reading R10).
 *   stream       cudaStream_t or NULL.
 * Buffers must not overlap.  With a 2-bit error the decoder deterministically
 * miscorrects (reading R9); for perfect codes no syndrome exceeds n, so there
 * is no uncorrectable status (reading R8). */
hamming_status hamming_decode(int m, const void *rx_dev, uint64_t n_codewords,
                              void *data_dev, uint8_t *syndromes_dev,
                              unsigned long long *corrected_dev, void *stream);

/* ----------------------------------------------------------- encode (f1) */

/* hamming_encode -- the transmitter's "exact reverse process":
 * data bits [c*k, c*k + k) -> codeword c at stream bits [c*n, c*n + n), data
 * at the non-power-of-two positions, even parity over every I_j (reading R2).
 * data_dev: hamming_data_bytes bytes (pad bits ignored); rx_dev:
 * hamming_coded_bytes bytes, fully overwritten (pad bits 0).  Both 16-byte
 * aligned, non-overlapping. */
hamming_status hamming_encode(int m, const void *data_dev, uint64_t n_codewords,
                              void *rx_dev, void *stream);

/* hamming_channel_generate -- seeded synthetic received packet (test and
 * benchmark input).  The same counter-based
 * generator is written independently in oracle/oracle.c and the two are
 * compared byte for byte.  For global codeword index g = c_first + c:
 *   u(g, q) = splitmix64_mix(seed + (4g + q + 1) * 0x9E3779B97F4A7C15)
 *   message = low k bits of u(g,0); codeword = encode(message);
 *   error event iff all != 0 or u(g,1) < thresh; weight 2 iff
 *   (u(g,2) >> 32) < q2thresh (q2thresh <= 2^32); positions
 *   p1 = 1 + umulhi(lo32(u(g,3)), n),
 *   p2 = 1 + ((p1 - 1) + 1 + umulhi(hi32(u(g,3)), n - 1)) mod n.
 * rx_dev: hamming_coded_bytes(m, n_codewords) bytes, 16-byte aligned, fully
 * overwritten.  c_first must be a multiple of 8 only if the caller wants to
 * concatenate separately generated ranges byte-wise. */
hamming_status hamming_channel_generate(int m, uint64_t seed, uint64_t c_first,
                                        uint64_t n_codewords, uint64_t thresh, int all,
                                        uint64_t q2thresh, void *rx_dev, void *stream);

/* ----------------------------------------------- host-buffer decode (f3) */

/* hamming_decode_host -- end-to-end decode of a packet that lives in HOST
 * memory, the paper's "asynchronous data transfer (ADT)" pipeline (P:L113-132,
 * Eq. 1, Fig. 5): the packet is cut into chunks of `chunk_codewords`
 * (a multiple of 1024), and for each chunk an H2D copy, the decode kernels
 * and the D2H copies are issued on one of `n_streams` (1..4) streams so that
 * transfers of chunk i+1 overlap the decode of chunk i.
 *   rx_host / data_host / syndromes_host (nullable): as in hamming_decode but
 *   host memory (pinned memory gives full PCIe bandwidth; pageable works).
 *   corrected_host: host uint64, overwritten.
 *   workspace_dev: device memory of hamming_host_workspace_bytes(m,
 *   chunk_codewords, n_streams, syndromes_host != NULL) bytes, 16-byte aligned,
 *   on the current device; the C ABI cannot check its size (the Python
 *   binding does).  The library's streams (created once per thread and device,
 *   reused) do not wait on any caller stream: the caller must have completed
 *   all work that touches the workspace (the binding synchronises its current
 *   stream first).
 * Synchronous: returns when all outputs are in host memory. */
size_t hamming_host_workspace_bytes(int m, uint64_t chunk_codewords, int n_streams,
                                    int with_syndromes);
hamming_status hamming_decode_host(int m, const void *rx_host, uint64_t n_codewords,
                                   void *data_host, uint8_t *syndromes_host,
                                   unsigned long long *corrected_host,
                                   void *workspace_dev, uint64_t chunk_codewords,
                                   int n_streams);

/* ------------------------------------------- SECDED: extended Hamming (f4) */

/* Extended Hamming / SECDED codes (2^m, 2^m-1-m), m in [3, 6] -- (8,4),
 * (16,11), (32,26), (64,57) -- SURVEY.md 8(f) f4, reading R17:
 * codeword c = stream bits [c 2^m, (c+1) 2^m); its bit 0 is the overall
 * (even) parity of all 2^m bits and bits 1..n (positions 1..n) are the
 * Hamming codeword of hamming_decode.  Decoding: s = syndrome over positions
 * 1..n, P = parity of all 2^m bits;
 *   P = 1: single error at position s (s = 0: the parity bit) -- corrected;
 *   P = 0, s != 0: double error DETECTED -- nothing is changed;
 *   P = 0, s = 0: clean.
 * flags_dev (N bytes or NULL): s | 0x40 if corrected | 0x80 if detected.
 * counts_dev: 2 device uint64, OVERWRITTEN with {corrected, detected}.
 * data_dev: as hamming_decode (k bits per codeword, pad bits 0).  Buffers
 * 16-byte aligned, non-overlapping. */
uint64_t hamming_secded_coded_bytes(int m, uint64_t n_codewords); /* N 2^m / 8; 0 on bad m */
hamming_status hamming_decode_secded(int m, const void *rx_dev, uint64_t n_codewords, void *data_dev,
                                     uint8_t *flags_dev, unsigned long long *counts_dev, void *stream);
hamming_status hamming_encode_secded(int m, const void *data_dev, uint64_t n_codewords, void *rx_dev,
                                     void *stream);
/* Seeded SECDED channel: the draws of hamming_channel_generate, flip positions
 * drawn over all 2^m bits: b1 = umulhi(lo32(u(g,3)), 2^m), b2 = (b1 + 1 +
 * umulhi(hi32(u(g,3)), 2^m - 1)) mod 2^m (bit index, 0 = the parity bit). */
hamming_status hamming_channel_generate_secded(int m, uint64_t seed, uint64_t c_first, uint64_t n_codewords,
                                               uint64_t thresh, int all, uint64_t q2thresh, void *rx_dev,
                                               void *stream);

/* ------------------------------------- packets: the paper's workload (f2) */

/* The paper's packets (Fig. 1): a message of msg_bytes bytes
 * (1..4096) is split into t segments (1..16) -- the first (8*msg_bytes mod t)
 * get ceil(8*msg_bytes/t) message bits, the rest floor (DESIGN.md reading
 * R14) -- and segment i is ONE shortened Hamming codeword of k_i message bits
 * and the minimal r_i with 2^r >= k + r + 1, n_i = k_i + r_i.  The
 * encoded packet is H_1 ... H_t concatenated bitwise, LSB-first.  Packet j
 * starts at byte j*rx_stride (rx_stride a multiple of 16, >= the coded bytes
 * rounded up to 16; for hamming_decode_packets also <= 100 KiB, since the
 * decoder stages whole strides in shared memory); its message at byte j*msg_stride.  HAMMING_E_ARG for a bad stride,
 * HAMMING_E_RANGE if n_packets * stride overflows. */
uint64_t hamming_packet_coded_bytes(uint32_t msg_bytes, int t); /* 0 on bad arguments */
hamming_status hamming_packet_layout(uint32_t msg_bytes, int t, uint32_t *seg_k_host, uint32_t *seg_n_host);

/* hamming_decode_packets -- per segment: syndrome, ED/EC:
 * s = 0 clean, 1 <= s <= n_i flip position s, s > n_i uncorrectable (the
 * segment is left as received, reading R15); RR and merger.
 *   syndromes_dev: n_packets*t uint16 or NULL; status_dev: n_packets bytes or
 *   NULL (0 clean, 1 corrected, 2 some segment uncorrectable); counts_dev: 2
 *   device uint64 or NULL, OVERWRITTEN with {segments corrected, segments
 *   uncorrectable}.  rx 16-byte aligned, syndromes 2-byte aligned, counts
 *   8-byte aligned (HAMMING_E_MISALIGNED); no two of rx, msg, syndromes,
 *   status, counts may overlap (HAMMING_E_OVERLAP).  All checks return
 *   before any launch. */
/* hamming_packet_launch_shape -- host only, no CUDA call: the launch shape
 * hamming_decode_packets would use for n_packets packets at rx_stride on a
 * GPU with sm_count SMs (the issue model): warps per CTA,
 * packets per warp batch, lanes per (packet, segment) item in pass S, CTAs
 * per SM the shared memory allows, and the shared-memory bytes per CTA.  All
 * outputs are host ints (any may be NULL).  HAMMING_E_ARG for a bad shape or
 * stride. */
hamming_status hamming_packet_launch_shape(uint32_t msg_bytes, int t, uint64_t rx_stride, uint64_t n_packets,
                                           int sm_count, int *warps, int *packets_per_batch, int *lanes_per_item,
                                           int *ctas_per_sm, int *smem_bytes);

hamming_status hamming_decode_packets(uint32_t msg_bytes, int t, const void *rx_dev, uint64_t rx_stride,
                                      uint64_t n_packets, void *msg_dev, uint64_t msg_stride,
                                      uint16_t *syndromes_dev, uint8_t *status_dev,
                                      unsigned long long *counts_dev, void *stream);

/* hamming_encode_packets -- the transmitter ("exact reverse process"):
 * messages (msg_stride apart) -> packets (rx_stride apart, pad bits 0). */
hamming_status hamming_encode_packets(uint32_t msg_bytes, int t, const void *msg_dev, uint64_t msg_stride,
                                      uint64_t n_packets, void *rx_dev, uint64_t rx_stride, void *stream);

/* hamming_packet_channel_generate -- seeded synthetic received packets (test
 * and benchmark input, the oracle's oracle_generate_packets written
 * independently): for global packet index g, key = mix(seed + (g+1) gamma),
 * u(g,q) = mix(key + (q+1) gamma); message byte b = byte (b&7) of u(g, b>>3);
 * W = ceil(msg_bytes/8); segment i gets one flip iff all or u(g, W+2i) < thresh,
 * at position 1 + umulhi(lo32(u(g, W+2i+1)), n_i) -- one error per segment,
 * the paper's t-error regime.  msg_dev (nullable) receives the sent messages,
 * msg_bytes apart. */
hamming_status hamming_packet_channel_generate(uint32_t msg_bytes, int t, uint64_t seed, uint64_t g_first,
                                               uint64_t n_packets, uint64_t thresh, int all, void *rx_dev,
                                               uint64_t rx_stride, void *msg_dev, void *stream);

/* --------------------------------------------------------------- helpers */

uint64_t hamming_coded_bytes(int m, uint64_t n_codewords); /* ceil(n*N/8), 0 on bad m */
uint64_t hamming_data_bytes(int m, uint64_t n_codewords);  /* ceil(k*N/8), 0 on bad m */
const char *hamming_status_string(hamming_status s);
const char *hamming_last_error(void);  /* thread-local text of the last failure */
int hamming_abi_version(void);         /* HAMMING_ABI_VERSION */

/* Introspection for benchmarks: how many kernel launches the last
 * successful device entry point on this thread issued, and the grid it used. */
int hamming_last_launch_count(void);
int hamming_last_grid_blocks(void);

#ifdef __cplusplus
}
#endif

#endif /* HAMMING_H_ */
