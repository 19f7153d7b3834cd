/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * Hamming decoder of Islam, Kim & Kim, "Computationally Efficient
 * Implementation of a Hamming Code Decoder using Graphics Processing Unit"
 * (arXiv 1412.6862; /root/reference/PAPER.md, cited below as P:L<line>).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1412_6862_b200/csrc/); neither side includes the other.
 *
 * Style rules (so a reader can check it against the paper by eye):
 *   - one bit at a time: codewords are unpacked into arrays of 0/1 bytes,
 *     bits[p] = value at 1-based position p ("H = {b; b=0|b=1}");
 *   - the syndrome is the XOR over each index set I_j, walked in ascending
 *     position order (P:L98 index sets; Algorithm 1 Step 4);
 *   - no popcount intrinsics, no SWAR, no lookup tables, no blocking.
 *
 * Readings of the paper (DESIGN.md "Readings" R1..R12 lists all of them):
 *   R2 even parity; R3 data bits fill the non-power-of-two positions in
 *   ascending order, message bit 1 first; R4 stream bit b is bit (b & 7) of
 *   byte b >> 3 (LSB-first); R5 syndrome bit j has weight 2^j; R6 there are
 *   r index sets I_0 .. I_{r-1}, r = number of powers of two <= n.
 *
 * Pins (tests/test_oracle_*.py, all -m "not gpu"): the paper's worked
 * example I_j(11), SPEC examples, brute-force nearest-codeword
 * decoding over all 2^n words for m <= 4, the closed form
 * syndrome = XOR of the positions of the set bits, minimum distance 3.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define ORACLE_MAX_N 4096 /* longest codeword the word-level routines accept */

/* ------------------------------------------------------------------ */
/* Code geometry                                                        */
/* ------------------------------------------------------------------ */

/* Number of parity (redundancy) bits for k data bits: the minimal r with
 * 2^r >= k + r + 1 ("|H_i| = 7+4 = 11 bits and |R| = 4"; SPEC
 * parity_bit_count).  Returns -1 for k < 1. */
int oracle_parity_bit_count(int k)
{
    if (k < 1) return -1;
    int r = 0;
    while ((1L << r) < (long)k + r + 1) r++;
    return r;
}

/* Number of parity positions in an n-bit codeword: the powers of two that
 * are <= n (positions 1, 2, 4, ...).  Returns -1 for n < 3. */
int oracle_parity_positions(int n)
{
    if (n < 3) return -1;
    int r = 0;
    while ((1L << r) <= n) r++;
    return r;
}

/* 1 if p is a power of two (a parity position), else 0. */
static int is_power_of_two(int p)
{
    int v = 1;
    while (v < p) v = v * 2;
    return v == p;
}

/* Index set I_j of an n-bit codeword: every position p in [1, n] whose
 * binary representation has bit j set, in ascending order; 2^j itself is
 * included (for n = 11, I_0 = {1,3,5,7,9,11}, I_1 = {2,3,6,7,10,11},
 * I_2 = {4,5,6,7}, I_3 = {8,9,10,11}).  Writes the positions to out (room
 * for n entries) and returns how many; -1 if j is out of range. */
int oracle_index_set(int j, int n, int *out)
{
    int r = oracle_parity_positions(n);
    if (r < 0 || j < 0 || j >= r || n > ORACLE_MAX_N) return -1;
    int count = 0;
    for (int p = 1; p <= n; p++) {
        if ((p >> j) & 1) {
            out[count] = p;
            count++;
        }
    }
    return count;
}

/* ------------------------------------------------------------------ */
/* One codeword, bit arrays (index 0 <-> position 1)                    */
/* ------------------------------------------------------------------ */

/* Syndrome (the paper's checksum vector C_i): bit j is the
 * XOR of the received bits over I_j; the value is sum_j c_j 2^j (R5).
 * bits[p-1] is the bit at position p.  Returns the value, or -1 on bad n. */
int oracle_syndrome_bits(int n, const uint8_t *bits)
{
    int r = oracle_parity_positions(n);
    if (r < 0 || n > ORACLE_MAX_N) return -1;
    int set[ORACLE_MAX_N];
    int s = 0;
    for (int j = 0; j < r; j++) {
        int len = oracle_index_set(j, n, set);
        int c = 0;
        for (int i = 0; i < len; i++) {
            c = c ^ (bits[set[i] - 1] & 1);   /* modulo-2 (XOR), Alg. 1 Step 4 */
        }
        s = s + c * (1 << j);
    }
    return s;
}

/* Error detection and correction ("error detection (ED), error
 * correction (EC)"): syndrome 0 means no error; 1 <= s <= n names the
 * erroneous position, which is flipped in place; s > n names a position
 * that does not exist -> uncorrectable (returns -1, bits untouched).
 * Returns 0 when nothing was flipped, 1 when bit s was flipped. */
int oracle_correct_bits(int n, uint8_t *bits, int s)
{
    if (s == 0) return 0;
    if (s < 0 || s > n) return -1;
    bits[s - 1] = (uint8_t)(bits[s - 1] ^ 1);
    return 1;
}

/* Redundancy removal ("redundancy remover (RR)"): keep the
 * bits at the non-power-of-two positions, ascending.  Returns k. */
int oracle_remove_redundancy_bits(int n, const uint8_t *bits, uint8_t *msg)
{
    int k = 0;
    for (int p = 1; p <= n; p++) {
        if (!is_power_of_two(p)) {
            msg[k] = bits[p - 1] & 1;
            k++;
        }
    }
    return k;
}

/* Encoder, "the exact reverse process" of decoding: message bit i
 * (i = 1..k) goes to the i-th non-power-of-two position (R3); parity
 * position 2^j gets the XOR of the other bits of I_j so that every index
 * set has even parity (R2).  k = n - r message bits are read. */
int oracle_encode_bits(int n, const uint8_t *msg, uint8_t *cw)
{
    int r = oracle_parity_positions(n);
    if (r < 0 || n > ORACLE_MAX_N) return -1;
    int i = 0;
    for (int p = 1; p <= n; p++) {
        if (is_power_of_two(p)) {
            cw[p - 1] = 0;
        } else {
            cw[p - 1] = msg[i] & 1;
            i++;
        }
    }
    int set[ORACLE_MAX_N];
    for (int j = 0; j < r; j++) {
        int len = oracle_index_set(j, n, set);
        int c = 0;
        for (int t = 0; t < len; t++) {
            if (set[t] != (1 << j)) c = c ^ cw[set[t] - 1];
        }
        cw[(1 << j) - 1] = (uint8_t)c;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Bit streams (R4: stream bit b is bit (b & 7) of byte b >> 3)         */
/* ------------------------------------------------------------------ */

static int get_bit(const uint8_t *buf, uint64_t b)
{
    return (buf[b >> 3] >> (b & 7)) & 1;
}

static void put_bit(uint8_t *buf, uint64_t b, int v)
{
    if (v) buf[b >> 3] = (uint8_t)(buf[b >> 3] | (1u << (b & 7)));
    else   buf[b >> 3] = (uint8_t)(buf[b >> 3] & ~(1u << (b & 7)));
}

/* Perfect code of order m: n = 2^m - 1, k = n - m.  m in [2, 12]. */
static int code_n(int m) { return (1 << m) - 1; }

/* Decode a packet of `count` concatenated n-bit codewords (codeword c =
 * stream bits [c*n, c*n + n), position p = stream bit c*n + p - 1), the
 * paper's splitter -> ED -> EC -> RR -> merger chain (Fig. 1):
 *   data_out bits [c*k, c*k + k) = the k recovered message bits of c,
 *   syn[c] = syndrome of c (may be NULL),
 *   *corrected = number of codewords with a nonzero syndrome.
 * The bits of data_out's last byte past k*count are written as 0.
 * Returns 0, or -1 on a bad argument, or -2 if a syndrome exceeds n
 * (impossible for perfect codes; kept for completeness, SPEC detect_and_
 * correct).  data_out must hold ceil(k*count/8) bytes. */
int oracle_decode(int m, const uint8_t *rx, uint64_t count,
                  uint8_t *data_out, uint8_t *syn, uint64_t *corrected)
{
    if (m < 2 || m > 12) return -1;
    int n = code_n(m);
    int k = n - m;
    uint8_t bits[ORACLE_MAX_N];
    uint8_t msg[ORACLE_MAX_N];
    uint64_t fixed = 0;
    for (uint64_t c = 0; c < count; c++) {
        for (int p = 1; p <= n; p++)                     /* splitter */
            bits[p - 1] = (uint8_t)get_bit(rx, c * (uint64_t)n + (uint64_t)(p - 1));
        int s = oracle_syndrome_bits(n, bits);           /* ED (checksum) */
        int flipped = oracle_correct_bits(n, bits, s);   /* EC */
        if (flipped < 0) return -2;
        if (s != 0) fixed++;
        oracle_remove_redundancy_bits(n, bits, msg);     /* RR */
        for (int i = 0; i < k; i++)                      /* merger */
            put_bit(data_out, c * (uint64_t)k + (uint64_t)i, msg[i]);
        if (syn) syn[c] = (uint8_t)s;
    }
    uint64_t total = count * (uint64_t)k;
    for (uint64_t b = total; b < ((total + 7) / 8) * 8; b++) put_bit(data_out, b, 0);
    if (corrected) *corrected = fixed;
    return 0;
}

/* Encode a packet: data bits [c*k, c*k + k) -> stream bits [c*n, c*n + n).
 * Bits of rx's last byte past n*count are written as 0. */
int oracle_encode(int m, const uint8_t *data, uint64_t count, uint8_t *rx)
{
    if (m < 2 || m > 12) return -1;
    int n = code_n(m);
    int k = n - m;
    uint8_t msg[ORACLE_MAX_N];
    uint8_t cw[ORACLE_MAX_N];
    for (uint64_t c = 0; c < count; c++) {
        for (int i = 0; i < k; i++)
            msg[i] = (uint8_t)get_bit(data, c * (uint64_t)k + (uint64_t)i);
        oracle_encode_bits(n, msg, cw);
        for (int p = 1; p <= n; p++)
            put_bit(rx, c * (uint64_t)n + (uint64_t)(p - 1), cw[p - 1]);
    }
    uint64_t total = count * (uint64_t)n;
    for (uint64_t b = total; b < ((total + 7) / 8) * 8; b++) put_bit(rx, b, 0);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Seeded synthetic channel                  */
/* ------------------------------------------------------------------ */

/* splitmix64 output function (Steele, Lea & Flood 2014), used as a
 * counter-based generator: u(c, q) = mix(seed + (4c + q + 1) * gamma). */
static uint64_t mix64(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t draw(uint64_t seed, uint64_t c, uint64_t q)
{
    return mix64(seed + (4 * c + q + 1) * 0x9E3779B97F4A7C15ULL);
}

/* Generate `count` received codewords whose global indices are
 * c_first .. c_first + count - 1 (the random draws depend only on the
 * global index, so any range can be regenerated on its own):
 *   message  = low k bits of u(c,0), message bit i = bit i-1;
 *   codeword = oracle_encode_bits(message);
 *   an error event happens iff `all` != 0 or u(c,1) < thresh;
 *   the event has weight 2 iff (u(c,2) >> 32) < q2thresh (q2thresh <= 2^32),
 *   else weight 1;
 *   w3 = lo32(u(c,3)), w4 = hi32(u(c,3)):
 *     p1 = 1 + floor(w3 * n / 2^32),
 *     p2 = 1 + ((p1 - 1) + 1 + floor(w4 * (n-1) / 2^32)) mod n   (p2 != p1);
 *   received = codeword with bit p1 (and p2 for weight 2) flipped.
 * rx gets ceil(n*count/8) bytes (pad bits 0).  sent (nullable) gets the
 * message stream, ceil(k*count/8) bytes.  err (nullable) gets 2 bytes per
 * codeword: p1, p2 (0 where there is no such flip). */
int oracle_generate(int m, uint64_t seed, uint64_t c_first, uint64_t count,
                    uint64_t thresh, int all, uint64_t q2thresh,
                    uint8_t *rx, uint8_t *sent, uint8_t *err)
{
    if (m < 2 || m > 6) return -1;
    int n = code_n(m);
    int k = n - m;
    uint8_t msg[64];
    uint8_t cw[64];
    for (uint64_t i = 0; i < count; i++) {
        uint64_t c = c_first + i;
        uint64_t u0 = draw(seed, c, 0);
        uint64_t u1 = draw(seed, c, 1);
        uint64_t u2 = draw(seed, c, 2);
        uint64_t u3 = draw(seed, c, 3);
        for (int b = 0; b < k; b++) msg[b] = (uint8_t)((u0 >> b) & 1);
        oracle_encode_bits(n, msg, cw);
        int p1 = 0, p2 = 0;
        if (all || u1 < thresh) {
            uint64_t w3 = u3 & 0xFFFFFFFFULL;
            uint64_t w4 = u3 >> 32;
            p1 = 1 + (int)((w3 * (uint64_t)n) >> 32);
            cw[p1 - 1] ^= 1;
            if ((u2 >> 32) < q2thresh) {
                p2 = 1 + (int)(((uint64_t)(p1 - 1) + 1 + ((w4 * (uint64_t)(n - 1)) >> 32)) % (uint64_t)n);
                cw[p2 - 1] ^= 1;
            }
        }
        for (int p = 1; p <= n; p++) put_bit(rx, i * (uint64_t)n + (uint64_t)(p - 1), cw[p - 1]);
        if (sent)
            for (int b = 0; b < k; b++) put_bit(sent, i * (uint64_t)k + (uint64_t)b, msg[b]);
        if (err) {
            err[2 * i] = (uint8_t)p1;
            err[2 * i + 1] = (uint8_t)p2;
        }
    }
    uint64_t total = count * (uint64_t)n;
    for (uint64_t b = total; b < ((total + 7) / 8) * 8; b++) put_bit(rx, b, 0);
    if (sent) {
        uint64_t tk = count * (uint64_t)k;
        for (uint64_t b = tk; b < ((tk + 7) / 8) * 8; b++) put_bit(sent, b, 0);
    }
    return 0;
}

/* The channel's error events alone, for packets too large to generate on the
 * host (C5: 8.7e9 codewords): the draws u(c,1) and u(c,2) of
 * oracle_generate, nothing else.  *events = #{c : all or u(c,1) < thresh},
 * *weight2 (nullable) = how many of them have (u(c,2) >> 32) < q2thresh.
 * With q2 = 0 every event is one flip, whose syndrome is the flipped
 * position (nonzero), so a decoder's corrected count must equal *events.
 * Returns 0. */
int oracle_count_events(uint64_t seed, uint64_t c_first, uint64_t count, uint64_t thresh, int all,
                        uint64_t q2thresh, uint64_t *events, uint64_t *weight2)
{
    uint64_t ev = 0, w2 = 0;
    for (uint64_t i = 0; i < count; i++) {
        uint64_t c = c_first + i;
        if (all || draw(seed, c, 1) < thresh) {
            ev++;
            if ((draw(seed, c, 2) >> 32) < q2thresh) w2++;
        }
    }
    *events = ev;
    if (weight2) *weight2 = w2;
    return 0;
}

/* ABI marker so tests can check they loaded the oracle, not something else. */
int oracle_version(void) { return 1; }

/* ================================================================== */
/* The paper's own workload: one packet of      */
/* msg_bytes message bytes is split into t segments ("splits the  */
/* message into t segments H_1 ... H_t, where t is the error tolerance")*/
/* and each segment is one shortened Hamming codeword with the minimal  */
/* r of 2^r >= k + r + 1 (P:L98 |H_i| = 7 + 4 = 11, |R| = 4).           */
/* ================================================================== */

/* Segment sizes (reading R14, SPEC make_layout): the first (bits mod t)
 * segments get ceil(bits/t) message bits, the rest floor(bits/t).  Writes
 * seg_k[t], seg_n[t]; returns the total coded bits, or -1. */
long oracle_packet_layout(uint32_t msg_bits, int t, uint32_t *seg_k, uint32_t *seg_n)
{
    if (t < 1 || msg_bits < (uint32_t)t) return -1;
    long total = 0;
    for (int i = 0; i < t; i++) {
        uint32_t k = msg_bits / (uint32_t)t + ((uint32_t)i < msg_bits % (uint32_t)t ? 1u : 0u);
        int r = oracle_parity_bit_count((int)k);
        if (r < 0 || k + (uint32_t)r > ORACLE_MAX_N * 4u) return -1;
        seg_k[i] = k;
        seg_n[i] = k + (uint32_t)r;
        total += (long)seg_n[i];
    }
    return total;
}

#define ORACLE_MAX_SEG 16384  /* longest shortened codeword the packet routines take */

/* Syndrome of a general n-bit word (n may exceed ORACLE_MAX_N): the same
 * definition as oracle_syndrome_bits -- bit j is the XOR over I_j -- walked
 * position by position. */
static int syndrome_long(int n, const uint8_t *bits)
{
    int r = oracle_parity_positions(n);
    int s = 0;
    for (int j = 0; j < r; j++) {
        int c = 0;
        for (int p = 1; p <= n; p++)
            if ((p >> j) & 1) c = c ^ (bits[p - 1] & 1);
        s = s + c * (1 << j);
    }
    return s;
}

static void encode_long(int n, const uint8_t *msg, uint8_t *cw)
{
    int r = oracle_parity_positions(n);
    int i = 0;
    for (int p = 1; p <= n; p++) {
        if (is_power_of_two(p)) cw[p - 1] = 0;
        else { cw[p - 1] = msg[i] & 1; i++; }
    }
    for (int j = 0; j < r; j++) {
        int c = 0;
        for (int p = 1; p <= n; p++)
            if (((p >> j) & 1) && p != (1 << j)) c = c ^ cw[p - 1];
        cw[(1 << j) - 1] = (uint8_t)c;
    }
}

/* Encode one packet: message bits (LSB-first bytes) -> splitter -> encoder per
 * segment -> concatenation H = H_1 + ... + H_t, LSB-first, pad bits 0. */
int oracle_encode_packet(uint32_t msg_bytes, int t, const uint8_t *msg, uint8_t *rx)
{
    uint32_t seg_k[64], seg_n[64];
    if (t > 64) return -1;
    long total = oracle_packet_layout(msg_bytes * 8u, t, seg_k, seg_n);
    if (total < 0) return -1;
    static __thread uint8_t m[ORACLE_MAX_SEG], cw[ORACLE_MAX_SEG];
    uint64_t mb = 0, cb = 0;
    for (int i = 0; i < t; i++) {
        if (seg_n[i] > ORACLE_MAX_SEG) return -1;
        for (uint32_t b = 0; b < seg_k[i]; b++) m[b] = (uint8_t)get_bit(msg, mb + b);
        encode_long((int)seg_n[i], m, cw);
        for (uint32_t p = 0; p < seg_n[i]; p++) put_bit(rx, cb + p, cw[p]);
        mb += seg_k[i];
        cb += seg_n[i];
    }
    for (uint64_t b = cb; b < ((cb + 7) / 8) * 8; b++) put_bit(rx, b, 0);
    return 0;
}

/* Decode one packet (Fig. 1: splitter -> ED/EC/RR per segment -> merger):
 *   syn[i]  = syndrome of segment i;
 *   s = 0: nothing; 1 <= s <= n_i: bit s flipped (corrected); s > n_i: the
 *   syndrome names a position that does not exist -> uncorrectable (SPEC
 *   detect_and_correct), the segment's bits are left as received (reading
 *   R15) and the packet status is 2;
 *   msg = merged message bits.  Returns the packet status: 0 clean,
 *   1 corrected, 2 uncorrectable; -1 on a bad argument. */
int oracle_decode_packet(uint32_t msg_bytes, int t, const uint8_t *rx, uint8_t *msg, uint16_t *syn)
{
    uint32_t seg_k[64], seg_n[64];
    if (t > 64) return -1;
    long total = oracle_packet_layout(msg_bytes * 8u, t, seg_k, seg_n);
    if (total < 0) return -1;
    static __thread uint8_t bits[ORACLE_MAX_SEG], m[ORACLE_MAX_SEG];
    uint64_t mb = 0, cb = 0;
    int status = 0;
    for (int i = 0; i < t; i++) {
        int n = (int)seg_n[i];
        if (n > ORACLE_MAX_SEG) return -1;
        for (int p = 0; p < n; p++) bits[p] = (uint8_t)get_bit(rx, cb + (uint64_t)p);   /* splitter */
        int s = syndrome_long(n, bits);                                                 /* ED */
        if (s != 0 && s <= n) {                                                         /* EC */
            bits[s - 1] ^= 1;
            if (status < 1) status = 1;
        } else if (s > n) {
            status = 2;
        }
        int k = oracle_remove_redundancy_bits(n, bits, m);                              /* RR */
        for (int b = 0; b < k; b++) put_bit(msg, mb + (uint64_t)b, m[b]);              /* merger */
        if (syn) syn[i] = (uint16_t)s;
        mb += seg_k[i];
        cb += (uint64_t)n;
    }
    return status;
}

/* Seeded packet channel (packets): for global
 * packet index g, key = mix(seed + (g+1) gamma) and u(g,q) = mix(key +
 * (q+1) gamma).  Message byte b = byte (b & 7) of u(g, b >> 3); W = number of
 * message draws = ceil(msg_bytes / 8); segment i has an error event iff all
 * or u(g, W + 2i) < thresh, at position 1 + umulhi(lo32(u(g, W + 2i + 1)), n_i)
 * (one flip per segment: the paper's t-error regime).
 * Packet j of the output starts at rx + j*stride (stride >= coded bytes);
 * msg (nullable) gets the sent messages, msg_bytes apart.  Returns 0 / -1. */
int oracle_generate_packets(uint32_t msg_bytes, int t, uint64_t seed, uint64_t g_first, uint64_t count,
                            uint64_t thresh, int all, uint8_t *rx, uint64_t stride, uint8_t *msg)
{
    uint32_t seg_k[64], seg_n[64];
    if (t > 64) return -1;
    long total = oracle_packet_layout(msg_bytes * 8u, t, seg_k, seg_n);
    if (total < 0 || stride < (uint64_t)((total + 7) / 8)) return -1;
    static __thread uint8_t m[ORACLE_MAX_SEG / 8 * 64];
    uint32_t W = (msg_bytes + 7) / 8;
    for (uint64_t j = 0; j < count; j++) {
        uint64_t g = g_first + j;
        uint64_t key = mix64(seed + (g + 1) * 0x9E3779B97F4A7C15ULL);
        for (uint32_t b = 0; b < msg_bytes; b++) {
            uint64_t u = mix64(key + ((uint64_t)(b >> 3) + 1) * 0x9E3779B97F4A7C15ULL);
            m[b] = (uint8_t)(u >> (8 * (b & 7)));
        }
        uint8_t *out = rx + j * stride;
        if (oracle_encode_packet(msg_bytes, t, m, out) != 0) return -1;
        uint64_t cb = 0;
        for (int i = 0; i < t; i++) {
            uint64_t ue = mix64(key + ((uint64_t)W + 2 * (uint64_t)i + 1) * 0x9E3779B97F4A7C15ULL);
            uint64_t up = mix64(key + ((uint64_t)W + 2 * (uint64_t)i + 2) * 0x9E3779B97F4A7C15ULL);
            if (all || ue < thresh) {
                uint64_t p = 1 + (((up & 0xFFFFFFFFULL) * (uint64_t)seg_n[i]) >> 32);
                uint64_t b = cb + p - 1;
                put_bit(out, b, get_bit(out, b) ^ 1);
            }
            cb += seg_n[i];
        }
        for (uint64_t b = (uint64_t)total; b < stride * 8; b++) put_bit(out, b, 0);
        if (msg) for (uint32_t b = 0; b < msg_bytes; b++) msg[j * msg_bytes + b] = m[b];
    }
    return 0;
}

/* ================================================================== */
/* Extended Hamming / SECDED (reading R17): a   */
/* codeword of 2^m bits whose bit 0 (position 0) is the overall parity */
/* over all 2^m bits (even) and whose positions 1..n, n = 2^m - 1, are */
/* the Hamming codeword.  Codeword c = stream bits [c 2^m, (c+1) 2^m). */
/* ================================================================== */

/* Decode: s = syndrome over positions 1..n (index sets, as above);
 * P = XOR of all 2^m bits.
 *   P = 1: one error -- at position s (s = 0: the parity bit itself) --
 *          corrected; flags bit 6.
 *   P = 0, s != 0: two errors detected, nothing corrected; flags bit 7.
 *   P = 0, s = 0: clean.
 * flags[c] = s | bit6 | bit7 (nullable); data as in oracle_decode;
 * *corrected / *detected count the two cases. */
int oracle_decode_secded(int m, const uint8_t *rx, uint64_t count, uint8_t *data_out, uint8_t *flags,
                         uint64_t *corrected, uint64_t *detected)
{
    if (m < 3 || m > 6) return -1;
    int n = code_n(m);
    int k = n - m;
    int w = n + 1;
    uint8_t bits[64];
    uint8_t msg[64];
    uint64_t fixed = 0, found = 0;
    for (uint64_t c = 0; c < count; c++) {
        for (int b = 0; b < w; b++) bits[b] = (uint8_t)get_bit(rx, c * (uint64_t)w + (uint64_t)b);
        int s = oracle_syndrome_bits(n, bits + 1);          /* positions 1..n */
        int P = 0;
        for (int b = 0; b < w; b++) P = P ^ bits[b];
        int f = 0;
        if (P == 1) {
            bits[s] ^= 1;                                    /* position s (0 = the parity bit) */
            f = 0x40;
            fixed++;
        } else if (s != 0) {
            f = 0x80;
            found++;
        }
        oracle_remove_redundancy_bits(n, bits + 1, msg);
        for (int i = 0; i < k; i++) put_bit(data_out, c * (uint64_t)k + (uint64_t)i, msg[i]);
        if (flags) flags[c] = (uint8_t)(s | f);
    }
    uint64_t total = count * (uint64_t)k;
    for (uint64_t b = total; b < ((total + 7) / 8) * 8; b++) put_bit(data_out, b, 0);
    if (corrected) *corrected = fixed;
    if (detected) *detected = found;
    return 0;
}

/* Encode: Hamming-encode positions 1..n, then bit 0 = XOR of positions 1..n. */
int oracle_encode_secded(int m, const uint8_t *data, uint64_t count, uint8_t *rx)
{
    if (m < 3 || m > 6) return -1;
    int n = code_n(m);
    int k = n - m;
    int w = n + 1;
    uint8_t msg[64], cw[64];
    for (uint64_t c = 0; c < count; c++) {
        for (int i = 0; i < k; i++) msg[i] = (uint8_t)get_bit(data, c * (uint64_t)k + (uint64_t)i);
        oracle_encode_bits(n, msg, cw + 1);
        int P = 0;
        for (int p = 1; p <= n; p++) P = P ^ cw[p];
        cw[0] = (uint8_t)P;
        for (int b = 0; b < w; b++) put_bit(rx, c * (uint64_t)w + (uint64_t)b, cw[b]);
    }
    return 0;
}

/* Seeded SECDED channel: the draws of oracle_generate, positions drawn over
 * all 2^m bits (bit index 0 = the parity bit):
 *   b1 = umulhi(lo32(u(g,3)), 2^m), b2 = (b1 + 1 + umulhi(hi32(u(g,3)), 2^m - 1)) mod 2^m;
 * err (nullable) records b1 + 1, b2 + 1 (0 = no flip). */
int oracle_generate_secded(int m, uint64_t seed, uint64_t c_first, uint64_t count,
                           uint64_t thresh, int all, uint64_t q2thresh,
                           uint8_t *rx, uint8_t *sent, uint8_t *err)
{
    if (m < 3 || m > 6) return -1;
    int n = code_n(m);
    int k = n - m;
    int w = n + 1;
    uint8_t msg[64], cw[64];
    for (uint64_t i = 0; i < count; i++) {
        uint64_t c = c_first + i;
        uint64_t u0 = draw(seed, c, 0);
        uint64_t u1 = draw(seed, c, 1);
        uint64_t u2 = draw(seed, c, 2);
        uint64_t u3 = draw(seed, c, 3);
        for (int b = 0; b < k; b++) msg[b] = (uint8_t)((u0 >> b) & 1);
        oracle_encode_bits(n, msg, cw + 1);
        int P = 0;
        for (int p = 1; p <= n; p++) P = P ^ cw[p];
        cw[0] = (uint8_t)P;
        int b1 = -1, b2 = -1;
        if (all || u1 < thresh) {
            b1 = (int)(((u3 & 0xFFFFFFFFULL) * (uint64_t)w) >> 32);
            cw[b1] ^= 1;
            if ((u2 >> 32) < q2thresh) {
                b2 = (int)(((uint64_t)b1 + 1 + (((u3 >> 32) * (uint64_t)(w - 1)) >> 32)) % (uint64_t)w);
                cw[b2] ^= 1;
            }
        }
        for (int b = 0; b < w; b++) put_bit(rx, i * (uint64_t)w + (uint64_t)b, cw[b]);
        if (sent)
            for (int b = 0; b < k; b++) put_bit(sent, i * (uint64_t)k + (uint64_t)b, msg[b]);
        if (err) {
            err[2 * i] = (uint8_t)(b1 + 1);
            err[2 * i + 1] = (uint8_t)(b2 + 1);
        }
    }
    if (sent) {
        uint64_t tk = count * (uint64_t)k;
        for (uint64_t b = tk; b < ((tk + 7) / 8) * 8; b++) put_bit(sent, b, 0);
    }
    return 0;
}
