"""Mutation check of the oracle's pins: apply plausible mistakes to
oracle/oracle.c one at a time, rebuild, run the -m "not gpu" oracle tests,
and require every mutant to be caught.  Restores the original on exit.

    python tools/mutate_oracle.py            # prints a markdown table
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
LIB = os.path.join(ROOT, "oracle", "liboracle.so")

MUTANTS = [
    ("syndrome bit weight 2^(j+1)", "s = s + c * (1 << j);\n    }\n    return s;\n}\n\n/* Error detection", "s = s + c * (1 << (j + 1));\n    }\n    return s;\n}\n\n/* Error detection"),
    ("index set misses its last member", "for (int p = 1; p <= n; p++) {\n        if ((p >> j) & 1) {", "for (int p = 1; p < n; p++) {\n        if ((p >> j) & 1) {"),
    ("index set uses bit j+1", "        if ((p >> j) & 1) {\n            out[count] = p;", "        if ((p >> (j + 1)) & 1) {\n            out[count] = p;"),
    ("correction flips position s+1", "bits[s - 1] = (uint8_t)(bits[s - 1] ^ 1);", "bits[s % n] = (uint8_t)(bits[s % n] ^ 1);"),
    ("correction ignores s == n", "if (s < 0 || s > n) return -1;", "if (s < 0 || s >= n) return -1;"),
    ("RR keeps position 1", "        if (!is_power_of_two(p)) {\n            msg[k] = bits[p - 1] & 1;", "        if (!is_power_of_two(p) || p == 1) {\n            msg[k] = bits[p - 1] & 1;"),
    ("odd parity in the encoder", "        cw[(1 << j) - 1] = (uint8_t)c;\n    }\n    return 0;", "        cw[(1 << j) - 1] = (uint8_t)(c ^ 1);\n    }\n    return 0;"),
    ("MSB-first bytes", "return (buf[b >> 3] >> (b & 7)) & 1;", "return (buf[b >> 3] >> (7 - (b & 7))) & 1;"),
    ("codeword stride n+1", "bits[p - 1] = (uint8_t)get_bit(rx, c * (uint64_t)n + (uint64_t)(p - 1));", "bits[p - 1] = (uint8_t)get_bit(rx, c * (uint64_t)(n + 1) + (uint64_t)(p - 1));"),
    ("count includes clean codewords", "if (s != 0) fixed++;", "fixed++;"),
    ("output pad not cleared", "for (uint64_t b = total; b < ((total + 7) / 8) * 8; b++) put_bit(data_out, b, 0);", ""),
    ("parity_bit_count off by one", "while ((1L << r) < (long)k + r + 1) r++;", "while ((1L << r) < (long)k + r) r++;"),
    ("generator p2 may equal p1", "p2 = 1 + (int)(((uint64_t)(p1 - 1) + 1 + ((w4 * (uint64_t)(n - 1)) >> 32)) % (uint64_t)n);", "p2 = 1 + (int)(((w4 * (uint64_t)n) >> 32));"),
    ("splitmix constant typo", "z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;", "z = (z ^ (z >> 27)) * 0x94D049BB133111EAULL;"),
    ("packet layout: larger segments last", "uint32_t k = msg_bits / (uint32_t)t + ((uint32_t)i < msg_bits % (uint32_t)t ? 1u : 0u);", "uint32_t k = msg_bits / (uint32_t)t + ((uint32_t)(t - 1 - i) < msg_bits % (uint32_t)t ? 1u : 0u);"),
    ("packet: uncorrectable segment still flipped", "        if (s != 0 && s <= n) {                                                         /* EC */", "        if (s != 0 && s <= 2 * n) {                                                     /* EC */"),
    ("packet generator flips p+1", "uint64_t b = cb + p - 1;", "uint64_t b = cb + p;"),
    ("packet generator event draw index off by one", "uint64_t ue = mix64(key + ((uint64_t)W + 2 * (uint64_t)i + 1) * 0x9E3779B97F4A7C15ULL);", "uint64_t ue = mix64(key + ((uint64_t)W + 2 * (uint64_t)i) * 0x9E3779B97F4A7C15ULL);"),
    ("packet generator message key g instead of g+1", "uint64_t key = mix64(seed + (g + 1) * 0x9E3779B97F4A7C15ULL);", "uint64_t key = mix64(seed + g * 0x9E3779B97F4A7C15ULL);"),
    ("count_events uses the message draw", "if (all || draw(seed, c, 1) < thresh) {\n            ev++;", "if (all || draw(seed, c, 0) < thresh) {\n            ev++;"),
    ("count_events weight-2 test on the low half", "if ((draw(seed, c, 2) >> 32) < q2thresh) w2++;", "if ((draw(seed, c, 2) & 0xFFFFFFFFULL) < q2thresh) w2++;"),
    ("generator p1 from the high half", "p1 = 1 + (int)((w3 * (uint64_t)n) >> 32);", "p1 = 1 + (int)((w4 * (uint64_t)n) >> 32);"),
]

TESTS = ["tests/test_oracle_pins.py", "tests/test_oracle_generator.py", "tests/test_oracle_packets.py",
         "tests/test_oracle_draws.py"]


def main():
    orig = open(SRC).read()
    backup = SRC + ".orig"
    shutil.copy(SRC, backup)
    rows = []
    try:
        for name, a, b in MUTANTS:
            if a not in orig:
                rows.append((name, "pattern not found"))
                continue
            open(SRC, "w").write(orig.replace(a, b, 1))
            if os.path.exists(LIB):
                os.remove(LIB)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *TESTS],
                               cwd=ROOT, capture_output=True, text=True)
            caught = r.returncode != 0
            first = ""
            for line in r.stdout.splitlines():
                if line.startswith("FAILED"):
                    first = line.split("::")[-1].split(" ")[0]
                    break
            rows.append((name, f"caught by {first}" if caught else "NOT CAUGHT"))
            print(name, "->", rows[-1][1], flush=True)
    finally:
        shutil.copy(backup, SRC)
        os.remove(backup)
        if os.path.exists(LIB):
            os.remove(LIB)
    print("\n| mutant | result |\n|---|---|")
    for name, res in rows:
        print(f"| {name} | {res} |")
    if any("NOT" in r or "not found" in r for _, r in rows):
        sys.exit(1)


if __name__ == "__main__":
    main()
