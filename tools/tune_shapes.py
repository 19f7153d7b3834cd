"""Launch-shape sweep: `python tools/tune_shapes.py build` compiles variants of
libhamming.so into build/tune/ (CPU box); `python tools/tune_shapes.py run`
times each on the GPU via HAMMING_LIB + tools/quick_bench.py."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tune_libs")  # ships to the GPU box (build/ is gpurun-ignored)

VARIANTS = {
    # m: list of (W, S, in_place)
    3: [(16, 12, 1), (32, 6, 1), (24, 8, 1), (8, 24, 1)],
    4: [(8, 8, 1), (12, 6, 1), (4, 16, 1)],
    5: [(8, 4, 1), (12, 3, 1), (16, 2, 1), (4, 8, 1), (8, 3, 1)],
    6: [(8, 3, 1)],
}


ENCODE_VARIANTS = {
    ("ENC", 3): [(16, 4), (8, 8), (16, 8), (24, 4)],
    ("ENC", 4): [(8, 8), (16, 4), (12, 4), (8, 4)],
    ("SENC", 3): [(8, 4), (16, 4), (16, 8)],
    ("SENC", 4): [(8, 4), (16, 3), (8, 8)],
    ("SENC", 5): [(8, 3), (12, 2), (4, 4)],
    ("SENC", 6): [(4, 2), (8, 2), (6, 2)],
}
SECDED_VARIANTS = {
    3: [(16, 8), (8, 12), (16, 4), (24, 4)],
    4: [(8, 8), (16, 3), (12, 4), (8, 12), (16, 4)],
    5: [(12, 3), (8, 4), (16, 2), (8, 3)],
    6: [(8, 3), (12, 2), (8, 2)],
}
M3_VARIANTS = [("DecodeLut3Op", 16, 12), ("DecodeLut3Op", 32, 6), ("DecodeLut3Op", 24, 8),
               ("DecodeLut3PairOp", 16, 10), ("DecodeLut3PairOp", 16, 3), ("DecodeLut3PairOp", 32, 5),
               ("DecodeLut3PairOp", 24, 6)]
# (63,57) decode and the probe ops (-DHAM_PROBE) at several shapes, for the sustained power probe
POWER6_VARIANTS = [(8, 3, 0, 0), (8, 3, 1, 100000), (8, 3, 1, 2000), (8, 3, 2, 32), (8, 3, 2, 256), (8, 3, 2, 1000)]
LONG_VARIANTS = [(16, 6), (12, 4), (8, 3)]  # (warps for m = 7, warps for m = 8)
PKT_VARIANTS = [(9216, 2, 1, 12), (12416, 2, 1, 8), (14464, 2, 1, 14), (16512, 2, 1, 8), (18560, 2, 1, 12), (20608, 2, 1, 10), (24704, 2, 1, 8), (28800, 2, 1, 7)]


def name(m, v):
    return f"m{m}_w{v[0]}_s{v[1]}_ip{v[2]}"


def build():
    from concurrent.futures import ThreadPoolExecutor

    from paper_1412_6862_b200 import build as b
    os.makedirs(OUT, exist_ok=True)
    for f in os.listdir(OUT):
        if not (len(sys.argv) > 2 and sys.argv[2] == "m3" and f.startswith("m3_")):
            continue
        os.remove(os.path.join(OUT, f))
    jobs = []
    for m, vs in VARIANTS.items():
        for v in vs:
            # the other m keep their defaults
            defs = [f"HAM_W{m}={v[0]}", f"HAM_S{m}={v[1]}", f"HAM_IP{m}={'true' if v[2] else 'false'}"]
            jobs.append((os.path.join(OUT, name(m, v) + ".so"), defs))
    if len(sys.argv) > 2 and sys.argv[2] == "encode":
        jobs = [(os.path.join(OUT, f"enc_{nm}{m}_w{w}_s{st}.so"), [f"HAM_{nm}_W{m}={w}", f"HAM_{nm}_S{m}={st}"])
                for (nm, m), vs in ENCODE_VARIANTS.items() for w, st in vs]
    if len(sys.argv) > 2 and sys.argv[2] == "secded":
        jobs = [(os.path.join(OUT, f"sec_m{m}_w{w}_s{st}.so"), [f"HAM_SEC_W{m}={w}", f"HAM_SEC_S{m}={st}"])
                for m, vs in SECDED_VARIANTS.items() for w, st in vs]
    if len(sys.argv) > 2 and sys.argv[2] == "packets":
        for f in os.listdir(OUT):
            if f.startswith("pkt_"):
                os.remove(os.path.join(OUT, f))
        jobs = [(os.path.join(OUT, f"pkt_{b}_{st}_{mb}_{w}.so"),
                 [f"HAM_PKT_BUDGET={b}", f"HAM_PKT_STAGES={st}", f"HAM_PKT_MSGBUF={mb}", f"HAM_PKT_WARPS={w}"])
                for b, st, mb, w in PKT_VARIANTS]
    if len(sys.argv) > 2 and sys.argv[2] == "power6":
        jobs = [(os.path.join(OUT, f"pw6_w{w}_s{st}_m{md}_{ns}.so"),
                 ["HAM_PROBE", f"HAM_W6={w}", f"HAM_S6={st}", f"HAM_WAIT_MODE={md}", f"HAM_WAIT_NS={ns}"])
                for w, st, md, ns in POWER6_VARIANTS]
    if len(sys.argv) > 2 and sys.argv[2] == "long":
        jobs = [(os.path.join(OUT, f"long_w{w7}_{w8}.so"), [f"HAM_LONG_W7={w7}", f"HAM_LONG_W8={w8}"])
                for w7, w8 in LONG_VARIANTS]
    if len(sys.argv) > 2 and sys.argv[2] == "m3":
        jobs = [(os.path.join(OUT, f"m3_{op}_w{w}_s{st}.so"), [f"HAM_M3_OP={op}", f"HAM_W3={w}", f"HAM_S3={st}"])
                for op, w, st in M3_VARIANTS]
    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        for path in ex.map(lambda j: b.build(force=True, out=j[0], defines=j[1]), jobs):
            print("built", path, flush=True)


def run():
    if len(sys.argv) > 2 and sys.argv[2] == "encode":
        for (nm, m), vs in ENCODE_VARIANTS.items():
            for w, st in vs:
                env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"enc_{nm}{m}_w{w}_s{st}.so"))
                print(nm, m, w, st, flush=True)
                subprocess.run([sys.executable, os.path.join(ROOT, "tools", "encode_bench.py"), "--m", str(m)], env=env)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "secded":
        for m, vs in SECDED_VARIANTS.items():
            for w, st in vs:
                env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"sec_m{m}_w{w}_s{st}.so"))
                subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_bench.py"), "--secded", "--m",
                                str(m), "--tag", f"w{w}_s{st}"], env=env)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "power6":
        for w, st, md, ns in POWER6_VARIANTS:
            env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"pw6_w{w}_s{st}_m{md}_{ns}.so"))
            print(f"== shape W={w} S={st} wait mode {md} ({ns} ns)", flush=True)
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "power_probe.py"), "--probe", "--only6",
                            "--no-copy"], env=env)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "long":
        for w7, w8 in LONG_VARIANTS:
            env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"long_w{w7}_{w8}.so"))
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_bench.py"), "--m", "7", "8",
                            "--tag", f"w{w7}_{w8}"], env=env)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "m3":
        for op, w, st in M3_VARIANTS:
            env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"m3_{op}_w{w}_s{st}.so"))
            for gib in ("2", "0.25"):
                subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_bench.py"), "--m", "3", "--gib", gib,
                                "--tag", f"{op}_w{w}_s{st}"], env=env)
        return
    if len(sys.argv) > 2 and sys.argv[2] == "packets":
        for b, st, mb, w in PKT_VARIANTS:
            env = dict(os.environ, HAMMING_LIB=os.path.join(OUT, f"pkt_{b}_{st}_{mb}_{w}.so"))
            print("budget", b, "stages", st, "msgbufs", mb, "warps", w, flush=True)
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "packets_bench.py"), "--M", "400", "800", "1200", "1600",
                            "2000", "--t", "2", "3", "5", "6"], env=env)
        return
    for m, vs in VARIANTS.items():
        for v in vs:
            path = os.path.join(OUT, name(m, v) + ".so")
            env = dict(os.environ, HAMMING_LIB=path)
            subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_bench.py"), "--m", str(m),
                            "--tag", name(m, v)], env=env)


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]]()
