"""Developer run: the suite's randomized parity tests of the register-gather
evaluators (tests/test_gpu_fuzz.py) on seeds beyond the suite's.
python tools/tools_fuzz_extended_gather.py [n_block] [n_single] [n_partitioned]"""
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import test_gpu_fuzz as G  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 300
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 100
npart = int(sys.argv[3]) if len(sys.argv) > 3 else 60
bad = []
for name, fn, lo, cnt in (("block", G.test_random_block_bitwise, 64, nb),
                          ("single", G.test_random_single_bitwise, 16, ns),
                          ("partitioned", G.test_random_partitioned_bitwise, 16, npart)):
    ok = 0
    for seed in range(lo, lo + cnt):
        try:
            fn(seed)
            ok += 1
        except BaseException as e:  # noqa: BLE001
            bad.append((name, seed, repr(e)[:160]))
    print(f"{name}: {ok} of {cnt} draws bitwise", flush=True)
print("failures:", bad, flush=True)
