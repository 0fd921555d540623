"""Runs the tcgen05 self-test modes on cuda:0 and prints max relative errors."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_08358_b200 as eb
L = eb.lib()
for mode in range(6):
    for K, N in [(16, 128), (64, 128), (128, 112), (128, 128), (64, 64)]:
        err = C.c_double(-1)
        st = L.ember_tc_selftest(0, mode, K, N, 7, C.byref(err))
        print(f"mode={mode} K={K} N={N} status={st} err={err.value:.3e} {L.ember_last_error().decode()}", flush=True)

for mode in (0, 1):
    for N in (64, 112, 128, 256):
        for nacc in (1, 2, 3, 4):
            if N * nacc > 256:
                continue
            c = C.c_double(-1)
            st = L.ember_tc_mmabench(0, mode + 16 * (nacc - 1), N, 4096, C.byref(c))
            print(f"mmabench mode={mode} N={N} nacc={nacc} status={st} cycles/mma={c.value:.1f} floor={128 * N / 256:.0f}",
                  flush=True)
