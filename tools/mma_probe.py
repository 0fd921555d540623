"""Cycles per tcgen05.mma (M=128, K=16, bf16) for the operand modes the contraction uses."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import paper_2101_08358_b200 as eb
L = eb.lib()
for mode in (0, 1, 2, 3):
    for N in (96, 112, 128, 192):
        for nacc in (1, 2):
            if N * nacc > 256:
                continue
            c = C.c_double(0)
            st = L.ember_tc_mmabench(0, mode + 16 * (nacc - 1), N, 4096, C.byref(c))
            print(f"mode={mode} N={N} nacc={nacc} status={st} cycles/mma={c.value:.1f} floor={128 * N / 256:.0f} "
                  f"{L.ember_last_error().decode()}", flush=True)
