"""Graph-store files: Python writer/reader and the C++ binary_io.h restatement
agree byte for byte; size errors raise (IoError in C++)."""
import os
import subprocess

import numpy as np
import pytest

from paper_2101_08358_b200 import storage

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_node_part_relations_edges_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    th, ac = rng.standard_normal((7, 8)).astype(np.float32), rng.random((7, 8)).astype(np.float32)
    storage.write_meta(str(tmp_path), 20, 3, 3, 8)
    storage.write_node_part(str(tmp_path), 1, th, ac)
    t2, a2 = storage.read_node_part(str(tmp_path), 1, 7, 8)
    assert t2.tobytes() == th.tobytes() and a2.tobytes() == ac.tobytes()
    raw = np.fromfile(tmp_path / "node_part_1.bin", np.float32)
    assert raw.tobytes() == th.tobytes() + ac.tobytes()  # theta immediately followed by acc
    storage.write_relations(str(tmp_path), th[:3], ac[:3])
    r1, r2 = storage.read_relations(str(tmp_path), 3, 8)
    assert r1.tobytes() == th[:3].tobytes() and r2.tobytes() == ac[:3].tobytes()
    e = rng.integers(0, 20, (11, 3)).astype(np.uint32)
    off = np.array([0, 4, 4, 11] + [11] * 6, np.uint64)
    storage.write_edges(str(tmp_path), "train", e, off)
    assert (storage.read_edges(str(tmp_path), "train") == e).all()
    assert (storage.read_bucket_offsets(str(tmp_path), 3) == off).all()
    with pytest.raises(OSError):
        storage.read_node_part(str(tmp_path), 1, 8, 8)  # wrong size
    assert storage.read_meta(str(tmp_path))["num_partitions"] == 3


@pytest.mark.parametrize("std", ["c++17", "c++20"])
def test_cpp_binary_io_reads_python_files(tmp_path, std):
    th = np.arange(12, dtype=np.float32).reshape(3, 4)
    storage.write_node_part(str(tmp_path), 0, th, -th)
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include <vector>
#include "ember/binary_io.h"
int main(int argc, char** argv) {
    std::string dir = argv[1];
    std::vector<float> v = ember::read_pod_file<float>(dir + "/node_part_0.bin");
    if (v.size() != 24 || v[5] != 5.f || v[17] != -5.f) return 1;
    std::vector<float> part(24);
    ember::read_pod_file_exact(dir + "/node_part_0.bin", part.data(), part.size());
    ember::write_pod_file(dir + "/copy.bin", part.data(), part.size());
    try {
        std::vector<float> bad(23);
        ember::read_pod_file_exact(dir + "/node_part_0.bin", bad.data(), bad.size());
        return 2;
    } catch (const ember::IoError&) {
    }
    try {
        ember::read_pod_file<double>(dir + "/missing.bin");
        return 3;
    } catch (const ember::IoError&) {
    }
    std::puts("ok");
    return 0;
}
''')
    exe = tmp_path / "t"
    subprocess.run(["g++", f"-std={std}", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", (out.returncode, out.stdout, out.stderr)
    assert (tmp_path / "copy.bin").read_bytes() == (tmp_path / "node_part_0.bin").read_bytes()
