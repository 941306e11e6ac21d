"""Regenerate the golden fixtures from the REFERENCE's own code.

  reference_kat.json  oracle/_ref/ref_kat: the reference's shipped headers
                      (proj/include/kinoplan/core/{rng,cost,types}.hpp) compiled
                      in place against oracle/ref_shim/Eigen/Core (oracle/Makefile).
  philox_kat.json     Philox4x32-10 vectors from PyTorch's independent
                      implementation (ATen/core/PhiloxRNGEngine.h); the first
                      three are the published Random123 known-answer vectors.

Needs /root/reference (this container only); the committed JSON travels.
Run:  make -C oracle && python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

PHILOX_SRC = r"""
#define private public
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
int main() {
  unsigned cases[][6] = {
    {0,0,0,0,0,0},
    {0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu,0xffffffffu},
    {0x243f6a88u,0x85a308d3u,0x13198a2eu,0x03707344u,0xa4093822u,0x299f31d0u},
    {5,42,7,0,2602,0}, {1000,1048575,31,1,123456789,1}, {3,17,9,0,1234,0}, {0,0,0,1,0,0}};
  printf("[");
  for (int i = 0; i < 7; ++i) {
    unsigned* c = cases[i];
    at::Philox4_32 e; at::detail::UINT4 ctr; at::detail::UINT2 k;
    for (int j = 0; j < 4; ++j) ctr[j] = c[j];
    k[0] = c[4]; k[1] = c[5];
    auto o = e.rand(ctr, k, 10);
    printf("%s{\"ctr\": [%u, %u, %u, %u], \"key\": [%u, %u], \"out\": [%u, %u, %u, %u]}", i ? ", " : "",
           c[0], c[1], c[2], c[3], c[4], c[5], o[0], o[1], o[2], o[3]);
  }
  printf("]\n");
}
"""


def main():
    kat = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_kat")], check=True, capture_output=True,
                         text=True).stdout
    data = json.loads(kat)
    data["_source"] = "oracle/_ref/ref_kat = /root/reference/proj/include/kinoplan/core/{rng,cost,types}.hpp"
    with open(os.path.join(HERE, "reference_kat.json"), "w") as f:
        json.dump(data, f, indent=1)
    import torch

    inc = os.path.join(os.path.dirname(torch.__file__), "include")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.cpp")
        with open(src, "w") as f:
            f.write(PHILOX_SRC)
        exe = os.path.join(d, "p")
        subprocess.run(["g++", "-std=c++17", "-I", inc, "-o", exe, src], check=True)
        ph = json.loads(subprocess.run([exe], check=True, capture_output=True, text=True).stdout)
    with open(os.path.join(HERE, "philox_kat.json"), "w") as f:
        json.dump({"_source": "torch ATen/core/PhiloxRNGEngine.h philox_engine::rand (10 rounds)", "cases": ph},
                  f, indent=1)
    print("wrote reference_kat.json, philox_kat.json")


if __name__ == "__main__":
    main()
