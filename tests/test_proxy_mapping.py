"""CPU check of the FIFO-channel -> proxy-thread map (csrc/common.cuh
proxy_thread_of) that the CPU proxy (which channels a thread serves,
csrc/proxy.cpp) and the LL receivers (whose per-thread signal counts they
wait for, csrc/ll.cu proxy_cmds_per_call) must agree on: every channel has one
owner, every command group of a call is counted exactly once, and the "phase"
map puts a whole phase on one thread.  A disagreement would leave a receiver
waiting for a signal no proxy thread ever publishes.
"""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

PROGRAM = r"""
#include <cstdio>
#include "common.cuh"
using epb::proxy_thread_of;
int main() {
  int bad = 0, cases = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int C : {4, 8, 16, 32, 64})
      for (int nth = 1; nth <= 8; ++nth) {
        const int half = C / 2 > 0 ? C / 2 : 1;
        for (int ch = 0; ch < C; ++ch) {  // one owner in range
          const int t = proxy_thread_of(ch, half, nth, mode);
          bad += t < 0 || t >= nth;
          if (mode == 1) bad += t != (ch < half ? 0 : 1 % nth);
        }
        for (int R : {1, 2, 4, 8})
          for (int per : {1, 2, 4}) {
            const int G = R * per;  // groups per call and direction (ll_groups)
            if (G > half) continue;
            for (int me = 0; me < R; ++me)
              for (int kind = 0; kind < 2; ++kind) {
                const int chan0 = kind ? half : 0;
                int total = 0;  // sum over threads of proxy_cmds_per_call
                for (int pt = 0; pt < nth; ++pt)
                  for (int b = me; b < G; b += R) total += proxy_thread_of(chan0 + b, half, nth, mode) == pt;
                bad += total != per;
                ++cases;
              }
          }
      }
  std::printf("%d %d\n", cases, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_proxy_thread_map_is_consistent(tmp_path):
    src = tmp_path / "map.cpp"
    src.write_text(PROGRAM)
    exe = tmp_path / "map"
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT / 'paper_2512_19849_b200' / 'csrc'}", f"-I{cuda_inc}",
                    str(src), "-o", str(exe)], check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    cases, bad = map(int, r.stdout.split())
    assert cases > 500 and bad == 0 and r.returncode == 0
