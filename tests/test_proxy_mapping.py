"""CPU check of the FIFO-channel -> proxy-thread map (csrc/common.cuh
proxy_thread_of) that the CPU proxy (which channels a thread serves,
csrc/proxy.cpp) and the LL receivers (whose per-thread signal counts they
wait for, csrc/ll.cu proxy_cmds_per_call) must agree on: every channel has one
owner, every command group of a call is counted exactly once, and the "phase"
map puts a whole phase on one thread.  A disagreement would leave a receiver
waiting for a signal no proxy thread ever publishes.

Also the SM copy engine's launch planning (csrc/pcopy_plan.h): per destination
the copies and signals keep their issue order, and no launch holds two jobs of
one destination (a signal could otherwise overtake the earlier copies).
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


PLAN_PROGRAM = r"""
#include <cstdio>
#include <random>
#include "pcopy_plan.h"
// Random sweeps of jobs -> pcopy_plan; check the invariants the proxy relies on.
int main() {
  std::mt19937 rng(7);
  int bad = 0, launches = 0;
  static uint64_t sigs[64];
  for (int trial = 0; trial < 3000; ++trial) {
    std::vector<PJob> jobs;
    const int nj = 1 + rng() % 20, R = 1 + rng() % 8;
    for (int j = 0; j < nj; ++j) {
      PJob J;
      J.dest = rng() % R;
      const int ns = rng() % 40;
      for (int s = 0; s < ns; ++s) {
        const uint64_t len = (rng() % 4 == 0) ? 0 : 16 * (1 + rng() % 20000);
        J.segs.push_back({reinterpret_cast<const char*>(0x1000 * (j * 64 + s)), reinterpret_cast<char*>(0x2000 * (j * 64 + s)), len});
        J.bytes += len;
      }
      J.nsig = rng() % 3;
      for (int k = 0; k < J.nsig; ++k) {
        J.sig[k] = &sigs[(j * 2 + k) % 64];
        J.val[k] = 1000 * j + k;
      }
      jobs.push_back(J);
    }
    const auto plan = pcopy_plan(jobs, 65536);
    launches += (int)plan.size();
    // flatten: per destination, the order of segments and signals must be the issue order, and
    // a signal must come in a later launch than every segment of the same job and of earlier jobs
    std::vector<std::vector<const void*>> seg_order(8), want_seg(8);
    std::vector<std::vector<uint64_t>> sig_order(8), want_sig(8);
    std::vector<int> last_seg_launch(8, -1);
    for (const PJob& J : jobs) {
      for (const auto& g : J.segs) want_seg[J.dest].push_back(g.src);
      for (int k = 0; k < J.nsig; ++k) want_sig[J.dest].push_back(J.val[k]);
    }
    for (size_t L = 0; L < plan.size(); ++L) {
      const epb_pcopy_batch& b = plan[L];
      bool seen[8] = {};
      int nb = 0;
      bad += b.njobs < 1 || b.njobs > kPcopyJobs || b.nsegs > kPcopySegs;
      for (int j = 0; j < b.njobs; ++j) {
        const epb_pcopy_job& q = b.jobs[j];
        bad += seen[q.dest];  // one job per destination per launch
        seen[q.dest] = true;
        bad += q.block0 != nb || q.blocks < 1 || q.blocks > 148;
        nb += q.blocks;
        for (int s = q.seg0; s < q.seg0 + q.nseg; ++s) {
          seg_order[q.dest].push_back(b.segs[s].src);
          last_seg_launch[q.dest] = (int)L;
        }
        if (q.sig) {
          sig_order[q.dest].push_back(q.sig_val);
          // every segment of this destination issued so far is in this launch or an earlier one
          bad += last_seg_launch[q.dest] > (int)L;
        }
      }
      bad += nb != b.nblocks;
    }
    for (int d = 0; d < 8; ++d) bad += seg_order[d] != want_seg[d] || sig_order[d] != want_sig[d];
    // a destination's second signal never shares a launch with its first
    for (size_t L = 0; L < plan.size(); ++L) {
      int cnt[8] = {};
      for (int j = 0; j < plan[L].njobs; ++j) cnt[plan[L].jobs[j].dest] += plan[L].jobs[j].sig != nullptr;
      for (int d = 0; d < 8; ++d) bad += cnt[d] > 1;
    }
  }
  std::printf("%d %d\n", launches, bad);
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_pcopy_plan_keeps_per_destination_order(tmp_path):
    src = tmp_path / "plan.cpp"
    src.write_text(PLAN_PROGRAM)
    exe = tmp_path / "plan"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT / 'paper_2512_19849_b200' / 'csrc'}",
                    "-I/usr/local/cuda/include", str(src), "-o", str(exe)], check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    launches, bad = map(int, r.stdout.split())
    assert launches > 3000 and bad == 0 and r.returncode == 0
