// pcopy_plan.h — how the CPU proxy's SM copy engine turns one sweep's jobs into
// copy-kernel launches (host only; proxy.cpp; tested on the CPU by
// tests/test_proxy_mapping.py).
//
// A job = one destination's copies (segments) in issue order, then up to two
// signals (the cumulative counts the receivers wait for).  Launches go to one
// stream and run in order; inside a launch all jobs run at once.  So:
//   * a launch holds at most one job per destination — a later job's signal
//     would otherwise run beside, and could overtake, the earlier job's copies;
//   * a job's second signal goes into a signal-only job of a later launch;
//   * a job with more segments than a launch holds is split, its signal on
//     the last part;
//   * <= kPcopyJobs jobs and <= kPcopySegs segments per launch;
//   * blocks per job = clamp(bytes / block_bytes, 1, 148).
#pragma once

#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.h"

struct PJob {
  int dest = -1;
  std::vector<epb_pcopy_seg> segs;
  uint64_t* sig[2] = {nullptr, nullptr};
  uint64_t val[2] = {0, 0};
  int nsig = 0;
  uint64_t bytes = 0;
};

inline std::vector<epb_pcopy_batch> pcopy_plan(const std::vector<PJob>& jobs, int64_t block_bytes) {
  std::vector<epb_pcopy_batch> out;
  epb_pcopy_batch b;
  bool seen[epb::kMaxRanks];
  auto reset = [&] {
    std::memset(&b, 0, sizeof(b));
    std::memset(seen, 0, sizeof(seen));
  };
  auto flush = [&] {
    if (b.njobs > 0) out.push_back(b);
    reset();
  };
  // one job into the current launch (a new launch when it does not fit)
  auto add = [&](int dest, const epb_pcopy_seg* segs, int nseg, uint64_t* sig, uint64_t val) {
    if (b.njobs == kPcopyJobs || seen[dest] || b.nsegs + nseg > kPcopySegs) flush();
    epb_pcopy_job& q = b.jobs[b.njobs++];
    q.dest = dest;
    q.seg0 = b.nsegs;
    q.nseg = nseg;
    uint64_t bytes = 0;
    for (int i = 0; i < nseg; ++i) {
      b.segs[b.nsegs++] = segs[i];
      bytes += segs[i].len;
    }
    q.blocks = (int)std::min<uint64_t>(148, std::max<uint64_t>(1, bytes / (uint64_t)std::max<int64_t>(1, block_bytes)));
    q.block0 = b.nblocks;
    b.nblocks += q.blocks;
    q.sig = sig;
    q.sig_val = val;
    seen[dest] = true;
  };
  reset();
  for (const PJob& J : jobs) {
    const int n = (int)J.segs.size();
    int s = 0;
    while (n - s > kPcopySegs) {  // split: the leading parts carry no signal
      add(J.dest, J.segs.data() + s, kPcopySegs, nullptr, 0);
      s += kPcopySegs;
    }
    add(J.dest, J.segs.data() + s, n - s, J.nsig > 0 ? J.sig[0] : nullptr, J.val[0]);
    if (J.nsig == 2) add(J.dest, nullptr, 0, J.sig[1], J.val[1]);
  }
  flush();
  return out;
}
