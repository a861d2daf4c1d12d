// ring.cpp — bounded SPSC command ring over the reference control array.
//
// Layout is kernels.py:23-31 verbatim (int64 words): TAIL@0, HEAD@8,
// COMPLETED@16, FLAGS@24, slots (lo, hi) from word 32.  Batch semantics
// follow kernels.py:61-104: push copies min(want - pushed, free) commands at a
// time and publishes TAIL; pop mirrors it on HEAD; both spin at most max_spin
// empty/full observations and then return a partial count.
//
// Difference from the reference, on purpose: the owner's
// counter is published with a release store and the peer's counter is read
// with an acquire load.  The reference uses plain numpy/numba stores and is
// correct only under x86-TSO with no compiler reordering (kernels.py:5-8).
// The same protocol is what the device producer (ll.cu) speaks over pinned
// host memory, so one consumer serves CPU and GPU producers alike.
//
// Extension: a producer that finds FLAG_SHUTDOWN set returns
// -EPB_ERR_SHUTDOWN ("push refused with a distinct shutdown
// signal"); the reference defines the flag (kernels.py:30) but never reads it.
#include <cstdint>

#include "ctx.h"

namespace {
inline int64_t load_acquire(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_ACQUIRE); }
inline int64_t load_relaxed(const int64_t* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
inline void store_release(int64_t* p, int64_t v) { __atomic_store_n(p, v, __ATOMIC_RELEASE); }
inline void cpu_relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}
}  // namespace

extern "C" int64_t epb_ring_push_batch(int64_t* ctl, int64_t cap, const int64_t* lo, const int64_t* hi,
                                       int64_t start, int64_t want, int64_t max_spin) {
  if (load_relaxed(&ctl[EPB_CTL_FLAGS]) & EPB_RING_FLAG_SHUTDOWN) return -EPB_ERR_SHUTDOWN;
  const int64_t mask = cap - 1;
  int64_t tail = load_relaxed(&ctl[EPB_CTL_TAIL]);
  int64_t pushed = 0, spins = 0;
  while (pushed < want) {
    const int64_t head = load_acquire(&ctl[EPB_CTL_HEAD]);
    const int64_t free_slots = cap - (tail - head);
    if (free_slots == 0) {
      if (++spins > max_spin) break;
      cpu_relax();
      continue;
    }
    const int64_t n = (want - pushed) < free_slots ? (want - pushed) : free_slots;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t s = EPB_CTL_SLOT0 + 2 * ((tail + i) & mask);
      ctl[s] = lo[start + pushed + i];
      ctl[s + 1] = hi[start + pushed + i];
    }
    tail += n;
    store_release(&ctl[EPB_CTL_TAIL], tail);
    pushed += n;
  }
  return pushed;
}

extern "C" int64_t epb_ring_pop_batch(int64_t* ctl, int64_t cap, int64_t* lo_out, int64_t* hi_out, int64_t start,
                                      int64_t want, int64_t max_spin) {
  const int64_t mask = cap - 1;
  int64_t head = load_relaxed(&ctl[EPB_CTL_HEAD]);
  int64_t popped = 0, spins = 0;
  while (popped < want) {
    const int64_t tail = load_acquire(&ctl[EPB_CTL_TAIL]);
    const int64_t avail = tail - head;
    if (avail == 0) {
      if (++spins > max_spin) break;
      cpu_relax();
      continue;
    }
    const int64_t n = (want - popped) < avail ? (want - popped) : avail;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t s = EPB_CTL_SLOT0 + 2 * ((head + i) & mask);
      lo_out[start + popped + i] = ctl[s];
      hi_out[start + popped + i] = ctl[s + 1];
    }
    head += n;
    store_release(&ctl[EPB_CTL_HEAD], head);
    popped += n;
  }
  return popped;
}

extern "C" int epb_ring_poll(const int64_t* ctl, int64_t cap, int64_t* lo, int64_t* hi) {
  const int64_t head = load_relaxed(&ctl[EPB_CTL_HEAD]);
  const int64_t tail = load_acquire(&ctl[EPB_CTL_TAIL]);
  if (tail == head) return 0;
  const int64_t s = EPB_CTL_SLOT0 + 2 * (head & (cap - 1));
  *lo = ctl[s];
  *hi = ctl[s + 1];
  return 1;
}

extern "C" int epb_ring_mark_completed(int64_t* ctl, int64_t upto) {
  if (upto > load_acquire(&ctl[EPB_CTL_HEAD])) return EPB_ERR_PROTOCOL;
  int64_t cur = load_relaxed(&ctl[EPB_CTL_COMPLETED]);
  while (upto > cur && !__atomic_compare_exchange_n(&ctl[EPB_CTL_COMPLETED], &cur, upto, true, __ATOMIC_RELEASE,
                                                    __ATOMIC_RELAXED)) {
  }
  return EPB_OK;
}

extern "C" int epb_ring_check_completion(const int64_t* ctl, int64_t idx) {
  return load_acquire(&ctl[EPB_CTL_COMPLETED]) > idx ? 1 : 0;
}

extern "C" int epb_ring_shutdown(int64_t* ctl) {
  __atomic_fetch_or(&ctl[EPB_CTL_FLAGS], (int64_t)EPB_RING_FLAG_SHUTDOWN, __ATOMIC_RELEASE);
  return EPB_OK;
}
