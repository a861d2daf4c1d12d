// barrier.cpp — the proxy's all-peer barrier (the Barrier TransferCmd).
//
// "the Proxy thread creates an intra-node shared memory to
// enforce a hierarchical barrier — synchronization among local peers first,
// then across nodes".  On one NVLink node the hierarchy has one level: the
// ranks' proxies rendezvous through a POSIX shared-memory segment that every
// rank of the job maps (its name is derived from all ranks' IPC handles, so it
// is unique per job and identical on every rank).  SPEC.md:274-282:
//   post: no participant returns before all have entered (per epoch);
//         all return when all call (liveness, watchdog-bounded).
// The protocol is an epoch flag per rank: rank r stores arrive[r] = e
// (release) and waits until arrive[q] >= e for every q (acquire).  Nothing is
// ever reset, so consecutive barriers need no sense reversal.
// SameRail scope (flag EPB_FLAG_SAME_RAIL_BARRIER): the rail peers of a rank
// are the same GPU index on other nodes; on one node that set is empty, so the
// barrier completes immediately ("1 rank ... returns immediately").
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "ctx.h"

struct epb_barrier {
  struct Shared {
    std::atomic<uint64_t> arrive[EPB_MAX_RANKS];
  };
  Shared* sh = nullptr;
  int world = 1, rank = 0;
  uint64_t epoch = 0;
  std::string name;
};

static_assert(std::atomic<uint64_t>::is_always_lock_free, "shared-memory barrier needs lock-free 64-bit atomics");

extern "C" int epb_barrier_open(const char* name, int world, int rank, epb_barrier_t** out) {
  if (!name || !out || world <= 0 || world > EPB_MAX_RANKS || rank < 0 || rank >= world)
    return epb_set_error(EPB_ERR_PROTOCOL, "bad barrier arguments");
  const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return epb_set_error(EPB_ERR_CONNECTION, std::string("shm_open failed for ") + name);
  const size_t bytes = sizeof(epb_barrier::Shared);
  if (ftruncate(fd, (off_t)bytes) != 0) {  // a new segment is zero-filled; an existing one keeps its size
    close(fd);
    return epb_set_error(EPB_ERR_CONNECTION, "ftruncate of the barrier segment failed");
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return epb_set_error(EPB_ERR_CONNECTION, "mmap of the barrier segment failed");
  auto* b = new epb_barrier();
  b->sh = static_cast<epb_barrier::Shared*>(p);
  b->world = world;
  b->rank = rank;
  b->name = name;
  b->epoch = b->sh->arrive[rank].load(std::memory_order_acquire);  // re-opened by the same rank: continue
  *out = b;
  return EPB_OK;
}

extern "C" int epb_barrier_wait(epb_barrier_t* b, int same_rail, double timeout_s) {
  if (!b) return epb_set_error(EPB_ERR_PROTOCOL, "null barrier");
  const uint64_t e = ++b->epoch;
  b->sh->arrive[b->rank].store(e, std::memory_order_release);
  if (same_rail) return EPB_OK;  // no rail peers on one node
  const auto t0 = std::chrono::steady_clock::now();
  for (int q = 0; q < b->world; ++q) {
    int spins = 0;
    while (b->sh->arrive[q].load(std::memory_order_acquire) < e) {
      if (++spins < 4096) continue;
      spins = 0;
      std::this_thread::yield();
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
        return epb_set_error(EPB_ERR_DEADLOCK, "proxy barrier timed out (rank " + std::to_string(q) + " absent)");
    }
  }
  return EPB_OK;
}

extern "C" int epb_barrier_close(epb_barrier_t* b, int unlink) {
  if (!b) return EPB_OK;
  munmap(b->sh, sizeof(epb_barrier::Shared));
  if (unlink) shm_unlink(b->name.c_str());
  delete b;
  return EPB_OK;
}

// Segment name shared by every rank of a job: FNV-1a over all IPC handles
// (multi-process) or over the process id and the group's first context
// (emulated ranks in one process).
std::string epb_barrier_name(const void* bytes, size_t n) {
  uint64_t h = 1469598103934665603ull;
  const unsigned char* p = static_cast<const unsigned char*>(bytes);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  char buf[48];
  std::snprintf(buf, sizeof(buf), "/epb_bar_%016llx", (unsigned long long)h);
  return buf;
}
