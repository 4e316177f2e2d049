// Internal device-side structures of the B200 temporal traversal engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>
#include <string>
#include <vector>

#include "../../include/tgxd.h"

namespace tgxd {

// Largest representable edge time. Keys are stored as start (Out) and -end
// (In), the strict bound adds 1 to a label, so times stay inside
// [0, 2^31 - 2] to keep every derived bound inside int32.
constexpr int64_t kTimeMax = 2147483646LL;
constexpr int32_t kInf = 0x7fffffff;  // unreached label in key space

// Fence stride of the selective index ("bucketed timeline"): fence[j] =
// key[32 j], so a fence probe narrows a search to one 128-byte key line.
constexpr uint32_t kFenceShift = 5;
constexpr uint32_t kFenceStride = 1u << kFenceShift;

// One direction of the device T-CSR. Segments are sorted by key ascending.
//   Out layout: key = start, val = end           (earliest arrival / fastest)
//   In layout : key = -end,  val = -start        (latest departure, mirrored)
// Keys live in their own array (searched, never streamed); neighbor and val
// are interleaved so the relax step reads one 8-byte word per edge and a
// short range touches as few 32-byte sectors as possible.
// With that mirror, both traversals are "relax val over edges whose key lies
// at or above the frontier vertex's bound", so one kernel family serves both.
struct DevCsr {
  const uint32_t* off = nullptr;  // n + 1
  const int32_t* key = nullptr;   // m: search keys (binary search / fences only)
  const uint2* pay = nullptr;     // m: relax payload {neighbor, val} (one 8-byte load)
  const int32_t* fence = nullptr; // ceil(m / 32): key[32 j]
  const int32_t* kmax = nullptr;  // n: last (largest) key of each segment, INT32_MIN if empty
  // n + 1: {off[v], kmax[v]} side by side — an expansion's segment bounds and
  // last key come from one 128-byte line (a random miss fetches the whole line)
  const uint2* okm = nullptr;
  uint32_t n = 0;
  uint32_t m = 0;
};

struct DeviceBuffer {
  void* p = nullptr;
  size_t bytes = 0;
  ~DeviceBuffer();
  cudaError_t ensure(size_t nbytes);
  void release();
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Per-query parameters in key space.
struct QueryParam {
  uint32_t root;  // vertex exempt from the ordering check (kNoRoot for none)
  int32_t klo;    // lowest admissible key (window start, mirrored for In)
  int32_t vhi;    // highest admissible val (window end, mirrored for In)
  int32_t depart; // fastest: departure of the current candidate
};
constexpr uint32_t kNoRoot = 0xffffffffu;

// Traversal workspace, sized for q_cap concurrent queries.
struct Workspace {
  uint64_t slots = 0;  // Q x n label slots currently allocated
  DeviceBuffer X, EP, R, fa, fb, chunks, smalls, ctl, params, seeds;
  uint64_t launches = 0;  // kernels this handle's queries launched (running total)
  // lazy label reset (api.cu launch): while `xinv` holds, every slot whose
  // expansion state is not the initial one has a finite label, and slots at
  // or above `xdirty` are untouched — so the next round-kernel query resets
  // only [0, xdirty) where X is finite instead of writing every slot
  bool xinv = false;
  uint64_t xdirty = 0;
  // the bytes of the query parameters / seeds last uploaded to params /
  // seeds (api.cu upload_query: a repeated query skips its two small
  // host-to-device copies)
  std::vector<char> up_qp, up_seeds;
  bool up_valid = false;
  uint64_t last_h2d = 0;  // bytes the last query moved host -> device
  // lane-per-query batches (lanes.cuh): vertex-major labels, ranges, dirty masks
  DeviceBuffer lxm, leb, ldirty;
  DeviceBuffer cand_lo, cand_cnt, cand_key, cand_n, timing_out;
  DeviceBuffer dep;    // split fastest sweeps: each sub-sweep's current departure
  // asynchronous engine: queued flags, vertex / chunk rings, control block
  DeviceBuffer axq, aunits, actl;
  uint64_t a_slots = 0, a_units = 0;
  // edge-state engine (edges.cuh): per-edge states, edge queues, results
  DeviceBuffer ereached, edep, eval, estamp, efa, efb, ectl, ey, esm;
  bool last_edge = false;
  bool last_async = false;
  bool last_handoff = false;  // round kernel may have handed its tail to a tail engine
  DeviceBuffer tstamp, tctl;  // cluster tail engine: per-slot stamps, control block
  uint64_t t_slots = 0;
  // early host copy (api.cu query_impl): the labels leave for the host while
  // the async tail runs; the tail's changed labels are patched afterwards
  bool early_req = false;   // set by the caller for one launch
  bool early_done = false;  // launch recorded early_ev (and the patch list)
  bool p24_req = false;     // the early copy reads 24-bit packed labels (p24)
  DeviceBuffer p24;
  uint64_t last_d2h = 0;    // bytes the last host-result query moved to the host
  DeviceBuffer chg, chg_n;
  unsigned long long chg_cap = 0;
  unsigned long long* trace_host = nullptr;  // mapped pinned trace (diagnostics)
  unsigned long long* trace_dev = nullptr;
  DeviceBuffer wtrace;
  uint32_t trace_cap = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // what the last query left in X (for tgxd_last_work)
  int last_kind = -1;
  uint32_t last_q = 0;
  int last_strict = 1;
  std::vector<QueryParam> last_params;
};

// Device control block (one per workspace), see traverse.cuh. The three
// work counters only ever grow during a query; each round works on the
// difference between its start and end values.
struct Control {
  // the six counters every block reads after a barrier, contiguous and
  // 16-byte aligned in pairs: three vector loads per block instead of six
  // (592 blocks read this line at once; traverse.cuh read_counters)
  unsigned long long pushes;        // frontier appends (queue position)
  unsigned long long improved;      // label improvements in non-pushing rounds
  unsigned long long chunks;        // big-range chunks emitted
  unsigned long long smalls;        // small ranges emitted
  unsigned long long edges;         // edges handed to the relax step
  unsigned long long pchunks;       // pull chunks emitted
  unsigned long long expansions;    // vertex expansions (the reference's for_each_window_edge calls)
  unsigned long long index_lookups; // expansions that used the fence index
  unsigned long long pull_scanned;  // reverse-layout entries scanned by pull rounds
  unsigned int rounds;
  unsigned int candidates;
  unsigned int error;               // watchdog tripped
  unsigned int handoff_flip;        // handoff: the queue holding the frontier (fb if 1)
  unsigned long long handoff_n;     // handoff: frontier size left to a tail engine
  unsigned long long handoff_kind;  // handoff: 1 the cluster tail engine, 2 the async engine
  unsigned long long t_end;         // globaltimer when the round kernel finished
  unsigned long long state[12];     // CTA-local rounds hand their state over here
  // grid barrier of the round kernel (traverse.cuh GridBarrier), own lines
  alignas(128) unsigned int bar_count;
  alignas(128) unsigned int bar_gen;
  unsigned int bar_pad[31];
};

}  // namespace tgxd

// Host-side widening pool: a few threads per graph handle that turn the
// int32 result chunks arriving in pinned staging into the caller's int64
// PathResult values while later chunks are still on the PCIe link.
struct WidenPool {
  std::vector<std::thread> threads;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  std::function<void(int)> job;  // called with the worker index
  uint64_t generation = 0;
  int pending = 0;
  bool stop = false;
  int size() const { return (int)threads.size(); }
  void start(int n) {
    for (int i = 0; i < n; ++i)
      threads.emplace_back([this, i] {
        uint64_t seen = 0;
        for (;;) {
          std::function<void(int)> f;
          {
            std::unique_lock<std::mutex> l(mu);
            cv.wait(l, [&] { return stop || generation != seen; });
            if (stop) return;
            seen = generation;
            f = job;
          }
          f(i);
          std::lock_guard<std::mutex> l(mu);
          if (--pending == 0) done_cv.notify_all();
        }
      });
  }
  void run(std::function<void(int)> f) {  // blocks until every worker ran f
    std::unique_lock<std::mutex> l(mu);
    job = std::move(f);
    pending = (int)threads.size();
    ++generation;
    cv.notify_all();
    done_cv.wait(l, [&] { return pending == 0; });
  }
  ~WidenPool() {
    {
      std::lock_guard<std::mutex> l(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : threads) t.join();
  }
};

struct tgxd_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t m_logical = 0;
  uint64_t m = 0;  // materialized per layout
  int directed = 1;
  uint64_t index_cutoff = 2048;
  uint64_t indexed[2] = {0, 0};
  tgxd::DeviceBuffer out_off, out_key, out_pay, out_fence, out_kmax, out_okm;
  tgxd::DeviceBuffer in_off, in_key, in_pay, in_fence, in_kmax, in_okm;
  tgxd::DeviceBuffer out2in;  // Out -> In position of each edge (shortest duration; lazy)
  // weighted shortest duration: per Out position the edge's weight as int64
  // (-1: not a non-negative integer, -2: >= 2^62); null = every weight 1
  tgxd::DeviceBuffer out_wbuf;
  const long long* out_w = nullptr;
  bool out2in_ready = false;
  uint32_t max_out_deg = 0;  // fastest: sizes the device candidate lists (lazy)
  std::vector<uint32_t> h_out_off;  // fastest: host copy of the Out offsets (lazy; split width)
  int span[2] = {0, 0};       // earliest start, latest end (lazy; batch splitting)
  bool span_known = false;
  bool max_out_deg_known = false;
  tgxd::DevCsr out, in;
  // selective-index cost model (costmodel.cuh), per direction, built on first use
  struct Hist {
    bool built = false;
    uint32_t count = 0;  // indexed vertices
    tgxd::DeviceBuffer ids, slot, hdr, counts, rows;
  } hist[2];
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  int coop_blocks = 0;
  int coop_blocks_async = 0;
  int coop_blocks_edge = 0;
  int coop_blocks_sd = 0;
  int coop_blocks_lanes = 0;
  int tail_per_sm = 3;       // CTAs per SM of the async tail continuation
  int tail_cluster = 0;      // CTAs of the cluster tail engine (0: async engine)
  int share = 1;             // views: handles meant to run side by side (grids divided)
  const tgxd_graph* parent = nullptr;  // views: the handle whose device graph is shared
  std::mutex mu;
  tgxd::Workspace ws;
  // pipelined host results (int32 chunks -> int64 on the host)
  int32_t* pinned = nullptr;  // cudaHostAlloc'd staging
  size_t pinned_n = 0;
  cudaEvent_t chunk_ev[16] = {};
  cudaStream_t copy_stream = nullptr;  // early host copies
  cudaEvent_t early_ev = nullptr;      // the round kernel is done
  unsigned long long* patch_host = nullptr;  // mapped: count, {slot, label} pairs
  volatile unsigned int* copy_flag_host = nullptr;  // mapped: the round kernel's copy signal
  unsigned int* copy_flag_dev = nullptr;
  unsigned long long* patch_dev = nullptr;
  size_t patch_cap = 0;
  WidenPool pool;
};
