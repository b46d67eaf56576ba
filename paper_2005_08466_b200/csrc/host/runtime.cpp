// haocl::HostContext on the CUDA C-ABI (include/haocl/runtime.hpp).
//
// Reference: proj/src/runtime.cpp. The handle tables, argument binding,
// launch validation, EMA profiling, timing fragments and message trace keep
// the reference's semantics; the transport changes:
//   * NodeLink/Channel (runtime.cpp:67-92)        -> a CUDA device + stream via hcl_*;
//   * stage_buffer's host-mediated migration      -> device-to-device NVLink copies
//     (runtime.cpp:220-249)                          (hcl_buffer_copy_peer);
//   * launch_on_queue's blocking RPC (253-309)    -> asynchronous hcl_launch; compute time
//                                                    from CUDA events, drained by finish().
// New: the partitioned NDRange launch (see runtime.hpp) with sharded buffers:
// every buffer tracks, per device, the allocated byte slice and the valid
// byte interval, so SPLIT_ROWS outputs stay on the devices that computed them
// and reads gather the pieces.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>

#include <nvtx3/nvToolsExt.h>

#include "haocl/runtime.hpp"
#include "hcl_cabi.h"
#include "hcl_host.h"

namespace hcl {
void set_last_error(const std::string& m);
extern thread_local bool t_launch_untimed;  // csrc/common.hpp
}

namespace haocl {

namespace {

// NVTX ranges around the host API's phases (launch, transfers, collectives,
// finish): visible in Nsight Systems / ncu range filters, no cost without a tool
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  Range(const char* prefix, const std::string& what) { nvtxRangePushA((std::string(prefix) + what).c_str()); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) { return std::chrono::duration<double, std::milli>(Clock::now() - t).count(); }

[[noreturn]] void fail(ErrorCode code, const std::string& m) { throw Error(code, m); }

// Turns a C-ABI return code back into the reference's exception.
void check(int rc) {
  if (rc == HCL_OK) return;
  int code = rc - HCL_ERR_BASE;
  if (code < 0 || code > 23) code = 0;
  throw Error(static_cast<ErrorCode>(code), hcl_last_error());
}

}  // namespace

void MessageTrace::record(TraceEvent e) {
  std::lock_guard lock(mutex_);
  events_.push_back(std::move(e));
}
std::vector<TraceEvent> MessageTrace::events() const {
  std::lock_guard lock(mutex_);
  return events_;
}
size_t MessageTrace::count_calls(const std::string& function, int device) const {
  std::lock_guard lock(mutex_);
  size_t n = 0;
  for (const auto& e : events_)
    if (e.function == function && (device < 0 || e.device == device)) ++n;
  return n;
}
void MessageTrace::clear() {
  std::lock_guard lock(mutex_);
  events_.clear();
}

struct HostContext::Impl {
  // Disjoint, non-adjacent byte intervals [first, end) kept in a sorted map.
  struct Ranges {
    std::map<uint64_t, uint64_t> m;  // first -> end
    bool empty() const { return m.empty(); }
    void clear() { m.clear(); }
    void add(uint64_t first, uint64_t len) {
      if (!len) return;
      uint64_t f = first, e = first + len;
      auto it = m.upper_bound(f);
      if (it != m.begin()) {
        auto pv = std::prev(it);
        if (pv->second >= f) it = pv;  // overlaps or touches the previous interval
      }
      while (it != m.end() && it->first <= e) {
        f = std::min(f, it->first);
        e = std::max(e, it->second);
        it = m.erase(it);
      }
      m.emplace(f, e);
    }
    void sub(uint64_t first, uint64_t len) {
      if (!len) return;
      const uint64_t f = first, e = first + len;
      auto it = m.upper_bound(f);
      if (it != m.begin() && std::prev(it)->second > f) --it;
      while (it != m.end() && it->first < e) {
        const uint64_t a = it->first, b = it->second;
        it = m.erase(it);
        if (a < f) m.emplace(a, f);
        if (b > e) {
          m.emplace(e, b);
          break;
        }
      }
    }
    // end of the interval holding `pos`, or 0 when no interval holds it
    uint64_t holds(uint64_t pos) const {
      auto it = m.upper_bound(pos);
      if (it == m.begin()) return 0;
      --it;
      return pos < it->second ? it->second : 0;
    }
    bool covers(uint64_t first, uint64_t len) const {
      if (!len) return true;
      const uint64_t e = holds(first);
      return e && e >= first + len;
    }
    // first interval start strictly after `pos` (UINT64_MAX if none)
    uint64_t next_start(uint64_t pos) const {
      auto it = m.upper_bound(pos);
      return it == m.end() ? UINT64_MAX : it->first;
    }
  };
  struct Piece {
    uint64_t alloc_first = 0, alloc_bytes = 0;
    Ranges valid;  // valid byte intervals inside the allocation
    bool allocated = false;
  };
  struct BufferRec {
    uint64_t size = 0;
    std::map<int, Piece> pieces;  // device gid -> piece
  };
  struct Launch {
    std::string kernel;
    uint64_t work = 0;
    cudaEvent_t start = nullptr, stop = nullptr;
    int gid = 0;
  };
  struct QueueRec {
    int gid = 0;
    std::string user;
    bool shared = true;
    double transfer_ms = 0.0, compute_ms = 0.0, modeled_ms = 0.0;
    std::vector<Launch> pending;
    // serializes finish() per queue; the table lock is never held across a
    // device synchronization (the reference's per-queue mutex, runtime.cpp:60-64)
    std::shared_ptr<std::mutex> op_mu = std::make_shared<std::mutex>();
  };
  struct ProgramRec {
    std::string bundle;
    std::vector<std::pair<std::string, uint32_t>> kernels;
  };
  struct KernelRec {
    uint64_t program = 0;
    std::string bundle;
    std::string name;
    uint32_t arity = 0;
    std::vector<uint8_t> kinds, classes;
    std::map<uint32_t, Arg> args;
    // last rate-driven split (hysteresis against EMA noise moving shards)
    std::vector<uint64_t> last_bounds, last_queues;
  };

  GlobalDeviceMap device_map;
  Scheduler scheduler;
  MessageTrace trace;
  std::recursive_mutex mu;
  std::map<uint64_t, BufferRec> buffers;
  std::map<uint64_t, QueueRec> queues;
  std::map<uint64_t, ProgramRec> programs;
  std::map<uint64_t, KernelRec> kernels;
  std::set<uint64_t> events;
  std::map<int, uint64_t> internal_queues;
  std::atomic<uint64_t> next_handle{1};
  std::mutex breakdown_mu;
  TimingBreakdown timings;

  uint64_t new_id() { return next_handle.fetch_add(1); }
  std::vector<std::pair<int, uint64_t>> mapped;  // (device, id) of IPC-mapped peer buffers

  Handle new_event() {
    uint64_t id = new_id();
    events.insert(id);
    return Handle{HandleKind::event, id};
  }

  int dev_index(int gid) const {
    const DeviceEntry* e = device_map.find(gid);
    if (!e) fail(ErrorCode::unknown_device, "device " + std::to_string(gid));
    return static_cast<int>(e->local_index);
  }

  BufferRec& buffer(uint64_t id) {
    auto it = buffers.find(id);
    if (it == buffers.end()) fail(ErrorCode::handle, "buffer handle " + std::to_string(id) + " is released or unknown");
    return it->second;
  }
  QueueRec& queue(uint64_t id) {
    auto it = queues.find(id);
    if (it == queues.end()) fail(ErrorCode::handle, "queue handle " + std::to_string(id) + " is released or unknown");
    return it->second;
  }
  KernelRec& kernel(uint64_t id) {
    auto it = kernels.find(id);
    if (it == kernels.end()) fail(ErrorCode::handle, "kernel handle " + std::to_string(id) + " is released or unknown");
    return it->second;
  }

  void add_transfer(QueueRec* q, double ms) {
    if (q) q->transfer_ms += ms;
    std::lock_guard lock(breakdown_mu);
    timings.transfer_ms += ms;
  }

  // -- residency --------------------------------------------------------------

  // Make the allocation of `id` on `gid` cover [first, first+len), preserving
  // the currently valid bytes of that device.
  Piece& ensure_alloc(uint64_t id, BufferRec& b, int gid, uint64_t first, uint64_t len) {
    Piece& p = b.pieces[gid];
    int dev = dev_index(gid);
    if (p.allocated && first >= p.alloc_first && first + len <= p.alloc_first + p.alloc_bytes) return p;
    uint64_t nf = first, ne = first + len;
    if (p.allocated) {
      nf = std::min(nf, p.alloc_first);
      ne = std::max(ne, p.alloc_first + p.alloc_bytes);
    }
    if (p.allocated && !p.valid.empty()) {
      // preserve every valid interval through a temporary buffer on the same device
      const uint64_t tmp = new_id(), of = p.alloc_first;
      check(hcl_buffer_alloc(dev, tmp, of, p.alloc_bytes));
      for (auto& [a, e] : p.valid.m) check(hcl_buffer_copy_peer(dev, tmp, a, dev, id, a, e - a));
      check(hcl_buffer_alloc(dev, id, nf, ne - nf));
      for (auto& [a, e] : p.valid.m) check(hcl_buffer_copy_peer(dev, id, a, dev, tmp, a, e - a));
      check(hcl_buffer_release(dev, tmp));
    } else {
      check(hcl_buffer_alloc(dev, id, nf, ne - nf));
      p.valid.clear();
    }
    trace.record({gid, "alloc_buffer", id});
    p.allocated = true;
    p.alloc_first = nf;
    p.alloc_bytes = ne - nf;
    return p;
  }

  static void set_valid(Piece& p, uint64_t first, uint64_t len) { p.valid.add(first, len); }

  // Other devices' copies of [first, first+len) are stale after a write there.
  static void invalidate_others(BufferRec& b, int gid, uint64_t first, uint64_t len) {
    for (auto& [g, p] : b.pieces)
      if (g != gid) p.valid.sub(first, len);
  }

  // Make bytes [first, first+len) of buffer `id` valid on `gid`, copying the
  // missing parts from devices that hold them (NVLink peer copies). Bytes no
  // device holds were never written: the zero-filled allocation stands for them.
  void ensure_valid(uint64_t id, BufferRec& b, int gid, uint64_t first, uint64_t len, QueueRec* q) {
    Piece& p = ensure_alloc(id, b, gid, first, len);
    if (p.valid.covers(first, len)) return;
    auto started = Clock::now();
    int dev = dev_index(gid);
    uint64_t pos = first, end = first + len;
    bool copied = false;
    while (pos < end) {
      if (uint64_t e = p.valid.holds(pos)) {
        pos = e;
        continue;
      }
      const uint64_t stop = std::min(end, p.valid.next_start(pos));
      int src = -1;
      uint64_t src_end = 0;
      for (auto& [g, o] : b.pieces) {
        if (g == gid) continue;
        if (uint64_t e = o.valid.holds(pos)) {
          src = g;
          src_end = e;
          break;
        }
      }
      if (src < 0) {  // skip to the next byte some other device holds
        uint64_t next = stop;
        for (auto& [g, o] : b.pieces)
          if (g != gid) next = std::min(next, o.valid.next_start(pos));
        pos = next;
        continue;
      }
      const uint64_t n = std::min(stop, src_end) - pos;
      check(hcl_buffer_copy_peer(dev, id, pos, dev_index(src), id, pos, n));
      trace.record({gid, "copy_peer", id});
      copied = true;
      pos += n;
    }
    set_valid(p, first, len);
    if (copied) add_transfer(q, ms_since(started));
  }

  void note_residency(uint64_t id, BufferRec& b) {
    std::vector<int> ids;
    for (auto& [g, p] : b.pieces)
      if (b.size && p.valid.covers(0, b.size)) ids.push_back(g);
    scheduler.note_resident(id, ids);
  }

  // -- launches -----------------------------------------------------------------

  struct Part {
    int gid;
    uint64_t queue;
    uint64_t lo, hi;
  };

  Handle launch_parts(KernelRec& k, const std::vector<Arg>& args, std::array<uint64_t, 3> global, uint32_t dims,
                      const std::vector<Part>& parts, bool whole) {
    Range range("hcl:launch ", k.name);
    const uint32_t n = k.arity;
    const uint64_t rows = global[0];
    // per-argument byte geometry
    std::vector<uint64_t> row_bytes(n, 0);
    for (uint32_t i = 0; i < n; ++i) {
      if (!args[i].is_buffer) continue;
      if (k.kinds[i] == HCL_ARG_SCALAR)
        fail(ErrorCode::argument, k.name + " argument " + std::to_string(i) + ": expected a scalar");
      BufferRec& b = buffer(args[i].buffer);
      if (!whole && k.classes[i] == HCL_PART_SPLIT_ROWS) {
        if (rows == 0 || b.size % rows)
          fail(ErrorCode::argument, k.name + " argument " + std::to_string(i) + ": buffer of " + std::to_string(b.size) +
                                        " bytes does not split into " + std::to_string(rows) + " rows");
        row_bytes[i] = b.size / rows;
      }
    }
    for (uint32_t i = 0; i < n; ++i)
      if (!args[i].is_buffer && k.kinds[i] != HCL_ARG_SCALAR)
        fail(ErrorCode::argument, k.name + " argument " + std::to_string(i) + ": expected a buffer");
    if (!whole)
      for (uint32_t i = 0; i < n; ++i)
        if (args[i].is_buffer && k.classes[i] == HCL_PART_REPLICATE &&
            (k.kinds[i] == HCL_ARG_OUT || k.kinds[i] == HCL_ARG_INOUT) && parts.size() > 1)
          fail(ErrorCode::argument, k.name + ": a replicated output cannot be partitioned");

    auto slice = [&](uint32_t i, const Part& part, uint64_t& first, uint64_t& len) {
      bool split = !whole && k.classes[i] == HCL_PART_SPLIT_ROWS;
      first = split ? part.lo * row_bytes[i] : 0;
      len = split ? (part.hi - part.lo) * row_bytes[i] : buffer(args[i].buffer).size;
    };
    // 1. stage every part (inputs made valid, outputs allocated) before any launch
    for (const Part& part : parts) {
      if (!whole && part.hi == part.lo) continue;
      QueueRec& q = queue(part.queue);
      for (uint32_t i = 0; i < n; ++i) {
        if (!args[i].is_buffer) continue;
        BufferRec& b = buffer(args[i].buffer);
        uint64_t first, len;
        slice(i, part, first, len);
        if (k.kinds[i] == HCL_ARG_OUT || k.classes[i] == HCL_PART_LOCAL)  // LOCAL: private workspace
          ensure_alloc(args[i].buffer, b, part.gid, first, len);
        else
          ensure_valid(args[i].buffer, b, part.gid, first, len, &q);
      }
    }
    // 1b. EXCHANGE / PEERS: each part's kernel stores its rows into every part's copy
    //     of the EXCHANGE output; its PEERS input lists the other copies' addresses
    std::vector<const Part*> live;
    for (const Part& part : parts)
      if (whole || part.hi > part.lo) live.push_back(&part);
    int xi = -1;
    for (uint32_t i = 0; i < n; ++i)
      if (args[i].is_buffer && k.classes[i] == HCL_PART_EXCHANGE) {
        if (xi >= 0) fail(ErrorCode::argument, k.name + ": one EXCHANGE output per kernel");
        xi = static_cast<int>(i);
      }
    const bool exchange = xi >= 0 && live.size() > 1;
    if (exchange) {
      for (size_t a = 0; a < live.size(); ++a)
        for (size_t c = a + 1; c < live.size(); ++c)
          if (live[a]->gid == live[c]->gid)
            fail(ErrorCode::argument, k.name + ": an EXCHANGE output needs one device per part");
      for (uint32_t i = 0; i < n; ++i) {
        if (!args[i].is_buffer || k.classes[i] != HCL_PART_PEERS) continue;
        if (i + 1 >= n || args[i + 1].is_buffer || args[i + 1].scalar != static_cast<int64_t>(live.size() - 1))
          fail(ErrorCode::argument, k.name + ": the PEERS count argument must equal parts - 1");
        BufferRec& pb = buffer(args[i].buffer);
        if (pb.size < 8 * (live.size() - 1)) fail(ErrorCode::size, k.name + ": PEERS buffer too small");
        for (const Part* p : live) {
          std::vector<uint64_t> addrs;
          for (const Part* o : live) {
            if (o == p) continue;
            void* ptr = nullptr;
            check(hcl_buffer_device_ptr(dev_index(o->gid), args[xi].buffer, &ptr, nullptr, nullptr));
            addrs.push_back(reinterpret_cast<uint64_t>(ptr));
          }
          check(hcl_buffer_write(dev_index(p->gid), args[i].buffer, 0, addrs.data(), addrs.size() * 8));
          set_valid(pb.pieces[p->gid], 0, pb.size);  // per-device contents: the others stay valid too
        }
      }
    }
    // 1c. EXCHANGE: a part's kernel stores into its peers' copies, whose
    //     allocation (stream-ordered alloc + zero fill on the peer's stream) and
    //     older readers must be complete first: every live stream waits for
    //     every other live stream's staging before any part launches
    if (exchange) {
      std::vector<std::pair<cudaStream_t, cudaEvent_t>> staged;
      for (const Part* p : live) {
        void* st = nullptr;
        check(hcl_device_stream(dev_index(p->gid), &st));
        int ordinal = 0;
        if (cudaStreamGetDevice(static_cast<cudaStream_t>(st), &ordinal) == cudaSuccess) cudaSetDevice(ordinal);
        cudaEvent_t ev = nullptr;
        cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cudaEventRecord(ev, static_cast<cudaStream_t>(st));
        staged.emplace_back(static_cast<cudaStream_t>(st), ev);
      }
      for (auto& [st, own] : staged)
        for (auto& [st2, ev] : staged)
          if (ev != own) cudaStreamWaitEvent(st, ev, 0);
      for (auto& [st, ev] : staged) cudaEventDestroy(ev);  // released once the waits resolve
    }
    // 2. launch every part asynchronously on its device stream
    std::vector<std::pair<cudaStream_t, cudaEvent_t>> part_done;
    std::vector<hcl_arg> cargs(n);
    for (uint32_t i = 0; i < n; ++i)
      cargs[i] = hcl_arg{static_cast<uint32_t>(k.kinds[i]), 0, args[i].scalar, args[i].buffer};
    for (const Part& part : parts) {
      if (!whole && part.hi == part.lo) continue;
      QueueRec& q = queue(part.queue);
      scheduler.note_dispatch(part.gid);
      Launch l;
      l.kernel = k.name;
      l.gid = part.gid;
      int dev = dev_index(part.gid);
      void* stream = nullptr;
      check(hcl_device_stream(dev, &stream));
      // the events must belong to the stream's GPU (several GPUs per process)
      int ordinal = 0;
      if (cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &ordinal) == cudaSuccess) cudaSetDevice(ordinal);
      cudaEventCreate(&l.start);
      cudaEventCreate(&l.stop);
      cudaEventRecord(l.start, static_cast<cudaStream_t>(stream));
      uint64_t goff[3] = {part.lo, 0, 0};
      uint64_t gsz[3] = {part.hi - part.lo, global[1], global[2]};
      trace.record({part.gid, "launch_kernel", 0});
      hcl::t_launch_untimed = true;  // l.start / l.stop time this part (one event pair, not two)
      int rc = hcl_launch(dev, k.name.c_str(), cargs.data(), n, goff, whole ? nullptr : gsz, dims, &l.work);
      hcl::t_launch_untimed = false;
      cudaEventRecord(l.stop, static_cast<cudaStream_t>(stream));
      part_done.emplace_back(static_cast<cudaStream_t>(stream), l.stop);
      scheduler.note_complete(part.gid);
      if (rc != HCL_OK) {
        cudaEventDestroy(l.start);
        cudaEventDestroy(l.stop);
        check(rc);
      }
      q.pending.push_back(l);
    }
    // 2b. EXCHANGE: every part wrote into every copy, so each device's stream
    //     waits for all parts before anything later touches the output there
    if (exchange)
      for (auto& [st, ev_own] : part_done)
        for (auto& [st2, ev] : part_done)
          if (ev != ev_own) cudaStreamWaitEvent(st, ev, 0);
    // 3. outputs: the launch produced the bytes U = union of the part slices
    //    (one interval); older copies of U anywhere are stale, bytes outside U
    //    keep their validity
    bool merged_topk = false;
    for (uint32_t i = 0; i < n; ++i) {
      if (!args[i].is_buffer || k.kinds[i] == HCL_ARG_IN) continue;
      BufferRec& b = buffer(args[i].buffer);
      if (k.classes[i] == HCL_PART_LOCAL) continue;  // device-private contents: no validity to track
      if (!whole && k.classes[i] == HCL_PART_REDUCE_SUM) {
        // sum the parts' int64 partials onto the first part's device
        std::vector<int> gids;
        for (const Part& part : parts)
          if (part.hi > part.lo) gids.push_back(part.gid);
        if (gids.empty()) continue;
        for (size_t a = 0; a < gids.size(); ++a)
          for (size_t c = a + 1; c < gids.size(); ++c)
            if (gids[a] == gids[c])
              fail(ErrorCode::argument, k.name + ": a REDUCE_SUM output needs one device per part");
        // binary tree: in round r part a folds part a + 2^r into itself; the
        // folds of one round run concurrently on their devices' streams and
        // integer sums make the result independent of the tree shape
        const int g0 = gids[0];
        const uint64_t id = args[i].buffer;
        for (size_t stride = 1; stride < gids.size(); stride *= 2)
          for (size_t a = 0; a + stride < gids.size(); a += 2 * stride) {
            const int da = dev_index(gids[a]);
            uint64_t tmp = new_id();
            check(hcl_buffer_alloc(da, tmp, 0, b.size));
            check(hcl_buffer_copy_peer(da, tmp, 0, dev_index(gids[a + stride]), id, 0, b.size));
            trace.record({gids[a], "copy_peer", id});
            hcl_arg ra[3] = {{HCL_ARG_INOUT, 0, 0, id}, {HCL_ARG_IN, 0, 0, tmp},
                             {HCL_ARG_SCALAR, 0, static_cast<int64_t>(b.size / 8), 0}};
            check(hcl_launch(da, "reduce_add_i64", ra, 3, nullptr, nullptr, 1, nullptr));
            check(hcl_buffer_release(da, tmp));
          }
        for (auto& [g, p] : b.pieces) p.valid.clear();
        b.pieces[g0].valid.add(0, b.size);
        continue;
      }
      if (k.classes[i] == HCL_PART_EXCHANGE) {  // whole on every participating device
        for (auto& [g, p] : b.pieces) p.valid.clear();
        for (const Part* p : live) b.pieces[p->gid].valid.add(0, b.size);
        continue;
      }
      if (!whole && k.classes[i] == HCL_PART_MERGE_TOPK) {
        // fold the parts' top-k lists onto the first part's device with the
        // kernel's "<name>_merge" companion (same arguments + the other part's
        // index and distance lists), in part order
        if (merged_topk) continue;  // both MERGE_TOPK outputs are folded together
        merged_topk = true;
        std::vector<uint32_t> mi;
        for (uint32_t j = 0; j < n; ++j)
          if (args[j].is_buffer && k.classes[j] == HCL_PART_MERGE_TOPK) mi.push_back(j);
        if (mi.size() != 2) fail(ErrorCode::argument, k.name + ": MERGE_TOPK needs one index and one distance output");
        std::vector<int> gids;
        for (const Part& part : parts)
          if (part.hi > part.lo) gids.push_back(part.gid);
        if (gids.empty()) continue;
        for (size_t a = 0; a < gids.size(); ++a)
          for (size_t c = a + 1; c < gids.size(); ++c)
            if (gids[a] == gids[c])
              fail(ErrorCode::argument, k.name + ": a MERGE_TOPK output needs one device per part");
        // binary tree of pairwise merges (the (dist, idx) merge is associative,
        // so any fold order equals the P-way merge); one round's merges run
        // concurrently on their devices
        const int g0 = gids[0];
        BufferRec& bi = buffer(args[mi[0]].buffer);
        BufferRec& bd = buffer(args[mi[1]].buffer);
        const std::string merge = k.name + "_merge";
        for (size_t stride = 1; stride < gids.size(); stride *= 2)
          for (size_t a = 0; a + stride < gids.size(); a += 2 * stride) {
            const int d0 = dev_index(gids[a]), da = dev_index(gids[a + stride]);
            uint64_t ti = new_id(), td = new_id();
            check(hcl_buffer_alloc(d0, ti, 0, bi.size));
            check(hcl_buffer_alloc(d0, td, 0, bd.size));
            check(hcl_buffer_copy_peer(d0, ti, 0, da, args[mi[0]].buffer, 0, bi.size));
            check(hcl_buffer_copy_peer(d0, td, 0, da, args[mi[1]].buffer, 0, bd.size));
            trace.record({gids[a], "copy_peer", args[mi[0]].buffer});
            trace.record({gids[a], "copy_peer", args[mi[1]].buffer});
            std::vector<hcl_arg> margs(cargs);
            margs[mi[0]].kind = HCL_ARG_INOUT;
            margs[mi[1]].kind = HCL_ARG_INOUT;
            margs.push_back(hcl_arg{HCL_ARG_IN, 0, 0, ti});
            margs.push_back(hcl_arg{HCL_ARG_IN, 0, 0, td});
            const int rc = hcl_launch(d0, merge.c_str(), margs.data(), static_cast<uint32_t>(margs.size()), nullptr,
                                      nullptr, 1, nullptr);
            hcl_buffer_release(d0, ti);
            hcl_buffer_release(d0, td);
            check(rc);
          }
        for (BufferRec* b2 : {&bi, &bd}) {
          for (auto& [g, p] : b2->pieces) p.valid.clear();
          b2->pieces[g0].valid.add(0, b2->size);
        }
        continue;
      }
      // every part's slice is now valid on its device and stale everywhere else
      for (const Part& part : parts) {
        if (!whole && part.hi == part.lo) continue;
        uint64_t first, len;
        slice(i, part, first, len);
        for (auto& [g, p] : b.pieces)
          if (g != part.gid) p.valid.sub(first, len);
      }
      for (const Part& part : parts) {
        if (!whole && part.hi == part.lo) continue;
        uint64_t first, len;
        slice(i, part, first, len);
        b.pieces[part.gid].valid.add(first, len);
      }
    }
    for (uint32_t i = 0; i < n; ++i)
      if (args[i].is_buffer && k.kinds[i] != HCL_ARG_IN) note_residency(args[i].buffer, buffer(args[i].buffer));
    return new_event();
  }

  KernelRec& bound_kernel(uint64_t kid, std::vector<Arg>& args) {
    KernelRec& k = kernel(kid);
    for (const auto& [index, value] : k.args)
      if (index >= k.arity)
        fail(ErrorCode::argument, "argument index " + std::to_string(index) + " out of range for a " +
                                      std::to_string(k.arity) + "-arg kernel");
    for (uint32_t i = 0; i < k.arity; ++i)
      if (!k.args.count(i)) fail(ErrorCode::argument, "kernel argument " + std::to_string(i) + " is unbound");
    for (uint32_t i = 0; i < k.arity; ++i) args.push_back(k.args.at(i));
    return k;
  }

  KernelRec temp_kernel(const std::string& name) {
    KernelRec k;
    k.name = name;
    uint8_t kinds[64], classes[64];
    int arity = 0;
    int rc = hcl_kernel_signature("core", name.c_str(), kinds, classes, 64, &arity);
    if (rc != HCL_OK) rc = hcl_kernel_signature("b200", name.c_str(), kinds, classes, 64, &arity);
    if (rc != HCL_OK) fail(ErrorCode::name, "unknown kernel '" + name + "'");
    k.arity = static_cast<uint32_t>(arity);
    k.kinds.assign(kinds, kinds + arity);
    k.classes.assign(classes, classes + arity);
    return k;
  }
};

HostContext::HostContext() : impl_(new Impl) {}
HostContext::HostContext(HostContext&&) noexcept = default;
HostContext& HostContext::operator=(HostContext&&) noexcept = default;
HostContext::~HostContext() {
  if (!impl_) return;
  for (auto& [dev, id] : impl_->mapped) hcl_buffer_release(dev, id);
  for (auto& [id, b] : impl_->buffers)
    for (auto& [g, p] : b.pieces)
      if (p.allocated) hcl_buffer_release(impl_->dev_index(g), id);
}

HostContext HostContext::init(const HostOptions& options) {
  auto started = Clock::now();
  HostContext ctx;
  Impl& impl = *ctx.impl_;
  impl.scheduler.configure(options.scheduler, options.kernel_map);
  int n = 0;
  check(hcl_init(options.cuda_ordinals.empty() ? nullptr : options.cuda_ordinals.data(),
                 static_cast<int>(options.cuda_ordinals.size()), &n));
  std::vector<std::pair<int, DeviceModel>> sched;
  for (int i = 0; i < n; ++i) {
    DeviceEntry e;
    e.global_id = i;
    e.local_index = static_cast<uint32_t>(i);
    e.cuda_ordinal = options.cuda_ordinals.empty() ? i : options.cuda_ordinals[i];
    int type = 1, sms = 0;
    double rel = 1.0;
    uint64_t hbm = 0;
    char name[128];
    check(hcl_device_info(i, &type, &rel, &sms, &hbm, name, sizeof(name)));
    e.name = name;
    e.model = DeviceModel{static_cast<DeviceType>(type), rel};
    impl.device_map.entries.push_back(e);
    sched.emplace_back(i, e.model);
  }
  impl.scheduler.sync_devices(sched);
  impl.timings.init_ms = ms_since(started);
  return ctx;
}

const GlobalDeviceMap& HostContext::device_map() const { return impl_->device_map; }

std::vector<int> HostContext::get_device_ids(std::optional<DeviceType> filter) const {
  std::vector<int> ids;
  for (const auto& e : impl_->device_map.entries)
    if (!filter || e.model.type == *filter) ids.push_back(e.global_id);
  return ids;
}

Handle HostContext::create_queue(int gid, std::string user_id, bool shared) {
  std::lock_guard lock(impl_->mu);
  if (!impl_->device_map.find(gid)) fail(ErrorCode::unknown_device, "device " + std::to_string(gid));
  uint64_t id = impl_->new_id();
  Impl::QueueRec q;
  q.gid = gid;
  q.user = std::move(user_id);
  q.shared = shared;
  impl_->queues.emplace(id, std::move(q));
  return Handle{HandleKind::queue, id};
}

Handle HostContext::create_buffer(uint64_t size) {
  std::lock_guard lock(impl_->mu);
  uint64_t id = impl_->new_id();
  impl_->buffers[id].size = size;
  return Handle{HandleKind::buffer, id};
}

Handle HostContext::create_program(const std::string& bundle) {
  std::lock_guard lock(impl_->mu);
  char names[4096];
  uint32_t arities[256];
  int n = 0;
  impl_->trace.record({0, "query_registry", 0});
  check(hcl_query_registry(bundle.c_str(), names, sizeof(names), arities, 256, &n));
  Impl::ProgramRec p;
  p.bundle = bundle;
  std::string csv = names;
  size_t pos = 0;
  for (int i = 0; i < n; ++i) {
    size_t c = csv.find(',', pos);
    p.kernels.emplace_back(csv.substr(pos, c == std::string::npos ? std::string::npos : c - pos), arities[i]);
    pos = c + 1;
  }
  uint64_t id = impl_->new_id();
  impl_->programs.emplace(id, std::move(p));
  return Handle{HandleKind::program, id};
}

Handle HostContext::create_kernel(Handle program, const std::string& kernel_name) {
  std::lock_guard lock(impl_->mu);
  if (program.kind != HandleKind::program) fail(ErrorCode::handle, "not a program handle");
  auto it = impl_->programs.find(program.id);
  if (it == impl_->programs.end()) fail(ErrorCode::handle, "program handle is released or unknown");
  const auto& ks = it->second.kernels;
  auto e = std::find_if(ks.begin(), ks.end(), [&](const auto& x) { return x.first == kernel_name; });
  if (e == ks.end()) {
    std::string names;
    for (const auto& x : ks) names += (names.empty() ? "" : ", ") + x.first;
    fail(ErrorCode::name, "unknown kernel '" + kernel_name + "' (available: " + names + ")");
  }
  Impl::KernelRec k = impl_->temp_kernel(kernel_name);
  k.program = program.id;
  k.bundle = it->second.bundle;
  uint64_t id = impl_->new_id();
  impl_->kernels.emplace(id, std::move(k));
  return Handle{HandleKind::kernel, id};
}

void HostContext::set_kernel_arg(Handle kernel, uint32_t index, int64_t scalar) {
  std::lock_guard lock(impl_->mu);
  if (kernel.kind != HandleKind::kernel) fail(ErrorCode::handle, "not a kernel handle");
  impl_->kernel(kernel.id).args[index] = Arg::of_i64(scalar);
}

void HostContext::set_kernel_arg(Handle kernel, uint32_t index, Handle buffer) {
  std::lock_guard lock(impl_->mu);
  if (kernel.kind != HandleKind::kernel) fail(ErrorCode::handle, "not a kernel handle");
  if (buffer.kind != HandleKind::buffer) fail(ErrorCode::handle, "argument is not a buffer handle");
  impl_->kernel(kernel.id).args[index] = Arg::of_handle(buffer.id);
}

Handle HostContext::enqueue_write_buffer(Handle queue, Handle buffer, std::span<const uint8_t> data, uint64_t offset,
                                         bool blocking) {
  Range range("hcl:write_buffer");
  int dev = -1;
  Handle ev;
  auto started = Clock::now();
  {
    std::lock_guard lock(impl_->mu);
    Impl::QueueRec& q = impl_->queue(queue.id);
    if (buffer.kind != HandleKind::buffer) fail(ErrorCode::handle, "not a buffer handle");
    Impl::BufferRec& b = impl_->buffer(buffer.id);
    if (offset + data.size() > b.size)
      fail(ErrorCode::size, "write of " + std::to_string(data.size()) + " bytes at offset " + std::to_string(offset) +
                                " into a " + std::to_string(b.size) + "-byte buffer");
    Impl::Piece& p = impl_->ensure_alloc(buffer.id, b, q.gid, offset, data.size());
    if (!data.empty()) {
      impl_->trace.record({q.gid, "write_buffer", buffer.id});
      if (blocking)
        dev = impl_->dev_index(q.gid);  // issued below, off the table lock
      else
        check(hcl_buffer_write_async(impl_->dev_index(q.gid), buffer.id, offset, data.data(), data.size()));
    }
    Impl::set_valid(p, offset, data.size());
    Impl::invalidate_others(b, q.gid, offset, data.size());
    impl_->note_residency(buffer.id, b);
    ev = impl_->new_event();
  }
  // a blocking copy from pageable memory waits for the buffer's earlier users:
  // other threads keep using the context meanwhile
  if (dev >= 0) check(hcl_buffer_write(dev, buffer.id, offset, data.data(), data.size()));
  std::lock_guard lock(impl_->mu);
  auto qi = impl_->queues.find(queue.id);
  impl_->add_transfer(qi == impl_->queues.end() ? nullptr : &qi->second, ms_since(started));
  return ev;
}

void HostContext::enqueue_read_buffer_into(Handle queue, Handle buffer, void* dst, uint64_t offset, uint64_t len,
                                           bool blocking) {
  Range range("hcl:read_buffer");
  struct Copy {
    int dev;
    uint64_t pos, n;
  };
  std::vector<Copy> copies;  // blocking pieces, issued off the table lock
  auto started = Clock::now();
  auto* out = static_cast<uint8_t*>(dst);
  {
    std::lock_guard lock(impl_->mu);
    Impl::QueueRec& q = impl_->queue(queue.id);
    if (buffer.kind != HandleKind::buffer) fail(ErrorCode::handle, "not a buffer handle");
    Impl::BufferRec& b = impl_->buffer(buffer.id);
    if (offset + len > b.size) fail(ErrorCode::size, "read past the end of the buffer");
    uint64_t pos = offset, end = offset + len;
    while (pos < end) {
      int src = -1;
      uint64_t src_end = 0;
      auto qi = b.pieces.find(q.gid);
      if (qi != b.pieces.end() && (src_end = qi->second.valid.holds(pos))) {
        src = q.gid;
      } else {
        for (auto& [g, o] : b.pieces)
          if ((src_end = o.valid.holds(pos))) {
            src = g;
            break;
          }
      }
      if (src < 0) {  // never written: zeros (SPEC design decision; runtime.cpp:496-497)
        uint64_t next = end;
        for (auto& [g, o] : b.pieces) next = std::min(next, o.valid.next_start(pos));
        std::memset(out + (pos - offset), 0, next - pos);
        pos = next;
        continue;
      }
      uint64_t n = std::min(end, src_end) - pos;
      impl_->trace.record({src, "read_buffer", buffer.id});
      if (blocking)
        copies.push_back({impl_->dev_index(src), pos, n});
      else
        check(hcl_buffer_read_async(impl_->dev_index(src), buffer.id, pos, out + (pos - offset), n));
      pos += n;
    }
  }
  for (const Copy& c : copies) check(hcl_buffer_read(c.dev, buffer.id, c.pos, out + (c.pos - offset), c.n));
  std::lock_guard lock(impl_->mu);
  auto qi = impl_->queues.find(queue.id);
  impl_->add_transfer(qi == impl_->queues.end() ? nullptr : &qi->second, ms_since(started));
}

std::vector<uint8_t> HostContext::enqueue_read_buffer(Handle queue, Handle buffer) {
  uint64_t size = buffer_size(buffer);
  std::vector<uint8_t> out(size);
  enqueue_read_buffer_into(queue, buffer, out.data(), 0, size);
  return out;
}

Handle HostContext::enqueue_ndrange_kernel(Handle queue, Handle kernel, std::array<uint64_t, 3> global_size,
                                           uint32_t dims) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  if (kernel.kind != HandleKind::kernel) fail(ErrorCode::handle, "not a kernel handle");
  std::vector<Arg> args;
  Impl::KernelRec& k = impl_->bound_kernel(kernel.id, args);
  for (uint32_t d = 0; d < dims && d < 3; ++d)
    if (global_size[d] < 1) fail(ErrorCode::argument, "global_size extents must be >= 1");
  // the reference carries global_size but runs the kernel whole (daemon.cpp:334)
  return impl_->launch_parts(k, args, global_size, dims, {{q.gid, queue.id, 0, global_size[0]}}, true);
}

std::vector<uint64_t> HostContext::partition_plan(Handle kernel, std::array<uint64_t, 3> global_size,
                                                  const std::vector<Handle>& queues, std::vector<uint64_t> weights) {
  std::lock_guard lock(impl_->mu);
  if (queues.empty()) fail(ErrorCode::argument, "partitioned launch needs at least one queue");
  Impl::KernelRec& k = impl_->kernel(kernel.id);
  if (weights.empty()) {
    std::vector<int> gids;
    for (const Handle& h : queues) gids.push_back(impl_->queue(h.id).gid);
    weights = impl_->scheduler.partition_weights(k.name, gids);
  }
  if (weights.size() != queues.size()) fail(ErrorCode::argument, "one weight per queue");
  return split_ranges(global_size[0], weights);
}

Handle HostContext::enqueue_ndrange_kernel(Handle kernel, std::array<uint64_t, 3> global_size, uint32_t dims,
                                           const std::vector<Handle>& queues, std::vector<uint64_t> weights,
                                           std::vector<uint64_t> bounds) {
  std::lock_guard lock(impl_->mu);
  for (uint32_t d = 0; d < dims && d < 3; ++d)
    if (global_size[d] < 1) fail(ErrorCode::argument, "global_size extents must be >= 1");
  if (bounds.empty()) {
    const bool profiled = weights.empty();
    bounds = partition_plan(kernel, global_size, queues, std::move(weights));
    if (profiled) {
      // Rate-driven split: keep the previous boundaries unless some boundary
      // moves by more than 2% of the range -- EMA noise must not migrate
      // shards between devices on every launch.
      Impl::KernelRec& kr = impl_->kernel(kernel.id);
      std::vector<uint64_t> qids;
      for (const Handle& h : queues) qids.push_back(h.id);
      if (kr.last_queues == qids && kr.last_bounds.size() == bounds.size() && kr.last_bounds.back() == bounds.back()) {
        const uint64_t tol = std::max<uint64_t>(1, global_size[0] / 50);
        bool small = true;
        for (size_t i = 0; i < bounds.size(); ++i) {
          const uint64_t d = bounds[i] > kr.last_bounds[i] ? bounds[i] - kr.last_bounds[i] : kr.last_bounds[i] - bounds[i];
          if (d > tol) small = false;
        }
        if (small) bounds = kr.last_bounds;
      }
      kr.last_bounds = bounds;
      kr.last_queues = qids;
    }
  } else {
    if (bounds.size() != queues.size() + 1 || bounds.front() != 0 || bounds.back() != global_size[0])
      fail(ErrorCode::argument, "bounds must hold parts+1 boundaries from 0 to global_size[0]");
    for (size_t i = 0; i + 1 < bounds.size(); ++i)
      if (bounds[i] > bounds[i + 1]) fail(ErrorCode::argument, "bounds must be nondecreasing");
  }
  std::vector<Arg> args;
  Impl::KernelRec& k = impl_->bound_kernel(kernel.id, args);
  std::vector<Impl::Part> parts;
  for (size_t i = 0; i < queues.size(); ++i)
    parts.push_back({impl_->queue(queues[i].id).gid, queues[i].id, bounds[i], bounds[i + 1]});
  return impl_->launch_parts(k, args, global_size, dims, parts, false);
}

Handle HostContext::enqueue_ndrange_range(Handle queue, Handle kernel, std::array<uint64_t, 3> global_size,
                                          uint32_t dims, uint64_t row_offset, uint64_t rows) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  for (uint32_t d = 0; d < dims && d < 3; ++d)
    if (global_size[d] < 1) fail(ErrorCode::argument, "global_size extents must be >= 1");
  if (row_offset + rows > global_size[0]) fail(ErrorCode::argument, "sub-range exceeds the global range");
  std::vector<Arg> args;
  Impl::KernelRec& k = impl_->bound_kernel(kernel.id, args);
  return impl_->launch_parts(k, args, global_size, dims, {{q.gid, queue.id, row_offset, row_offset + rows}}, false);
}

}  // namespace haocl

extern "C" {
int hcl_nccl_init(int dev, int nranks, int rank, const uint8_t* id_bytes);
int hcl_allgatherv(int dev, uint64_t buffer_id, const uint64_t* bounds);
int hcl_allreduce_sum_i64(int dev, uint64_t buffer_id, uint64_t offset, uint64_t count);
int hcl_broadcast(int dev, uint64_t buffer_id, uint64_t offset, uint64_t bytes, int root);
}

namespace haocl {

void HostContext::init_collectives(Handle queue, int rank, int nranks, const std::vector<uint8_t>& id) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  if (id.size() < 128) fail(ErrorCode::argument, "NCCL unique id is 128 bytes");
  check(hcl_nccl_init(impl_->dev_index(q.gid), nranks, rank, id.data()));
}

void HostContext::enqueue_allgather(Handle queue, Handle buffer, const std::vector<uint64_t>& bounds) {
  Range range("hcl:allgather");
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::BufferRec& b = impl_->buffer(buffer.id);
  if (bounds.size() < 2 || bounds.back() > b.size) fail(ErrorCode::argument, "allgather bounds exceed the buffer");
  auto started = Clock::now();
  Impl::Piece& p = impl_->ensure_alloc(buffer.id, b, q.gid, bounds.front(), bounds.back() - bounds.front());
  impl_->trace.record({q.gid, "allgather", buffer.id});
  check(hcl_allgatherv(impl_->dev_index(q.gid), buffer.id, bounds.data()));
  Impl::set_valid(p, bounds.front(), bounds.back() - bounds.front());
  impl_->add_transfer(&q, ms_since(started));
}

std::vector<uint8_t> HostContext::share_buffer(Handle queue, Handle buffer) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::BufferRec& b = impl_->buffer(buffer.id);
  std::vector<uint8_t> h(64);
  check(hcl_buffer_alloc_shared(impl_->dev_index(q.gid), buffer.id, b.size, h.data()));
  Impl::Piece& p = b.pieces[q.gid];  // zero-filled, whole buffer, nothing written yet
  p.allocated = true;
  p.alloc_first = 0;
  p.alloc_bytes = b.size;
  p.valid.clear();
  impl_->trace.record({q.gid, "alloc_buffer", buffer.id});
  return h;
}

void HostContext::bind_external(Handle queue, Handle buffer, uint64_t device_ptr) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::BufferRec& b = impl_->buffer(buffer.id);
  if (!device_ptr) fail(ErrorCode::argument, "bind_external: null device pointer");
  check(hcl_buffer_bind_external(impl_->dev_index(q.gid), buffer.id, reinterpret_cast<void*>(device_ptr), 0, b.size));
  Impl::Piece& p = b.pieces[q.gid];
  p.allocated = true;
  p.alloc_first = 0;
  p.alloc_bytes = b.size;
  p.valid.clear();
  impl_->trace.record({q.gid, "alloc_buffer", buffer.id});
}

uint64_t HostContext::open_shared_buffer(Handle queue, const std::vector<uint8_t>& ipc_handle, uint64_t bytes) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  if (ipc_handle.size() < 64) fail(ErrorCode::argument, "open_shared_buffer: IPC handles are 64 bytes");
  const int dev = impl_->dev_index(q.gid);
  const uint64_t id = impl_->new_id() | (1ull << 61);  // device-level mapping, outside the buffer table
  check(hcl_buffer_open_shared(dev, id, ipc_handle.data(), bytes));
  impl_->mapped.push_back({dev, id});
  void* p = nullptr;
  check(hcl_buffer_device_ptr(dev, id, &p, nullptr, nullptr));
  return reinterpret_cast<uint64_t>(p);
}

void HostContext::enqueue_barrier(Handle queue, const std::vector<Handle>& completed) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  impl_->trace.record({q.gid, "barrier", 0});
  check(hcl_nccl_barrier(impl_->dev_index(q.gid)));
  for (const Handle& h : completed) {
    Impl::BufferRec& b = impl_->buffer(h.id);
    Impl::Piece& p = impl_->ensure_alloc(h.id, b, q.gid, 0, b.size);
    Impl::set_valid(p, 0, b.size);
    Impl::invalidate_others(b, q.gid, 0, b.size);
  }
}

void HostContext::enqueue_allreduce_sum_i64(Handle queue, Handle buffer) {
  Range range("hcl:allreduce");
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::BufferRec& b = impl_->buffer(buffer.id);
  impl_->ensure_valid(buffer.id, b, q.gid, 0, b.size, &q);
  impl_->trace.record({q.gid, "allreduce", buffer.id});
  check(hcl_allreduce_sum_i64(impl_->dev_index(q.gid), buffer.id, 0, b.size / 8));
}

void HostContext::enqueue_broadcast(Handle queue, Handle buffer, int root) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::BufferRec& b = impl_->buffer(buffer.id);
  Impl::Piece& p = impl_->ensure_alloc(buffer.id, b, q.gid, 0, b.size);
  impl_->trace.record({q.gid, "broadcast", buffer.id});
  check(hcl_broadcast(impl_->dev_index(q.gid), buffer.id, 0, b.size, root));
  p.valid.clear();
  p.valid.add(0, b.size);
}

std::pair<int, Handle> HostContext::submit_task(const KernelTask& task) {
  std::lock_guard lock(impl_->mu);
  Impl::KernelRec k = impl_->temp_kernel(task.kernel_name);
  if (task.args.size() != k.arity)
    fail(ErrorCode::argument, task.kernel_name + ": expected " + std::to_string(k.arity) + " bound arguments");
  if (task.placement.mode == Placement::Mode::auto_policy && !impl_->scheduler.has_policy(task.placement.policy))
    fail(ErrorCode::policy, "unknown policy '" + task.placement.policy + "'");
  TaskEstimate est;
  double work = 1.0;
  for (size_t i = 0; i < task.args.size(); ++i)
    if (task.args[i].is_buffer) {
      uint64_t size = impl_->buffer(task.args[i].buffer).size;
      (k.kinds[i] == HCL_ARG_OUT ? est.out_bytes : est.in_bytes) += size;
    }
  // work estimate: the reference's formulas (kernels.cpp:285-298) where they apply
  std::vector<int64_t> sc;
  for (const auto& a : task.args)
    if (!a.is_buffer) sc.push_back(a.scalar);
  if ((task.kernel_name == "matmul" || task.kernel_name.rfind("gemm", 0) == 0) && sc.size() >= 3)
    work = 2.0 * sc[0] * sc[1] * sc[2];
  else if (task.kernel_name == "vecadd" && !sc.empty())
    work = static_cast<double>(sc[0]);
  else if (task.kernel_name == "knn" && sc.size() >= 3)
    work = static_cast<double>(sc[2]) * sc[0] * sc[1];
  est.work_units = work;
  int chosen = impl_->scheduler.schedule(task, est);
  uint64_t qid;
  auto it = impl_->internal_queues.find(chosen);
  if (it != impl_->internal_queues.end()) {
    qid = it->second;
  } else {
    qid = create_queue(chosen).id;
    impl_->internal_queues[chosen] = qid;
  }
  Handle ev = impl_->launch_parts(k, task.args, task.global_size, task.dims, {{chosen, qid, 0, task.global_size[0]}}, true);
  return {chosen, ev};
}

Handle HostContext::launch_task(Handle queue, const KernelTask& task) {
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  Impl::KernelRec k = impl_->temp_kernel(task.kernel_name);
  if (task.args.size() != k.arity)
    fail(ErrorCode::argument, task.kernel_name + ": expected " + std::to_string(k.arity) + " bound arguments");
  return impl_->launch_parts(k, task.args, task.global_size, task.dims, {{q.gid, queue.id, 0, task.global_size[0]}}, true);
}

TimingFragment HostContext::finish(Handle queue) {
  Range range("hcl:finish");
  std::shared_ptr<std::mutex> op;
  {
    std::lock_guard lock(impl_->mu);
    op = impl_->queue(queue.id).op_mu;
  }
  std::lock_guard serial(*op);  // one finish per queue at a time
  std::vector<Impl::Launch> done;
  int dev = 0;
  {
    std::lock_guard lock(impl_->mu);
    Impl::QueueRec& q = impl_->queue(queue.id);
    dev = impl_->dev_index(q.gid);
    done.swap(q.pending);
  }
  // device synchronization without the table lock: other queues keep enqueueing
  check(hcl_finish(dev, nullptr));
  std::vector<float> ms(done.size(), 0.f);
  for (size_t i = 0; i < done.size(); ++i) {
    cudaEventSynchronize(done[i].stop);
    cudaEventElapsedTime(&ms[i], done[i].start, done[i].stop);
    cudaEventDestroy(done[i].start);
    cudaEventDestroy(done[i].stop);
  }
  std::lock_guard lock(impl_->mu);
  Impl::QueueRec& q = impl_->queue(queue.id);
  for (size_t i = 0; i < done.size(); ++i) {
    const Impl::Launch& l = done[i];
    q.compute_ms += ms[i];
    const DeviceEntry* e = impl_->device_map.find(l.gid);
    double modeled = static_cast<double>(l.work) /
                     ((e ? e->model.relative_throughput : 1.0) * impl_->scheduler.options().baseline_rate) * 1000.0;
    q.modeled_ms += modeled;
    {
      std::lock_guard lb(impl_->breakdown_mu);
      impl_->timings.compute_ms += ms[i];
      impl_->timings.modeled_compute_ms += modeled;
    }
    if (ms[i] > 0.f && l.work > 0)
      impl_->scheduler.record_profile(l.gid, l.kernel, static_cast<double>(l.work), ms[i] / 1000.0);
  }
  TimingFragment f{q.transfer_ms, q.compute_ms, q.modeled_ms};
  q.transfer_ms = q.compute_ms = q.modeled_ms = 0.0;
  return f;
}

void HostContext::release(Handle h) {
  std::lock_guard lock(impl_->mu);
  switch (h.kind) {
    case HandleKind::buffer: {
      Impl::BufferRec& b = impl_->buffer(h.id);
      for (auto& [g, p] : b.pieces)
        if (p.allocated) {
          impl_->trace.record({g, "release_object", h.id});
          check(hcl_buffer_release(impl_->dev_index(g), h.id));
        }
      impl_->buffers.erase(h.id);
      impl_->scheduler.drop_resident(h.id);
      return;
    }
    case HandleKind::queue: {
      Impl::QueueRec& q = impl_->queue(h.id);
      if (!q.pending.empty()) check(hcl_finish(impl_->dev_index(q.gid), nullptr));
      for (auto& l : q.pending) {
        cudaEventDestroy(l.start);
        cudaEventDestroy(l.stop);
      }
      for (auto it = impl_->internal_queues.begin(); it != impl_->internal_queues.end();)
        it = it->second == h.id ? impl_->internal_queues.erase(it) : std::next(it);
      impl_->queues.erase(h.id);
      return;
    }
    case HandleKind::program:
      if (!impl_->programs.erase(h.id)) fail(ErrorCode::handle, "program handle is released or unknown");
      return;
    case HandleKind::kernel:
      if (!impl_->kernels.erase(h.id)) fail(ErrorCode::handle, "kernel handle is released or unknown");
      return;
    case HandleKind::event:
      if (!impl_->events.erase(h.id)) fail(ErrorCode::handle, "event handle is released or unknown");
      return;
    case HandleKind::context:
      fail(ErrorCode::handle, "the context is not a releasable handle");
  }
}

TimingBreakdown HostContext::breakdown() const {
  std::lock_guard lock(impl_->breakdown_mu);
  return impl_->timings;
}

void HostContext::add_data_creation_ms(double ms) {
  std::lock_guard lock(impl_->breakdown_mu);
  impl_->timings.data_creation_ms += ms;
}

MessageTrace& HostContext::trace() { return impl_->trace; }
Scheduler& HostContext::scheduler() { return impl_->scheduler; }

void HostContext::set_device_sm_budget(int gid, int sms) {
  std::lock_guard lock(impl_->mu);
  const int dev = impl_->dev_index(gid);
  check(hcl_device_set_sm_budget(dev, sms));
  double rel = 1.0;
  check(hcl_device_info(dev, nullptr, &rel, nullptr, nullptr, nullptr, 0));
  auto st = impl_->scheduler.snapshot();
  std::vector<std::pair<int, DeviceModel>> devs;
  for (auto& d : st.devices)
    devs.push_back({d.global_id, d.global_id == gid ? DeviceModel{d.model.type, rel} : d.model});
  impl_->scheduler.sync_devices(devs);
}

uint64_t HostContext::buffer_size(Handle buffer) const {
  std::lock_guard lock(impl_->mu);
  if (buffer.kind != HandleKind::buffer) fail(ErrorCode::handle, "not a buffer handle");
  return impl_->buffer(buffer.id).size;
}

int HostContext::queue_device(Handle queue) const {
  std::lock_guard lock(impl_->mu);
  return impl_->queue(queue.id).gid;
}

void* HostContext::buffer_device_ptr(Handle buffer, int gid, uint64_t* first_byte, uint64_t* bytes) const {
  std::lock_guard lock(impl_->mu);
  impl_->buffer(buffer.id);
  void* p = nullptr;
  check(hcl_buffer_device_ptr(impl_->dev_index(gid), buffer.id, &p, first_byte, bytes));
  return p;
}

}  // namespace haocl

// ---------------------------------------------------------------------------
// C entry points (include/hcl_host.h)

struct hcl_context {
  haocl::HostContext ctx;
};

namespace {
template <typename F>
int ctx_guarded(F&& f) {
  try {
    f();
    return HCL_OK;
  } catch (const haocl::Error& e) {
    hcl::set_last_error(e.what());
    return HCL_ERR_BASE + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    hcl::set_last_error(std::string("internal: ") + e.what());
    return HCL_ERR_BASE;
  }
}
using haocl::Handle;
using haocl::HandleKind;
Handle H(HandleKind k, uint64_t id) { return Handle{k, id}; }
}  // namespace

extern "C" {

int hcl_ctx_init(const int* ordinals, int n, const hcl_scheduler_options* opts, hcl_context** out) {
  return ctx_guarded([&] {
    haocl::HostOptions o;
    if (ordinals && n > 0) o.cuda_ordinals.assign(ordinals, ordinals + n);
    if (opts) {
      o.scheduler.baseline_rate = opts->baseline_rate;
      o.scheduler.net_bandwidth = opts->net_bandwidth;
      o.scheduler.ema_alpha = opts->ema_alpha;
    }
    *out = new hcl_context{haocl::HostContext::init(o)};
  });
}

int hcl_ctx_destroy(hcl_context* ctx) {
  delete ctx;
  return HCL_OK;
}

int hcl_ctx_get_device_ids(hcl_context* ctx, int* ids, int cap, int* n) {
  return ctx_guarded([&] {
    auto v = ctx->ctx.get_device_ids();
    *n = static_cast<int>(v.size());
    for (int i = 0; i < *n && i < cap; ++i) ids[i] = v[i];
  });
}

int hcl_ctx_create_queue(hcl_context* ctx, int gid, const char* user, int shared, uint64_t* queue) {
  return ctx_guarded([&] { *queue = ctx->ctx.create_queue(gid, user ? user : "default", shared != 0).id; });
}
int hcl_ctx_create_buffer(hcl_context* ctx, uint64_t size, uint64_t* buffer) {
  return ctx_guarded([&] { *buffer = ctx->ctx.create_buffer(size).id; });
}
int hcl_ctx_create_program(hcl_context* ctx, const char* bundle, uint64_t* program) {
  return ctx_guarded([&] { *program = ctx->ctx.create_program(bundle).id; });
}
int hcl_ctx_create_kernel(hcl_context* ctx, uint64_t program, const char* name, uint64_t* kernel) {
  return ctx_guarded([&] { *kernel = ctx->ctx.create_kernel(H(HandleKind::program, program), name).id; });
}
int hcl_ctx_set_kernel_arg_i64(hcl_context* ctx, uint64_t kernel, uint32_t index, int64_t value) {
  return ctx_guarded([&] { ctx->ctx.set_kernel_arg(H(HandleKind::kernel, kernel), index, value); });
}
int hcl_ctx_set_kernel_arg_buffer(hcl_context* ctx, uint64_t kernel, uint32_t index, uint64_t buffer) {
  return ctx_guarded([&] { ctx->ctx.set_kernel_arg(H(HandleKind::kernel, kernel), index, H(HandleKind::buffer, buffer)); });
}
int hcl_ctx_enqueue_write_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, const void* data, uint64_t len,
                                 uint64_t offset, uint64_t* event) {
  return ctx_guarded([&] {
    auto ev = ctx->ctx.enqueue_write_buffer(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer),
                                            std::span<const uint8_t>(static_cast<const uint8_t*>(data), len), offset);
    if (event) *event = ev.id;
  });
}
int hcl_ctx_enqueue_read_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, void* dst, uint64_t offset,
                                uint64_t len) {
  return ctx_guarded([&] {
    ctx->ctx.enqueue_read_buffer_into(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer), dst, offset, len);
  });
}
int hcl_ctx_enqueue_write_buffer_async(hcl_context* ctx, uint64_t queue, uint64_t buffer, const void* data,
                                       uint64_t len, uint64_t offset, uint64_t* event) {
  return ctx_guarded([&] {
    auto ev = ctx->ctx.enqueue_write_buffer(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer),
                                            std::span<const uint8_t>(static_cast<const uint8_t*>(data), len), offset,
                                            false);
    if (event) *event = ev.id;
  });
}
int hcl_ctx_enqueue_read_buffer_async(hcl_context* ctx, uint64_t queue, uint64_t buffer, void* dst, uint64_t offset,
                                      uint64_t len) {
  return ctx_guarded([&] {
    ctx->ctx.enqueue_read_buffer_into(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer), dst, offset, len,
                                      false);
  });
}
int hcl_ctx_enqueue_ndrange_kernel(hcl_context* ctx, uint64_t queue, uint64_t kernel, const uint64_t global[3],
                                   uint32_t dims, uint64_t* event) {
  return ctx_guarded([&] {
    std::array<uint64_t, 3> g = {1, 1, 1};
    if (global) g = {global[0], global[1], global[2]};
    auto ev = ctx->ctx.enqueue_ndrange_kernel(H(HandleKind::queue, queue), H(HandleKind::kernel, kernel), g, dims);
    if (event) *event = ev.id;
  });
}
int hcl_ctx_enqueue_ndrange_partitioned(hcl_context* ctx, uint64_t kernel, const uint64_t global[3], uint32_t dims,
                                        const uint64_t* queues, int nqueues, const uint64_t* weights,
                                        const uint64_t* bounds, uint64_t* event) {
  return ctx_guarded([&] {
    std::vector<Handle> qs;
    for (int i = 0; i < nqueues; ++i) qs.push_back(H(HandleKind::queue, queues[i]));
    std::vector<uint64_t> w, b;
    if (weights) w.assign(weights, weights + nqueues);
    if (bounds) b.assign(bounds, bounds + nqueues + 1);
    auto ev = ctx->ctx.enqueue_ndrange_kernel(H(HandleKind::kernel, kernel), {global[0], global[1], global[2]}, dims,
                                              qs, w, b);
    if (event) *event = ev.id;
  });
}
int hcl_ctx_enqueue_ndrange_range(hcl_context* ctx, uint64_t queue, uint64_t kernel, const uint64_t global[3],
                                  uint32_t dims, uint64_t row_offset, uint64_t rows, uint64_t* event) {
  return ctx_guarded([&] {
    auto ev = ctx->ctx.enqueue_ndrange_range(H(HandleKind::queue, queue), H(HandleKind::kernel, kernel),
                                             {global[0], global[1], global[2]}, dims, row_offset, rows);
    if (event) *event = ev.id;
  });
}
int hcl_ctx_init_collectives(hcl_context* ctx, uint64_t queue, int rank, int nranks, const uint8_t* id) {
  return ctx_guarded([&] {
    ctx->ctx.init_collectives(H(HandleKind::queue, queue), rank, nranks, std::vector<uint8_t>(id, id + 128));
  });
}
int hcl_ctx_enqueue_allgather(hcl_context* ctx, uint64_t queue, uint64_t buffer, const uint64_t* bounds,
                              int nranks) {
  return ctx_guarded([&] {
    ctx->ctx.enqueue_allgather(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer),
                               std::vector<uint64_t>(bounds, bounds + nranks + 1));
  });
}
int hcl_ctx_enqueue_allreduce_sum_i64(hcl_context* ctx, uint64_t queue, uint64_t buffer) {
  return ctx_guarded([&] { ctx->ctx.enqueue_allreduce_sum_i64(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer)); });
}
int hcl_ctx_share_buffer(hcl_context* ctx, uint64_t queue, uint64_t buffer, uint8_t* ipc_handle) {
  return ctx_guarded([&] {
    auto h = ctx->ctx.share_buffer(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer));
    std::memcpy(ipc_handle, h.data(), h.size());
  });
}
int hcl_ctx_open_shared_buffer(hcl_context* ctx, uint64_t queue, const uint8_t* ipc_handle, uint64_t bytes,
                               uint64_t* device_address) {
  return ctx_guarded([&] {
    *device_address = ctx->ctx.open_shared_buffer(H(HandleKind::queue, queue),
                                                  std::vector<uint8_t>(ipc_handle, ipc_handle + 64), bytes);
  });
}
int hcl_ctx_bind_external(hcl_context* ctx, uint64_t queue, uint64_t buffer, uint64_t device_ptr) {
  return ctx_guarded([&] {
    ctx->ctx.bind_external(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer), device_ptr);
  });
}
int hcl_ctx_enqueue_barrier(hcl_context* ctx, uint64_t queue, const uint64_t* completed, int n) {
  return ctx_guarded([&] {
    std::vector<Handle> bs;
    for (int i = 0; i < n; ++i) bs.push_back(H(HandleKind::buffer, completed[i]));
    ctx->ctx.enqueue_barrier(H(HandleKind::queue, queue), bs);
  });
}
int hcl_ctx_enqueue_broadcast(hcl_context* ctx, uint64_t queue, uint64_t buffer, int root) {
  return ctx_guarded([&] { ctx->ctx.enqueue_broadcast(H(HandleKind::queue, queue), H(HandleKind::buffer, buffer), root); });
}
int hcl_ctx_partition_plan(hcl_context* ctx, uint64_t kernel, const uint64_t global[3], const uint64_t* queues,
                           int nqueues, const uint64_t* weights, uint64_t* bounds) {
  return ctx_guarded([&] {
    std::vector<Handle> qs;
    for (int i = 0; i < nqueues; ++i) qs.push_back(H(HandleKind::queue, queues[i]));
    std::vector<uint64_t> w;
    if (weights) w.assign(weights, weights + nqueues);
    auto b = ctx->ctx.partition_plan(H(HandleKind::kernel, kernel), {global[0], global[1], global[2]}, qs, w);
    std::memcpy(bounds, b.data(), b.size() * sizeof(uint64_t));
  });
}
int hcl_ctx_submit_task(hcl_context* ctx, const char* kernel, const uint8_t* is_buffer, const int64_t* values,
                        int nargs, const char* policy, int explicit_device, int* chosen, uint64_t* event) {
  return ctx_guarded([&] {
    haocl::KernelTask t;
    t.kernel_name = kernel;
    for (int i = 0; i < nargs; ++i)
      t.args.push_back(is_buffer[i] ? haocl::Arg::of_handle(static_cast<uint64_t>(values[i])) : haocl::Arg::of_i64(values[i]));
    t.placement = (policy && *policy) ? haocl::Placement::auto_with(policy) : haocl::Placement::explicit_on(explicit_device);
    auto [c, ev] = ctx->ctx.submit_task(t);
    if (chosen) *chosen = c;
    if (event) *event = ev.id;
  });
}
int hcl_ctx_finish(hcl_context* ctx, uint64_t queue, double* transfer_ms, double* compute_ms, double* modeled_ms) {
  return ctx_guarded([&] {
    auto f = ctx->ctx.finish(H(HandleKind::queue, queue));
    if (transfer_ms) *transfer_ms = f.transfer_ms;
    if (compute_ms) *compute_ms = f.compute_ms;
    if (modeled_ms) *modeled_ms = f.modeled_ms;
  });
}
int hcl_ctx_release(hcl_context* ctx, uint8_t kind, uint64_t id) {
  return ctx_guarded([&] { ctx->ctx.release(H(static_cast<HandleKind>(kind), id)); });
}
int hcl_ctx_breakdown(hcl_context* ctx, double out[5]) {
  return ctx_guarded([&] {
    auto b = ctx->ctx.breakdown();
    out[0] = b.init_ms;
    out[1] = b.data_creation_ms;
    out[2] = b.transfer_ms;
    out[3] = b.compute_ms;
    out[4] = b.modeled_compute_ms;
  });
}
int hcl_ctx_add_data_creation_ms(hcl_context* ctx, double ms) {
  return ctx_guarded([&] { ctx->ctx.add_data_creation_ms(ms); });
}
int hcl_ctx_buffer_size(hcl_context* ctx, uint64_t buffer, uint64_t* size) {
  return ctx_guarded([&] { *size = ctx->ctx.buffer_size(H(HandleKind::buffer, buffer)); });
}
int hcl_ctx_buffer_device_ptr(hcl_context* ctx, uint64_t buffer, int gid, void** ptr, uint64_t* first_byte,
                              uint64_t* bytes) {
  return ctx_guarded([&] { *ptr = ctx->ctx.buffer_device_ptr(H(HandleKind::buffer, buffer), gid, first_byte, bytes); });
}
int hcl_ctx_trace_count(hcl_context* ctx, const char* function, int device, uint64_t* count) {
  return ctx_guarded([&] { *count = ctx->ctx.trace().count_calls(function, device); });
}
int hcl_ctx_trace_clear(hcl_context* ctx) {
  return ctx_guarded([&] { ctx->ctx.trace().clear(); });
}
int hcl_ctx_sched_record_profile(hcl_context* ctx, int gid, const char* kernel, double work, double seconds) {
  return ctx_guarded([&] { ctx->ctx.scheduler().record_profile(gid, kernel, work, seconds); });
}
int hcl_ctx_sched_rate(hcl_context* ctx, int gid, const char* kernel, double* rate) {
  return ctx_guarded([&] {
    auto st = ctx->ctx.scheduler().snapshot();
    const auto* d = st.find(gid);
    if (!d) throw haocl::Error(haocl::ErrorCode::unknown_device, "device " + std::to_string(gid));
    auto it = d->profiled_rate.find(kernel);
    *rate = it == d->profiled_rate.end() ? 0.0 : it->second;
  });
}
int hcl_ctx_sched_schedule(hcl_context* ctx, const char* kernel, const char* policy, int explicit_device,
                           double work, uint64_t in_bytes, uint64_t out_bytes, int* chosen) {
  return ctx_guarded([&] {
    haocl::KernelTask t;
    t.kernel_name = kernel;
    t.placement = (policy && *policy) ? haocl::Placement::auto_with(policy) : haocl::Placement::explicit_on(explicit_device);
    *chosen = ctx->ctx.scheduler().schedule(t, haocl::TaskEstimate{work, in_bytes, out_bytes});
  });
}
int hcl_ctx_sched_save_profiles(hcl_context* ctx, const char* path) {
  return ctx_guarded([&] {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw haocl::Error(haocl::ErrorCode::argument, std::string("cannot write ") + path);
    const std::string t = ctx->ctx.scheduler().export_profiles();
    const bool ok = std::fwrite(t.data(), 1, t.size(), f) == t.size();
    std::fclose(f);
    if (!ok) throw haocl::Error(haocl::ErrorCode::argument, std::string("short write to ") + path);
  });
}
int hcl_ctx_sched_load_profiles(hcl_context* ctx, const char* path, int* loaded) {
  return ctx_guarded([&] {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw haocl::Error(haocl::ErrorCode::argument, std::string("cannot read ") + path);
    std::string t;
    char buf[4096];
    for (size_t n; (n = std::fread(buf, 1, sizeof buf, f)) > 0;) t.append(buf, n);
    std::fclose(f);
    const size_t n = ctx->ctx.scheduler().import_profiles(t);
    if (loaded) *loaded = static_cast<int>(n);
  });
}
int hcl_ctx_set_sm_budget(hcl_context* ctx, int gid, int sms) {
  return ctx_guarded([&] { ctx->ctx.set_device_sm_budget(gid, sms); });
}
int hcl_ctx_sched_set_model(hcl_context* ctx, int gid, double relative_throughput) {
  return ctx_guarded([&] {
    auto st = ctx->ctx.scheduler().snapshot();
    std::vector<std::pair<int, haocl::DeviceModel>> devs;
    for (auto& d : st.devices)
      devs.push_back({d.global_id, d.global_id == gid ? haocl::DeviceModel{d.model.type, relative_throughput} : d.model});
    ctx->ctx.scheduler().sync_devices(devs);
  });
}
int hcl_ctx_sched_partition_weights(hcl_context* ctx, const char* kernel, const int* gids, int n, uint64_t* weights) {
  return ctx_guarded([&] {
    auto w = ctx->ctx.scheduler().partition_weights(kernel, std::vector<int>(gids, gids + n));
    std::memcpy(weights, w.data(), w.size() * sizeof(uint64_t));
  });
}

}  // extern "C"
