// Node daemon: the reference's remote-node path in front
// of the C-ABI. It speaks the HaoCL wire protocol the reference host runtime
// uses (HCL1 frames, proj/include/haocl/wire.hpp:6-13; one TCP port for
// messages and message+1 for data, proj/include/haocl/net.hpp:1-6), so an
// unmodified reference HostContext can drive this box's B200s:
//
//   Ping -> Pong                               (connection handshake, net.cpp)
//   DeviceIdRequest -> DeviceIdResponse       (the logical devices of hcl_init)
//   DataTransfer chunks -> DataAck            (reassembly with overlap check,
//                                              proj/src/daemon.cpp:21-69)
//   ApiCallRequest alloc_buffer / read_buffer / release_object /
//                  query_registry / launch_kernel      (daemon.cpp:159-352)
//   Shutdown                                   (drain and stop)
//
// The B200 difference is where buffers live: the reference daemon keeps every
// buffer as host bytes and copies each input into the kernel call
// (daemon.cpp:313). Here a buffer's bytes stay resident in HBM on the device
// that last wrote it; host bytes are materialised only when the host reads
// the buffer back, inputs move between GPUs with NVLink peer copies, and
// repeated launches on one device re-use the resident copy.
//
// Errors travel as ErrorReply{code, message} with the reference's ErrorCode
// numbering (error.hpp:11-36); C-ABI failures map rc - HCL_ERR_BASE.

#include <arpa/inet.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <poll.h>
#include <sys/socket.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <bit>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/hcl_cabi.h"
#include "../common.hpp"

namespace hcl {
void set_last_error(const std::string& m);
namespace {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return HCL_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return HCL_ERR_BASE + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    set_last_error(std::string("internal: ") + e.what());
    return HCL_ERR_BASE;
  }
}

// ---- wire codec (big-endian, HCL1) ----------------------------------------

enum Kind : uint8_t {
  kApiCallRequest = 1,
  kApiCallResponse = 2,
  kDeviceIdRequest = 3,
  kDeviceIdResponse = 4,
  kDataTransfer = 5,
  kDataAck = 6,
  kErrorReply = 7,
  kPing = 8,
  kPong = 9,
  kShutdown = 10,
};
enum Tag : uint8_t { kI32 = 1, kI64 = 2, kF32 = 3, kF64 = 4, kBytes = 5, kString = 6, kHandle = 7 };
constexpr size_t kHeader = 18;  // magic 4, version 1, kind 1, call_id 8, len 4
constexpr uint8_t kVersion = 1;

// ErrorCode values of the wire contract (proj/include/haocl/error.hpp:11-36)
enum Code : uint16_t {
  kInternal = 0, kProtocol = 1, kVersionErr = 2, kMalformed = 3, kEncoding = 4, kUnknownCall = 5,
  kPrecondition = 7, kReassembly = 8, kArgument = 9, kName = 10, kSizeErr = 18, kUnknownDevice = 20,
};

struct WireError {
  uint16_t code;
  std::string msg;
};
[[noreturn]] void werr(uint16_t code, std::string msg) { throw WireError{code, std::move(msg)}; }

struct Value {
  uint8_t tag = kI32;
  int64_t i = 0;        // i32, i64, handle (as bits)
  double f = 0.0;       // f32, f64
  std::string s;        // bytes, string
};

class Out {
 public:
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void u16(uint16_t v) { u8(v >> 8), u8(v & 0xff); }
  void u32(uint32_t v) {
    for (int sh = 24; sh >= 0; sh -= 8) u8(static_cast<uint8_t>(v >> sh));
  }
  void u64(uint64_t v) {
    for (int sh = 56; sh >= 0; sh -= 8) u8(static_cast<uint8_t>(v >> sh));
  }
  void blob(const void* p, size_t n) {
    if (n > 0xffffffffull) werr(kEncoding, "blob exceeds 32-bit length prefix");
    u32(static_cast<uint32_t>(n));
    const uint8_t* c = static_cast<const uint8_t*>(p);
    b.insert(b.end(), c, c + n);
  }
  void value(const Value& v) {
    u8(v.tag);
    switch (v.tag) {
      case kI32: u32(static_cast<uint32_t>(static_cast<int32_t>(v.i))); break;
      case kI64: case kHandle: u64(static_cast<uint64_t>(v.i)); break;
      case kF32: u32(std::bit_cast<uint32_t>(static_cast<float>(v.f))); break;
      case kF64: u64(std::bit_cast<uint64_t>(v.f)); break;
      default: blob(v.s.data(), v.s.size()); break;
    }
  }
};

class In {
 public:
  In(const uint8_t* p, size_t n) : p_(p), n_(n) {}
  const uint8_t* take(size_t k) {
    if (k > n_ - at_) werr(kMalformed, "body truncated");
    const uint8_t* r = p_ + at_;
    at_ += k;
    return r;
  }
  uint8_t u8() { return *take(1); }
  uint32_t u32() {
    const uint8_t* q = take(4);
    return (uint32_t(q[0]) << 24) | (uint32_t(q[1]) << 16) | (uint32_t(q[2]) << 8) | q[3];
  }
  uint64_t u64() {
    const uint8_t* q = take(8);
    uint64_t v = 0;
    for (int k = 0; k < 8; ++k) v = (v << 8) | q[k];
    return v;
  }
  std::string str() {
    const uint32_t k = u32();
    const uint8_t* q = take(k);
    return std::string(reinterpret_cast<const char*>(q), k);
  }
  Value value() {
    Value v;
    v.tag = u8();
    switch (v.tag) {
      case kI32: v.i = static_cast<int32_t>(u32()); break;
      case kI64: case kHandle: v.i = static_cast<int64_t>(u64()); break;
      case kF32: v.f = std::bit_cast<float>(u32()); break;
      case kF64: v.f = std::bit_cast<double>(u64()); break;
      case kBytes: case kString: v.s = str(); break;
      default: werr(kMalformed, "unknown value tag " + std::to_string(v.tag));
    }
    return v;
  }
  size_t left() const { return n_ - at_; }
  const uint8_t* here() const { return p_ + at_; }

 private:
  const uint8_t* p_;
  size_t n_, at_ = 0;
};

struct Frame {
  uint8_t kind = 0;
  uint64_t call_id = 0;
  std::vector<uint8_t> body;
};

std::vector<uint8_t> encode(uint8_t kind, uint64_t call_id, const std::vector<uint8_t>& body) {
  if (body.size() > 0xffffffffull) werr(kEncoding, "body exceeds the 4-byte length field");
  Out o;
  o.b.reserve(kHeader + body.size());
  for (char c : {'H', 'C', 'L', '1'}) o.u8(static_cast<uint8_t>(c));
  o.u8(kVersion);
  o.u8(kind);
  o.u64(call_id);
  o.u32(static_cast<uint32_t>(body.size()));
  o.b.insert(o.b.end(), body.begin(), body.end());
  return o.b;
}

std::vector<uint8_t> error_frame(uint64_t call_id, uint16_t code, const std::string& msg) {
  Out o;
  o.u16(code);
  o.blob(msg.data(), msg.size());
  return encode(kErrorReply, call_id, o.b);
}

// ---- sockets ---------------------------------------------------------------

bool send_all(int fd, const std::vector<uint8_t>& bytes) {
  size_t at = 0;
  while (at < bytes.size()) {
    const ssize_t n = ::send(fd, bytes.data() + at, bytes.size() - at, MSG_NOSIGNAL);
    if (n <= 0) {
      if (n < 0 && errno == EINTR) continue;
      return false;
    }
    at += static_cast<size_t>(n);
  }
  return true;
}

// Buffered frame reader over one connection. next() returns nullopt when the
// peer closed; a bad magic or version throws WireError after dropping the
// buffered bytes (the connection keeps serving, as net.cpp does).
class FrameReader {
 public:
  explicit FrameReader(int fd) : fd_(fd) {}
  std::optional<Frame> next(const std::atomic<bool>& stop) {
    for (;;) {
      if (buf_.size() >= 4 && std::memcmp(buf_.data(), "HCL1", 4) != 0) {
        buf_.clear();
        werr(kProtocol, "bad magic");
      }
      if (buf_.size() < 4)
        for (size_t k = 0; k < buf_.size(); ++k)
          if (buf_[k] != static_cast<uint8_t>("HCL1"[k])) {
            buf_.clear();
            werr(kProtocol, "bad magic");
          }
      if (buf_.size() >= kHeader) {
        if (buf_[4] != kVersion) {
          const uint8_t v = buf_[4];
          buf_.clear();
          werr(kVersionErr, "unsupported protocol version " + std::to_string(v));
        }
        In h(buf_.data() + 6, 12);
        Frame f;
        f.kind = buf_[5];
        f.call_id = h.u64();
        const uint32_t len = h.u32();
        if (buf_.size() >= kHeader + len) {
          f.body.assign(buf_.begin() + kHeader, buf_.begin() + kHeader + len);
          buf_.erase(buf_.begin(), buf_.begin() + kHeader + len);
          return f;
        }
      }
      pollfd pfd{fd_, POLLIN, 0};
      const int rc = ::poll(&pfd, 1, 200);
      if (rc < 0 && errno != EINTR) return std::nullopt;
      if (rc <= 0) {
        if (stop.load()) return std::nullopt;
        continue;
      }
      uint8_t chunk[1 << 16];
      const ssize_t n = ::recv(fd_, chunk, sizeof(chunk), 0);
      if (n <= 0) {
        if (n < 0 && errno == EINTR) continue;
        return std::nullopt;
      }
      buf_.insert(buf_.end(), chunk, chunk + n);
    }
  }

 private:
  int fd_;
  std::vector<uint8_t> buf_;
};

// ---- buffer store: host bytes + HBM residency -------------------------------

struct Entry {
  uint64_t size = 0;
  std::vector<uint8_t> host;  // valid when host_valid
  bool host_valid = true;
  int owner = -1;             // device holding the newest bytes when !host_valid
  uint64_t version = 1;
  std::map<int, uint64_t> on_dev;  // device -> version of its resident copy
  bool session = false;            // DataTransfer reassembly in progress
  uint64_t session_total = 0;
  std::vector<std::pair<uint64_t, uint64_t>> got;  // merged received intervals
};

// C-ABI buffer ids of the daemon: the wire ids in their own id space, so a
// daemon sharing a process (and its devices) with a local HostContext never
// collides with that context's buffers
constexpr uint64_t kIdSpace = 1ull << 62;
uint64_t cid(uint64_t wire_id) { return wire_id ^ kIdSpace; }
// launch outputs are written under cid(id) ^ kStagedSpace, then swapped in
constexpr uint64_t kStagedSpace = 1ull << 60;

void check(int rc) {
  if (rc != HCL_OK) werr(static_cast<uint16_t>(rc - HCL_ERR_BASE), hcl_last_error());
}

class NodeDaemon {
 public:
  NodeDaemon(std::string host, int port) : host_(std::move(host)), port_(port) {
    int n = 0;
    if (hcl_device_count(&n) != HCL_OK) n = 0;
    for (int d = 0; d < n; ++d) {
      int type = 1, sms = 0;
      double rel = 1.0;
      uint64_t hbm = 0;
      hcl_device_info(d, &type, &rel, &sms, &hbm, nullptr, 0);
      rel_.push_back(rel);
      max_buffer_ = std::max(max_buffer_, hbm);
      dev_mu_.push_back(std::make_unique<std::mutex>());
    }
    listen_fd_[0] = listen_on(port_);
    listen_fd_[1] = listen_on(port_ + 1);
    for (int k = 0; k < 2; ++k) accept_thr_.emplace_back([this, k] { accept_loop(listen_fd_[k]); });
  }

  ~NodeDaemon() { stop_and_join(); }

  void request_stop() {
    std::lock_guard<std::mutex> l(stop_mu_);
    stopping_.store(true);
    stop_cv_.notify_all();
  }

  // blocks until a Shutdown message or request_stop(); the owner frees the
  // daemon with shutdown() once every waiter has returned
  void wait() {
    std::unique_lock<std::mutex> l(stop_mu_);
    ++waiters_;
    stop_cv_.wait(l, [this] { return stopping_.load(); });
    --waiters_;
    stop_cv_.notify_all();
  }

  void shutdown() {
    request_stop();
    {
      std::unique_lock<std::mutex> l(stop_mu_);
      stop_cv_.wait(l, [this] { return waiters_ == 0; });
    }
    stop_and_join();
  }

 private:
  int listen_on(int port) {
    const int fd = ::socket(AF_INET, SOCK_STREAM, 0);
    if (fd < 0) fail(ErrorCode::internal, std::string("socket: ") + std::strerror(errno));
    int one = 1;
    ::setsockopt(fd, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_port = htons(static_cast<uint16_t>(port));
    if (::inet_pton(AF_INET, host_.c_str(), &a.sin_addr) != 1) {
      ::close(fd);
      fail(ErrorCode::argument, "node daemon: bad IPv4 address '" + host_ + "'");
    }
    if (::bind(fd, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0 || ::listen(fd, 64) != 0) {
      const std::string why = std::strerror(errno);
      ::close(fd);
      if (listen_fd_[0] >= 0) ::close(listen_fd_[0]);
      listen_fd_[0] = -1;
      fail(ErrorCode::argument, "node daemon: cannot listen on " + host_ + ":" + std::to_string(port) + ": " + why);
    }
    return fd;
  }

  void accept_loop(int lfd) {
    while (!stopping_.load()) {
      pollfd pfd{lfd, POLLIN, 0};
      if (::poll(&pfd, 1, 200) <= 0) continue;
      const int fd = ::accept(lfd, nullptr, nullptr);
      if (fd < 0) continue;
      int one = 1;
      ::setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
      std::lock_guard<std::mutex> l(conn_mu_);
      if (stopping_.load()) {
        ::close(fd);
        return;
      }
      conn_thr_.emplace_back([this, fd] { serve(fd); });
    }
  }

  void serve(int fd) {
    FrameReader rd(fd);
    for (;;) {
      std::optional<Frame> f;
      try {
        f = rd.next(stopping_);
      } catch (const WireError& e) {
        if (!send_all(fd, error_frame(0, e.code, e.msg))) break;
        continue;
      }
      if (!f) break;
      std::optional<std::vector<uint8_t>> reply;
      try {
        reply = handle(*f);
      } catch (const WireError& e) {
        reply = error_frame(f->call_id, e.code, e.msg);
      } catch (const Error& e) {
        reply = error_frame(f->call_id, static_cast<uint16_t>(e.code()), e.what());
      } catch (const std::exception& e) {
        reply = error_frame(f->call_id, kInternal, e.what());
      }
      if (reply && !send_all(fd, *reply)) break;
      if (f->kind == kShutdown) break;
    }
    ::close(fd);
  }

  void stop_and_join() {
    request_stop();
    for (auto& t : accept_thr_)
      if (t.joinable()) t.join();
    accept_thr_.clear();
    for (int& fd : listen_fd_)
      if (fd >= 0) ::close(fd), fd = -1;
    for (size_t i = 0;; ++i) {
      std::thread t;
      {
        std::lock_guard<std::mutex> l(conn_mu_);
        if (i >= conn_thr_.size()) break;
        t = std::move(conn_thr_[i]);
      }
      if (t.joinable()) t.join();
    }
    std::lock_guard<std::mutex> l(store_mu_);
    for (auto& [id, e] : store_)
      for (auto& [d, v] : e.on_dev) hcl_buffer_release(d, cid(id));
    store_.clear();
  }

  // ---- dispatch ----

  std::optional<std::vector<uint8_t>> handle(const Frame& f) {
    switch (f.kind) {
      case kPing:
        return encode(kPong, f.call_id, {});
      case kDeviceIdRequest: {
        Out o;
        o.u32(static_cast<uint32_t>(rel_.size()));
        for (size_t d = 0; d < rel_.size(); ++d) {
          o.u32(static_cast<uint32_t>(d));
          o.u8(1);  // gpu
          o.u64(std::bit_cast<uint64_t>(rel_[d]));
        }
        return encode(kDeviceIdResponse, f.call_id, o.b);
      }
      case kDataTransfer: {
        In in(f.body.data(), f.body.size());
        const uint64_t id = in.u64(), off = in.u64(), total = in.u64();
        const size_t len = in.left();
        if (off > total || len > total - off) werr(kMalformed, "data package exceeds total_len");
        check_size(total, "data transfer");
        const auto done = put_chunk(id, off, total, in.here(), len);
        if (!done) return std::nullopt;  // only the completing chunk is acknowledged
        Out o;
        o.u64(id);
        o.u64(*done);
        return encode(kDataAck, f.call_id, o.b);
      }
      case kApiCallRequest: {
        In in(f.body.data(), f.body.size());
        const std::string fn = in.str();
        const uint32_t nargs = in.u32();
        std::vector<Value> args;
        for (uint32_t k = 0; k < nargs; ++k) args.push_back(in.value());
        const uint32_t nrefs = in.u32();
        for (uint32_t k = 0; k < nrefs; ++k) {
          in.u64();
          if (in.u8() > 2) werr(kMalformed, "bad buffer direction");
        }
        std::vector<Value> res = call(fn, args);
        Out o;
        o.u32(static_cast<uint32_t>(res.size()));
        for (const Value& v : res) o.value(v);
        return encode(kApiCallResponse, f.call_id, o.b);
      }
      case kShutdown:
        request_stop();
        return std::nullopt;
      default:
        werr(kMalformed, "unexpected message kind " + std::to_string(f.kind));
    }
  }

  static uint64_t handle_arg(const Value& v, const char* what) {
    if (v.tag != kHandle) werr(kArgument, std::string(what) + " expects a handle");
    return static_cast<uint64_t>(v.i);
  }

  std::vector<Value> call(const std::string& fn, const std::vector<Value>& a) {
    if (fn == "alloc_buffer") {
      if (a.size() != 2 || a[1].tag != kI64) werr(kArgument, "alloc_buffer expects (id, size)");
      if (a[1].i < 0) werr(kArgument, "alloc_buffer: negative size");
      alloc(handle_arg(a[0], "alloc_buffer"), static_cast<uint64_t>(a[1].i));
      return {};
    }
    if (fn == "read_buffer") {
      if (a.size() != 1) werr(kArgument, "read_buffer expects (id)");
      Value v;
      v.tag = kBytes;
      v.s = read(handle_arg(a[0], "read_buffer"));
      return {v};
    }
    if (fn == "release_object") {
      if (a.size() != 1) werr(kArgument, "release_object expects (id)");
      release(handle_arg(a[0], "release_object"));
      return {};
    }
    if (fn == "query_registry") {
      if (a.size() != 1 || a[0].tag != kString) werr(kArgument, "query_registry expects (bundle)");
      return registry(a[0].s);
    }
    if (fn == "launch_kernel") return launch(a);
    werr(kUnknownCall, "unknown-call '" + fn + "'");
  }

  std::vector<Value> registry(const std::string& bundle) {
    std::vector<char> names(1 << 16);
    std::vector<uint32_t> ar(256);
    int n = 0;
    check(hcl_query_registry(bundle.c_str(), names.data(), static_cast<int>(names.size()), ar.data(),
                             static_cast<int>(ar.size()), &n));
    std::vector<Value> out;
    Value cnt;
    cnt.i = n;
    out.push_back(cnt);
    std::string csv(names.data());
    size_t at = 0;
    for (int k = 0; k < n; ++k) {
      const size_t comma = csv.find(',', at);
      Value name, arity;
      name.tag = kString;
      name.s = csv.substr(at, comma == std::string::npos ? std::string::npos : comma - at);
      arity.i = ar[k];
      out.push_back(name);
      out.push_back(arity);
      at = comma == std::string::npos ? csv.size() : comma + 1;
    }
    return out;
  }

  // ---- store operations ----

  // bring the newest bytes of e to the host (caller holds store_mu_)
  void pull_host(uint64_t id, Entry& e) {
    if (e.host_valid) return;
    e.host.resize(e.size);
    if (e.size) check(hcl_buffer_read(e.owner, cid(id), 0, e.host.data(), e.size));
    e.host_valid = true;
  }

  // sizes come from the network: a buffer never exceeds one device's HBM
  // (HCL_NODE_MAX_BUFFER lowers the cap), else a size error instead of an
  // attempt to allocate it on the host
  void check_size(uint64_t bytes, const char* what) const {
    uint64_t cap = max_buffer_ ? max_buffer_ : (1ull << 40);
    if (const char* e = std::getenv("HCL_NODE_MAX_BUFFER")) cap = std::min<uint64_t>(cap, std::strtoull(e, nullptr, 10));
    if (bytes > cap)
      werr(kSizeErr, std::string(what) + ": " + std::to_string(bytes) + " bytes exceeds the node's buffer cap of " +
                         std::to_string(cap));
  }

  void alloc(uint64_t id, uint64_t size) {
    check_size(size, "alloc_buffer");
    std::lock_guard<std::mutex> l(store_mu_);
    Entry& e = store_[id];
    if (e.size >= size) return;
    pull_host(id, e);
    e.host.resize(size, 0);
    e.size = size;
    ++e.version;  // resident device copies are shorter now
  }

  std::optional<uint64_t> put_chunk(uint64_t id, uint64_t off, uint64_t total, const uint8_t* p, size_t len) {
    std::lock_guard<std::mutex> l(store_mu_);
    Entry& e = store_[id];
    if (!e.session) {
      pull_host(id, e);
      e.session = true;
      e.session_total = total;
      e.got.clear();
      if (e.size < total) {
        e.host.resize(total, 0);
        e.size = total;
      }
      ++e.version;  // device copies are stale from here on
    }
    if (total != e.session_total)
      werr(kReassembly, "total_len changed mid-transfer for buffer " + std::to_string(id));
    const uint64_t b = off, end = off + len;
    for (const auto& [lo, hi] : e.got) {
      const uint64_t olo = std::max(b, lo), ohi = std::min(end, hi);
      if (olo < ohi && std::memcmp(e.host.data() + olo, p + (olo - b), ohi - olo) != 0)
        werr(kReassembly, "overlapping chunk with different bytes in buffer " + std::to_string(id));
    }
    if (len) {
      std::memcpy(e.host.data() + b, p, len);
      e.got.emplace_back(b, end);
      std::sort(e.got.begin(), e.got.end());
      std::vector<std::pair<uint64_t, uint64_t>> m;
      for (const auto& iv : e.got) {
        if (!m.empty() && iv.first <= m.back().second)
          m.back().second = std::max(m.back().second, iv.second);
        else
          m.push_back(iv);
      }
      e.got.swap(m);
    }
    const bool covered = e.session_total == 0 ||
                         (e.got.size() == 1 && e.got[0].first == 0 && e.got[0].second == e.session_total);
    if (!covered) return std::nullopt;
    e.session = false;
    e.got.clear();
    return e.session_total;
  }

  std::string read(uint64_t id) {
    std::lock_guard<std::mutex> l(store_mu_);
    auto it = store_.find(id);
    if (it == store_.end()) werr(kPrecondition, "buffer " + std::to_string(id) + " not in store");
    if (it->second.session) werr(kPrecondition, "buffer " + std::to_string(id) + " is mid-reassembly");
    pull_host(id, it->second);
    return std::string(reinterpret_cast<const char*>(it->second.host.data()), it->second.size);
  }

  void release(uint64_t id) {
    std::lock_guard<std::mutex> l(store_mu_);
    auto it = store_.find(id);
    if (it == store_.end()) return;
    for (auto& [d, v] : it->second.on_dev) hcl_buffer_release(d, cid(id));
    store_.erase(it);
  }

  // make device d's copy of an input current (caller holds store_mu_)
  void stage_in(int d, uint64_t id, Entry& e) {
    auto r = e.on_dev.find(d);
    if (r != e.on_dev.end() && r->second == e.version) return;
    check(hcl_buffer_alloc(d, cid(id), 0, e.size));
    if (e.size) {
      if (e.host_valid)
        check(hcl_buffer_write(d, cid(id), 0, e.host.data(), e.size));
      else
        check(hcl_buffer_copy_peer(d, cid(id), 0, e.owner, cid(id), 0, e.size));  // NVLink, no host hop
    }
    e.on_dev[d] = e.version;
  }

  std::vector<Value> launch(const std::vector<Value>& a) {
    // layout of make_launch_kernel (proj/src/api.cpp:43-71)
    if (a.size() < 9) werr(kMalformed, "launch_kernel: short argument list");
    auto want = [&](size_t k, uint8_t tag) -> const Value& {
      if (a[k].tag != tag) werr(kArgument, "launch_kernel: argument " + std::to_string(k) + " has the wrong type");
      return a[k];
    };
    const std::string kernel = want(0, kString).s;
    const int dev = static_cast<int>(want(3, kI32).i);
    const uint32_t dims = static_cast<uint32_t>(want(4, kI32).i);
    const int32_t nargs = static_cast<int32_t>(want(8, kI32).i);
    if (nargs < 0 || a.size() != 9 + static_cast<size_t>(nargs))
      werr(kMalformed, "launch_kernel: argument count mismatch");
    if (dev < 0 || dev >= static_cast<int>(rel_.size()))
      werr(kUnknownDevice, "local device " + std::to_string(dev));
    // the kernel's signature: the reference's core bundle first, then this repo's
    uint8_t kinds[64], parts[64];
    int arity = 0;
    if (hcl_kernel_signature("core", kernel.c_str(), kinds, parts, 64, &arity) != HCL_OK &&
        hcl_kernel_signature("b200", kernel.c_str(), kinds, parts, 64, &arity) != HCL_OK)
      werr(kName, "unknown kernel '" + kernel + "'");
    if (arity != nargs) werr(kArgument, kernel + ": arity mismatch");

    std::lock_guard<std::mutex> dl(*dev_mu_[dev]);
    std::vector<hcl_arg> args(static_cast<size_t>(nargs));
    std::vector<uint64_t> outs;
    std::vector<std::pair<uint64_t, uint64_t>> fresh;  // (output id, staging device id)
    {
      std::lock_guard<std::mutex> l(store_mu_);
      for (int k = 0; k < nargs; ++k) {
        const Value& v = a[9 + static_cast<size_t>(k)];
        hcl_arg& h = args[static_cast<size_t>(k)];
        h.kind = kinds[k];
        if (kinds[k] == HCL_ARG_SCALAR) {
          if (v.tag != kI64 && v.tag != kI32)
            werr(kArgument, kernel + ": argument " + std::to_string(k) + " must be an integer scalar");
          h.scalar = v.i;
          continue;
        }
        if (v.tag != kHandle)
          werr(kArgument, kernel + ": argument " + std::to_string(k) + " must be a buffer handle");
        const uint64_t id = static_cast<uint64_t>(v.i);
        h.buffer_id = cid(id);
        auto it = store_.find(id);
        if (kinds[k] == HCL_ARG_OUT) {
          if (it == store_.end()) werr(kPrecondition, "output buffer " + std::to_string(id) + " not allocated");
          // fresh zero-filled HBM (the reference zero-fills outputs, kernels.cpp:43-48),
          // under a staging id: the buffer's current copy survives a failed launch
          const uint64_t staged = cid(id) ^ kStagedSpace;
          hcl_buffer_release(dev, staged);
          check(hcl_buffer_alloc(dev, staged, 0, it->second.size));
          h.buffer_id = staged;
          fresh.push_back({id, staged});
          continue;
        }
        if (it == store_.end() || it->second.session)
          werr(kPrecondition, "input buffer " + std::to_string(id) + " not complete");
        stage_in(dev, id, it->second);
        if (kinds[k] == HCL_ARG_INOUT) outs.push_back(id);
      }
    }
    uint64_t work = 0;
    double ms = 0.0;
    int rc = hcl_launch(dev, kernel.c_str(), args.data(), static_cast<uint32_t>(nargs), nullptr, nullptr,
                        dims ? dims : 1, &work);
    if (rc == HCL_OK) rc = hcl_finish(dev, &ms);
    if (rc != HCL_OK) {  // the outputs keep their previous contents
      for (const auto& [id, staged] : fresh) hcl_buffer_release(dev, staged);
      check(rc);
    }
    for (const auto& [id, staged] : fresh) {  // commit: the staged allocations become the outputs
      check(hcl_buffer_swap(dev, cid(id), staged));
      hcl_buffer_release(dev, staged);
      outs.push_back(id);
    }
    {
      std::lock_guard<std::mutex> l(store_mu_);
      for (uint64_t id : outs) {
        auto it = store_.find(id);
        if (it == store_.end()) continue;  // released meanwhile
        Entry& e = it->second;
        ++e.version;
        e.host_valid = false;
        e.owner = dev;
        e.on_dev.clear();
        e.on_dev[dev] = e.version;
      }
    }
    Value c, m, w;
    c.tag = kF64;
    c.f = ms / 1e3;
    m.tag = kF64;
    m.f = static_cast<double>(work) / (rel_[static_cast<size_t>(dev)] * 1e9);  // kBaselineWorkRate
    w.tag = kI64;
    w.i = static_cast<int64_t>(work);
    return {c, m, w};
  }

  std::string host_;
  int port_;
  int listen_fd_[2] = {-1, -1};
  std::vector<double> rel_;
  uint64_t max_buffer_ = 0;  // largest device HBM: the cap on network-supplied sizes
  std::vector<std::unique_ptr<std::mutex>> dev_mu_;
  std::atomic<bool> stopping_{false};
  int waiters_ = 0;
  std::mutex stop_mu_;
  std::condition_variable stop_cv_;
  std::mutex conn_mu_;
  std::vector<std::thread> accept_thr_, conn_thr_;
  std::mutex store_mu_;
  std::map<uint64_t, Entry> store_;
};

}  // namespace
}  // namespace hcl

// ---- C-ABI ------------------------------------------------------------------

extern "C" {

int hcl_node_start(const char* host, int message_port, void** node) {
  return hcl::guard([&] {
    if (!node) hcl::fail(hcl::ErrorCode::argument, "hcl_node_start: node is NULL");
    if (message_port <= 0 || message_port >= 65535)
      hcl::fail(hcl::ErrorCode::argument, "hcl_node_start: message port must be in [1, 65534]");
    *node = new hcl::NodeDaemon(host ? host : "127.0.0.1", message_port);
  });
}

int hcl_node_wait(void* node) {
  return hcl::guard([&] {
    if (!node) hcl::fail(hcl::ErrorCode::argument, "hcl_node_wait: node is NULL");
    static_cast<hcl::NodeDaemon*>(node)->wait();
  });
}

int hcl_node_stop(void* node) {
  return hcl::guard([&] {
    if (!node) return;
    auto* d = static_cast<hcl::NodeDaemon*>(node);
    d->shutdown();
    delete d;
  });
}

}  // extern "C"
