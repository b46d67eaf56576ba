// TEST INFRASTRUCTURE ONLY (built into oracle/_ref by oracle/Makefile, never
// shipped): the reference's own host runtime and bench layer, compiled in
// place from /root/reference/proj/src, pointed at a node daemon of THIS repo
// (paper_2005_08466_b200.node) instead of the reference's CPU daemon.
//
//   ref_bench_remote <node_port> <n_devices> <benchmark> <partition> [key=value ...]
//
// Builds the cluster config "node n0 127.0.0.1:<node_port> gpu 1.0" (one line
// per device, proj/include/haocl/config.hpp:4-10), HostContext::init (the
// Ping/Pong handshake and the DeviceIdRequest exchange), then
// haocl::bench::run_benchmark -- the unmodified reference path: seeded inputs,
// block_range partitioning over the parts, per-part buffers and launches, and
// in-process oracle verification -- and prints the RunReport JSON.
// Keys: m k n rows cols density vertices edges knn_r knn_q knn_d knn_k length seed type.

#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

#include "haocl/bench.hpp"
#include "haocl/config.hpp"
#include "haocl/runtime.hpp"

int main(int argc, char** argv) {
  if (argc < 5) {
    std::cerr << "usage: ref_bench_remote <node_port> <n_devices> <benchmark> <partition> [key=value ...]\n";
    return 2;
  }
  const int port = std::atoi(argv[1]), ndev = std::atoi(argv[2]);
  std::string type = "gpu";  // type=cpu to drive the reference's own daemon (ref_node)
  for (int i = 5; i < argc; ++i)
    if (std::string(argv[i]).rfind("type=", 0) == 0) type = std::string(argv[i]).substr(5);
  std::ostringstream conf;
  conf << "host 127.0.0.1:" << (port + 50) << "\n";
  for (int d = 0; d < ndev; ++d) conf << "node n0 127.0.0.1:" << port << " " << type << " 1.0\n";
  haocl::bench::BenchParams p;
  p.benchmark = argv[3];
  p.partition = std::atoi(argv[4]);
  for (int i = 5; i < argc; ++i) {
    std::string kv = argv[i];
    const auto eq = kv.find('=');
    if (eq == std::string::npos) continue;
    const std::string key = kv.substr(0, eq), v = kv.substr(eq + 1);
    const long long x = std::atoll(v.c_str());
    if (key == "m") p.m = x;
    else if (key == "k") p.k = x;
    else if (key == "n") p.n = x;
    else if (key == "rows") p.rows = x;
    else if (key == "cols") p.cols = x;
    else if (key == "density") p.density = std::atof(v.c_str());
    else if (key == "vertices") p.vertices = x;
    else if (key == "edges") p.edges = x;
    else if (key == "knn_r") p.knn_r = x;
    else if (key == "knn_q") p.knn_q = x;
    else if (key == "knn_d") p.knn_d = x;
    else if (key == "knn_k") p.knn_k = x;
    else if (key == "length") p.length = x;
    else if (key == "seed") p.seed = static_cast<uint64_t>(x);
  }
  try {
    auto ctx = haocl::HostContext::init(haocl::ClusterConfig::parse(conf.str()));
    auto report = haocl::bench::run_benchmark(ctx, p);
    std::cout << report.to_json() << std::endl;
    return report.verify_pass ? 0 : 1;
  } catch (const haocl::Error& e) {
    std::cerr << "haocl error " << static_cast<int>(e.code()) << ": " << e.what() << "\n";
    return 3;
  }
}
