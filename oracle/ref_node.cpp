// TEST INFRASTRUCTURE ONLY (built into oracle/_ref by oracle/Makefile): the
// reference's own node daemon (haocl::run_daemon, proj/src/daemon.cpp) with
// n cpu devices of relative throughput 1.0 and all host threads per device --
// what `haocl node` runs (proj/tools/haocl_main.cpp, whose CLI11 dependency
// is absent here). The CPU baseline arm of scripts/remote_compare.py.
//
//   ref_node <message_port> <n_devices> [threads_per_device]

#include <cstdlib>
#include <iostream>
#include <thread>

#include "haocl/daemon.hpp"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: ref_node <message_port> <n_devices> [threads_per_device]\n";
    return 2;
  }
  const int port = std::atoi(argv[1]), ndev = std::atoi(argv[2]);
  haocl::DaemonOptions opt;
  opt.threads_per_device = argc > 3 ? std::atoi(argv[3]) : static_cast<int>(std::thread::hardware_concurrency());
  std::vector<haocl::DeviceModel> devs(static_cast<size_t>(ndev));
  std::cout << "ref node serving " << ndev << " cpu device(s) on 127.0.0.1:" << port << std::endl;
  haocl::run_daemon(haocl::Endpoint::at("127.0.0.1", static_cast<uint16_t>(port)), devs, opt);
  return 0;
}
