// Immutable kernel registry (the reference's core_kernels/find_kernel/
// kernel_names/bundle_exists, proj/include/haocl/kernels.hpp:37-40,
// proj/src/kernels.cpp:13-33, 248-266). Two bundles:
//   "core" — the reference's kernels in its buffer encodings (fp64/int64),
//            bit-exact with the reference;
//   "b200" — the BASELINE workloads (bf16/tf32/fp32 GEMM, PageRank SpMV,
//            k-means, 3x3 conv) in B200-native encodings.
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"

namespace hcl {

void register_core(std::vector<KernelDef>& r);
void register_gemm(std::vector<KernelDef>& r);
void register_graph(std::vector<KernelDef>& r);
void register_kmeans(std::vector<KernelDef>& r);
void register_conv(std::vector<KernelDef>& r);
void register_kmeans_tc(std::vector<KernelDef>& r);

const std::vector<KernelDef>& registry() {
  static const std::vector<KernelDef> defs = [] {
    std::vector<KernelDef> r;
    register_core(r);
    register_gemm(r);
    register_graph(r);
    register_kmeans(r);
    register_conv(r);
    register_kmeans_tc(r);
    return r;
  }();
  return defs;
}

bool bundle_exists(const std::string& bundle) { return bundle == "core" || bundle == "b200"; }

const KernelDef* find_kernel(const std::string& bundle, const std::string& name) {
  if (!bundle_exists(bundle)) return nullptr;
  for (const auto& k : registry())
    if (bundle == k.bundle && name == k.name) return &k;
  return nullptr;
}

const KernelDef* find_kernel_any(const std::string& name) {
  for (const auto& k : registry())
    if (name == k.name) return &k;
  return nullptr;
}

}  // namespace hcl
