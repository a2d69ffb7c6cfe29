// Kernel shapes compiled into the library (instantiated in kernels_resident.cu and
// kernels_cluster.cu so nvcc builds them as separate translation units).
#pragma once

#include "dr_cluster.cuh"
#include "dr_kernel.cuh"
#include "dr_node.cuh"
#include "dr_stream.cuh"

namespace fibra_b200 {

using KernelFn = void (*)(DrParams);
using ClusterFn = void (*)(ClusterParams);
using StreamFn = void (*)(StreamParams);

struct Variant {     // resident kernel: one CTA per RVE
  int T, FPT, NPT, MINB;
  KernelFn fn[4][2];  // [law + 2 * buckling_off][uniform EA]
};

struct ClusterVariant {  // cluster kernel: one cluster of C CTAs per RVE (per-CTA shape)
  int T, FPT, NPT;
  ClusterFn fn[4][2];
};

struct NodeVariant {  // node-centric kernel: one CTA per RVE, NPT node slots per thread
  int T, NPT, MINB;
  KernelFn fn[4][2];
};

struct StreamVariant {  // HBM-streaming kernel: one cluster per RVE, per-CTA shape
  int T, NPT;
  StreamFn fn[4][2];
};

extern const Variant kVariants[];
extern const StreamVariant kStreamVariants[];
extern const int kNumStreamVariants;
extern const NodeVariant kNodeVariants[];
extern const int kNumNodeVariants;
extern const int kNumVariants;
extern const ClusterVariant kClusterVariants[];
extern const int kNumClusterVariants;

}  // namespace fibra_b200
