// paracycle_b200 C ABI implementation (see include/paracycle_b200.h).
//
// Host-side orchestration of the PTL-cycled parabolic advance:
//   pc_cycle  == ptl.cycle_operator: one F+argmax pass, the
//   Eq. 5 pair kernel, ONE 64-byte device->host read per cycle, then either
//   s fused STS stage kernels (RKL2/RKG2) or a device-driven Jacobi-PCG solve.
// Integer decisions (s, coefficient tables, remaining-time bookkeeping) are
// computed here with the same expressions as oracle/schemes.py and
// oracle/ptl.py (host code compiled with -ffp-contract=off).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <string>
#include <mutex>
#include <unordered_set>
#include <vector>

#include "../../include/paracycle_b200.h"
#include "gen.cuh"
#include "march.cuh"
#include "smarch.cuh"
#include "vmarch.cuh"
#include "tma_march.cuh"
#include "sts.cuh"
#include "persist.cuh"

#include <cudaTypedefs.h>
#include "nccl_shim.h"

using namespace pc;

// the C ABI, in dependency order (one translation unit)
#include "capi_objects.cuh"
#include "capi_fields.cuh"
#include "capi_ops.cuh"
#include "capi_sts.cuh"
#include "capi_pcg.cuh"
#include "capi_cycle.cuh"
#include "capi_gen.cuh"
