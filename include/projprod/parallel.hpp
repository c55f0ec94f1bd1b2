// Host-side mirror of the reference's slice-loop helper
// (/root/reference/proj/include/projprod/parallel.hpp:8-16, src/parallel.cpp:13-57).
//
// The engine itself does not loop over slices on the host: every facewise
// step is one batched grid (or one persistent kernel) on the GPU, and
// PROJPROD_DEVICES caps the devices the multi-GPU driver uses. These two
// functions are kept for callers of the reference API that run their own
// independent host loops (generators, per-slice post-processing).
#pragma once

#include <cstddef>
#include <functional>

namespace projprod {

// min(hardware_concurrency, PROJPROD_THREADS); an unset or unparsable
// PROJPROD_THREADS adds no cap, values below 1 count as 1.
int max_threads();

// fn(i) for every i in [0, n), iterations independent: contiguous index ranges
// on at most max_threads() workers (a single worker runs in the caller).
// The first exception a worker throws is rethrown here after all have joined.
void parallel_for(std::ptrdiff_t n, const std::function<void(std::ptrdiff_t)>& fn);

}  // namespace projprod
