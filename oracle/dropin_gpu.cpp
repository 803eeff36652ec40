// Test infrastructure: the reference's hot-path entry points re-implemented on
// the B200 library, with the REFERENCE'S OWN SIGNATURES, so that the
// reference's unit tests (tests/test_fmm.cpp, tests/test_mlfmm.cpp, compiled
// unmodified) run against the GPU path. This is the "link unchanged" drop-in
// of SURVEY §8(b): a maintainer builds the library with these definitions in
// place of mlfmm_matvec (mlfmm.cpp:361-406), fmm_matvec_single
// (fmm.cpp:123-213), direct_matvec (fmm.cpp:30-75) and direct_matvec_hybrid
// (fmm.cpp:77-113); oracle/Makefile does it by compiling the reference's
// mlfmm.cpp / fmm.cpp with those four functions renamed to *_cpu (upsweep / couple / downsweep, the stage
// diagnostics, stay the reference's CPU code).
#include <vector>

#include "blfmm/fmm.hpp"
#include "blfmm/mlfmm.hpp"
#include "blfmm_gpu.hpp"

namespace blfmm {

SumResult mlfmm_matvec(const SumRequest& req, const BoxTree& tree, const LevelGrids& grids) {
  return gpu::mlfmm_matvec(req, tree, grids);
}

SumResult fmm_matvec_single(const SumRequest& req, const BoxTree& tree) {
  return gpu::fmm_matvec_single(req, tree);
}

SumResult direct_matvec(const RadialKernel& k, const PointSet& ps,
                        const std::vector<double>& weights, bool use_bandlimited, double sigma,
                        int refinement) {
  return gpu::direct_matvec(k, ps, weights, use_bandlimited, sigma, refinement);
}

SumResult direct_matvec_hybrid(const RadialKernel& k, const PointSet& ps, const BoxTree& tree,
                               const std::vector<double>& weights, double sigma, int refinement) {
  return gpu::direct_matvec_hybrid(k, ps, tree, weights, sigma, refinement);
}

}  // namespace blfmm
