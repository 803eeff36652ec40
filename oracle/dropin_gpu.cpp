// Test infrastructure: the reference's hot-path entry points re-implemented on
// the B200 library, with the REFERENCE'S OWN SIGNATURES, so that the
// reference's unit tests (tests/test_fmm.cpp, tests/test_mlfmm.cpp, compiled
// unmodified) run against the GPU path. This is the "link unchanged" drop-in
// of SURVEY §8(b): a maintainer builds the library with these definitions in
// place of mlfmm_matvec (mlfmm.cpp:361-406), fmm_matvec_single
// (fmm.cpp:123-213) and direct_matvec (fmm.cpp:30-75); oracle/Makefile does
// it by compiling the reference's mlfmm.cpp / fmm.cpp with those three
// functions renamed to *_cpu (upsweep / couple / downsweep, the stage
// diagnostics, stay the reference's CPU code).
#include <vector>

#include "blfmm/fmm.hpp"
#include "blfmm/mlfmm.hpp"
#include "blfmm_gpu.hpp"

namespace blfmm {

// the reference's own implementation, renamed at compile time
SumResult direct_matvec_cpu(const RadialKernel& k, const PointSet& ps,
                            const std::vector<double>& weights, bool use_bandlimited, double sigma,
                            int refinement);

SumResult mlfmm_matvec(const SumRequest& req, const BoxTree& tree, const LevelGrids& grids) {
  return gpu::mlfmm_matvec(req, tree, grids);
}

SumResult fmm_matvec_single(const SumRequest& req, const BoxTree& tree) {
  return gpu::fmm_matvec_single(req, tree);
}

SumResult direct_matvec(const RadialKernel& k, const PointSet& ps,
                        const std::vector<double>& weights, bool use_bandlimited, double sigma,
                        int refinement) {
  if (use_bandlimited)  // the 1-D band-limited table oracle is CPU setup code
    return direct_matvec_cpu(k, ps, weights, true, sigma, refinement);
  return gpu::direct_matvec(k, ps, weights, false, sigma, refinement);
}

}  // namespace blfmm
