// Oracle-build aid only: Boost is absent from this image, and the reference
// uses exactly one Boost routine (boost::math::gamma_p, proj/src/dist.cpp:17).
// Forward it to the shared definition so the reference build and the engine
// build Scenario A's demand pmf from identical arithmetic.
#pragma once
#include "../../../../../paper_2303_10672_b200/csrc/gamma_p.h"

namespace boost {
namespace math {
inline double gamma_p(double a, double x) { return pvi_gamma_p(a, x); }
}  // namespace math
}  // namespace boost
