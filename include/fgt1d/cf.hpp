#pragma once
// Near-best rational (Caratheodory-Fejer) SOE of the Gaussian.  The reference
// builds it at run time (proj/src/cf.cpp:63-194, needs Eigen); here cf_soe(n)
// is a lookup into the compiled-in tables (tools/gen_soe_tables.py), same
// values, same (Re t, Im t) order, same domain_error for n outside 2..14.
#include "fgt1d/soe.hpp"

namespace fgt {

SoeApprox cf_soe(int n);

// Table lookup by tolerance (north_star): folded CF SOE with the fewest modes
// whose documented transform error (proj/README.md:184-189) is <= tol.
SoeApprox soe_for_tolerance(double tol);

}  // namespace fgt
