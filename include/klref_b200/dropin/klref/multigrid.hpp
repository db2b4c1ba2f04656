// Drop-in replacement of the reference's proj/include/klref/multigrid.hpp: the
// B200 facade (include/klref_b200/klref.hpp) declares the whole hot-path API
// (hhg, fem, multigrid, estimator).  Put include/klref_b200/dropin before the
// reference's include directory; macro_mesh.hpp, errors.hpp, amr.hpp,
// mesh_io.hpp and problems.hpp keep coming from the reference.
#ifndef KLREF_B200_DROPIN_MULTIGRID_HPP
#define KLREF_B200_DROPIN_MULTIGRID_HPP
#include "klref_b200/klref.hpp"
#endif
