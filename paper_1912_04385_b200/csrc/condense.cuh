// condense.cuh -- static condensation state (condense_exact.cu).
#pragma once
#include "mprec.cuh"

namespace mg {

// ReducedSystem (condense.hpp:83-90) on the device: the reduced A in BSR with
// its pattern, b, and what back_substitute needs (the J22 factors, J21, r2).
struct Condensed {
    int nc = 0, np = 0, n2 = 0;
    Pattern pat;
    DBuf<double> a_val, b;
    DBuf<int> sec_off, perm;
    std::vector<int> h_sec;
    DBuf<int64_t> lu_off;
    DBuf<double> lu, j21, r2;
};

// condense.cpp:206-241 (throws Error(MPREC_SINGULAR_BLOCK, .., cell))
void condense(Ctx& c, const mprec_global_jacobian& j, Condensed& out);
// condense.cpp:243-258 on device vectors (d1: nc*np, d2: n2)
void back_substitute(Ctx& c, const Condensed& h, const double* d1_dev, double* d2_dev);

}  // namespace mg
