// gates.cpp -- fp64 gate matrices of the Sycamore gate set.
// Entries are the closed forms of reading V2-V4:
//   sqrt(X) = 1/2 [[1+i, 1-i], [1-i, 1+i]]
//   sqrt(Y) = 1/2 [[1+i, -1-i], [1+i, 1+i]]
//   sqrt(W) = [[1/2+i/2, -i/sqrt2], [1/sqrt2, 1/2+i/2]],  W = (X+Y)/sqrt2
//   Rz(phi) = diag(e^{-i phi/2}, e^{+i phi/2})
//   fSim(theta, phi) = [[1,0,0,0],[0,c,-is,0],[0,-is,c,0],[0,0,0,e^{-i phi}]]
// Row-major; 2-qubit basis index b_q0 + 2*b_q1.
#include <cmath>

#include "internal.h"

namespace rcs {

void gate_matrix(const Gate& g, cplx* m) {
    const double h = 0.5;
    const double r = 0.70710678118654752440084436210484903928;   // 1/sqrt(2)
    switch (g.kind) {
        case RCS_GATE_SX:
            m[0] = {h, h};  m[1] = {h, -h};
            m[2] = {h, -h}; m[3] = {h, h};
            return;
        case RCS_GATE_SY:
            m[0] = {h, h};  m[1] = {-h, -h};
            m[2] = {h, h};  m[3] = {h, h};
            return;
        case RCS_GATE_SW:
            m[0] = {h, h};  m[1] = {0.0, -r};
            m[2] = {r, 0.0}; m[3] = {h, h};
            return;
        case RCS_GATE_RZ: {
            const double c = std::cos(0.5 * g.phi), s = std::sin(0.5 * g.phi);
            m[0] = {c, -s}; m[1] = {0.0, 0.0};
            m[2] = {0.0, 0.0}; m[3] = {c, s};
            return;
        }
        default: {  // fSim
            for (int i = 0; i < 16; i++) m[i] = {0.0, 0.0};
            const double c = std::cos(g.theta), s = std::sin(g.theta);
            m[0] = {1.0, 0.0};
            m[5] = {c, 0.0};
            m[6] = {0.0, -s};
            m[9] = {0.0, -s};
            m[10] = {c, 0.0};
            m[15] = {std::cos(g.phi), -std::sin(g.phi)};
            return;
        }
    }
}

}  // namespace rcs
