// Leaf-block Jacobi preconditioner of the BEM GMRES (bem_prec.cu)
#pragma once
#include "fmm.cuh"

namespace ebem {

struct LeafBlockPrec {
    static constexpr int BMAX = 52;    // panels per diagonal block (a leaf's targets in runs of at most BMAX): 156 unknowns, inverted in shared memory
    int nblocks = 0, maxn = 0;
    int64_t entries = 0;               // doubles in M
    DBuf<int4> blocks;                 // (first sorted target, panels, offset hi, offset lo)
    DBuf<double> M;                    // the inverted blocks, row-major, back to back
    void release() {
        nblocks = maxn = 0;
        entries = 0;
        blocks.release();
        M.release();
    }
};

// forms and inverts the blocks for the boundary-condition types bc; false (P released) when
// they do not fit half of the free device memory or a block is singular
bool leafblock_build(const Tree& t, int64_t npanels, int nq, const float* cent, const float* qp, const float* qn,
                     const float* qw, const int32_t* bc, const double* DU, const double* DP, const Material& m,
                     LeafBlockPrec& P, cudaStream_t s);
// out = M^-1 v (panel vectors [npanels x 3], caller order)
void leafblock_apply(const Tree& t, const LeafBlockPrec& P, const double* v, double* out, cudaStream_t s);

}  // namespace ebem
