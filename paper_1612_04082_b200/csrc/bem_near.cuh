// BEM near-field operator in HBM (see bem_near.cu)
#pragma once
#include "fmm.cuh"

namespace ebem {

struct NearMat {
    bool ready = false;
    long long entries = 0;        // floats in M
    DBuf<int> col_first, ncol;    // per target leaf (eval order): first column, column count
    DBuf<int> seg_start;          // per column: first entry in the sorted (leaf, panel) list
    DBuf<int> col_panel;          // per column: panel index
    DBuf<long long> moff;         // per target leaf: offset of its [9][rows][ncol] block in M
    DBuf<float> M;
    DBuf<int32_t> bc;             // boundary-condition types the blocks were built for
    void release() {
        ready = false;
        entries = 0;
        for (DBuf<int>* b : {&col_first, &ncol, &seg_start, &col_panel}) b->release();
        moff.release();
        M.release();
        bc.release();
    }
};

bool near_matrix_enabled();
// builds (or keeps, when bc is unchanged) the near operator of the BEM tree; false when it
// does not fit the memory budget (the near-field kernel is used then)
bool near_matrix_build(const Tree& t, int nq, int64_t npanels, const int32_t* bc, const Material& m, NearMat& N,
                       cudaStream_t s);
// near[sorted target][3] = N x (x: panel vector [npanels x 3], caller order), fp64
void near_matrix_apply(const Tree& t, const NearMat& N, const double* x, double* near, cudaStream_t s);

}  // namespace ebem
