// BEM panel operators in HBM: near field, S2M and S2L check potentials (see bem_near.cu)
#pragma once
#include "fmm.cuh"

namespace ebem {

struct PanelOp {
    enum Kind { NEAR = 0, S2M = 1, S2L = 2 };
    Kind kind = NEAR;
    bool ready = false;
    long long entries = 0;        // floats in M
    DBuf<int> col_first, ncol;    // per row set: first column, column count
    DBuf<int> seg_start;          // per column: first entry in the sorted (set, panel) list
    DBuf<int> col_panel;          // per column: panel index
    DBuf<int> vals;               // build scratch: sorted sources of the (set, panel) list
    DBuf<long long> moff;         // per row set: offset of its [9][rows][ncol] block in M
    DBuf<float> M;
    DBuf<int32_t> bc;             // boundary-condition types the blocks were built for
    void release() {
        ready = false;
        entries = 0;
        for (DBuf<int>* b : {&col_first, &ncol, &seg_start, &col_panel, &vals}) b->release();
        moff.release();
        M.release();
        bc.release();
    }
};
using NearMat = PanelOp;

bool near_matrix_enabled();
bool check_matrix_enabled();
// builds (or keeps, when bc is unchanged) one panel operator of the BEM tree; false when it
// does not fit the memory budget (the kernel path is used then)
bool panel_op_build(const Tree& t, PanelOp::Kind kind, int nq, int64_t npanels, const int32_t* bc,
                    const Material& m, PanelOp& N, cudaStream_t s);
// near: near[sorted target][3] = N x (fp64);  S2M / S2L: check potential rows of N x written
// as the TF32 split to Qb / Qs (row = set index, leading dimension ldq)
void panel_op_apply(const Tree& t, const PanelOp& N, const double* x, double* near, float* Qb, float* Qs, int ldq,
                    cudaStream_t s);
bool near_matrix_build(const Tree& t, int nq, int64_t npanels, const int32_t* bc, const Material& m, NearMat& N,
                       cudaStream_t s);
// near[sorted target][3] = N x (x: panel vector [npanels x 3], caller order), fp64
void near_matrix_apply(const Tree& t, const NearMat& N, const double* x, double* near, cudaStream_t s);

}  // namespace ebem
