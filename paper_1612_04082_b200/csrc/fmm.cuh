// Tree, plan and pass declarations of the B200 KIFMM (Sec. 2.2).
//
// Representation ("well-conditioned KIFMM state"): the paper's
// equivalent densities phi (line 147) are never stored in fp32.  Each box keeps the
// rotated check potential
//     z_B = Q_u1^T q_u(B)   (upward)      w_B = Q_d1^T q_d(B)   (downward)
// where [K_uc<-ue ; a I] = Q_u R_u is the QR factorisation of the Tikhonov-augmented
// check-to-equivalent kernel matrix at unit scale (Q_u1 = its first 3 n_c rows), so
// phi = r R_u^-1 z.  The M2M / M2L / L2L operators of line 149 become composites
//     M2M_c = Q_u1^T (1/2 K(uc_P, ue_C)) R_u^-1,  M2L_o = Q_d1^T K(dc_B, ue_A) R_u^-1,
//     L2L_c = Q_d1^T K(dc_C, de_P) R_d^-1
// computed once in fp64 and applied in fp32: they map well-scaled vectors to
// well-scaled vectors (|z| <= |q|), so fp32 rounding is not amplified by the
// ill-conditioned solve.  phi is only formed (in fp64) for the leaf evaluations
// L2T and M2T.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <functional>
#include <map>
#include <memory>
#include <mutex>

#include "../../include/elastobem.h"
#include "common.cuh"

namespace ebem {

// 2^(12 - floor(log2 amax)): the power-of-two row scale of the FP16 operand splits (tc_gemm.cu,
// reading R14), 1 for an all-zero (or non-finite) row
__device__ __forceinline__ float pow2_scale(float amax) {
    if (!(amax > 0.f) || !isfinite(amax)) return 1.f;
    return scalbnf(1.f, 12 - ilogbf(amax));
}

constexpr int MAXLEVEL = 20;
constexpr double RAD_UE = 1.05, RAD_UC = 2.95, RAD_DE = 2.95, RAD_DC = 1.05;
constexpr int NV_OFFSETS = 316;        // 7^3 - 3^3 M2L translation vectors

// ------------------------------------------------------------------ plan (operators)
struct Plan {
    int p = 0, pc = 0;          // equivalent / check surface points per edge (pc = p + 1)
    int ne = 0, nc = 0;         // surface point counts
    int me = 0, mc = 0;         // 3 ne, 3 nc (vector lengths)
    int lde = 0, ldc = 0;       // row strides (me, mc rounded up to a multiple of 4: 16-B TMA rows)
    double rcond = 0;
    Material mat{};
    DBuf<float> s_e, s_c;       // unit surface grids [ne*3], [nc*3] (fp32 copies)
    DBuf<double> s_e64, s_c64;
    DBuf<float4> s_e4;          // unit equivalent surface as float4 (fp32 far field)
    DBuf<float> Qu1T, Qd1T;     // [me x ldc] row-major: z = Qu1T q
    DBuf<double> Ruinv, Rdinv;  // [me x me] row-major upper triangular: phi = r Rinv z
    DBuf<float> M2M, L2L;       // [8][me x lde]
    DBuf<float> M2L;            // [316][me x lde]
    // exact-TF32 head / remainder splits of the operators (3xTF32 tensor-core path)
    DBuf<float> Qu1T_b, Qu1T_s, Qd1T_b, Qd1T_s, M2M_b, M2M_s, L2L_b, L2L_s, M2L_b, M2L_s;
    CUtensorMap mQu1T_b, mQu1T_s, mQd1T_b, mQd1T_s, mM2M_b, mM2M_s, mL2L_b, mL2L_s, mM2L_b, mM2L_s;
    // scaled FP16 head / remainder copies of the M2L operators (3xFP16 path, tc_gemm.cu): row
    // stride ldh halves (me rounded up to 8: 16-B rows), one power-of-two scale for the set
    // (m2l_hinv undoes it)
    DBuf<__half> M2L_hb, M2L_hs, M2M_hb, M2M_hs, L2L_hb, L2L_hs, Qu1T_hb, Qu1T_hs;
    CUtensorMap mM2L_hb, mM2L_hs, mM2M_hb, mM2M_hs, mL2L_hb, mL2L_hs, mQu1T_hb, mQu1T_hs;
    int ldh = 0, ldch = 0;      // half row strides of the me- and mc-long rows
    float m2l_hinv = 1.f, m2m_hinv = 1.f, l2l_hinv = 1.f, qu_hinv = 1.f;
    int off_index[343];         // (ox+3)*49+(oy+3)*7+(oz+3) -> 0..315 or -1
};

std::shared_ptr<Plan> get_plan(int p, const Material& m, cudaStream_t s);

// ------------------------------------------------------------------ pair lists
// Work grouped by operator: pairs (target row, source row) sorted by op.
struct OpPairs {
    int nops = 0;
    int64_t npairs = 0;
    DBuf<int> op_ptr;            // [nops+1]
    DBuf<int2> pairs;            // [npairs] (target row, source row)
    std::vector<int> op_ptr_h;   // host copy (launch sizing)
    int max_per_op = 0;
    int ntiles = 0;              // tensor-core tiles (op, first pair, #pairs, row block)
    int tile_mode = 0;           // tile shape: 0 128 rows x 128 pairs (precise), 1 256 x 128 (fast /
                                 // drained two-slice), 2 128 x 256 (wide, full-chain), 3 two-slice tiles in cluster order
    int tile_cs = 1;             // CTAs per cluster tile (tile_mode 3: tc_pairs_mc_kernel), else 1
    int tile_bke = 32;           // K elements per 128-B chunk the tiles were cut for: 32 (TF32) or 64 (FP16)
    DBuf<int> tiles;
};

// a level chain (M2M or L2L) run as one cooperative launch (tc_gemm.cu, tc_chain_kernel)
struct ChainArgs {
    int nlev;
    int lvl_tile[MAXLEVEL + 1];          // tiles of chain level i: [lvl_tile[i], lvl_tile[i + 1])
    long long row0[MAXLEVEL], nrows[MAXLEVEL];   // source rows split before level i
    long long tail_row0, tail_rows;      // rows split after the last level (upward chain)
};
struct Chain {
    int nlev = 0;
    std::vector<int> lvl_tile;
    std::vector<int64_t> row0, nrows;
    DBuf<int> tiles;
    DBuf<int2> pairs;
    DBuf<unsigned> bar;                  // grid-barrier counter (cleared before each launch), level times
};

// ------------------------------------------------------------------ tree
struct Tree {
    int64_t nsrc = 0, ntrg = 0, npts = 0;
    int max_pts = 0, p = 0;
    double w_direct = 1.0;               // R11: W box summed directly below w_direct x n_e sources
    Material mat{};
    bool has_normals = false, has_weights = false;
    double origin[3] = {0, 0, 0}, side = 1;
    int nlevels = 0, nboxes = 0, nleaves = 0;
    std::vector<int> level_start;       // host [nlevels+1]

    // points, sorted by Morton key (stable: sources first, then targets)
    DBuf<long long> keys;               // [npts]
    DBuf<int> perm;                     // sorted pos -> original point index
    DBuf<int> src_perm, trg_perm;       // sorted source/target pos -> original index
    DBuf<float> src_xyz, src_nrm, src_w, trg_xyz;   // sorted copies

    // boxes (level then Morton order)
    DBuf<int> level, anchor, parent, child, pbeg, pend;
    DBuf<int> sbeg, send, tbeg, tend;   // ranges in the sorted source / target arrays
    DBuf<int> nsrc_sub, ntrg_sub;       // sources / targets in the subtree (= in range)
    DBuf<long long> bkey;               // Morton key of the box at its level
    DBuf<int> is_leaf;
    DBuf<int> colleague;                // [nboxes*27] same-level neighbours (-1 absent)
    DBuf<int> lst_off[4], lst_idx[4];   // U, V, W, X lists (CSR, ascending ids)
    int64_t lst_n[4] = {0, 0, 0, 0};

    // execution plan
    std::shared_ptr<Plan> plan;
    int n_up = 0;                        // boxes carrying z (level >= 2, sources in subtree)
    DBuf<int> up_slot;                   // box -> row in Z (-1 none)
    int n_dn = 0;                        // boxes carrying w (level >= 2, targets in subtree)
    DBuf<int> dn_slot;                   // box -> row in W (-1 none)
    // S2M: leaves with sources (rows of Z); S2L: boxes with X lists (rows of W)
    int n_s2m = 0, n_s2l = 0;
    DBuf<int> s2m_box, s2l_box;
    DBuf<int> x_src_off, x_src_idx;       // S2L: per s2l box, the X-list leaves (source boxes)
    OpPairs q2z_up, q2z_dn;              // check potential -> z / w (single op)
    std::vector<OpPairs> m2m;            // per level (parents at that level), 8 ops
    OpPairs m2l;                         // all levels, 316 ops
    std::vector<OpPairs> l2l;            // per level (children at that level), 8 ops
    Chain m2m_chain, l2l_chain;          // the same, one cooperative launch per pass (ml_chain)
    bool ml_chain = false;
    // leaf evaluation
    int n_eval = 0;                      // leaves with targets
    DBuf<int> eval_box;                  // [n_eval]
    DBuf<int> eval_l2t_slot;             // row in PHI_D (-1 if leaf level < 2)
    DBuf<int> far_box, far_l2t_slot;     // the same leaves in the far-field kernel's order
    int n_phid = 0;                      // leaves with L2T
    DBuf<int> phid_box;                  // [n_phid] (box ids) for the fp64 phi reconstruction
    int n_phiu = 0;                      // boxes appearing in some W list (with sources)
    DBuf<int> phiu_box, phiu_slot;       // [n_phiu] box ids; box -> row in PHI_U (-1)
    OpPairs phid_pairs, phiu_pairs;      // single-op pairs for the fp64 reconstruction GEMM
    DBuf<double> phid_scale, phiu_scale; // half-width r of the box of each PHI row
    std::vector<int> up_lstart, dn_lstart;  // per level: first Z / W row (rows are level-major)
    bool use_tc = true;                  // tcgen05 3xTF32 translations (else SIMT fp32)
    bool far64 = false;                  // L2T / M2T in fp64 (set for p >= 9 and by the BEM operator)
    bool tc_fast = false;                // p <= 8 plain matvec: two-slice full-K tensor-core kernel
    bool ml_fast = false;                // Q2Z / M2M / L2L on the fast kernel too

    // profiling (fmm_set_profiling / fmm_phase_stats): 0 off; 1 phases one after another on
    // the caller's stream (solo times); 2 in situ: the normal two-stream schedule, each phase
    // bracketed by timing events on the stream it is launched on.  Every profiled evaluation
    // records into the next of PROF_RING event sets; fmm_phase_stats averages the sets
    // recorded since profiling was switched on (at most the last PROF_RING).
    static constexpr int NPHASE = 11, PROF_RING = 64;
    int profile = 0;
    struct ProfSet {
        cudaEvent_t b[NPHASE] = {}, e[NPHASE] = {};
        cudaEvent_t from[NPHASE] = {};   // the event a phase's time is measured from
        bool used[NPHASE] = {};
    };
    std::vector<ProfSet> prof_ring;
    int prof_count = 0;                  // evaluations recorded since fmm_set_profiling
    int phase_launches[NPHASE] = {};
    // algorithmic work counts (schedule time)
    double w_s2m_inter = 0, w_s2l_inter = 0, w_p2p_inter = 0, w_l2t_inter = 0, w_m2t_inter = 0;
    double w_s2m_src = 0, w_s2l_src = 0, w_p2p_src = 0;
    int64_t w_m2m_pairs = 0, w_l2l_pairs = 0;
    int w_m2l_ops = 0;
    ~Tree() {
        for (auto& ps : prof_ring)
            for (int i = 0; i < NPHASE; ++i) {
                if (ps.b[i]) cudaEventDestroy(ps.b[i]);
                if (ps.e[i]) cudaEventDestroy(ps.e[i]);
            }
        for (cudaEvent_t e : {ev_fork, ev_s2l, ev_near, ev_joinA, ev_m2l, ev_zz, ev_wz})
            if (e) cudaEventDestroy(e);
        if (sA) cudaStreamDestroy(sA);
        if (sB) cudaStreamDestroy(sB);
    }

    // workspace (allocated at build time; evaluation allocates nothing)
    DBuf<float4> rec_disp, rec_stress;   // prepared sources, tree order
    DBuf<float> Q, Qd;                   // check potentials [n_s2m x mc] (S2M), [n_s2l x mc] (S2L)
    DBuf<double> Z, W;                   // [n_up x lde], [n_dn x lde] accumulators: fp64 atomics make
                                         // the sum order-independent at fp32 precision (deterministic)
    DBuf<float> Qb, Qs, Qdb, Qds, Zb, Zs, Wb, Ws;   // TF32 head / remainder copies (B operands)
    CUtensorMap mQb, mQs, mQdb, mQds, mZb, mZs, mWb, mWs;
    // 3xFP16 M2L: row-scaled fp16 head / remainder copies of the Z rows and the factors undoing
    // each row's scale (split once per evaluation, after the upward pass)
    DBuf<__half> Zhb, Zhs, Whb, Whs;
    DBuf<float> Zhinv, Whinv;
    bool m2l_f16 = false;                // M2L operands in FP16 (EBEM_M2L_F16, default on)
    bool ml_f16 = false;                 // M2M / L2L on the fast kernel in FP16 too (split level by level)
    bool ml_drain = false;               // ... with drained accumulation (p = 7, 8; ml_fast false)
    DBuf<__half> Qhb, Qhs;               // FP16 split of the S2M check potentials (written by the S2M kernel)
    DBuf<float> Qhinv;
    bool q2z_f16 = false;                // upward Q2Z on FP16 operands (not with the BEM's stored S2M operator)
    DBuf<double> PHID, PHIU;             // [n_phid x me], [n_phiu x me] (fp64 far field)
    DBuf<float4> PHIDF, PHIUF;           // [n_phid x ne], [n_phiu x ne] (fp32 far field, scaled)
    DBuf<float> near_sorted;             // [ntrg x 6] near field, sorted target order
    // BEM operator inside GMRES (bem.cu): the near hook writes the near field in fp64 to
    // near_sorted_d (near_f64), and the fp64 far field writes its sum to out_d instead of the
    // float output, so the Krylov vectors meet no fp32 rounding outside the FMM's far field
    DBuf<double> near_sorted_d;
    bool near_f64 = false;
    double* out_d = nullptr;
    std::function<void(cudaStream_t)> near_hook;   // replaces the near-field kernel (BEM near operator)
    std::function<void(cudaStream_t)> s2m_hook;    // replaces the S2M check potentials (BEM S2M operator)
    std::function<void(cudaStream_t)> s2l_hook;    // replaces the S2L check potentials (BEM S2L operator)
    bool force_serial = false;                     // one stream (the BEM inside GMRES, measured faster)
    DBuf<int> ssplit;                    // BEM: per leaf, first source of the second boundary-condition group
    int split_mode = 0;                  // 0 off; 1: [sbeg, ssplit) single layer, rest double layer; 2 reverse
    DBuf<int> near_off, near_idx;        // per box: source boxes summed directly (U + direct X/W)
    DBuf<int> m2t_off, m2t_idx;          // per box: W-list boxes evaluated from their equivalent density
    // two-stream schedule (fmm_evaluate): created on first use
    cudaStream_t sA = nullptr, sB = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_s2l = nullptr, ev_near = nullptr, ev_joinA = nullptr, ev_m2l = nullptr,
                ev_zz = nullptr, ev_wz = nullptr;
    int64_t device_bytes = 0;
};

// w_direct: W entries whose box holds fewer sources than w_direct x n_e are summed directly (R11)
Tree* build_tree(const float* src, const float* nrm, const float* w, int64_t nsrc, const float* trg,
                 int64_t ntrg, int max_pts, int p, const Material& m, cudaStream_t s, double w_direct = 1.0);
void fmm_evaluate(Tree& t, int kernel, const float* f, const float* g, float* out, cudaStream_t s);
void tree_info(const Tree& t, ebem_tree_info* info);
int64_t tree_export(const Tree& t, int what, void* buf, int64_t cap);
int phase_stats(Tree& t, int kernel, ebem_phase_stat* out, int cap);
void set_profiling(Tree& t, int mode);
struct Bem;
Bem* bem_create(const float* verts, int64_t n, int nq, int max_pts, int p, const Material& m, cudaStream_t s);
void bem_free(Bem* B);
void bem_apply(Bem& B, const int32_t* bc, const float* x, float* y, cudaStream_t s);
void bem_rhs(Bem& B, const int32_t* bc, const float* val, float* b, cudaStream_t s);
int bem_gmres(Bem& B, const int32_t* bc, const float* val, float* x, int m, int max_iter, double tol,
              int32_t* iters, double* resid, int precond, cudaStream_t s);
int bem_history(const Bem& B, int what, double* buf, int cap);

// ------------------------------------------------------------------ primitives (linalg.cu)
// exclusive scan of n ints (out may alias in); returns the total on the host (syncs)
int64_t exclusive_scan_i32(const int* in, int* out, int64_t n, cudaStream_t s);
// stable LSD radix sort of (key, value) pairs on the low `bits` bits of the keys
void radix_sort_pairs(long long* keys, int* vals, int64_t n, int bits, cudaStream_t s);
// C[b] = alpha * A[b] * B[b] (+ beta C[b]); row-major; fp64; batch strides in elements
void gemm_f64(int m, int n, int k, double alpha, const double* A, int64_t sA, int lda,
              const double* B, int64_t sB, int ldb, double beta, double* C, int64_t sC, int ldc,
              int batch, cudaStream_t s);
// pairs GEMM: Y[t] += Mat[op] * X[src] for every pair (t, src) of every op; Mat row-major
// [M x K]; X rows of length ldx >= K; Y rows of length ldy >= M.  fp32.
template <class XT>
void gemm_pairs_f32(const OpPairs& P, const float* mats, int M, int K, int ldm, const XT* X, int ldx,
                    double* Y, int ldy, cudaStream_t s);
// tensor-core path (tc_gemm.cu)
void tc_make_map_a(CUtensorMap* m, const float* base, int nops, int M, int K, int ld);
void tc_make_map_b(CUtensorMap* m, const float* base, int64_t rows, int K, int ld);
template <class XT>
void tc_split_rows(const XT* X, int ld, int64_t row0, int64_t nrows, int K, float* Xb, float* Xs,
                   cudaStream_t s);
void tree_precise(Tree& t, cudaStream_t s);
void tree_partition_sources(Tree& t, const int32_t* bc, int nq, cudaStream_t s);
void tree_m2l_fast(Tree& t, bool fast, cudaStream_t s);
void tc_build_tiles(OpPairs& P, int M, int K, int mode, int bke = 32, int cs = 1);
void tc_make_map_a_h(CUtensorMap* m, const __half* base, int nops, int M, int K, int ldh);
float tc_split_ops_h(const float* X, int ld, int64_t nrows, int K, __half* Xh, __half* Xr, int ldh, cudaStream_t s);
void tc_split_rows_h(const double* X, int ldx, int64_t row0, int64_t nrows, int K, __half* Xh, __half* Xr, int ldh,
                     float* inv_scale, cudaStream_t s);
void tc_build_chain(Chain& ch, const std::vector<const OpPairs*>& levels, const std::vector<int64_t>& row0,
                    const std::vector<int64_t>& nrows, int M, int K, cudaStream_t s);
// X: fp64 state rows (ldx), split into Xb / Xs level by level ([row0, row0 + nrows) before
// each level, [tail_row0, tail_row0 + tail_rows) after the last); Y += translations
void tc_chain_run(const Chain& ch, const CUtensorMap& Ab, const CUtensorMap& As, const double* X, int ldx, float* Xb,
                  float* Xs, int M, int K, double* Y, int ldy, int64_t tail_row0, int64_t tail_rows, cudaStream_t s);
int tc_fast_tile_mode(int M);                  // full-chain tile shape for M operator rows: 1 two-slice, 2 wide
int tc_fast_smem_bytes();                     // dynamic shared memory of one fast translation CTA
int beside_translation_pad(const void* kernel);   // fmm.cu: stream-B co-residency padding
void tc_pairs_gemm_fast(const OpPairs& P, const CUtensorMap& Ab, const CUtensorMap& As, const void* Bb,
                        const void* Bs, int ldb, int M, int K, double* Y, int ldy, bool drain, cudaStream_t s,
                        bool f16 = false, const float* bscale = nullptr, float ascale_inv = 1.f);
void tc_pairs_gemm(const OpPairs& P, const CUtensorMap& Ab, const CUtensorMap& As, const CUtensorMap& Bb,
                   const CUtensorMap& Bs, int M, int K, double* Y, int ldy, cudaStream_t s);
// fp64 variant with per-pair scale (r of the box, looked up from scale[t])
void gemm_pairs_f64(const OpPairs& P, const double* mat, int M, int K, const double* X, int ldx,
                    const double* scale, double* Y, int ldy, cudaStream_t s);
// the same with fp32 output in the far-field layout: row t = M/3 float4 (cf * value, 0)
void gemm_pairs_f64_to_f32(const OpPairs& P, const double* mat, int M, int K, const double* X, int ldx,
                           const double* scale, double cf, float4* Y, int ldy, cudaStream_t s);
void build_op_pairs(OpPairs& P, int nops, const std::vector<int>& op, const std::vector<int2>& pr,
                    cudaStream_t s);

}  // namespace ebem
