/*
 * mrlbm_gpu.h — C-ABI of the B200-native adaptive multiresolution lattice
 * Boltzmann (MR-LBM) time step.
 *
 * The reference (/root/reference/proj/core) is a header-only C++20 library with
 * no FFI; its "interface" is the SPEC data contracts.  Each entry point below
 * replaces one of them (file:line into /root/reference):
 *
 *   mrlbm_scheme_spec  <- SchemeSpec      SPEC.md:267-273 (q, eta^h, lambda, M, S,
 *                                         equilibrium, conserved moments)
 *                         DenseMatrix     dense_matrix.hpp:13-127 (M, M^-1 row-major)
 *   mrlbm_run_config   <- RunConfig       SPEC.md:512-515 (J_min, J_bar, epsilon,
 *                                         mu_guess, gamma), grading width SPEC.md:108,
 *                         DomainBox       cell.hpp:121-196 (base_cells, extents),
 *                         boundary kinds  SPEC.md:317-320 (+ periodic, velocity BB)
 *   mrlbm_create       <- run(config) initialisation
 *   mrlbm_load_leaves  <- FieldSet on S(Lambda) in CellIndex slot order
 *                         cell_set.hpp:326-354 (lexicographic, last axis fastest)
 *   mrlbm_step         <- one Algorithm-1 iteration
 *                         (adapt G∘H∘T, transfer, stream, collide, obstacle)
 *   mrlbm_read_leaves  <- FieldSet read-back (same slot order)
 *   mrlbm_last_error   <- C++ exceptions of the reference (std::invalid_argument,
 *                         std::domain_error, std::out_of_range; cell.hpp:85,107,
 *                         dense_matrix.hpp:62,81, prediction.hpp:38) become status
 *                         codes + message; no exception crosses the ABI.
 *
 * Ownership: inputs are copied; outputs go to caller buffers sized with
 * mrlbm_level_count.  The context owns all device memory and one CUDA stream.
 * Threading: one host thread per context; not reentrant.
 */
#ifndef MRLBM_GPU_H
#define MRLBM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRLBM_MAX_Q 16
#define MRLBM_MAX_LEVELS 16

/* status codes (SPEC.md:566 exit codes 0/2/3 extended) */
enum {
    MRLBM_OK = 0,
    MRLBM_ERR_CONFIG = 2,   /* ~ std::invalid_argument */
    MRLBM_ERR_NUMERIC = 3,  /* non-finite value / equilibrium domain */
    MRLBM_ERR_CUDA = 4,
    MRLBM_ERR_CAPACITY = 5, /* mesh invariant violated (unresolved stencil) */
    MRLBM_ERR_STATE = 6     /* call order (e.g. step before commit) */
};

/* boundary kinds per domain face (x-, x+, y-, y+, z-, z+) */
enum {
    MRLBM_BC_COPY = 0,              /* f^h(ghost) = f^{h*} of the adjacent interior leaf */
    MRLBM_BC_BOUNCE_BACK = 1,       /* f^h(ghost) = f^{h†*}            */
    MRLBM_BC_ANTI_BOUNCE_BACK = 2,  /* f^h(ghost) = -f^{h†*}            */
    MRLBM_BC_PERIODIC = 3,          /* wrap (not in SPEC; needed by config 3)          */
    MRLBM_BC_VELOCITY_BOUNCE_BACK = 4 /* f^{h†*} + bc_add[face][h] (moving wall/inlet) */
};

/* equilibrium maps m^eq(conserved moments) */
enum {
    MRLBM_EQ_BURGERS_D1Q2 = 1,     /* m^eq = (u, u^2/2)                       */
    MRLBM_EQ_EULER_D1Q3X3 = 2,     /* 3 x D1Q3: (u_i, F_i(u), lambda^2 u_i)   */
    MRLBM_EQ_ADVECTION_D2Q4 = 3,   /* (u, a u, b u, 0); eq_params = {a, b}    */
    MRLBM_EQ_EULER_D2Q4X4 = 4,     /* 4 x D2Q4: (u_i, Fx_i, Fy_i, 0)          */
    MRLBM_EQ_NS_D2Q9 = 5,          /* Lallemand-Luo; eq_params = {cs2, variant} */
    MRLBM_EQ_ADVECTION_D3Q6 = 6    /* (u, Vx u, Vy u, Vz u, 0, 0); eq_params = {Vx, Vy, Vz}
                                              */
};

/* SchemeSpec */
typedef struct mrlbm_scheme_spec {
    int32_t d;                 /* 1, 2 or 3 (3: the D3Q6 path) */
    int32_t q;                 /* populations, <= MRLBM_MAX_Q */
    int32_t nblocks;           /* vectorial schemes: M is block diagonal, q/nblocks per block */
    int32_t equilibrium;       /* MRLBM_EQ_* */
    double lambda;             /* lattice velocity dx/dt */
    int32_t eta[MRLBM_MAX_Q][3];        /* logical velocities */
    double M[MRLBM_MAX_Q * MRLBM_MAX_Q];    /* row-major q x q */
    double Minv[MRLBM_MAX_Q * MRLBM_MAX_Q]; /* row-major q x q, DenseMatrix::inverse order */
    double s[MRLBM_MAX_Q];     /* relaxation rates, 0 for conserved moments */
    double eq_params[8];       /* per equilibrium kind */
} mrlbm_scheme_spec;

/* RunConfig + DomainBox + boundaries + obstacle */
typedef struct mrlbm_run_config {
    int32_t j_min, j_max;      /* coarsest / finest level */
    int64_t base_cells[3];     /* cells per axis at j_min (DomainBox) */
    double origin[3];          /* domain origin (domain units) */
    double epsilon;            /* threshold; 0 = uniform mode */
    int32_t mu;                /* regularity guess mu_guess in [0, 2 gamma + 1] */
    int32_t gamma;             /* prediction half width (only 1) */
    int32_t graduation;        /* grading box half width (only 1 = gamma) */
    int32_t bc_kind[6];
    double bc_add[6][MRLBM_MAX_Q];
    int32_t obstacle;          /* 0 none, 1 disc (config 5) */
    int32_t obstacle_subsamples; /* per axis (16) */
    double obstacle_center[3];
    double obstacle_radius;
    double obstacle_feq[MRLBM_MAX_Q]; /* M^-1 m^eq(rho0, 0, 0) */
} mrlbm_run_config;

typedef struct mrlbm_step_stats {
    int32_t levels;                        /* j_max - j_min + 1 */
    int64_t leaves[MRLBM_MAX_LEVELS];      /* |S(Lambda)| per level after the last step */
    int64_t internal[MRLBM_MAX_LEVELS];    /* complete-tree internal cells */
    int64_t virtual_cells[MRLBM_MAX_LEVELS]; /* ghost + reconstruction-band cells */
    int64_t fallback_leaves;               /* leaves streamed by the recursive path */
    int64_t leaf_updates;                  /* sum over steps of |S(Lambda(t+dt))| */
    double ms_total;                       /* device time of the steps (CUDA events) */
    double ms_phase[8];                    /* see MRLBM_PHASE_* (only when profiling on) */
    int64_t bytes_model;                   /* algorithmic fp64 bytes of the last step (SURVEY 8d model) */
    int64_t bytes_stream;                  /* algorithmic bytes of the last step's stream+collide phase */
    int64_t kernel_launches;               /* CUDA kernels this call launched (graph nodes included) */
    /* algorithmic fp64 bytes of the LAST step per phase (MRLBM_PHASE_*), SURVEY 8d model with the
       old-tree counts taken before that step and N_G = 0 (virtual cells are not compulsory traffic):
       project 8q(N_S,old + 2 N_I,old), details 8q(N_S,old + N_I,old), flags / compact 0 (integer),
       transfer 8q(3 N_S,new + N_I,new), stream 8q(2 N_S,new); bytes_model = their sum */
    int64_t bytes_phase[8];
} mrlbm_step_stats;

enum {
    MRLBM_PHASE_PROJECT = 0,   /* K1 */
    MRLBM_PHASE_DETAILS = 1,   /* K2 */
    MRLBM_PHASE_FLAGS = 2,     /* K3: closure, enlarge, grade */
    MRLBM_PHASE_COMPACT = 3,   /* K4 */
    MRLBM_PHASE_TRANSFER = 4,  /* K5 + K6 + virtual values */
    MRLBM_PHASE_STREAM = 5,    /* K7/K8 stream + collide (+ obstacle) */
    MRLBM_PHASE_COUNT = 6
};

/* Near-threshold tie record (BASELINE north_star: "except where a detail lies within
   1e-12 relative of its threshold; any such case is logged").
   The thresholds stay inclusive (metric >= threshold keeps). */
typedef struct mrlbm_tie_record {
    int32_t step;        /* 1-based step since mrlbm_commit in which the group was tested */
    int32_t level;       /* level l of the sibling group (its parent lies at l - 1)       */
    int32_t cell[3];     /* parent cell coordinates at level l - 1 (unused axes 0)        */
    int32_t which;       /* 0: keep threshold eps_l = 2^{d(l-J)} eps (Eq. 10);
                            1: blow-up threshold 2^{mu+d} eps_l           */
    double metric;       /* group metric max |d| over siblings and populations */
    double threshold;
} mrlbm_tie_record;

typedef struct mrlbm_ctx mrlbm_ctx;

int mrlbm_create(const mrlbm_scheme_spec* scheme, const mrlbm_run_config* cfg, mrlbm_ctx** out);
/* leaves of one level: n cells, idx = n*d int32 coordinates (CellIndex order),
   f = q*n doubles, SoA (f[h*n + i]).  Call for every level, then mrlbm_commit. */
int mrlbm_load_leaves(mrlbm_ctx* ctx, int level, int64_t n, const int32_t* idx, const double* f);
int mrlbm_commit(mrlbm_ctx* ctx);
int mrlbm_step(mrlbm_ctx* ctx, int nsteps, mrlbm_step_stats* stats);
int mrlbm_level_count(mrlbm_ctx* ctx, int level, int64_t* n);
int mrlbm_read_leaves(mrlbm_ctx* ctx, int level, int32_t* idx, double* f);
/* Tie log since commit (or the last reset): every group metric m with
   |m - t| <= 1e-12 t for t = eps_l or 2^{mu+d} eps_l (t > 0), sorted by
   (step, level, cell, which).  n = records logged; at most cap are copied.  Status 5
   when more records were logged than the device buffer holds (65536).  reset != 0
   clears the log.  The oracle logs the same records (tests/test_ties.py). */
int mrlbm_tie_log(mrlbm_ctx* ctx, mrlbm_tie_record* out, int cap, int64_t* n, int reset);
/* Profiling of the following mrlbm_step calls (eager launches instead of the step graph):
   on = 1: a CUDA event after every kernel, everything on one stream (mrlbm_profile_text,
           ms_phase); on = 2: phase events only, the step's independent launches forked onto
           side streams as in the graph (ms_phase adds up to the step); 0: off. */
int mrlbm_set_profiling(mrlbm_ctx* ctx, int on);
int mrlbm_set_graph(mrlbm_ctx* ctx, int on);
/* per-kernel device times accumulated over profiled steps: lines "kernel level ms launches" */
int mrlbm_profile_text(mrlbm_ctx* ctx, char* buf, int cap, int reset);
void* mrlbm_stream_handle(mrlbm_ctx* ctx);   /* cudaStream_t of the context */
int mrlbm_synchronize(mrlbm_ctx* ctx);
const char* mrlbm_last_error(const mrlbm_ctx* ctx);
void mrlbm_destroy(mrlbm_ctx* ctx);

/* ---- diagnostics (the reference has no implementation) ---- */
/* cells of the finest level (the full finest grid), n = prod(base_cells) * 2^(d (j_max - j_min)) */
int mrlbm_finest_count(const mrlbm_ctx* ctx, int64_t* n);
/* Zero-detail reconstruction f^^ of the current state on the full finest grid
   (§4.4): f[h*n + lin], lin lexicographic (axis 0 slow).
   f == NULL keeps it on the device only. */
int mrlbm_reconstruct_finest(mrlbm_ctx* ctx, double* f);
/* Additional error E[m] = sum |m^^ - m_ref| / sum |m_ref| over the finest grid
   (SPEC.md:450-458), m = sum_h row[h] f^h, both contexts
   reconstructed on their devices (the reference is typically an epsilon = 0 run
   on the full finest mesh, the uniform solver of SPEC.md:326-334).  A zero
   reference moment (sum < 1e-300) reports the absolute error.
   sums (optional, 2 doubles) = {sum |m^^ - m_ref|, sum |m_ref|}. */
int mrlbm_additional_error(mrlbm_ctx* adaptive, mrlbm_ctx* reference, const double* row, double* E,
                           double* sums);

/* ---- config-5 integral diagnostics ---- */
/* Obstacle force tracking.  capacity_steps > 0 records, for each following step, the
   force on the obstacle F = sum over leaves of alpha * q * |cell| / dt: the momentum the
   obstacle blend removes per unit time (SPEC.md:476 design decision),
   q = post-collision momentum moments (m_1, m_2), dt = 2^-J_bar / lambda.  Summed on the
   device in a fixed order (deterministic).  0 turns it off.  Needs the D2Q9 obstacle
   configuration (status 2 otherwise). */
int mrlbm_set_force_tracking(mrlbm_ctx* ctx, int capacity_steps);
/* per-step forces recorded since tracking was enabled: fx[i], fy[i] for i < min(n, cap);
   n = steps recorded (status 5 when n exceeds the capacity given to set_force_tracking) */
int mrlbm_force_history(mrlbm_ctx* ctx, double* fx, double* fy, int cap, int* n);
/* C_D = 2 F_x / (rho0 u0^2 L), C_L = 2 F_y / (rho0 u0^2 L) */
int mrlbm_drag_lift(double fx, double fy, double rho0, double u0, double L, double* cd, double* cl);
/* Strouhal number St = L f / u0 of a lift series sampled every dt (PAPER.md:1380-1383,
   SPEC.md:477-485): samples [skip, n) are detrended (least-squares line), Hann-windowed
   and transformed by a direct DFT; f = the bin of the largest non-zero-frequency
   power.  df (optional) = the frequency resolution 1 / ((n - skip) dt).  Status 3
   ("no dominant peak") when the detrended series is flat or the peak power is below
   4x the mean power of the other bins; status 2 for fewer than 8 samples. */
int mrlbm_strouhal(const double* cl, int64_t n, int64_t skip, double dt, double u0, double L, double* st,
                   double* df);

/* Flattened reconstruction table:
   sum over the E (side=0) or A (side=1) finest cells of a leaf at gap g of the
   zero-detail reconstruction == sum_i w_i f(l, k + off_i).  Lexicographic
   offsets, non-zero weights only.  offsets: cap*d int32, weights: cap doubles. */
int mrlbm_stream_table(int d, int gap, const int32_t eta[3], int side, int cap,
                       int32_t* offsets, double* weights, int* n);

/* Exactness sets of that table (Decision D.13): dep_box = {xlo, xhi, ylo, yhi} of
   the level-l cells the zero-detail recursion touches (must lie in the domain),
   par_offsets = parents of the level-(l+1) cells it touches (must not be internal). */
int mrlbm_stream_table_sets(int d, int gap, const int32_t eta[3], int side, int cap, int32_t* dep_box,
                            int32_t* par_offsets, int* npar);

/* Host-side builders for the five BASELINE configurations (Decisions).
   config_id 1..5 (config 3 with epsilon override 0 = the uniform run).
   j_max_override > 0 replaces J_bar (parity tests run reduced sizes);
   eps_override >= 0 replaces epsilon. */
int mrlbm_build_config(int config_id, int j_max_override, double eps_override,
                       mrlbm_scheme_spec* scheme, mrlbm_run_config* cfg);
/* number of steps N = ceil(T / dt) for the config at its J_bar */
int64_t mrlbm_config_steps(int config_id, const mrlbm_run_config* cfg);
/* Initial datum on the full finest mesh at equilibrium:
   f = M^-1 m^eq(u0(cell centre)), SoA q x N, N = cells at j_max in CellIndex order. */
int mrlbm_initial_finest(int config_id, const mrlbm_scheme_spec* scheme,
                         const mrlbm_run_config* cfg, uint64_t seed, double* f);

#ifdef __cplusplus
}
#endif
#endif /* MRLBM_GPU_H */
