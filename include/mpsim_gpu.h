/*
 * mpsim_gpu.h — C ABI of the B200-native MPS gate-application engine.
 *
 * Drop-in boundary for the reference mpsim simulator API (arXiv 2601.04422
 * TN-Sim; /root/reference/proj). Every entry point cites the reference
 * interface it replaces. Plain pointers and sizes only; complex numbers are
 * interleaved (re, im) doubles; matrices and site tensors are row-major with
 * the last index fastest (tensor.hpp:17-18, :116-125); a site is (Dl, 2, Dr)
 * with flat index (l*2 + p)*Dr + r (mps.hpp:36-40).
 *
 * Status codes (the reference's C++ exceptions, mapped like
 * exit_code_for_error, runner.cpp:330-341):
 *   MPSIM_OK 0, MPSIM_EINVAL 1 (std::invalid_argument / ConfigError),
 *   MPSIM_EPARSE 2 (ParseError, front end only), MPSIM_ENUMERIC 3
 *   (mpsim::NumericError), MPSIM_ELOGIC 4 (std::logic_error), MPSIM_ECUDA 5
 *   (device/runtime failure). mpsim_gpu_last_error() returns the message of
 *   the calling thread's last failure.
 *
 * Threading: a state handle is not thread-safe (the reference MpsState is
 * shared only through execute_parallel's disjoint-span contract,
 * gate_apply.hpp:20-24); batching disjoint gates is done inside
 * mpsim_gpu_apply_layer / mpsim_gpu_execute.
 */
#ifndef MPSIM_GPU_H_
#define MPSIM_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPSIM_OK 0
#define MPSIM_EINVAL 1
#define MPSIM_EPARSE 2 /* mpsim::ParseError, errors.hpp:22-37 */
#define MPSIM_ENUMERIC 3
#define MPSIM_ELOGIC 4
#define MPSIM_ECUDA 5

#define MPSIM_UNBOUNDED INT64_MAX /* kUnbounded, tensor.hpp:44 */

#define MPSIM_NONLOCAL_SWAP 0     /* NonlocalMethod::Swap, gate_apply.hpp:71 */
#define MPSIM_NONLOCAL_BONDPROP 1 /* NonlocalMethod::BondProp */

typedef struct mpsim_gpu_state mpsim_gpu_state;

/* TruncationPolicy, gate_apply.hpp:35-38 (max_bond >= 1, cutoff in [0,1)). */
typedef struct {
  int64_t max_bond;
  double cutoff;
} mpsim_policy;

/* ApplyReport, gate_apply.hpp:40-44. */
typedef struct {
  double discarded_weight;
  int64_t new_bond;
  int32_t svd_count;
  int32_t reserved;
} mpsim_report;

/* FusedGate, circuit.hpp:71-81: q1 = -1 for a one-qubit gate. Two-qubit
 * gates take (q0, q1) in any order with the 4x4 matrix in the (q0, q1)
 * basis (row = 2*bit(q0) + bit(q1)); (high, low) orders are folded by SWAP
 * conjugation (gates.cpp:206, gate_apply.cpp:156-159). u holds 4 (2x2) or
 * 16 (4x4) interleaved complex entries. */
typedef struct {
  int32_t q0;
  int32_t q1;
  double u[32];
} mpsim_gate;

/* ExecStats, executor.hpp:44-57. */
typedef struct {
  int64_t peak_bond;
  double total_discarded_weight;
  int32_t layers;
  int32_t gates;          /* local gates executed after SWAP lowering */
  int64_t kernel_launches; /* device kernels launched by the call */
  double device_ms;        /* CUDA-event time of the call on the state's stream */
} mpsim_exec_stats;

const char* mpsim_gpu_last_error(void);

/* ---- state (MpsState, mps.hpp:33-75) ---------------------------------- */
/* |0...0> on n qubits (mps.cpp:99-110). chi_hint sizes the padded site
 * store; it grows on demand. device = CUDA ordinal. */
int mpsim_gpu_state_create(int32_t n_qubits, int64_t chi_hint, int32_t device, mpsim_gpu_state** out);
int mpsim_gpu_state_destroy(mpsim_gpu_state* s);
int mpsim_gpu_state_copy(const mpsim_gpu_state* s, mpsim_gpu_state** out); /* mps.cpp:112-130 */
int mpsim_gpu_num_qubits(const mpsim_gpu_state* s, int32_t* out);
int mpsim_gpu_bond_dims(const mpsim_gpu_state* s, int64_t* out /* n+1 */); /* mps.hpp:49-52 */
int mpsim_gpu_chi_capacity(const mpsim_gpu_state* s, int64_t* out);
int mpsim_gpu_ortho_center(const mpsim_gpu_state* s, int32_t* out /* -1 unknown */); /* mps.hpp:57-60 */
int mpsim_gpu_set_ortho_center(mpsim_gpu_state* s, int32_t c);
int mpsim_gpu_set_bond_dim(mpsim_gpu_state* s, int32_t i, int64_t d); /* mps.hpp:50 */
int mpsim_gpu_validate(const mpsim_gpu_state* s); /* mps.cpp:150-169 */
/* Host export/import of one site (MpsState::site(i), mps.hpp:45-46):
 * get with out == NULL only reports dims; set replaces site i and records
 * bonds i and i+1 (test_util.cpp:104-106). */
int mpsim_gpu_get_site(const mpsim_gpu_state* s, int32_t i, int64_t* dl, int64_t* dr, double* out);
int mpsim_gpu_set_site(mpsim_gpu_state* s, int32_t i, int64_t dl, int64_t dr, const double* data);

/* ---- site-sharded chains (multi-GPU) -----------------------
 * A shard holds a contiguous site range of a longer chain, so its boundary
 * bonds may exceed 1 (validate then skips the "boundary bonds are 1" check).
 * Boundary sites move between shards as whole padded slots (chi x 2 x chi
 * complex128, contiguous) over NCCL; site_slot exposes the device address of
 * a slot and set_site_dims records the extents of a slot written that way. */
int mpsim_gpu_set_open_boundaries(mpsim_gpu_state* s, int32_t open);
int mpsim_gpu_site_slot(const mpsim_gpu_state* s, int32_t i, void** device_ptr, int64_t* chi);
int mpsim_gpu_set_site_dims(mpsim_gpu_state* s, int32_t i, int64_t dl, int64_t dr);

/* ---- multi-GPU chains: one process per GPU, NCCL over NVLink ---------------
 * Replaces execute_parallel's worker pool (executor.cpp:99-232) for a chain
 * that spans GPUs, and the paper's TAMM/GlobalArrays layer distribution
 * (SURVEY 8(e)). Rank r owns global sites [lo, hi) (even,
 * cost-weighted cut points) plus a ghost slot for the straddling gate of odd
 * layers; boundary sites and query environments move by NCCL send/recv on the
 * shard's stream (NCCL is loaded at run time, libnccl.so.2). Results are bit
 * for bit those of one GPU. The unique id comes from rank 0
 * (mpsim_gpu_nccl_unique_id) and reaches the other ranks out of band (MPI,
 * a TCP store, a file: the caller's choice, as with ncclCommInitRank). */
typedef struct mpsim_gpu_shard mpsim_gpu_shard;
#define MPSIM_REDUCE_SUM 0
#define MPSIM_REDUCE_MAX 1
#define MPSIM_REDUCE_MIN 2
/* host planning, no device: world + 1 bounds; chi <= 0 = even split */
int mpsim_shard_bounds(int32_t n_qubits, int32_t world, int64_t chi, int32_t* out);
/* one layer of local gates (global indices) -> the gates shard [lo, hi) runs
 * (local indices; the straddling gate on (hi-1, hi) uses the ghost slot hi-lo)
 * and whether it lends its first site left / borrows its right neighbour's */
int mpsim_shard_partition_layer(const mpsim_gate* gates, int32_t count, int32_t lo, int32_t hi, int32_t rank,
                                int32_t world, mpsim_gate* local, int32_t* n_local, int32_t* straddle_left,
                                int32_t* straddle_right);
int mpsim_gpu_nccl_unique_id(void* id_out /* 128 bytes */);
/* |0...0> shard of an n-qubit chain; nccl_id may be NULL when world == 1 */
int mpsim_gpu_shard_create(int32_t n_qubits, int64_t chi, int32_t rank, int32_t world, const void* nccl_id,
                           int32_t device, mpsim_gpu_shard** out);
int mpsim_gpu_shard_destroy(mpsim_gpu_shard* s);
/* owned range and the local state (borrowed: sites [0, hi-lo) + ghost) */
int mpsim_gpu_shard_info(const mpsim_gpu_shard* s, int32_t* lo, int32_t* hi, mpsim_gpu_state** local_state);
/* global site index i in [lo, hi) (MpsState::site(i) import / export) */
int mpsim_gpu_shard_set_site(mpsim_gpu_shard* s, int32_t i, int64_t dl, int64_t dr, const double* data);
int mpsim_gpu_shard_get_site(mpsim_gpu_shard* s, int32_t i, int64_t* dl, int64_t* dr, double* out);
int mpsim_gpu_shard_bond_dims(mpsim_gpu_shard* s, int64_t* out /* hi - lo + 1: bonds lo .. hi */);
/* one layer of disjoint local gates in global indices (every rank passes the
 * same layer): exchange in, one batched launch sequence, exchange out;
 * stats->device_ms spans all three (CUDA events on the shard stream) */
int mpsim_gpu_shard_apply_layer(mpsim_gpu_shard* s, const mpsim_gate* gates, int32_t count,
                                const mpsim_policy* policy, mpsim_exec_stats* stats);
/* execute_parallel over the whole chain: decompose_nonlocal + layerize
 * (fusion.cpp:137-190) on every rank, then the layers in order; stats are
 * reduced over the ranks (peak bond max, discarded weight sum) */
int mpsim_gpu_shard_execute(mpsim_gpu_shard* s, const mpsim_gate* gates, int32_t count, const mpsim_policy* policy,
                            mpsim_exec_stats* stats);
/* queries over the whole chain (every rank calls; every rank gets the result):
 * amplitudes of count full-length bit strings (mps.cpp:204-221), overlap of two
 * chains sharded alike (mps.cpp:223-239), norm (mps.cpp:189-202), <O_q> (P9) */
int mpsim_gpu_shard_amplitudes(mpsim_gpu_shard* s, const char* bits, int32_t count, double* out);
int mpsim_gpu_shard_overlap(mpsim_gpu_shard* a, mpsim_gpu_shard* b, double* out);
int mpsim_gpu_shard_norm(mpsim_gpu_shard* s, double* out);
int mpsim_gpu_shard_expect_1q(mpsim_gpu_shard* s, const double* op2x2, int32_t q, double* out);
/* move_center (mps.cpp:177-187) with the same QR steps in the same order */
int mpsim_gpu_shard_move_center(mpsim_gpu_shard* s, int32_t center);
int mpsim_gpu_shard_ortho_center(const mpsim_gpu_shard* s, int32_t* out);
/* perfect sampling (Sampler::sample, sampler.cpp:35-143) of the whole chain:
 * shot chunks (chunk, 0 = 4096) walk rank to rank; ordered counts afterwards
 * through mpsim_gpu_shard_sample_result (same on every rank) */
int mpsim_gpu_shard_sample(mpsim_gpu_shard* s, uint64_t shots, uint64_t seed, uint64_t chunk, int32_t* unique);
int mpsim_gpu_shard_sample_result(const mpsim_gpu_shard* s, int32_t i, char* bits /* n chars */, uint64_t* count);
/* plumbing for harnesses: element-wise all-reduce of host doubles, barrier */
int mpsim_gpu_shard_allreduce(mpsim_gpu_shard* s, double* values, int32_t count, int32_t op);
int mpsim_gpu_shard_barrier(mpsim_gpu_shard* s);

/* ---- gate application (gate_apply.hpp:48-78) --------------------------- */
int mpsim_gpu_apply_1q(mpsim_gpu_state* s, const double* u2x2, int32_t q, mpsim_report* rep);
/* apply_2q_local (q1 == q0+1), apply_2q_swap / apply_2q_bondprop otherwise. */
int mpsim_gpu_apply_2q(mpsim_gpu_state* s, const double* u4x4, int32_t q0, int32_t q1, int32_t method,
                       const mpsim_policy* policy, mpsim_report* rep);
/* One batched launch sequence for a set of gates on pairwise disjoint spans
 * (one layer of LayerPlan, circuit.hpp:85-95): local 2q and 1q gates only.
 * reports (nullable) receives one ApplyReport per gate, in input order. */
int mpsim_gpu_apply_layer(mpsim_gpu_state* s, const mpsim_gate* gates, int32_t count,
                          const mpsim_policy* policy, mpsim_report* reports);
/* execute_serial semantics (executor.cpp:73-97) over a fused gate list:
 * method SWAP lowers non-local gates (fusion.cpp:137-161), layerizes
 * (fusion.cpp:163-190) and runs every layer as one batched launch sequence
 * — bit-identical to gate-by-gate order because layer gates touch disjoint
 * sites. method BONDPROP runs gate by gate. reports (nullable): one per
 * input gate (aggregated over a SWAP chain as apply_2q_swap does). */
int mpsim_gpu_execute(mpsim_gpu_state* s, const mpsim_gate* gates, int32_t count, const mpsim_policy* policy,
                      int32_t method, mpsim_exec_stats* stats, mpsim_report* reports);

/* ---- truncated SVD of a plain matrix (svd(), svd.hpp:79-110) -------------
 * a: rows x cols row-major; outputs k (kept rank), s (k, descending),
 * u (rows x k), vdag (k x cols), w (discarded weight). u/vdag nullable;
 * s needs min(rows, cols) slots. Same batched Jacobi kernels as the gate
 * path, one matrix at a time. */
int mpsim_gpu_svd(int32_t rows, int32_t cols, const double* a, int64_t max_rank, double cutoff, int32_t device,
                  int64_t* k, double* s, double* u, double* vdag, double* w);

/* ---- queries (mps.hpp:79-100) ------------------------------------------ */
int mpsim_gpu_norm(const mpsim_gpu_state* s, double* out);                       /* mps.cpp:189-202 */
/* count bit strings of n chars '0'/'1' packed back to back (mps.cpp:204-221) */
int mpsim_gpu_amplitudes(const mpsim_gpu_state* s, const char* bits, int32_t count, double* out);
int mpsim_gpu_overlap(const mpsim_gpu_state* a, const mpsim_gpu_state* b, double* out); /* mps.cpp:223-239 */
int mpsim_gpu_to_statevector(const mpsim_gpu_state* s, int32_t max_qubits, double* out); /* mps.cpp:241-256 */
int mpsim_gpu_move_center(mpsim_gpu_state* s, int32_t center);                    /* mps.cpp:177-187 */
/* Environment forms for site-sharded chains (SURVEY 8(e) queries): a shard
 * continues its left neighbour's environment over its local sites [i0, i1)
 * and hands its own to the right. amplitudes_env: row environments of count
 * bit strings (n_local chars each, only [i0, i1) read; mps.cpp:204-221);
 * env_in host count x D_left complex (NULL = chain start), env_out host
 * count x D_right. transfer_env: E' = sum_p A_p^H E B_p (mps.cpp:189-202,
 * :223-239), op2x2 (nullable) applied to y at local site q (the P9
 * expectation form); env_in host D_left(x) x D_left(y) row-major (NULL =
 * [[1]]), env_out D_right(x) x D_right(y). */
/* move_center pieces for sharded chains (mps.cpp:57-95): left steps over
 * sites [i0, i1) (site i -> Q, R into site i+1), right steps over sites i1
 * down to i0 >= 1 (site i -> Q^H, R^H into site i-1); the ortho centre
 * becomes unknown. site_norm2: squared Frobenius norm of one site (the
 * zero-norm centre check, mps.cpp:183-185). */
int mpsim_gpu_sweep_left(mpsim_gpu_state* s, int32_t i0, int32_t i1);
int mpsim_gpu_sweep_right(mpsim_gpu_state* s, int32_t i0, int32_t i1);
int mpsim_gpu_site_norm2(const mpsim_gpu_state* s, int32_t i, double* out);
int mpsim_gpu_amplitudes_env(const mpsim_gpu_state* s, int32_t i0, int32_t i1, const char* bits, int32_t count,
                             const double* env_in, double* env_out);
int mpsim_gpu_transfer_env(const mpsim_gpu_state* x, const mpsim_gpu_state* y, int32_t i0, int32_t i1,
                           const double* op2x2, int32_t q, const double* env_in, double* env_out);
/* <psi| O_q |psi> for a 2x2 operator (the P9 definition: overlap(psi,
 * apply_1q(copy psi, O, q))); out = complex. */
int mpsim_gpu_expect_1q(const mpsim_gpu_state* s, const double* op2x2, int32_t q, double* out);
/* <psi| O_a (x) O_b |psi> for one-site operators on two distinct qubits. */
int mpsim_gpu_expect_2q(const mpsim_gpu_state* s, const double* op_a, int32_t qa, const double* op_b,
                        int32_t qb, double* out);

/* ---- sampling (Sampler, sampler.hpp:50-86) ------------------------------- */
typedef struct mpsim_gpu_sampler mpsim_gpu_sampler;
int mpsim_gpu_sampler_create(const mpsim_gpu_state* s, int32_t memoize, uint64_t max_cache_entries,
                             mpsim_gpu_sampler** out); /* sampler.cpp:35-66 */
int mpsim_gpu_sampler_destroy(mpsim_gpu_sampler* sp);
/* Draws shots (sampler.cpp:80-143); afterwards *unique distinct strings are
 * available, in lexicographic order, through mpsim_gpu_sampler_result. */
int mpsim_gpu_sample(mpsim_gpu_sampler* sp, uint64_t shots, uint64_t seed, int32_t* unique);
int mpsim_gpu_sampler_result(const mpsim_gpu_sampler* sp, int32_t i, char* bits /* n chars */, uint64_t* count);
int mpsim_gpu_sampler_stats(const mpsim_gpu_sampler* sp, uint64_t* cache_hits, uint64_t* cache_size);
int mpsim_gpu_sampler_clear_cache(mpsim_gpu_sampler* sp);
/* The sampler's site walk over sites [i0, i1) of an already canonicalised
 * state (a shard of a right-canonical chain): u holds shots x
 * (i1 - i0) variates (the reference's shot-major stream restricted to these
 * sites); env_in (host, u_in x D_left complex, NULL = chain start with one
 * node) and node_in (shots, NULL = all 0) carry the distinct prefixes of the
 * sites to the left. Outputs: *u_out distinct prefixes at i1, env_out (host,
 * capacity shots x D_right complex, nullable) their normalised
 * environments, node_out (shots) each shot's prefix, bits_out (shots x
 * (i1 - i0) chars) each shot's bits on these sites. */
int mpsim_gpu_sample_segment(const mpsim_gpu_state* s, int32_t i0, int32_t i1, uint64_t shots, const double* u,
                             int32_t u_in, const double* env_in, const int32_t* node_in, int32_t* u_out,
                             double* env_out, int32_t* node_out, char* bits_out);
/* As mpsim_gpu_sample_segment, but env_in / env_out are device pointers on
 * the state's device (the rank-to-rank prefix environments stay in HBM and go
 * straight to NCCL send/recv; SURVEY 8(e) "Queries"). The caller orders any
 * producer of env_in before the call; env_out is complete on return. */
int mpsim_gpu_sample_segment_dev(const mpsim_gpu_state* s, int32_t i0, int32_t i1, uint64_t shots, const double* u,
                                 int32_t u_in, const double* env_in, const int32_t* node_in, int32_t* u_out,
                                 double* env_out, int32_t* node_out, char* bits_out);
/* count variates of std::mt19937_64(seed) after skipping skip draws, as
 * (x >> 11) * 2^-53 (generators.cpp:31-33, sampler.cpp:115). Host only. */
int mpsim_uniform_variates(uint64_t seed, uint64_t skip, uint64_t count, double* out);

/* ---- instrumentation ----------------------------------------------------- */
/* Kernel launches and device time accumulated on the state's stream since
 * the last reset (bench.py's gpu_launches / roofline legs). */
int mpsim_gpu_counters(const mpsim_gpu_state* s, int64_t* launches, double* device_ms, int64_t* svd_sweeps);
/* The dominant kernel's share: Jacobi sweep launches (one persistent launch
 * per sweep) and their CUDA-event time, and the algorithmic flops of the work
 * done (SURVEY 8(d):
 * svd = 32 M N^2 per decomposed theta, gate = full F_2q per applied gate). */
int mpsim_gpu_kernel_counters(const mpsim_gpu_state* s, int64_t* jacobi_launches, double* jacobi_ms,
                              double* svd_flops, double* gate_flops);
/* Host<->device bytes moved by the gate path (descriptors in, reports and
 * convergence flags out) since the last reset. */
int mpsim_gpu_transfer_counters(const mpsim_gpu_state* s, int64_t* h2d_bytes, int64_t* d2h_bytes);
int mpsim_gpu_reset_counters(mpsim_gpu_state* s);
int mpsim_gpu_synchronize(mpsim_gpu_state* s);

/* ---- host front end --------------------------------------
 * OpenQASM 2.0 subset parser (qasm_parser.cpp), u4 sidecar (runner.cpp:
 * 129-190), fusion / SWAP lowering / layering (fusion.cpp:79-190), circuit
 * generators (generators.cpp:52-145) and the run pipeline with its JSON
 * record (runner.cpp:219-328, docs/run_output.schema.json). Parse, fuse,
 * plan and generate are host-only (no device touched). Errors map like
 * exit_code_for_error (runner.cpp:330-341): ConfigError -> MPSIM_EINVAL,
 * ParseError -> MPSIM_EPARSE (location via mpsim_last_parse_location),
 * NumericError -> MPSIM_ENUMERIC. Library-allocated outputs are released
 * with mpsim_free. */

/* GateKind, circuit.hpp:33-38 (same order) */
enum {
  MPSIM_GATE_H = 0, MPSIM_GATE_X, MPSIM_GATE_Y, MPSIM_GATE_Z, MPSIM_GATE_S, MPSIM_GATE_SDG, MPSIM_GATE_T,
  MPSIM_GATE_TDG, MPSIM_GATE_RX, MPSIM_GATE_RY, MPSIM_GATE_RZ, MPSIM_GATE_U1, MPSIM_GATE_U2, MPSIM_GATE_U3,
  MPSIM_GATE_CX, MPSIM_GATE_CZ, MPSIM_GATE_SWAP, MPSIM_GATE_U4
};

/* PrimOp, circuit.hpp:48-56 (q1 = -1 for one-qubit ops; U4 matrices are not echoed). */
typedef struct {
  int32_t kind;
  int32_t q0;
  int32_t q1;
  int32_t nparams;
  double params[3];
} mpsim_prim_op;

/* Circuit, circuit.hpp:58-63 */
typedef struct {
  int32_t n_qubits;
  int32_t n_clbits;
  int32_t has_measure_all;
  int32_t n_ops;
} mpsim_circuit_info;

void mpsim_free(void* p);
/* parse_qasm (circuit.hpp:108-110, qasm_parser.cpp): ops (nullable) receives
 * the first max_ops ops. */
int mpsim_parse_qasm(const char* text, mpsim_circuit_info* info, mpsim_prim_op* ops, int32_t max_ops);
/* ParseError::line() / column() of the calling thread's last MPSIM_EPARSE. */
int mpsim_last_parse_location(int32_t* line, int32_t* column);
/* parse_qasm + inject_sidecar (runner.cpp:165-190; sidecar_json nullable,
 * u4-sidecar-v1 text) + fuse_circuit (fusion.cpp:79-135). Fused two-qubit
 * gates have q0 < q1 and the matrix in the (q0, q1) basis; flipped[i]
 * (FusedGate::flipped) records a (high, low) origin. */
int mpsim_fuse_qasm(const char* qasm, const char* sidecar_json, int32_t* n_qubits, mpsim_gate** gates,
                    int32_t** flipped, int32_t* count);
/* decompose_nonlocal + layerize (fusion.cpp:137-190): the lowered local
 * gates in layer order; layer_of[i] = layer of out[i]. */
int mpsim_plan_layers(const mpsim_gate* gates, int32_t count, int32_t n_qubits, mpsim_gate** out,
                      int32_t** layer_of, int32_t* out_count, int32_t* n_layers);
/* ghz_qasm / brickwork_qasm (generators.cpp:52-145); haar != 0 draws
 * seeded Haar 4x4 entanglers into *sidecar_json (u4-sidecar-v1), else the
 * entangler is cx and *sidecar_json is NULL. */
int mpsim_gen_ghz_qasm(int32_t n, int32_t measure, char** qasm);
int mpsim_gen_brickwork_qasm(int32_t n, int32_t depth, uint64_t seed, int32_t measure, int32_t haar, char** qasm,
                             char** sidecar_json);

/* Backend, runner.hpp:38 */
#define MPSIM_BACKEND_MPS_SERIAL 0
#define MPSIM_BACKEND_MPS_PARALLEL 1
#define MPSIM_BACKEND_STATEVECTOR 2

/* RunConfig, runner.hpp:46-62 (+ device / chi_hint for the GPU state). */
typedef struct {
  const char* qasm_path;    /* read from file when non-empty */
  const char* qasm_text;    /* used when qasm_path is empty */
  const char* sidecar_path; /* explicit sidecar file; else <qasm_path>.u4.json when present */
  const char* sidecar_json; /* inline sidecar text (instead of a file) */
  const char* input_label;  /* echoed as config.input */
  int32_t backend;
  int32_t nonlocal;         /* MPSIM_NONLOCAL_* */
  int64_t max_bond;         /* 0 = unbounded */
  double cutoff;
  uint64_t shots;
  uint64_t seed;
  int32_t workers;
  int32_t memoize;
  uint64_t cache_cap;
  int32_t statevector_cap;
  int32_t device;
  int64_t chi_hint;
} mpsim_run_config;
void mpsim_run_config_defaults(mpsim_run_config* c);
/* run_circuit + run_output_to_json (runner.cpp:219-328): *json = the result
 * record (docs/run_output.schema.json), keys sorted like nlohmann::json. */
int mpsim_gpu_run_circuit(const mpsim_run_config* c, char** json);

#ifdef __cplusplus
}
#endif

#endif /* MPSIM_GPU_H_ */
