/*
 * es_b200.h -- C ABI of the B200 exact-simulation (ES) engine.
 *
 * Drop-in boundary for the reference ES engine (cecprove/es.py).  The
 * reference has no FFI; its seam is the Python function contract
 * ("the identical InstrProgram abstraction is the seam where
 * a device kernel would attach").  Each entry point below
 * replaces one reference interface, cited per function.  Plain pointers and
 * sizes only; the Python host layer (paper_2512_06627_b200/es.py) binds it
 * with ctypes, which drops the GIL for the duration of each call.
 *
 * Ownership: the caller owns every input array for the duration of a call.
 * The library owns device buffers, streams and JIT modules (released by
 * es_shutdown).  All entry points are re-entrant across host threads.
 *
 * Errors: every int-returning entry point returns ES_OK (0) or a negative
 * ES_E* code; es_last_error() gives a thread-local message.
 */
#ifndef ES_B200_H
#define ES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* op codes of the reference program (es.py:27-30) */
#define ES_OP_LOAD_PI 0
#define ES_OP_AND 1
#define ES_OP_XOR 2
#define ES_OP_OUTPUT 3

/* reference ceiling (es.py:25) */
#define ES_MAX_PIS 40

/* return codes */
#define ES_OK 0
#define ES_E_TOO_MANY_INPUTS (-1) /* TooManyInputs (es.py:39-40, 97-98) */
#define ES_E_CUDA (-2)            /* CUDA / JIT failure; es_last_error() says which */
#define ES_E_BAD_PROGRAM (-3)     /* malformed program or graph */
#define ES_E_BAD_ARG (-4)         /* e.g. workers < 1 (es.py:260-261) */
#define ES_E_NO_DEVICE (-5)       /* no CUDA device visible */
#define ES_E_WITNESS (-6)         /* witness failed re-check (es.py:360-361 AssertionError) */
#define ES_E_AIGER (-7)           /* AigerError: cyclic AND definitions (aiger.py:81-90) */
#define ES_E_AIGER_HEADER (-8)    /* MalformedHeader (aiger.py:17, 29-41, 114-189) */
#define ES_E_AIGER_LATCHES (-9)   /* LatchesUnsupported (aiger.py:21, 52-53) */
#define ES_E_AIGER_DANGLING (-10) /* DanglingLiteral (aiger.py:25, 86, 97, 110, 190) */

/* EsResult.verdict (es.py:34-36) */
#define ES_EXHAUSTED_ZERO 0
#define ES_COUNTEREXAMPLE 1
#define ES_BUDGET_EXCEEDED 2

/* reason attached to ES_BUDGET_EXCEEDED */
#define ES_REASON_NONE 0
#define ES_REASON_TIMEOUT 1
#define ES_REASON_CANCELLED 2

/* engines */
#define ES_ENGINE_AUTO 0   /* JIT straight-line kernel when it pays, else interpreter */
#define ES_ENGINE_JIT 1    /* K1: per-program LOP3 straight-line kernel (registers) */
#define ES_ENGINE_INTERP 2 /* K2: shared-memory interpreter of the program */

/*
 * The reference InstrProgram as structure-of-arrays -- exactly the arrays
 * es.py:_encode builds (es.py:232-249), with negations as 0/1 bytes.
 * InstrProgram (es.py:66-73) / Instr (es.py:43-63).
 */
typedef struct es_prog {
    int32_t num_instrs;
    int32_t num_registers; /* peak live registers (es.py:163) */
    int32_t num_pis;
    const int8_t *op;
    const int32_t *dst;
    const int32_t *src0; /* -1 = constant-0 rail (OUTPUT only) */
    const uint8_t *neg0;
    const int32_t *src1;
    const uint8_t *neg1;
    const int32_t *pi; /* 1-based PI index, LOAD_PI only */
} es_prog;

/* Options of one run (run_exhaustive's workers/budget/cancel, es.py:252-253). */
typedef struct es_run_opts {
    int32_t device;         /* CUDA ordinal (when n_devices == 0) */
    int32_t engine;         /* ES_ENGINE_* */
    double budget_s;        /* < 0: none; 0.0 -> BUDGET_EXCEEDED before any work */
    const volatile int32_t *cancel_flag; /* host flag polled between slices; may be NULL */
    double slice_ms;        /* target device time per launch slice (budget/cancel granularity) */
    int32_t block_threads;  /* 0: default */
    int32_t flags;          /* ES_FLAG_* */
    int32_t cofactor_pis;   /* ES_COFACTOR_* or k = 1..5 (K1 only) */
    int32_t n_devices;      /* > 0: sweep on devices[0..n_devices) (one host thread each; an
                             * ordinal may repeat); 0: on `device` only */
    const int32_t *devices;
    int32_t jit_parts;      /* K1 build: 0 = policy (cold runs write the body's SASS directly
                             * or split it so ptxas compiles its phases on parallel host threads),
                             * 1 = one straight-line body, >= 2 = split into that many phases,
                             * -1 = direct SASS, no ptxas (es_sass.cpp; a program that does not
                             * fit its template gets the split build) */
} es_run_opts;

/*
 * es_run_opts.cofactor_pis -- K1 cofactor copies.  k word PIs (PI >= 6, chosen
 * by smallest transitive fanout) are fixed per copy instead of per word, so
 * one kernel iteration evaluates 2^k words: the logic outside their fanout
 * once, the folded logic inside it once per copy.  Verdict and witness are
 * unchanged (minimum index); only the speed and the JIT cost differ.
 */
#define ES_COFACTOR_AUTO 0         /* minimise estimated JIT + sweep time (tiers up on reuse) */
#define ES_COFACTOR_NONE (-1)      /* one word per iteration */
#define ES_COFACTOR_THROUGHPUT (-2) /* maximise sweep rate; JIT cost ignored */

/* es_run_opts.flags: reserved (0) */

/* EsResult (es.py:76-84) plus engine statistics. */
typedef struct es_result {
    int32_t verdict;            /* ES_EXHAUSTED_ZERO | ES_COUNTEREXAMPLE | ES_BUDGET_EXCEEDED */
    int32_t reason;             /* ES_REASON_* (BUDGET_EXCEEDED only) */
    int32_t engine;             /* engine that ran (ES_ENGINE_JIT / _INTERP) */
    int32_t num_luts;           /* LOP3 ops per 32-pattern word after mapping (JIT) */
    uint64_t witness_index;     /* pattern p, PI i+1 = bit i of p (es.py:315-320) */
    uint64_t patterns_evaluated;/* reference workers=1 accounting (es.py:313, 333) */
    uint64_t patterns_swept;    /* patterns this engine actually simulated */
    double compile_ms;          /* host map + schedule + codegen */
    double jit_ms;              /* PTX -> SASS + module load (0 on a cache hit) */
    double device_ms;           /* CUDA-event time of the kernel slices */
    double wall_ms;             /* whole call */
    int32_t launches;           /* kernel launches issued */
    int32_t regs_per_thread;    /* JIT kernel register count */
    int32_t cofactor_pis;       /* K1 cofactor PIs used (0: none) */
    int32_t jit_opt;            /* ptxas -O level of the K1 kernel (1: cold runs, 3: throughput) */
    int32_t witness_minimal;    /* COUNTEREXAMPLE: 1 = witness_index is the minimum failing pattern
                                 * (always, except when a budget/cancel stop cut a cofactored sweep
                                 * short before every smaller pattern was swept: then the witness is
                                 * valid but may not be the minimum, and patterns_evaluated =
                                 * patterns_swept) */
    int32_t n_devices;          /* GPUs the sweep ran on */
    int32_t phases;             /* K1: 2 when a counterexample above a cofactored chunk's range
                                 * needed a second sweep below it (non-contiguous chunks) */
    int32_t phase2_cofactor_pis;/* cofactor PIs of the second phase's variant (phases == 2) */
    int32_t phase2_copies;      /* > 0: the second phase ran the first phase's cofactor set
                                 * restricted to copies 0..phase2_copies-1 */
    int32_t jit_parts;          /* K1: phases of the kernel's split build (1: one body; -1: direct
                                 * SASS, jit_opt 0) */
} es_result;

/*
 * compile_program (es.py:87-163): the reference schedule, instruction for
 * instruction (cone marking, fanin refcounts, lazy PI loads, LIFO register
 * reuse).  Input: the XAG as packed gates, literal = node*2+neg (xag.py:28-33),
 * kind 0 = AND, 1 = XOR (xag.py:16-18).  Output arrays must hold
 * num_pis + num_gates + 1 entries.  Returns the instruction count (> 0) or
 * ES_E_TOO_MANY_INPUTS / ES_E_BAD_PROGRAM.
 */
int32_t es_compile(int32_t num_pis, int32_t num_gates, const uint8_t *kind,
                   const uint32_t *in0, const uint32_t *in1, uint32_t out_lit,
                   int8_t *op, int32_t *dst, int32_t *src0, uint8_t *neg0,
                   int32_t *src1, uint8_t *neg1, int32_t *pi,
                   int32_t *num_registers);

/*
 * run_exhaustive (es.py:252-339): sweep all 2^num_pis patterns and return the
 * MINIMUM-index pattern whose output is 1 (== the reference's workers=1
 * witness), EXHAUSTED_ZERO, or BUDGET_EXCEEDED.  One call may drive several
 * GPUs (es_run_opts.devices; the reference's workers, es.py:272-331): the
 * pattern space is dealt to them chunk by chunk and one minimum word in the
 * first device's memory, shared as NVLink peer memory, gives every GPU the
 * global early exit.
 */
int32_t es_run(const es_prog *prog, const es_run_opts *opts, es_result *out);

/* Visible CUDA devices (0 when there is no driver or GPU; never an error). */
int32_t es_device_count(int32_t *n);

/*
 * Batched run_exhaustive over many independent programs (the sweep's
 * sub-miter stream, sweep.py:225-255): one interpreter launch covers all
 * jobs.  outs[i] receives job i's result.
 */
int32_t es_run_batch(int32_t n_jobs, const es_prog *progs, const es_run_opts *opts,
                     es_result *outs);

/*
 * Sharded sweep for one rank of a multi-GPU job.  Prepares the
 * JIT kernel for `prog` and returns an opaque session.  es_session_launch
 * enqueues, on `stream` (a cudaStream_t, e.g. torch's current stream), the
 * kernel over global chunks [chunk_begin, chunk_end) restricted to
 * chunk % world == rank; it atomically lowers *best (a device uint64 the
 * caller owns, initialised to 2^num_pis) to the minimum failing pattern it
 * finds and skips chunks above *best.  The caller reduces *best across ranks
 * (NCCL MIN) between launches.  Asynchronous: no host synchronisation.
 */
typedef struct es_session es_session;
int32_t es_session_open(const es_prog *prog, const es_run_opts *opts, es_session **out);
int32_t es_session_geometry(const es_session *s, uint64_t *n_chunks, uint64_t *patterns_per_chunk,
                            int32_t *num_luts, int32_t *regs_per_thread);
int32_t es_session_launch(es_session *s, void *stream, uint64_t *best_dev,
                          uint64_t chunk_begin, uint64_t chunk_end, int32_t rank,
                          int32_t world);
void es_session_close(es_session *s);

/*
 * Sub-miter batches: extract the cone-local miter
 * of each candidate pair of a parent XAG exactly as extract_submiter does
 * (sweep.py:92-158; merges = the sweep's proven-node map, node -> packed
 * literal), compile each with the reference schedule (es.py:87-163), on
 * n_threads host threads (0 = all), then run them all in one batched device
 * sweep.  es_batch_run re-checks every witness on its sub-miter (es.py:360)
 * and returns ES_E_WITNESS on a mismatch.  Jobs over 40 PIs report
 * verdict ES_BUDGET_EXCEEDED with reason -1 (ineligible, es.py:350-351).
 */
typedef struct es_batch es_batch;
int32_t es_batch_extract(int32_t num_pis, int32_t num_gates, const uint8_t *kind,
                         const uint32_t *in0, const uint32_t *in1, int32_t n_merges,
                         const int32_t *merge_node, const uint32_t *merge_lit, int32_t n_pairs,
                         const int32_t *a, const int32_t *b, const uint8_t *polarity,
                         int32_t n_threads, es_batch **out);
/* Build the interpreter programs (cofactor depth, schedule) of every job that
 * lacks one; es_batch_run does it on demand, this lets callers time it. */
int32_t es_batch_prepare(es_batch *b, int32_t n_threads);
/* evaluate (eval.py:22-36): the single output of a packed XAG (as es_compile)
 * on pattern `pattern` (PI i+1 = bit i, <= 64 PIs): returns 0 or 1, or an
 * error code.  es_check's witness re-check (es.py:360-361). */
int32_t es_xag_eval(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, uint32_t out_lit, uint64_t pattern);
/* Per-job interpreter program shape after es_batch_prepare: slot-file rows,
 * records (gates + OUT records) and cofactor depth; -1 for unprepared jobs.
 * The runtime groups launches by slots (<=44: 4 words/thread, <=88: 2, else). */
int32_t es_batch_k2_stats(const es_batch *b, int32_t *num_slots, int32_t *num_records,
                          int32_t *cofactor_pis);
/* Per-job shared-memory traffic of one interpreter pass (after accumulator
 * forwarding): slot loads, and slot stores including the PI words written at
 * the start of the pass; -1 for unprepared jobs (the bench's K2 roofline). */
int32_t es_batch_k2_traffic(const es_batch *b, int32_t *loads, int32_t *stores);
int32_t es_batch_size(const es_batch *b);
int32_t es_batch_info(const es_batch *b, int32_t i, int32_t *num_pis, int32_t *num_gates,
                      uint64_t *hash, int32_t *num_instrs, int32_t *num_registers, int32_t *G);
/* Per-job arrays for the whole batch (each may be NULL). */
int32_t es_batch_table(const es_batch *b, int32_t *num_pis, int32_t *num_gates, int32_t *G,
                       uint64_t *hash);
int32_t es_batch_xag(const es_batch *b, int32_t i, uint8_t *kind, uint32_t *in0, uint32_t *in1,
                     uint32_t *out_lit, int32_t *pi_map);
int32_t es_batch_select(es_batch *b, int32_t n, const int32_t *idx);
int32_t es_batch_run(es_batch *b, const es_run_opts *opts, es_result *outs);
/* Move every sub-miter of src to the end of dst (src becomes empty). */
int32_t es_batch_merge(es_batch *dst, es_batch *src);
void es_batch_free(es_batch *b);

/*
 * Shared minimum word for the NVLink peer path: rank 0 allocates a
 * device word and exports a 64-byte CUDA IPC handle; every other rank opens it
 * (peer access is enabled lazily, so on an NVSwitch box the word is a peer
 * GPU's memory reached over NVLink).  Pass the opened pointer as `best_dev` to
 * es_session_launch: every rank's kernel then atomicMin's (system scope) into
 * and early-exits on the one word, with no per-slice collective.
 */
int32_t es_ipc_alloc(int32_t device, void **dev_ptr, uint8_t *handle64);
int32_t es_ipc_open(int32_t device, const uint8_t *handle64, void **dev_ptr);
int32_t es_ipc_close(int32_t device, void *dev_ptr, int32_t owner);
int32_t es_word_write(int32_t device, void *dev_ptr, uint64_t value);
int32_t es_word_read(int32_t device, void *dev_ptr, uint64_t *value);
/* Device-side verdict barrier on an exchange slot ([0] minimum word, [8]
 * arrival counter; es_ipc_alloc'd): enqueued on `stream` after a rank's
 * es_session_launch, es_peer_arrive_wait counts the rank in, waits on the
 * device until all `world` ranks have, and writes the final minimum to
 * out_dev (device or mapped memory) -- no host synchronisation, no
 * collective.  es_peer_arm re-arms a slot (minimum all-ones, counter 0);
 * rank 0 arms the slot of verdict s+1 while verdict s runs (three slots
 * rotate: the armed one was last used at verdict s-2). */
int32_t es_peer_arm(void *stream, void *word_dev);
int32_t es_peer_arrive_wait(void *stream, void *word_dev, int32_t world, void *out_dev);

/*
 * K3: word-parallel random simulation (the sweep's
 * candidate-class discovery and refinement).  simulate (sim.py:21-38): the
 * XAG as packed gates (as es_compile), pi_words = num_pis x words uint64
 * (row i drives PI i+1, bit b of word w = pattern 64w+b), node_words =
 * (1+num_pis+num_gates) x words, row-major, the reference's array exactly.
 * device_ms (may be NULL) = the simulation kernels' CUDA-event time.
 */
int32_t es_sim(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
               const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
               uint64_t *node_words, double *device_ms);
/* ones_fraction(simulate(...)) numerators (sim.py:45-48; the stability /
 * entropy features, features.py:165-180): ones[v] = number of 1-bits of node
 * v over all words*64 patterns, num_nodes int64.  The node matrix stays on
 * the device. */
int32_t es_sim_ones(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                    const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                    int64_t *ones, double *device_ms);
/* The same on device buffers, enqueued on `stream` (a cudaStream_t) without
 * host synchronisation.  *prog_cache (may be NULL) keeps the compiled gate
 * program between calls on the same XAG; free it with es_sim_prog_free. */
int32_t es_sim_device(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                      const uint32_t *in1, const uint64_t *d_pi_words, int64_t words, void *stream,
                      uint64_t *d_node_words, void **prog_cache);
void es_sim_prog_free(void *prog_cache);
/* Host only: logic levels of the simulation program (batches never span one). */
int32_t es_sim_levels(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                     const uint32_t *in1);
/* random_simulate + build_pe_classes (sweep.py:54-81) under the given drive:
 * class_id[node] = class index in representative (smallest member) order,
 * -1 for a singleton; polarity[node] = the canonical polarity (the
 * complemented row's bytes compare smaller).  Arrays have num_nodes entries. */
int32_t es_sim_classes(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, const uint64_t *pi_words, int64_t words, int32_t device,
                       int32_t *class_id, uint8_t *polarity, int32_t *n_classes, double *device_ms);

/*
 * AIGER ingest.  es_aiger_parse = parse_aiger
 * (aiger.py:44-194) of ASCII "aag" or binary "aig" bytes, optionally followed
 * by detect_xors (transform.py:79-119) -- the CLI's _load_circuit
 * (cli.py:63-76).  The circuit is built with the reference's structural
 * hashing, so it is gate-for-gate the reference's Xag; read it back with
 * es_xag_size / es_xag_read (packed literals node*2+neg, kind 0 AND 1 XOR).
 */
typedef struct es_xag es_xag;
int32_t es_aiger_parse(const uint8_t *data, int64_t len, int32_t detect_xors, es_xag **out);
int32_t es_detect_xors(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits,
                       es_xag **out);
int32_t es_xag_size(const es_xag *x, int32_t *num_pis, int32_t *num_gates, int32_t *num_outputs);
int32_t es_xag_read(const es_xag *x, uint8_t *kind, uint32_t *in0, uint32_t *in1, uint32_t *out_lits);
void es_xag_free(es_xag *x);
/* write_aiger (aiger.py:197-225): ASCII AIGER, XOR as three ANDs; returns
 * the byte count (buf may be NULL to size it). */
int64_t es_aiger_write(int32_t num_pis, int32_t num_gates, const uint8_t *kind, const uint32_t *in0,
                       const uint32_t *in1, int32_t num_outputs, const uint32_t *out_lits, char *buf,
                       int64_t cap);

/* Engine-internal views for tests and profiling. */
/* LUT-3 mapping statistics of a program: LOP3s per word, schedule peak live. */
int32_t es_map_stats(const es_prog *prog, int32_t *num_luts, int32_t *peak_live,
                     int32_t *num_gates);
/* Per-word ops of the K1 body by pipe: LUTs issued as LOP3 (ALU pipe) and
 * as IMAD (FMA pipe, f(x, word-uniform selector)); lop3 + imad = num_luts. */
int32_t es_map_pipes(const es_prog *prog, int32_t *lop3, int32_t *imad);
/* Evaluate the mapped+scheduled LUT program on the CPU for words [w0, w0+nw)
 * (32 patterns per word, the kernel's layout): writes the output words.
 * Lets GPU-less CI check the mapper bit-exactly. */
int32_t es_map_eval(const es_prog *prog, uint64_t w0, uint64_t nw, uint32_t *out_words);
/* K2 interpreter program of `prog`: gates, slots (PI + recycled), stores
 * issued and operands forwarded from the accumulator. */
int32_t es_k2_stats(const es_prog *prog, int32_t *num_gates, int32_t *num_slots,
                    int32_t *stores, int32_t *acc_reads);
/* CPU model of the K2 program over words [w0, w0+nw) (bit-exact with K2). */
int32_t es_k2_eval(const es_prog *prog, uint64_t w0, uint64_t nw, uint32_t *out_words);
/* K2 with k forced cofactor PIs (0..6), and the depth K2 picks by itself
 * (the fewest shared-memory wavefronts per word, <= 88 slots). */
int32_t es_k2_eval_k(const es_prog *prog, int32_t k, uint64_t w0, uint64_t nw, uint32_t *out_words);
int32_t es_k2_cofactor_pis(const es_prog *prog);
/* The same views for the K1 variant with k cofactor PIs (0..5, chosen as
 * es_run does: the k word PIs of smallest transitive fanout).  es_map_eval_k
 * takes FULL word indices (cofactor PIs included) and returns the output of
 * the copy each word belongs to, so it is comparable with es_map_eval. */
int32_t es_map_stats_k(const es_prog *prog, int32_t k, int32_t *num_luts, int32_t *peak_live,
                       int32_t *num_gates, int32_t *cof_pis /* k entries, may be NULL */);
int32_t es_map_pipes_k(const es_prog *prog, int32_t k, int32_t *lop3, int32_t *imad);
int32_t es_map_eval_k(const es_prog *prog, int32_t k, uint64_t w0, uint64_t nw, uint32_t *out_words);
int64_t es_emit_ptx_k(const es_prog *prog, int32_t k, int32_t block_threads, char *buf, int64_t cap);
/* The restricted variant of the second phase of a non-equivalent search: the
 * k-PI cofactor set evaluating only copies 0..copies-1 (0 = all).  eval gives
 * 0 for words of the other copies. */
int32_t es_map_stats_kc(const es_prog *prog, int32_t k, int32_t copies, int32_t *num_luts,
                        int32_t *peak_live);
int32_t es_map_eval_kc(const es_prog *prog, int32_t k, int32_t copies, uint64_t w0, uint64_t nw,
                       uint32_t *out_words);
/* The K1 body alone (the LOP3/IMAD block es_emit_ptx_k splices into the
 * skeleton; inputs %lo %hi %one, outputs %o [%c]) with the shared-memory
 * overflow slots of es_spill.cpp applied for a register budget of
 * `spill_budget` values (0: none) at `block_threads` threads.  slots = the
 * shared-memory words per thread it needs (may be NULL).  buf NULL -> size. */
int64_t es_emit_body_k(const es_prog *prog, int32_t k, int32_t spill_budget, int32_t block_threads,
                       int32_t *slots, char *buf, int64_t cap);
/* The direct-SASS K1 cubin for `prog` with k cofactor PIs (es_sass.cpp; no
 * ptxas): the K1 skeleton ptxas compiled at build time with the program's
 * own sm_100a body written over its placeholder function.  block_threads:
 * 128 (k = 0) or 256 (k > 0).  stats (may be NULL): body instructions, LOP3,
 * IMAD, peak registers, modelled issue cycles, and the template's word-index
 * (lo, hi) and result (o0, o1) registers.  Returns the cubin's size (buf
 * NULL) or < 0 when the program does not fit a template. */
int64_t es_sass_cubin(const es_prog *prog, int32_t k, int32_t block_threads, int32_t *stats /* 9 */,
                      char *buf, int64_t cap);
/* A K4 module without a GPU (k4_skeleton.cu, es_sass.cpp): the direct-SASS
 * bodies of n programs (program i with cof_k[i] cofactor PIs, the same PI
 * choice as es_sass_cubin) written behind the K4 skeleton's indirect branch
 * of template `variant` (0: one CTA per SM, ~230 body registers; 1: two CTAs,
 * ~90); body i is jump-table entry i.  stats (n x 4, may be NULL): per body its
 * instructions, then the template's word-index (lo, hi) and result (o0) ...
 * as es_sass_cubin's fields 5..8 in stats[4 * n .. 4 * n + 3].  Returns the
 * cubin's size (buf NULL) or < 0 (a body does not fit). */
int64_t es_k4_cubin(const es_prog *progs, int32_t n, const int32_t *cof_k, int32_t variant, int32_t *stats,
                    char *buf, int64_t cap);
int64_t es_jit_check_k(const es_prog *prog, int32_t k, int32_t block_threads, int32_t *regs_per_thread,
                       int32_t *spill_bytes, char *log, int64_t log_cap);
/* Split build without a GPU: the k-cofactor body cut into `parts` phases,
 * compiled on parallel host threads and linked (es_split.cpp).  Returns the
 * linked cubin's bytes or < 0; smem_bytes = the slot file per CTA, slots =
 * shared-memory slots per thread, loads = slot loads per iteration. */
int64_t es_jit_check_split(const es_prog *prog, int32_t k, int32_t parts, int32_t block_threads,
                           int32_t *regs_per_thread, int32_t *smem_bytes, int32_t *slots, int32_t *loads,
                           double *ms);
/* The PTX the JIT path would compile for `prog` (buf NULL -> returns size).
 * block_threads: 128/256/512. */
int64_t es_emit_ptx(const es_prog *prog, int32_t block_threads, char *buf, int64_t cap);
/* Compile PTX to SASS without a GPU (build-time check); returns cubin bytes or < 0. */
int64_t es_jit_check(const es_prog *prog, int32_t block_threads, int32_t *regs_per_thread,
                     int32_t *spill_bytes, char *log, int64_t log_cap);

/* Measured ALU-pipe peak: lane-LOP3 operations per second on `device` (one
 * lane-op evaluates one 2/3-input gate over 32 patterns).  The roofline
 * denominator of the bench. */
int32_t es_alu_peak(int32_t device, double *lane_ops_per_s, double *ms);
/* Measured FMA-pipe integer peak: lane-IMAD operations per second (the K1
 * body's x*S+T LUTs and their coefficients; the second integer pipe K1 is
 * bound by). */
int32_t es_fma_peak(int32_t device, double *lane_ops_per_s, double *ms);
/* Measured shared-memory load bandwidth of the whole GPU (bytes/s): the
 * denominator of the K2 interpreter's shared-memory roofline. */
int32_t es_smem_peak(int32_t device, double *bytes_per_s, double *ms);

const char *es_last_error(void);
const char *es_version(void);
void es_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* ES_B200_H */
