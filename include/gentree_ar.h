/* gentree_ar.h — C-ABI of the B200-native GenModel/GenTree AllReduce library.
 *
 * Implements the data-parallel hot path of arXiv 2409.04202 ("Revisiting the Time Cost
 * Model of AllReduce"): fit GenModel (§3.4), generate a plan with GenTree (§4.2,
 * Algorithms 1-2) and execute it on device buffers (the ReduceScatter step(s) with fan-in
 * chosen by GenModel, then the AllGather = the RS reversed) with hand-written
 * sm_100a kernels that pull peer chunks over NVLink from CUDA-IPC-mapped buffers and push
 * results with P2P stores under flag synchronisation.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (the reference text),
 * readings "Qn" = the register in DESIGN.md.
 *
 * Conventions for every entry point:
 *   - return value is a status: AR_OK (0), AR_EINVAL (1) for validation/domain errors
 *     (SPEC exit code 1), AR_ESYS (2) for CUDA / system errors (SPEC exit code 2);
 *     nothing is thrown or aborted across the ABI;
 *   - ar_last_error() returns a thread-local message for the last failing call on this
 *     thread, valid until the next call;
 *   - all pointer arguments are borrowed for the duration of the call unless stated;
 *   - GenModel quantities are in seconds and bytes (β, γ, δ, ε in seconds per byte; the
 *     topology document keeps Table 5's per-float units and is converted by /4, exactly).
 */
#ifndef GENTREE_AR_H
#define GENTREE_AR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AR_OK 0
#define AR_EINVAL 1
#define AR_ESYS 2

#define AR_F32 0  /* IEEE binary32 data, fp32 accumulation */
#define AR_BF16 1 /* bfloat16 data, fp32 accumulation, one RNE rounding per stored partial (Q2) */

#define AR_MAX_RANKS 64     /* ranks of one communicator (2..64) */
#define AR_BLOB_BYTES 512   /* size of one exported registration blob */

const char *ar_last_error(void);
const char *ar_version(void);

/* ------------------------------------------------------------------ GenModel */

/* GenModel parameters, per byte.  When has_combined != 0 only the fitted
 * (2β+γ) = `combined` is known: evaluation then uses β = combined/2, γ = 0. */
typedef struct {
  double alpha, beta, gamma, delta, epsilon;
  int32_t w_t;
  int32_t has_combined;
  double combined;
} gm_params;

/* Per-term time (seconds) of a plan or closed form. */
typedef struct {
  double latency, bandwidth, compute, memory, incast, total;
} gm_breakdown;

/* One Co-located-PS benchmark observation: n ranks, `bytes` per rank,
 * mean AllReduce time in seconds. */
typedef struct {
  int32_t n;
  int32_t reserved;
  uint64_t bytes;
  double seconds;
} gm_measurement;

/* §3.4 fit (procedure S:441-458): for each w_t in [wt_min, wt_max], NNLS for
 * (α, k = 2β+γ, δ, ε) on the CPS row of Table 2; the lowest SSE wins (ties, within 1e-6
 * relative, go to the smaller w_t).  If link_bytes_per_s > 0, β = 1/link_bytes_per_s and
 * γ = k − 2β (AR_EINVAL if negative); otherwise out->has_combined = 1.
 * rows: n_rows observations, repeated (n, bytes) pairs are averaged.  `sse` may be NULL.
 * Errors: AR_EINVAL if fewer than 4 distinct (n, bytes) rows, fewer than 2 distinct n or
 * bytes, or an empty w_t range. */
int genmodel_fit(const gm_measurement *rows, size_t n_rows, int32_t wt_min, int32_t wt_max,
                 double link_bytes_per_s, gm_params *out, double *sse);

/* Fit of the NVLS plan row ("modelled in GenModel as a new plan row,
 * with α and β fitted in C3"; reading NV1): NNLS for (α, β) in
 * T(n, s) = 2α + ((n+1)·s/n)·β over rows of measured NVLS AllReduce times (allreduce_exec_nvls).
 * out: alpha, beta set; gamma = delta = epsilon = 0, w_t = 1, has_combined = 0 (usable with
 * genmodel_closed_form("nvls", ...)).  Repeated (n, bytes) rows are averaged.  `sse` may be
 * NULL.  Errors: AR_EINVAL on a bad row or fewer than 2 distinct sizes. */
int genmodel_fit_nvls(const gm_measurement *rows, size_t n_rows, gm_params *out, double *sse);

/* The same NNLS for (α, β) on the A and B coefficients of another measured-protocol row:
 * kind "nvls" (= genmodel_fit_nvls), "oneshot" (reading OS1: the executor's one-shot
 * small-message path, T = α + 2(N−1)S·β) or "ll128" (the LL128 two-shot path,
 * T = α + (16/15)·2(N−1)S/N·β).  AR_EINVAL for another kind. */
int genmodel_fit_row(const char *kind, const gm_measurement *rows, size_t n_rows, gm_params *out, double *sse);

/* Table 2 closed form (readings Q5-Q7) of `kind` ("cps", "ring", "rhd", "rb",
 * "hcps:f0,f1,...", "nvls" = the in-switch row of reading NV1, "oneshot" = the small-message
 * row of reading OS1, "ll128" = the mid-size two-shot row) for n ranks and `bytes`
 * per rank, evaluated in the fixed float64 order of DESIGN.md.  Errors: AR_EINVAL for
 * n < 2, unknown kind, bad factorization. */
int genmodel_closed_form(const char *kind, int32_t n, uint64_t bytes, const gm_params *params,
                         gm_breakdown *out);

/* ------------------------------------------------------------------ GenTree */

typedef struct gt_plan gt_plan; /* opaque, immutable, library-owned, thread-shareable */

/* Build an AllReduce plan for `count` elements of `dtype` per rank on the tree described by
 * `topology_json` (SPEC's document format; NUL-terminated).  Ranks are the servers in
 * depth-first pre-order.  params == NULL uses each link's own parameters from the
 * document; otherwise `params` is used for every link and server.  force_kind == NULL (or
 * "") runs GenTree's selection; otherwise every switch uses that kind ("cps", "ring",
 * "rhd", "hcps:f0,f1,..", or "rb" on a single-switch topology); "norearrange" runs GenTree's
 * selection without the data-rearrangement optimisation — tab:gentreesimu's
 * GenTree*, "the special plan without data rearrangement".  The plan is verified
 * (conservation invariant) before it is returned.  *out must be released with
 * gt_plan_free.  Errors: AR_EINVAL on a malformed/invalid topology, count < 1, unknown
 * dtype or kind, or a forced kind that does not fit a switch. */
int gentree_plan(const char *topology_json, uint64_t count, int32_t dtype, const gm_params *params,
                 const char *force_kind, gt_plan **out);

/* GenTree with the NVLS plan kind as an extra candidate (reading NV1;
 * the paper's min-GenModel selection): builds gentree_plan's plan, and on a
 * single-switch topology with dtype AR_F32 replaces it by the NVLS plan when the NVLS row
 * predicts less time than the path the executor would run the plan on (the communicator's
 * cut-offs, ar_comm_get_paths / ar_default_paths): the LL128 row (`ll128_params`) when
 * given, the plan is one-shot eligible, N <= 8, count·esize >= 8N and
 * min(ll128_min_bytes, oneshot_max_bytes) < count·esize <= ll128_max_bytes; else the one-shot
 * row (reading OS1, `oneshot_params`) when given, the plan is one-shot eligible and
 * count·esize <= oneshot_max_bytes; else the executed-plan prediction
 * (genmodel_choose_nvls).  NULL row params leave that path out.  NVLS plans (also
 * force_kind "nvls" in gentree_plan; fp32 only, single switch) have the CPS data movement
 * and "switch_reduce": true in their JSON; every element ends as the correctly rounded fp32
 * sum of the ranks' inputs (reading NV2, measured) — the oracle's exactsum, bit for bit.
 * They run through allreduce_exec on a communicator with an attached NVLS buffer
 * (ar_comm_attach_nvls; dptr = that buffer).  params and nvls_params are required. */
int gentree_plan_nvls(const char *topology_json, uint64_t count, int32_t dtype, const gm_params *params,
                      const gm_params *nvls_params, const gm_params *oneshot_params, uint64_t oneshot_max_bytes,
                      const gm_params *ll128_params, uint64_t ll128_min_bytes, uint64_t ll128_max_bytes,
                      gt_plan **out);

/* Convenience: single switch with `world` ranks and uniform `params` (required). */
int gentree_plan_single_switch(int32_t world, uint64_t count, int32_t dtype, const gm_params *params,
                               const char *force_kind, gt_plan **out);

/* Canonical plan JSON (sorted keys, compact; byte-identical to the oracle's).  Writes at most
 * cap bytes including the NUL; *needed (if non-NULL) receives the full size incl. NUL.
 * AR_EINVAL if cap is too small (buf then holds nothing useful). */
int gt_plan_to_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed);
/* GenTree decision report (per switch: chosen kind, candidate totals, rearranged children,
 * start/finish times), JSON, same buffer protocol. */
int gt_plan_report_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed);
/* Shape of a plan. */
int gt_plan_info(const gt_plan *plan, int32_t *n_ranks, int32_t *n_steps, uint64_t *count, int32_t *dtype);
/* Per-step GenModel of the plan as executed (a6): params == NULL uses
 * the topology's links as traversed by each step (max α/β/ε, min w_t; reading Q16). */
int genmodel_predict(const gt_plan *plan, const gm_params *params, gm_breakdown *out);
void gt_plan_free(gt_plan *plan);

/* Incast-aware flow-level simulation of the plan (procedure
 * S:382-424, readings FS1-FS3 in DESIGN.md): per step, the transfers are routed on the tree,
 * α = the max over used links, the communication time comes from max-min fair rate sharing
 * recomputed at every flow completion, each directed link with capacity 1/β',
 * β' = β + max(w − w_t, 0)·ε and w = 1 + the distinct source ranks of its active flows, and
 * the compute time is the slowest server's Σ (k−1)|b|γ + (k+1)|b|δ.  topology_json == NULL
 * simulates on the plan's own topology, otherwise on that document (same number of servers;
 * rank r = the r-th server in DFS pre-order) — e.g. a flat plan routed over a tree.
 * params == NULL uses the topology's own links and servers (a plan from gt_plan_from_json
 * without a document then needs params: it is simulated on a single switch).  out: latency = Σα, bandwidth = the communication time with
 * ε = 0, incast = the rest of the communication time, compute/memory = the slowest server's γ
 * and δ parts, total.  step_times (optional, cap entries) receives each step's time;
 * *n_steps (optional) the number of steps.  Errors: AR_EINVAL for null plan/out or invalid
 * params. */
int gt_plan_simulate(const gt_plan *plan, const char *topology_json, const gm_params *params, gm_breakdown *out,
                     double *step_times, size_t cap, size_t *n_steps);

/* Build a plan from its canonical JSON (the gt_plan_to_json format): ranks, block
 * indices and transfer sizes are validated and no op of a step may write a (rank, block)
 * another op of the step reads or writes (AR_EINVAL otherwise).  *is_allreduce (optional)
 * is set to 1 iff the plan also passes the AllReduce conservation check;
 * data-movement plans that are not AllReduces (e.g. the x-to-x fan-in probe of P:418) are
 * accepted, and run through ar_exec_movement_plan (allreduce_exec refuses them).
 * genmodel_predict needs explicit params. */
int gt_plan_from_json(const char *plan_json, gt_plan **out, int32_t *is_allreduce);

/* GenModel of the plan as the B200 executor runs it (reading A6x): the same
 * per-step formula applied to the lowered steps — after the last RS level is fused
 * with the first AG level — with one α per flag round (entry + one per executed step) and
 * B = max over ranks of max(bytes in, bytes out) per step, since NVLink is full duplex and a
 * fused step moves RS and AG traffic at the same time.  `params` is required (uniform).
 * Bit-identical to oracle/genmodel.py predict_executed (which derives the executed steps from
 * the plan and the stated fusion rule, not from these tables; tests/test_parity_planner.py). */
int genmodel_predict_executed(const gt_plan *plan, const gm_params *params, gm_breakdown *out);

/* The same for a plan whose ranks ALL share one GPU (emulated communicator; config C5's
 * "8 ranks per GPU" on one device; reading A6e): the ranks' data movement goes through one
 * HBM, so each executed step costs α + C·γ + D·δ with D = Σ over ranks and ops of
 * (sources + destinations)·bytes and C = Σ (k − 1)·bytes (no link term). */
int genmodel_predict_executed_shared(const gt_plan *plan, const gm_params *params, gm_breakdown *out);

/* Plan-vs-NVLS selection by GenModel: *t_plan = the executed-plan
 * prediction of `plan` under plan_params (genmodel_predict_executed), *t_nvls = the "nvls"
 * closed form at the plan's (n, bytes) under nvls_params; *use_nvls = 1 iff t_nvls < t_plan
 * (ties keep the plan, whose result is bit-reproducible).  t_plan/t_nvls may be NULL.
 * Errors: AR_EINVAL for null plan/params/use_nvls or invalid params. */
int genmodel_choose_nvls(const gt_plan *plan, const gm_params *plan_params, const gm_params *nvls_params,
                         int32_t *use_nvls, double *t_plan, double *t_nvls);

/* ------------------------------------------------------------------ communicator */

typedef struct ar_comm ar_comm; /* opaque; one per process and device; single-threaded */

/* Multi-process communicator: this process is `rank` of `world` (2..64) and drives CUDA
 * device `cuda_device`.  Allocates this rank's flag page.  Errors: AR_EINVAL for bad
 * rank/world, AR_ESYS on CUDA failure. */
int ar_comm_create(int32_t rank, int32_t world, int32_t cuda_device, ar_comm **out);

/* Multi-level execution (SURVEY §8(f) NEXT #3, config C5's "8 ranks/GPU" across GPUs):
 * process `proc` of `nproc` hosts the ranks_per_proc consecutive ranks
 * proc·ranks_per_proc … proc·ranks_per_proc + ranks_per_proc − 1 of a world of
 * nproc·ranks_per_proc ranks on `cuda_device`.  Its registered buffer holds those ranks'
 * buffers at ar_rank_stride_bytes(count, dtype) apart (as for an emulated comm); peers'
 * buffers are IPC-mapped, so a plan's leaf levels move data inside HBM and its upper levels
 * over NVLink, all in one cooperative launch per process.  ar_comm_register / open_peers
 * exchange one blob per process (blobs = nproc × AR_BLOB_BYTES, process order).
 * ranks_per_proc = 1 is ar_comm_create(proc, nproc, ...).  Errors: AR_EINVAL for bad
 * arguments, nproc == 1 (use ar_comm_create_local) or world > AR_MAX_RANKS. */
int ar_comm_create_multi(int32_t proc, int32_t nproc, int32_t ranks_per_proc, int32_t cuda_device, ar_comm **out);

/* Emulated communicator: all `world` ranks live in this process on one device (each rank's
 * buffer is a separate region of device memory; "8 ranks/GPU" of config C5).  The executor
 * runs all ranks in one cooperative launch, with the same step tables and flag protocol;
 * single-step (CPS-shaped) plans run flag-free over every SM instead (ar_flat_kernel, same
 * bits; AR_FLAT=0 disables). */
int ar_comm_create_local(int32_t world, int32_t cuda_device, ar_comm **out);

/* Number of CTAs per rank used by the step-table kernel (0 = automatic).  Same value on all
 * ranks (checked by ar_comm_open_peers); multi-process comms: call before ar_comm_register —
 * AR_EINVAL once peers are open.  The flat and one-shot paths size their own grids and ignore
 * it; the LL128 path uses at most its occupancy per SM (2) times this many CTAs. */
int ar_comm_set_ctas(ar_comm *comm, int32_t ctas);

/* Export `bytes` of device memory at `dptr` (16-byte aligned; may be an interior pointer of
 * a cudaMalloc allocation, e.g. a torch tensor) for peer access.  Writes AR_BLOB_BYTES to
 * blob_out (CUDA IPC handles of the allocation and of this rank's flag page + offsets).
 * The caller gathers the blobs of all ranks (in rank order) and passes them to
 * ar_comm_open_peers.  The memory stays caller-owned and must outlive the registration.
 * Not used by emulated communicators. */
int ar_comm_register(ar_comm *comm, void *dptr, size_t bytes, void *blob_out);
/* Map every peer's registered buffer (and flag page, first time) into this process.
 * blobs = nproc * AR_BLOB_BYTES (= world * AR_BLOB_BYTES for ar_comm_create), process
 * order, from ar_comm_register on every process for the
 * same logical buffer (same size).  Collective: call on all ranks before the first
 * allreduce_exec on that buffer.  This process's own blob selects the local registration
 * (same allocation handle, offset and size).  The blobs carry the settings every rank must
 * share — CTA count (ar_comm_set_ctas), flag-page geometry, one-shot scratch size and path
 * cut-offs — and AR_EINVAL is returned if any rank differs; after this call
 * ar_comm_set_ctas may no longer change the CTA count.  Peers in the SAME process (several
 * communicators in one process, e.g. one per rank on one GPU for single-GPU testing of this
 * path) are mapped by their raw device pointers, since CUDA IPC handles cannot be opened by
 * the exporting process; each such communicator's kernels must then run on their own stream
 * with ar_comm_set_ctas(...) * world <= the SM count, so that all ranks' persistent kernels
 * are resident together. */
int ar_comm_open_peers(ar_comm *comm, const void *blobs);
/* Asynchronous device error of earlier executions (flag wait timeout = AR_ESYS), cleared on
 * read.  Synchronises the communicator's device. */
int ar_comm_get_async_error(ar_comm *comm);
int ar_comm_destroy(ar_comm *comm);

/* Bytes between consecutive ranks' buffers of an emulated communicator:
 * count * element size rounded up to 256. */
uint64_t ar_rank_stride_bytes(uint64_t count, int32_t dtype);

/* ------------------------------------------------------------------ execution */

/* In-place AllReduce (SUM) of `count` elements of `dtype` at `dptr` by executing `plan`
 * (lowered once per (plan, comm) to a device step table).  Multi-process comm: dptr is this
 * rank's registered buffer (ar_comm_register + ar_comm_open_peers).  Emulated comm: dptr
 * is the base of world consecutive rank buffers, rank r's at dptr + r *
 * ar_rank_stride_bytes(count, dtype).  Asynchronous and ordered on `stream` (a
 * cudaStream_t; NULL = legacy default stream).  Calls on one communicator must be ordered
 * with respect to each other (one stream, or explicit events): a launch reads the flag epoch
 * and the tile counters (dynamic tile scheduling of CPS-shaped plans) that the
 * previous launch left.  Every element of every rank's buffer ends
 * equal to the plan's left-to-right fp32 sum of the ranks' inputs (bit-exact to the CPU
 * oracle).  One rank per GPU, CPS-shaped plans take a flag-free path by size: the LL128
 * two-shot kernel (flags inside 128-byte lines, its own block partition: any count,
 * 8-byte-aligned buffer) when the message lies in its range (ar_comm_get_paths), else the
 * one-shot kernel up to the one-shot cut-off, else the step-table kernel — all with the
 * plan's bits (ar_comm_last_kernel tells which); the flag-free paths need no registration but
 * a buffer that holds count elements.  Errors: AR_EINVAL for plan/comm world mismatch,
 * count/dtype different from the plan's, unregistered, too small or misaligned buffer; AR_ESYS
 * on launch failure. */
int allreduce_exec(const gt_plan *plan, ar_comm *comm, void *dptr, uint64_t count, int32_t dtype,
                   void *stream);

/* Reduction operators of allreduce_exec_op.  AR_OP_AVG (DESIGN.md
 * reading AV1): the last ReduceScatter op writing each block divides its fp32 sum by the
 * world size N with one correctly rounded IEEE fp32 division, before the store's rounding
 * (bf16: RNE of the fp32 quotient); the AllGather then copies that value, so every rank ends
 * with the same bits.  On an NVLS plan (fp32): the switch's correctly rounded sum divided by N
 * with one correctly rounded division before the multicast store. */
#define AR_OP_SUM 0
#define AR_OP_AVG 1

/* allreduce_exec with an explicit operator (AR_OP_SUM = allreduce_exec).  Same contract and
 * errors; AR_EINVAL for an unknown op. */
int allreduce_exec_op(const gt_plan *plan, ar_comm *comm, void *dptr, uint64_t count, int32_t dtype, int32_t op,
                      void *stream);

/* Data-movement plans (measurement probes, e.g. the C3-ii fan-in tests: plans loaded with
 * gt_plan_from_json that are not AllReduces).  allreduce_exec and allreduce_exec_op reject
 * a plan that failed symbolic verification with AR_EINVAL; this entry runs it through the same
 * executor (copies and reduces of the plan's steps, same flag protocol).  Plans whose ops
 * exceed AR_MAX_RANKS sources or destinations are rejected (AR_EINVAL) in either entry. */
int ar_exec_movement_plan(const gt_plan *plan, ar_comm *comm, void *dptr, uint64_t count, int32_t dtype,
                          void *stream);

/* The same, end to end from host memory: copies `host` (pinned recommended; for an emulated
 * comm world consecutive rank buffers at the same stride) into dptr, executes, copies the
 * result back into `host`, all on `stream`. */
int allreduce_exec_host(const gt_plan *plan, ar_comm *comm, void *dptr, void *host, uint64_t count,
                        int32_t dtype, void *stream);

/* Device kernels launched by the last allreduce_exec of this comm (per rank, per call). */
int ar_comm_last_launch_count(ar_comm *comm, int32_t *kernels);
/* Name of the kernel the last allreduce_exec of this comm launched: "ar_exec_kernel" (the
 * step-table kernel and its flag protocol), "ar_ll_kernel" (one-shot small-message path),
 * "ar_ll128_kernel" (mid-size two-shot path), "ar_flat_kernel" (emulated single-step plans)
 * or "nvls_kernel" (NVLS plans); "" before the first call.  Static storage. */
const char *ar_comm_last_kernel(ar_comm *comm);

/* Path cut-offs (bytes per rank) of CPS-shaped plans on a one-rank-per-GPU communicator:
 * messages in (ll128_min, ll128_max] take the LL128 two-shot kernel (N <= 8, 8-byte-aligned
 * buffer); otherwise messages up to oneshot_max take the one-shot kernel;
 * everything else the step-table kernel.  ar_default_paths gives the defaults for `world`
 * ranks, measured on 2 and 4 B200s (one-shot to 1.5 MiB/(N−1); LL128 from 768 KiB/(N−1),
 * at most 384 KiB, to 64 MiB/N); AR_LL_MAX_KB, AR_LL128_MIN_KB and AR_LL128_MAX_KB override
 * them at communicator creation.  ar_comm_get_paths reports a communicator's effective
 * values (ll128_min already capped by oneshot_max; zeros where a path is unavailable:
 * emulated or several-ranks-per-GPU communicators, N > 8 for LL128).  NULL outputs are
 * skipped.  Errors: AR_EINVAL for world outside [2, AR_MAX_RANKS] / a NULL comm. */
int ar_default_paths(int32_t world, uint64_t *oneshot_max_bytes, uint64_t *ll128_min_bytes, uint64_t *ll128_max_bytes);
int ar_comm_get_paths(ar_comm *comm, uint64_t *oneshot_max_bytes, uint64_t *ll128_min_bytes, uint64_t *ll128_max_bytes);

/* Largest message (bytes per rank) run through the one-shot small-message path (default the
 * measured cut-off 1.5 MiB/(N−1); e.g. set it to GenModel's crossover of the "oneshot" row and
 * the executed-plan prediction; messages the LL128 path takes (ar_comm_get_paths) do not reach
 * it).  0 disables the path.  AR_EINVAL above the scratch capacity
 * allocated at creation or on a communicator without one (emulated / several ranks per GPU). */
int ar_comm_set_oneshot_max(ar_comm *comm, uint64_t bytes);

/* Tracing: when enabled, thread 0 of every CTA writes %globaltimer (ns) at kernel
 * start, after each step's waits, after its ops, after its notifies, and at exit, into
 * slots_per_cta stamps per CTA ([local rank][cta][slot]; slot 0 = start, 1+3i / 2+3i / 3+3i =
 * step i after waits / ops / notify, last = end; unused slots hold stale values).  Costs a few
 * global stores per step; off by default.  read: synchronises the device, copies the stamps
 * of the last call into `out` (cap elements); AR_EINVAL if tracing is off or cap is short. */
int ar_comm_set_trace(ar_comm *comm, int32_t enable);
int ar_comm_read_trace(ar_comm *comm, uint64_t *out, size_t cap, size_t *n, int32_t *slots_per_cta,
                       int32_t *ctas_per_rank);

/* Inspection (host only, no GPU needed): the per-rank device step tables allreduce_exec
 * runs for `plan` — after op merging, RS/AG fusion and the dependency analysis — as JSON
 * {"ranks":[{"steps":[{"slot":s,"ops":[{"off","len","src":[..],"dst":[..]}],
 * "waits":[[rank,slot,kind,p_off,p_len,c_off,c_len],..],"notify":[..]}]}]}.  Slot 0 = entry;
 * slot s+1 = after plan step s; the last step of each rank (exit) has only paired waits.
 * kind 0 = paired (the producer's CTA with my index), 1 = every producer CTA, 2 = range: the
 * producer CTAs whose slice of op [p_off, p_off+p_len) intersects my slice of the consumer op
 * [c_off, c_off+c_len) (elements; slices: whole 16-byte vectors split evenly over the CTAs, CTA
 * 0 adds the unaligned head, the last CTA the tail).  Same buffer protocol as gt_plan_to_json
 * (the size query itself returns AR_EINVAL with *needed set). */
int ar_plan_lowering_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed);

/* ------------------------------------------------------------------ NVLS plan kind (NEXT #1) */

/* In-switch reduction (NVLink SHARP) for a single NVSwitch domain: the Co-located-PS step
 * with the fan-in-N reduce done by the switch (multimem.ld_reduce) and the broadcast
 * by switch multicast (multimem.st) — ~S bytes per GPU and direction instead of 2(N−1)/N·S.
 * The switch picks the summation order, so results are not bit-comparable to a plan-order
 * oracle: they equal the exact sum on integer-valued inputs and are within the fp32/bf16
 * accumulation bound otherwise.  Setup is collective, one process per GPU:
 *   1. ar_nvls_create on every rank (rank 0 creates the multicast object of `bytes` + a flag
 *      area and exports it as a POSIX fd) -> blob_out (AR_BLOB_BYTES);
 *   2. gather the blobs (rank order), ar_nvls_attach on every rank (non-zero ranks import the
 *      fd with pidfd_getfd; every rank adds its device), then a host barrier;
 *   3. ar_nvls_bind on every rank (allocate, bind, map unicast + multicast) -> the unicast
 *      device pointer of this rank's `bytes`-byte buffer (library-owned; freed by destroy),
 *      then a host barrier before the first allreduce_exec_nvls.
 * allreduce_exec_nvls: in-place SUM of the first `count` elements (fp32 any count, bf16 even
 * counts; whole 16-byte vectors split evenly over the ranks, the tail on the last rank),
 * stream-ordered, graph-capturable.  Errors: AR_EINVAL for bad
 * arguments, AR_ESYS for CUDA/driver failures (e.g. multicast unsupported). */
typedef struct ar_nvls ar_nvls;
int ar_nvls_create(int32_t rank, int32_t world, int32_t cuda_device, uint64_t bytes, ar_nvls **out,
                   void *blob_out);
int ar_nvls_attach(ar_nvls *nvls, const void *blobs);
int ar_nvls_bind(ar_nvls *nvls, void **uc_ptr_out);
int allreduce_exec_nvls(ar_nvls *nvls, uint64_t count, int32_t dtype, void *stream);
int ar_nvls_get_async_error(ar_nvls *nvls);
int ar_nvls_destroy(ar_nvls *nvls);
/* Attach this rank's NVLS buffer to a one-rank-per-GPU communicator: allreduce_exec then runs
 * NVLS plans (gentree_plan_nvls / force_kind "nvls") on it, dptr = the buffer's unicast
 * pointer from ar_nvls_bind, any count up to its size (fp32; bf16 even counts).  The comm does
 * not own it.  AR_EINVAL for emulated / several-ranks-per-GPU comms. */
int ar_comm_attach_nvls(ar_comm *comm, ar_nvls *nvls);

/* ------------------------------------------------------------------ inputs and harness */

/* Fill `count` elements at dptr with the seeded synthetic generator G(seed, rank, i),
 * i = start..start+count-1 (mode 0 gradient, 1 integer,
 * 2 specials).  Independent CUDA implementation of synth/generator.py. */
int ar_fill_synthetic(void *dptr, uint64_t count, int32_t dtype, uint64_t seed, int32_t rank,
                      int32_t mode, uint64_t start, void *stream);

/* Eq. 6 micro-benchmark kernel: out = ((in[0] + in[1]) + ...) + in[k-1]
 * elementwise, fp32 accumulation, k = 1..64 device pointers (array in host memory),
 * one read of each input and one write of out per element. */
int ar_local_reduce(void *const *inputs, int32_t k, void *out, uint64_t count, int32_t dtype, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* GENTREE_AR_H */
