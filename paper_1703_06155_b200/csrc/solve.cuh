// Device view of one level of a factor chain for the substitutions (solve.cu).
#pragma once

#include "device.cuh"

namespace h2g {

struct SolveTargetD {
  int seg, c0, c1;
};
struct SolveContribD {
  int m, entry;
};

struct SolveLevel {
  int nl;
  int bmax;
  const int* bsz;
  const long long* pos;
  const int* kfin;
  const int* C_ptr;
  const int* C_nb;
  const cplx* chain;
  const long long* Qt_off;
  const long long* L11_off;
  const long long* U11_off;
  const long long* Linv_off;
  const long long* Uinv_off;
  const long long* Lbar_off;
  const long long* Ubar_off;
  const long long* Lself_off;
  const long long* Uself_off;
};


// Batch schedule of one level for the persistent substitution kernels.
struct SolveSched {
  int nbat;
  const int* batch_ptr;   // [nbat + 1] into batch_cl
  const int* batch_cl;
  const int* batch_maxc;  // [nbat] max neighbour columns of a record
  const int* fs_ptr;      // [nbat + 1] into fs
  const SolveTargetD* fs;
  const SolveContribD* fc;
};

// Dataflow schedule of one level's substitutions (k_fwd_flow / k_bwd_flow).
struct SolveFlow {
  // forward: items in elimination order (>= 0 record, < 0 target -1-f),
  // writer index of every record / target on its segment
  int nf;
  const int* f_items;
  const int* rec_widx;
  const int* fs_widx;
  // backward: items (>= 0 record, < 0 gather slot -1-s)
  int nb;
  const int* b_items;
  const int* slot_m;             // record of the slot
  const int* slot_c;             // C entry (global index) or -1: self block
  const unsigned char* slot_final;  // neighbour processed later in the forward order: wait for its backward record
  const long long* slot_off;     // partial offset (complex per rhs)
  const int* rec_slot0;          // first slot of a record
  const int* rec_nslot;
  const int* reader_need;        // slots that read the record's retained part before it rotates it
  // split records (large blocks): number of rotation slabs, 0 = unsplit
  const int* rec_ns_f;
  const int* rec_ns_b;
  // fine levels (pull != 0): a record applies the updates of its earlier
  // neighbours to its own segment itself (targets rec_fs[rec_fs_ptr[t] ..],
  // in batch order) instead of one work item per (segment, batch)
  int pull;
  const int* rec_fs_ptr;
  const int* rec_fs;
};

// Right-hand sides beyond what the shared-memory segment buffers hold are cut
// into groups of rchunk columns; the dataflow kernels run the groups side by
// side (grid y), each with its own counter block.
struct FlowGroups {
  int rchunk;             // columns per group
  int cstride;            // ints between the counter blocks of two groups (>= 4 nl + 1)
  long long part_stride;  // complex between the backward partial buffers of two groups
};

// Whole level, all batches, one cooperative launch per direction; part holds
// max_b nb * (maxc_b + 1) * bmax * nrhs gathered backward partials.
void launch_fwd_level(const SolveLevel& S, const SolveSched& P, cplx* y, long long ldy, int nrhs, int explicit_inv, cudaStream_t s);
void launch_bwd_level(const SolveLevel& S, const SolveSched& P, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part, cudaStream_t s);
// Dataflow versions (no grid-wide barriers). cnt: >= 4 nl + 1 ints per group
// (G.cstride apart, reset by the launch); nrhs counts all columns from y; *fail is set when a dependency wait stalls (never reset here).
// tmp: n x nrhs scratch (ld ldy) holding the split records' segments between
// their slab and head items.
void launch_fwd_flow(const SolveLevel& S, const SolveSched& P, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, int* cnt,
                     int* fail, cplx* tmp, const FlowGroups& G, cudaStream_t s);
void launch_bwd_flow(const SolveLevel& S, const SolveFlow& F, cplx* y, long long ldy, int nrhs, int explicit_inv, cplx* part, int* cnt, int* fail,
                     cplx* tmp, const FlowGroups& G, cudaStream_t s);
void launch_permute(const long long* src, long long len, cplx* y, cplx* tmp, long long ldy, int nrhs, int scatter, cudaStream_t s);
void launch_root_trsv(const cplx* A, int n, cplx* y, long long ldy, int nrhs, int upper, cudaStream_t s);
void launch_finite(const cplx* y, long long total, int* bad, cudaStream_t s);

}  // namespace h2g
