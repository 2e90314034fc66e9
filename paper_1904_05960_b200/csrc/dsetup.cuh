// dsetup.cuh -- distributed setup primitives (dsetup.cu).
//
// A distributed setup keeps every operator in its GLOBAL row space with only
// the rank's own rows populated ("partial" CSR): the single-GPU setup kernels
// then run unchanged on the owned rows, and each product sums its middle
// index in the same global order as on one GPU, so every owned row comes out
// bitwise equal to the single-GPU row.  Per-point arrays (splits, measures,
// MIS status, C numbering) are replicated: each rank computes its owned
// segment and all-gathers it.  The exchange steps are the ones the algorithm
// needs: rows of the transposes (S^T for the MIS neighbourhoods, R = P^T)
// assembled at their owners, ghost rows of A and P fetched for the Galerkin
// products, and a full all-gather of a level once it is small (the coarse
// end of every AMG hierarchy is then set up redundantly on every rank).
#pragma once

#include <vector>

#include "common.cuh"

namespace pmgr {

struct Transport;

struct DistSetup {
    Transport *tr = nullptr;
    int rank = 0, nranks = 1;
    std::vector<int64_t> start;   // owned global row ranges of the space being built (nranks + 1)
    int64_t replicate_below = 0;  // spaces with at most this many rows are gathered to every rank
    int64_t lo() const { return start[rank]; }
    int64_t hi() const { return start[rank + 1]; }
    DistSetup with(const std::vector<int64_t> &st) const {
        DistSetup d = *this;
        d.start = st;
        return d;
    }
};

// owned ranges of the sub-space {i : (is_c[i] != 0) == want} (order kept)
std::vector<int64_t> ds_sub_bounds(const std::vector<int64_t> &start, const int8_t *is_c, int64_t n, bool want,
                                   cudaStream_t s);
int64_t ds_allsum(const DistSetup &d, int64_t v, cudaStream_t s);
int64_t ds_allmax(const DistSetup &d, int64_t v, cudaStream_t s);
// rows [lo, hi) of A in A's global row space (every other row empty)
void ds_partial_rows(const Csr &A, int64_t lo, int64_t hi, Csr &out, cudaStream_t s);
// X's rows (any, global row space over d's space) sent to their owners; each
// owned row of `out` concatenates the pieces of every rank in rank order.
// X.v may be null (pattern only; out.v stays empty).
void ds_rows_to_owners(const DistSetup &d, const Csr &X, Csr &out, cudaStream_t s);
// Y (partial over d's space) plus the rows `want` (sorted global ids owned by
// other ranks) fetched from their owners, in Y's global row space
void ds_fetch_rows(const DistSetup &d, const Csr &Y, const std::vector<int64_t> &want, Csr &Yext, cudaStream_t s);
// every rank's rows: the full operator on every rank
void ds_gather_rows(const DistSetup &d, const Csr &X, Csr &full, cudaStream_t s);
// replicate a per-point array: every rank's owned segment to every rank
void ds_gather_segment(const DistSetup &d, void *arr, size_t elem_bytes, cudaStream_t s);
// sorted distinct columns outside [clo, chi) of rows [rlo, rhi) of X
std::vector<int64_t> ds_cols_outside(const Csr &X, int64_t rlo, int64_t rhi, int64_t clo, int64_t chi,
                                     cudaStream_t s);
// csr_finalize with the statistics of the whole (distributed) operator, so
// every rank picks the single-GPU operator's SpMV lane group and long rows
void ds_finalize(const DistSetup *d, Csr &A, cudaStream_t s, bool build_sj = true);
// 1 / diag(A) on rows [lo, hi); first row with a zero or missing diagonal (-1: none)
int64_t ds_diag_inverse(const Csr &A, int64_t lo, int64_t hi, double *dinv, cudaStream_t s);

}  // namespace pmgr
