// Host-side helpers: bit-exact init_sparse, text I/O, CSC and chunk tables.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"

namespace lspb {

uint64_t derive_seed(uint64_t master, uint64_t tag, uint64_t index);
void init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val);
// Throws `code` (LSP_EINVAL or LSP_EIO) on an invalid projector.
void validate_projector(int n_rows, int d, int r, const int32_t* pos, const double* val,
                        int code);
std::string save_projector_text(int n_rows, int d, int r, const int32_t* pos,
                                const double* val);
void load_projector_text(const std::string& text, int* n_rows, int* d, int* r, int32_t* pos,
                         double* val);
int64_t subsample_size(double gamma, double beta, int m, int n, int total_steps, double delta);
void build_csc(int n_rows, int d, int r, const int32_t* pos, std::vector<int32_t>& ptr,
               std::vector<int32_t>& rows, std::vector<int32_t>& perm);
void build_chunks(int n_rows, int d, int bm, const std::vector<int32_t>& csc_ptr,
                  const std::vector<int32_t>& csc_rows, const std::vector<int32_t>& csc_perm,
                  std::vector<int32_t>& split, std::vector<int32_t>& row_in_chunk,
                  std::vector<int32_t>& perm);

// Fixed-slot stage-1 table (compress_slots.cu).  Per (row chunk c, bin a) the
// first K entries of the bin in the chunk (rows ascending) fill
// slot_row/slot_perm[(c*dpad + a)*K + t] (row -1 / perm -1 = padding); the
// bin's further entries go to the overflow list of (c, a/bpw), in bin then
// row order, with ovf_bin = a % bpw.  ovf_split[c*(dpad/bpw) + w] is the
// first overflow entry of (c, w).  dpad = d rounded up to 32; bpw divides 32.
struct SlotHost {
  std::vector<int32_t> slot_row, slot_perm, ovf_split, ovf_row, ovf_bin, ovf_perm;
};
void build_slots(int n_rows, int d, int bm, int K, int bpw, const std::vector<int32_t>& csc_ptr,
                 const std::vector<int32_t>& csc_rows, const std::vector<int32_t>& csc_perm,
                 SlotHost& out);
// Entries that would not fit K slots per (chunk, bin), i.e. the overflow size.
long long count_overflow(int n_rows, int d, int bm, int K, const std::vector<int32_t>& csc_ptr,
                         const std::vector<int32_t>& csc_rows);

}  // namespace lspb
