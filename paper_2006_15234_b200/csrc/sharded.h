// Multi-GPU bond-sharded row absorb behind the C ABI.
//
// One process per GPU; the ranks of a communicator split every column
// einsumsvd of two_layer_apply_row (proj/src/contraction.cpp:269-311) along
// the boundary-MPS bond, and NCCL collectives (loaded at run time from
// libnccl.so.2, the one torch already mapped when it is in the process) run on
// the library's own stream, stream-ordered with the GEMMs: no host round trip
// per collective.  Algorithm: paper_2006_15234_b200/sharded.py (the same
// schedule, tested on gloo groups), DESIGN.md §6.
#pragma once

#include <memory>
#include <utility>

#include "peps.h"

namespace pepsb {

struct NcclComm;  // opaque: ncclComm_t + rank / world

// ncclGetUniqueId (rank 0; the caller broadcasts the 128 bytes to the others).
void comm_unique_id(unsigned char out[128]);
// ncclCommInitRank for this context's device; replaces any previous communicator.
void comm_init(Ctx& ctx, const unsigned char id[128], int rank, int world);
void comm_destroy(Ctx& ctx);
int comm_rank(const Ctx& ctx);
int comm_world(const Ctx& ctx);

// contraction.cpp:269-311 with every column einsumsvd whose outgoing bond is at
// least the world size split across the ranks (t on the column side, s on the
// pending tensor); inputs and the emitted boundary are replicated.
BoundaryD two_layer_apply_row_sharded(Ctx& ctx, const BoundaryD& top, const PepsStateD& bra, const PepsStateD& ket,
                                      int row, const ContractOptD& opt, uint64_t seed_tag);
// contraction.cpp:313-338: first row replicated, every later row absorb
// bond-sharded, closing chain_scalar (mps.cpp:102-110) replicated.
std::pair<double, double> contract_two_layer_sharded(Ctx& ctx, const PepsStateD& bra, const PepsStateD& ket,
                                                     const ContractOptD& opt);

}  // namespace pepsb
