// The list step of a device-resident driver in one C call (nbx_list_step):
// grid -> search -> exclusions -> prune -> force layout, enqueued back to back
// so that the GPU never waits on the host between phases (the Python driver
// paid ~30-60 us of interpreter time between each of them per rebuild).
#include "internal.cuh"

using namespace nbx;

extern "C" int nbx_list_step(const double* positions, int64_t n, const double box[3], int32_t m, int64_t cells,
                             double r_list, double r_inner, const uint8_t* halo, const int32_t* atom_mol,
                             const int32_t* mol_first, const int32_t* mol_atoms, int32_t flags, void* stream,
                             nbx_grid_t** grid_out, nbx_list_t** list_out) {
  if (!grid_out || !list_out) {
    set_error("nbx_list_step: null output");
    return NBX_ERR_PARAM;
  }
  *grid_out = nullptr;
  *list_out = nullptr;
  if (atom_mol && (!mol_first || !mol_atoms)) {
    set_error("nbx_list_step: molecule topology needs atom_mol, mol_first and mol_atoms");
    return NBX_ERR_PARAM;
  }
  nbx_grid_t* grid = nullptr;
  nbx_list_t* built = nullptr;
  nbx_list_t* pruned = nullptr;
  int st = nbx_grid_build(positions, n, box, m, cells, stream, &grid);
  if (!st) st = nbx_pairlist_build_ex(grid, box, r_list, halo, stream, &built);
  if (!st && atom_mol) st = nbx_list_exclude(built, grid, atom_mol, mol_first, mol_atoms, stream, nullptr);
  if (!st && (flags & NBX_STEP_PRUNE)) {
    st = nbx_pairlist_prune_inner(built, grid, nbx_grid_clustered_positions(grid), box, r_inner, stream, &pruned);
    if (!st) {
      nbx_list_free(built);
      built = pruned;
    }
  }
  if (!st) {
    if (cudaError_t e = force_prepare(static_cast<List*>(built), to_stream(stream))) {
      set_error("nbx_list_step: %s", cudaGetErrorString(e));
      st = NBX_ERR_CUDA;
    }
  }
  if (st) {
    nbx_list_free(built);
    nbx_grid_free(grid);
    return st;
  }
  *grid_out = grid;
  *list_out = built;
  return NBX_OK;
}
