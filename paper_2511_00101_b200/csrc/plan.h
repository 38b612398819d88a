// plan.h -- segment scheduler data structures (host planner <-> device kernels).
//
// The planner turns a segmented batch (Alg. 1 Require: the packed hidden
// states plus the F / P / D segment descriptors and offsets) into work items for the kernels
// (DESIGN.md "Canonical plan").  Tiles are 128 rows (one tcgen05 M=128 accumulator).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/smlm.h"

namespace smlm {

constexpr int kTileM = 128;

enum TileFlags : int {
    kTileShort = 1,  // rows of several short segments; per-row adapters via blocks
    kTileFT = 2,     // long tile of a FINETUNE segment (V_save is written)
    kTileLora = 4,   // long tile whose segment has an adapter (slot >= 0)
};

// ---- device-visible records (POD, identical layout on host and device) ----
struct alignas(16) DevTile {
    int row0;
    int rows;
    int slot;   // long: adapter slot or -1; short: -1
    int flags;  // TileFlags
    float scale;  // long: effective s = slot_scale * seg_scale
    int blk0;   // short: first block index
    int nblk;   // short: number of adapter blocks
    int seg;    // segment index (long / backward tiles)
};

struct alignas(16) DevBlock {  // one adapter inside a short tile
    int slot;
    int tile;       // short tile index (position in the short-tile list)
    int row_begin;  // first entry in the short-row list
    int nrows;
};

struct alignas(16) DevShortRow {  // a short row that has an adapter, grouped by block
    int row;
    float scale;
    int ft;     // 1 if the row belongs to a FINETUNE segment (V_save written)
    int pos;    // row - tile.row0 (position inside the 128-row tile)
};

struct alignas(16) DevGroup {  // backward: one adapter with fine-tune rows
    int slot;
    int tile_begin;  // into the backward tile list
    int n_tiles;
    int tokens;
};

// ---- host plan ----
struct Plan {
    std::vector<DevTile> long_tiles;
    std::vector<DevTile> short_tiles;
    std::vector<DevBlock> blocks;
    std::vector<DevShortRow> short_rows;
    std::vector<DevTile> bwd_tiles;  // fine-tune tiles in reduction order
    std::vector<DevGroup> groups;    // slots >= 0 with fine-tune rows, ascending
    int ft_rows = 0;
};

// Validate the batch and build the canonical plan.  slot_ok[capacity] marks registered slots,
// slot_scale[capacity] their static scale.  Returns SMLM_OK or an error status (msg set).
int build_plan(const smlm_batch *b, int capacity, const uint8_t *slot_ok, const float *slot_scale,
               int l_long, bool backward, Plan &plan, std::string &msg);

// Export as 6-word int32 records.
void export_plan(const Plan &plan, const smlm_batch *b, bool backward, std::vector<int32_t> &out);

}  // namespace smlm
