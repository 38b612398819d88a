// planner.cpp -- host segment scheduler: (segment, adapter, tile) -> work items.
//
// Paper context: §3.3 (SMLM processes all input-LoRA pairs of one linear
// layer in one call, four request kinds) and Alg. 1 P:326-346 (segment descriptors and
// offsets).  The rules are in DESIGN.md "Canonical plan"; oracle/plan.py re-derives them
// independently and tests/test_plan.py compares the two bit-exactly.
#include <math.h>

#include <algorithm>

#include "plan.h"

namespace smlm {

static int fail(std::string &msg, int code, const std::string &m) {
    msg = m;
    return code;
}

int build_plan(const smlm_batch *b, int capacity, const uint8_t *slot_ok, const float *slot_scale,
               int l_long, bool backward, Plan &p, std::string &msg) {
    p = Plan();
    if (!b) return fail(msg, SMLM_E_INVALID, "batch is NULL");
    if (b->S < 0 || b->G < 0) return fail(msg, SMLM_E_INVALID, "negative S or G");
    if (b->G == 0) {
        if (b->S != 0) return fail(msg, SMLM_E_INVALID, "G == 0 but S != 0");
        return SMLM_OK;
    }
    if (!b->seg_offsets || !b->seg_slot || !b->seg_mode)
        return fail(msg, SMLM_E_INVALID, "segment arrays must be non-NULL");
    if (!(b->dropout_p >= 0.0f && b->dropout_p < 1.0f))
        return fail(msg, SMLM_E_INVALID, "dropout_p must be in [0, 1)");
    const int32_t *off = b->seg_offsets;
    if (off[0] != 0) return fail(msg, SMLM_E_INVALID, "seg_offsets[0] must be 0");
    if (off[b->G] != b->S) return fail(msg, SMLM_E_INVALID, "seg_offsets[G] must equal S");
    for (int g = 0; g < b->G; ++g) {
        if (off[g + 1] < off[g]) return fail(msg, SMLM_E_INVALID, "seg_offsets must be non-decreasing");
        int m = b->seg_mode[g];
        if (m < SMLM_FINETUNE || m > SMLM_DECODE)
            return fail(msg, SMLM_E_INVALID, "seg_mode outside 0..3 at segment " + std::to_string(g));
        int s = b->seg_slot[g];
        if (s < -1 || s >= capacity)
            return fail(msg, SMLM_E_SLOT, "seg_slot out of range at segment " + std::to_string(g));
        if (s >= 0 && !(slot_ok && slot_ok[s]))
            return fail(msg, SMLM_E_SLOT, "slot " + std::to_string(s) + " is not registered");
        if (b->seg_scale) {
            float sc = b->seg_scale[g];
            if (!(sc > 0.0f) || !isfinite(sc))
                return fail(msg, SMLM_E_INVALID, "seg_scale must be finite and > 0");
        }
    }
    auto eff = [&](int g) -> float {
        int s = b->seg_slot[g];
        if (s < 0) return 0.0f;
        float v = slot_scale ? slot_scale[s] : 1.0f;
        if (b->seg_scale) v *= b->seg_scale[g];
        return v;
    };
    if (l_long < 1) l_long = 1;

    // ---- forward: long tiles (segment order, k ascending) ----
    for (int g = 0; g < b->G; ++g) {
        int len = off[g + 1] - off[g];
        if (len <= 0 || len < l_long) continue;
        for (int k = 0; k * kTileM < len; ++k) {
            DevTile t{};
            t.row0 = off[g] + k * kTileM;
            t.rows = std::min(kTileM, len - k * kTileM);
            t.slot = b->seg_slot[g];
            t.flags = (t.slot >= 0 ? kTileLora : 0) |
                      (b->seg_mode[g] == SMLM_FINETUNE && t.slot >= 0 ? kTileFT : 0);
            t.scale = eff(g);
            t.seg = g;
            p.long_tiles.push_back(t);
        }
    }
    // ---- forward: short runs -> tiles of <= 128 consecutive rows -> adapter blocks ----
    {
        struct R { int row, slot, g; };
        std::vector<std::vector<R>> runs;
        std::vector<R> cur;
        for (int g = 0; g < b->G; ++g) {
            int len = off[g + 1] - off[g];
            if (len == 0) continue;
            if (len >= l_long) {
                if (!cur.empty()) { runs.push_back(cur); cur.clear(); }
                continue;
            }
            for (int t = off[g]; t < off[g + 1]; ++t) cur.push_back({t, b->seg_slot[g], g});
        }
        if (!cur.empty()) runs.push_back(cur);
        std::vector<int> idx;
        idx.reserve(kTileM);
        for (auto &run : runs) {
            for (size_t i = 0; i < run.size(); i += kTileM) {
                size_t n = std::min<size_t>(kTileM, run.size() - i);
                DevTile t{};
                t.row0 = run[i].row;
                t.rows = (int)n;
                t.slot = -1;
                t.flags = kTileShort;
                t.seg = -1;
                t.blk0 = (int)p.blocks.size();
                // adapter blocks: the tile's rows with a slot, stably sorted by slot (ascending slot,
                // rows in run order inside a block) -- no per-slot containers
                idx.clear();
                for (size_t j = i; j < i + n; ++j)
                    if (run[j].slot >= 0) idx.push_back((int)j);
                std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return run[x].slot < run[y].slot; });
                int tile_index = (int)p.short_tiles.size();
                for (size_t q = 0; q < idx.size();) {
                    const int slot = run[idx[q]].slot;
                    DevBlock blk{};
                    blk.slot = slot;
                    blk.tile = tile_index;
                    blk.row_begin = (int)p.short_rows.size();
                    size_t q2 = q;
                    for (; q2 < idx.size() && run[idx[q2]].slot == slot; ++q2) {
                        const R *r = &run[idx[q2]];
                        DevShortRow sr{};
                        sr.row = r->row;
                        sr.scale = eff(r->g);
                        sr.ft = b->seg_mode[r->g] == SMLM_FINETUNE ? 1 : 0;
                        sr.pos = r->row - t.row0;
                        p.short_rows.push_back(sr);
                    }
                    blk.nrows = (int)(q2 - q);
                    p.blocks.push_back(blk);
                    q = q2;
                }
                t.nblk = (int)p.blocks.size() - t.blk0;
                p.short_tiles.push_back(t);
            }
        }
    }
    // ---- backward: fine-tune tiles ordered by (slot asc, segment, k); per-slot groups ----
    if (backward) {
        std::vector<int> ft;
        for (int g = 0; g < b->G; ++g)
            if (b->seg_mode[g] == SMLM_FINETUNE && off[g + 1] > off[g]) ft.push_back(g);
        std::vector<int> slots;
        for (int g : ft) slots.push_back(b->seg_slot[g]);
        std::sort(slots.begin(), slots.end());
        slots.erase(std::unique(slots.begin(), slots.end()), slots.end());
        for (int s : slots) {
            DevGroup grp{};
            grp.slot = s;
            grp.tile_begin = (int)p.bwd_tiles.size();
            for (int g : ft) {
                if (b->seg_slot[g] != s) continue;
                int len = off[g + 1] - off[g];
                for (int k = 0; k * kTileM < len; ++k) {
                    DevTile t{};
                    t.row0 = off[g] + k * kTileM;
                    t.rows = std::min(kTileM, len - k * kTileM);
                    t.slot = s;
                    t.flags = kTileFT | (s >= 0 ? kTileLora : 0);
                    t.scale = eff(g);
                    t.seg = g;
                    p.bwd_tiles.push_back(t);
                    grp.tokens += t.rows;
                }
            }
            grp.n_tiles = (int)p.bwd_tiles.size() - grp.tile_begin;
            p.ft_rows += grp.tokens;
            if (s >= 0) p.groups.push_back(grp);
        }
    }
    return SMLM_OK;
}

void export_plan(const Plan &p, const smlm_batch *b, bool backward, std::vector<int32_t> &out) {
    out.clear();
    auto rec = [&](int a, int c, int d, int e, int f, int g) {
        out.push_back(a); out.push_back(c); out.push_back(d);
        out.push_back(e); out.push_back(f); out.push_back(g);
    };
    if (!backward) {
        for (auto &t : p.long_tiles) rec(0, t.seg, t.row0, t.rows, t.slot, b->seg_mode[t.seg]);
        for (size_t i = 0; i < p.short_tiles.size(); ++i) {
            const DevTile &t = p.short_tiles[i];
            rec(1, (int)i, t.row0, t.rows, t.nblk, 0);
            for (int k = 0; k < t.nblk; ++k) {
                const DevBlock &blk = p.blocks[t.blk0 + k];
                rec(2, (int)i, k, blk.slot, blk.nrows, 0);
            }
        }
    } else {
        for (auto &t : p.bwd_tiles) rec(3, t.slot, t.seg, t.row0, t.rows, 0);
        for (auto &g : p.groups) rec(4, g.slot, g.tokens, g.n_tiles, 0, 0);
    }
}

}  // namespace smlm
