// Library-wide status plumbing and table packing.
#include <cstdio>

#include "common.cuh"

namespace nvol {

static thread_local const char *g_last_error = "ok";
static thread_local char g_buf[512];

void set_error(const char *msg) { g_last_error = msg; }

// Ordered-reduction mode (nvol_set_deterministic): every reduction of the
// SIMT training path runs in a fixed order, so a run is bitwise repeatable.
int g_deterministic = 0;

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_buf, sizeof(g_buf), "%s: %s", what, cudaGetErrorString(e));
        g_last_error = g_buf;
        return NVOL_ECUDA;
    }
    return NVOL_OK;
}

int pack_tables(GridTables &t, const int64_t *level_off, const int64_t *level_res,
                const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels,
                int32_t n_feat) {
    NVOL_REQUIRE(n_levels >= 1 && n_levels <= NVOL_MAX_LEVELS, "n_levels must be in [1, 32]");
    NVOL_REQUIRE(n_feat == 1 || n_feat == 2 || n_feat == 4 || n_feat == 8,
                 "n_features_per_level must be in {1,2,4,8}");
    NVOL_REQUIRE(level_off && level_res && level_entries && level_dense, "null level table");
    t.n_levels = n_levels;
    t.n_feat = n_feat;
    for (int l = 0; l < n_levels; ++l) {
        NVOL_REQUIRE(level_res[l] >= 1 && level_res[l] < (1ll << 30), "level resolution out of range");
        NVOL_REQUIRE(level_entries[l] >= 1, "level entries must be >= 1");
        if (!level_dense[l]) {
            NVOL_REQUIRE((level_entries[l] & (level_entries[l] - 1)) == 0,
                         "hashed level entries must be a power of two");
        }
        t.res[l] = (int32_t)level_res[l];
        t.dense[l] = level_dense[l] ? 1 : 0;
        t.entries[l] = level_entries[l];
        t.offset[l] = level_off[l];
    }
    return NVOL_OK;
}

}  // namespace nvol

extern "C" {

int nvol_set_deterministic(int32_t on) {
    nvol::g_deterministic = on ? 1 : 0;
    return NVOL_OK;
}

int nvol_abi_version(void) { return 4; }  // 4: training NaN state (see nvol.h "NaN contract")

const char *nvol_last_error(void) { return nvol::g_last_error; }

}  // extern "C"
