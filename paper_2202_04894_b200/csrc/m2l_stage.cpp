// Host helpers of the staged M2L (K7 v13, defmm_m2l_stage_*): greedy packing
// of a CTA's classes into shared-memory stages.
#include <cstdint>
#include <vector>

#include "../../include/defmm_b200.h"

extern "C" int defmm_stage_pack(int64_t ncls, const int64_t* cls_cta, const int64_t* cls_ptr,
                                const int64_t* cls_sym, int64_t n_sym_ids, int32_t ns_cap,
                                int64_t* cls_stage_rel) {
    if (ncls < 0 || ns_cap < 8) return -1;
    // stamp[sym] = id of the stage that last staged the symbol (stages numbered globally)
    std::vector<int64_t> stamp((size_t)n_sym_ids, -1);
    int64_t stage_id = -1, in_stage = 0, rel = 0, cur_cta = -1;
    for (int64_t c = 0; c < ncls; ++c) {
        const int64_t a = cls_ptr[c], b = cls_ptr[c + 1];
        if (b - a > ns_cap) return -2;
        if (cls_cta[c] != cur_cta) {  // first class of a CTA opens its stage 0
            cur_cta = cls_cta[c];
            ++stage_id;
            in_stage = 0;
            rel = 0;
        }
        int64_t fresh = 0;
        for (int64_t j = a; j < b; ++j) fresh += stamp[(size_t)cls_sym[j]] != stage_id;
        if (in_stage + fresh > ns_cap) {  // next stage of the same CTA
            ++stage_id;
            in_stage = 0;
            ++rel;
            fresh = b - a;
        }
        for (int64_t j = a; j < b; ++j) stamp[(size_t)cls_sym[j]] = stage_id;
        in_stage += fresh;
        cls_stage_rel[c] = rel;
    }
    return 0;
}
