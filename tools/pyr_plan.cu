// Host-only: print the pyramid plan (stages, tiles, buffer capacities, shared
// memory) ft_build_pyramids would use for a W x H image.
//   nvcc -std=c++17 -o tools/pyr_plan tools/pyr_plan.cu && tools/pyr_plan 752 480 8 1.2 148
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "../paper_2509_10757_b200/csrc/ft_pyr.cuh"
using namespace ft;
int main(int argc, char **argv) {
    const int W = argc > 1 ? atoi(argv[1]) : 752, H = argc > 2 ? atoi(argv[2]) : 480;
    const int L = argc > 3 ? atoi(argv[3]) : 8;
    const double sc = argc > 4 ? atof(argv[4]) : 1.2;
    const int gb = argc > 5 ? atoi(argv[5]) : 1 << 30;
    PyrGeom g{};
    g.n_levels = L;
    long long off = 0;
    for (int l = 0; l < L; ++l) {
        const double p = pow(sc, l);
        g.widths[l] = (int)floor(W / p);
        g.heights[l] = (int)floor(H / p);
        g.offsets[l] = off;
        off += (long long)g.widths[l] * g.heights[l];
    }
    pyr_geom_scales(g);
    PyrPlan p{};
    if (!pyr_make_plan(g, p, gb)) { printf("plan failed\n"); return 1; }
    const size_t smem = pyr_plan_capacities(g, p);
    for (int s = 0; s < p.n_stages; ++s) printf("stage %d: end %d tiles %dx%d\n", s, p.stage_end[s], p.ty[s], p.tx[s]);
    printf("cap_region %d hsum %d smooth %d h %d rows %d cols %d smem %zu\n", p.cap_region, p.cap_hsum,
           p.cap_smooth, p.cap_h, p.cap_rows, p.cap_cols, smem);
    // computed pixels per level (sum of tile regions) vs the level's pixels
    double tot_c = 0, tot_o = 0, tot_in = 0;
    for (int s = 0; s < p.n_stages; ++s) {
        const int first = (s == 0 ? 0 : p.stage_end[s - 1]) + 1, last = p.stage_end[s];
        for (int l = first; l <= last; ++l) {
            double c = 0;
            for (int ty = 0; ty < p.ty[s]; ++ty)
                for (int tx = 0; tx < p.tx[s]; ++tx)
                    c += (double)(p.reg_y[l][ty][1] - p.reg_y[l][ty][0]) * (p.reg_x[l][tx][1] - p.reg_x[l][tx][0]);
            const double o = (double)g.widths[l] * g.heights[l];
            printf("level %d: computed %.0f px, level %.0f px, ratio %.2f\n", l, c, o, c / o);
            tot_c += c;
            tot_o += o;
        }
        double in = 0;
        for (int ty = 0; ty < p.ty[s]; ++ty)
            for (int tx = 0; tx < p.tx[s]; ++tx)
                in += (double)(p.in_y[s][ty][1] - p.in_y[s][ty][0]) * (p.in_x[s][tx][1] - p.in_x[s][tx][0]);
        tot_in += in;
    }
    printf("total computed %.0f / output %.0f = %.2f ; stage inputs loaded %.0f px\n", tot_c, tot_o, tot_c / tot_o, tot_in);
    return 0;
}
