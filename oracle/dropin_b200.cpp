// Drop-in translation unit (TEST INFRASTRUCTURE for the drop-in proof):
// defines fassmvs::estimate_bundle, dog_mask, geometric_consistency_mask and
// every stage-level function of the reference API and the CLI's output stage
// (colorize_*, write_pfm, write_png) on top of the B200 library through the
// public adapter include/fassmvs_b200.hpp. oracle/Makefile links it with the
// unmodified reference sources -- pipeline.cpp compiled with
// -Destimate_bundle=estimate_bundle_cpu so its CPU definition steps aside --
// and with the reference's own unit suite and acceptance program, which then
// exercise the B200 path through the reference's API.
#define FASSMVS_B200_DEFINE_ESTIMATE_BUNDLE
#define FASSMVS_B200_DEFINE_POSTFILTER
#define FASSMVS_B200_DEFINE_STAGES
#define FASSMVS_B200_DEFINE_OUTPUT
#include "fassmvs_b200.hpp"
