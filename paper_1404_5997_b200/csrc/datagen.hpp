// SPEC data_gen on the GPU (see datagen.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hpsim_b200.h"

namespace hp {

void datagen_validate(const hp_dataset_spec& s);
// datagen_validate plus [first, first + count) inside [0, num_examples) (UsageError).
void datagen_check_range(const hp_dataset_spec& s, int64_t first, int64_t count);
// Examples [first, first + count) of the dataset into device memory: x
// [count][C][H][W] (the reference's NCHW batch layout), t [count][L] one-hot.
void datagen_launch(const hp_dataset_spec& s, int64_t first, int64_t count, float* x, float* t, cudaStream_t st);
int64_t datagen_class_of(const hp_dataset_spec& s, int64_t i);

}  // namespace hp
