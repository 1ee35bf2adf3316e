// rpg_fit.h — internal interface of the K3 fit kernels (rpg_fit.cu).
#pragma once
#include <cstdint>
