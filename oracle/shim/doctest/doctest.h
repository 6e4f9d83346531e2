// doctest-subset shim (angle-bracket include path) — TEST INFRASTRUCTURE ONLY.
#pragma once
#include "../doctest.h"
