// Oracle build only (oracle/Makefile): resolves this repo's
// "fuseplan/minibatch.hpp" to the reference's own declaration of
// balance_minibatch, so the C-ABI adapter calls the reference implementation.
#pragma once
#include "fuseplan/workflow.hpp"
