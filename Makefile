# Builds the in-tree C-ABI library paper_1805_01407_b200/_lib/libslp_b200.so
# (sm_100a only).  The CPU oracle (oracle/) is numpy and needs no build.
NVCC ?= /usr/local/cuda/bin/nvcc
CSRC := paper_1805_01407_b200/csrc
LIBDIR := paper_1805_01407_b200/_lib
OBJDIR := build/obj$(if $(VARIANT),_$(VARIANT),)
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS = -O3 -std=c++17 $(ARCH) $(NVFLAGS_LINE) -Xcompiler -fPIC -Xcompiler -Wall -Xptxas -v -I include $(EXTRA)
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -I include

# A/B variant builds (VARIANT=name) leave out the run-time parameter
# (custom-engine) instances and -lineinfo: they only time registry kernels,
# and must stay small enough to ship to the GPU box next to the main library
INST := $(wildcard $(CSRC)/slp_inst_*.cu)
ifneq ($(VARIANT),)
INST := $(filter-out $(CSRC)/slp_inst_rt%.cu,$(INST))
override EXTRA += -DSLP_NO_RT_INSTANCES
NVFLAGS_LINE :=
else
NVFLAGS_LINE := -lineinfo
endif
OBJS := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(INST)) $(OBJDIR)/slp_api.o $(OBJDIR)/slp_host.o
HDRS := $(wildcard $(CSRC)/*.h $(CSRC)/*.cuh) include/slp_b200.h

all: $(LIBDIR)/libslp_b200.so

# A/B experiment builds: make variant VARIANT=name EXTRA="-DSLP_ROT_POLICY=0"
variant: variants/libslp_$(VARIANT).so

variants/libslp_$(VARIANT).so: $(OBJS)
	@mkdir -p variants
	$(NVCC) -shared $(ARCH) -cudart static -o $@ $(OBJS)

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ > $@.ptxas.log 2>&1 || (cat $@.ptxas.log; false)

$(OBJDIR)/slp_host.o: $(CSRC)/slp_host.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	g++ $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/libslp_b200.so: $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) -shared $(ARCH) -cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(LIBDIR)/*.so

.PHONY: all clean variant
