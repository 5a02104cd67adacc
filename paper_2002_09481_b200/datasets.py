"""Synthetic benchmark inputs.

``synthetic_cifar10`` reproduces the reference's deterministic CIFAR-shaped
generator (``/root/reference/pkg/src/axemu/datasets.py:20-36``: ten 8x8-blocky
class templates from a fixed seed, 70% template + 30% uniform noise, snapped
to the byte grid) so benchmark batches are byte-identical to what the
reference harness would feed.  ``uniform_images`` is the ImageNet-shaped
U[0,1) input of the ResNet-50 configuration.
"""

from __future__ import annotations

import numpy as np

_TEMPLATE_SEED = 20908


def class_templates() -> np.ndarray:
    base = np.random.default_rng(_TEMPLATE_SEED).uniform(0.0, 1.0, (10, 4, 4, 3))
    return base.repeat(8, axis=1).repeat(8, axis=2).astype(np.float32)


def synthetic_cifar10(n: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    templates = class_templates()
    labels = rng.integers(0, 10, n)
    noise = rng.uniform(0.0, 1.0, (n, 32, 32, 3)).astype(np.float32)
    mixed = np.clip(0.7 * templates[labels] + 0.3 * noise, 0.0, 1.0)
    images = (np.rint(mixed * 255.0) / 255.0).astype(np.float32)
    return images, labels.astype(np.uint8)


def uniform_images(n: int, size: int = 224, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, (n, size, size, 3)).astype(np.float32)
